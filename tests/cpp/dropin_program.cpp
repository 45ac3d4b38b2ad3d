// A program written against the reference's C++ operator API only
// (#include "sparsek/..."; proj/include/sparsek/*.hpp). It is compiled twice:
//   * against the reference itself (its headers + sources, oracle/Makefile
//     target `dropin`, CPU)      -> oracle/_ref/dropin_ref
//   * against this repository's drop-in headers (include/sparsek/*.hpp) and
//     libsparsek_b200.so (GPU) -> tests/cpp/dropin_b200
// and both runs' outputs are compared by tests/test_dropin_gpu.py. Every line
// of output is "name count v0 v1 ..." with %.17g values.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "sparsek/attention.hpp"
#include "sparsek/cache.hpp"
#include "sparsek/selection.hpp"
#include "sparsek/sparsek_op.hpp"
#include "sparsek/stream.hpp"

using namespace sparsek;

static FILE* g_out = nullptr;

template <class V>
static void put(const std::string& name, const V& v) {
    std::fprintf(g_out, "%s %zu", name.c_str(), (size_t)v.size());
    for (const auto& x : v) std::fprintf(g_out, " %.17g", (double)x);
    std::fprintf(g_out, "\n");
}
static void put1(const std::string& name, double x) { put(name, std::vector<double>{x}); }

template <class T>
static MatT<T> rnd(Rng& r, size_t rows, size_t cols, double scale) {
    MatT<T> m(rows, cols);
    for (auto& x : m.data) x = static_cast<T>(scale * r.normal());
    return m;
}

static void ops_section() {
    Rng r(1001);
    std::vector<double> z(40);
    for (auto& x : z) x = r.normal();
    for (double k : {1.0, 3.5, 12.0}) {
        const std::string tag = "op_k" + std::to_string((int)(k * 10));
        SparseKSolution s = sparsek::sparsek(z, KBudget(k));
        put(tag + "_p", s.p);
        put1(tag + "_tau", s.tau);
        put(tag + "_counts", std::vector<double>{(double)s.u_count, (double)s.w_count, (double)s.degenerate});
        put(tag + "_support", s.support);
        std::vector<double> v(z.size());
        for (size_t i = 0; i < v.size(); ++i) v[i] = std::sin(0.3 * (double)i);
        put(tag + "_jvp", sparsek_jvp(s, v));
        PartialSortStats st;
        for (size_t cap : {size_t(std::ceil(k)), size_t(20), size_t(39)}) {
            SparseKSolution ps = sparsek_partial(z, KBudget(k), cap, &st);
            put(tag + "_partial_p_" + std::to_string(cap), ps.p);
        }
        put(tag + "_partial_stats", std::vector<double>{(double)st.calls, (double)st.fallbacks});
        put(tag + "_topk", topk_hard(z, (size_t)k));
        StResult sr = sparsek_st(z, KBudget(k));
        put(tag + "_st_fwd", sr.forward);
    }
    // the reference's own examples (test_sparsek_op.cpp:131-162)
    SparseKSolution a = sparsek::sparsek({0.9, 0.5, 0.1}, KBudget(2.0));
    put("ex_p", a.p);
    put1("ex_tau", a.tau);
}

static void stream_section() {
    Rng r(2002);
    StreamState s(KBudget(6.5));
    std::vector<double> taus, ins, evc, evs;
    for (int t = 0; t < 300; ++t) {
        const double z = r.normal() + 0.01 * t;
        StreamStepResult st = s.push(z);
        taus.push_back(st.tau);
        ins.push_back(st.inserted);
        evc.push_back((double)st.evicted.size());
        for (size_t e : st.evicted) evs.push_back((double)e);
        if (t == 150) {
            std::vector<std::uint8_t> blob;
            s.serialize(blob);
            size_t used = 0;
            s = StreamState::deserialize(blob.data(), blob.size(), &used);
            put1("stream_blob_used", (double)used);
        }
    }
    put("stream_tau", taus);
    put("stream_inserted", ins);
    put("stream_evcount", evc);
    put("stream_evicted", evs);
    SparseKSolution sol = s.solution();
    put("stream_sol_p", sol.p);
    put("stream_sol_idx", sol.indices);
    put("stream_counts", std::vector<double>{(double)s.t(), (double)s.survivor_count(), (double)s.saturated_count()});
    SelectionMask m = stream_mask(s);
    put("mask_hard", m.hard);
    put("mask_soft", m.soft);
    put("mask_idx", m.indices);
    std::vector<double> evd;
    for (size_t i = 0; i < 300; ++i) evd.push_back(s.is_evicted(i));
    put("stream_is_evicted", evd);
}

template <class T>
static void attention_section(const std::string& tag) {
    Rng r(3003);
    const size_t L = 96, D = 16, H = 2;
    AttnConfig cfg;
    cfg.k = 6.5;
    cfg.window = 8;
    cfg.heads = H;
    ScoringParams sc;
    sc.w_score.resize(D);
    for (auto& w : sc.w_score) w = r.normal() / 4.0;
    AttnParams<T> P{rnd<T>(r, D, D, 0.15), rnd<T>(r, D, D, 0.15), rnd<T>(r, D, D, 0.15), rnd<T>(r, D, D, 0.15)};
    MatT<T> x = rnd<T>(r, L, D, 1.0);
    MatT<T> g = rnd<T>(r, L, D, 1.0);
    AttnTape<T> tape;
    MatT<T> y = sparsek_attention(x, P, sc, cfg, &tape);
    put(tag + "_y", y.data);
    put(tag + "_tape_q", tape.q.data);
    put(tag + "_tape_hc", tape.head_concat.data);
    put(tag + "_tape_u", tape.u);
    put(tag + "_tape_raw", tape.raw);
    put(tag + "_tape_tau", tape.tau_push);
    std::vector<double> nsel, att, gate;
    for (const auto& q : tape.queries) {
        nsel.push_back(q.n_sel);
        for (auto a : q.att) att.push_back(a);
        for (auto gg : q.gate) gate.push_back(gg);
    }
    put(tag + "_tape_nsel", nsel);
    put(tag + "_tape_att", att);
    put(tag + "_tape_gate", gate);
    AttnGrads<T> gr = sparsek_attention_backward(tape, g, P, sc);
    put(tag + "_dx", gr.dx.data);
    put(tag + "_dwq", gr.dwq.data);
    put(tag + "_dwk", gr.dwk.data);
    put(tag + "_dwv", gr.dwv.data);
    put(tag + "_dwo", gr.dwo.data);
    put(tag + "_dws", gr.dw_score);
    // Algorithm 3: the recurrence chunk by chunk (no tape) == one pass
    MatT<T> yc = chunked_forward(x, 20, P, sc, cfg);
    put(tag + "_chunked_y", yc.data);
    // chunked training: outputs and chunk-local gradients
    AttnTape<T> ct;
    MatT<T> yct = chunked_forward(x, 32, P, sc, cfg, &ct);
    put(tag + "_chunked_tape_y", yct.data);
    AttnGrads<T> cg = sparsek_attention_backward(ct, g, P, sc);
    put(tag + "_chunked_dx", cg.dx.data);
    put(tag + "_chunked_dws", cg.dw_score);
    // decode: a prompt through forward_chunk, then generate_step per row
    SparseKvCache<T> cache(cfg, D, sc);
    MatT<T> prompt(40, D);
    std::copy(x.data.begin(), x.data.begin() + 40 * D, prompt.data.begin());
    MatT<T> yp = cache.forward_chunk(prompt, P);
    std::vector<double> dec(yp.data.begin(), yp.data.end());
    std::vector<double> peaks;
    for (size_t i = 40; i < L; ++i) {
        std::vector<T> row(x.row(i), x.row(i) + D);
        std::vector<T> yo = generate_step(cache, row, P);
        dec.insert(dec.end(), yo.begin(), yo.end());
    }
    put(tag + "_decode_y", dec);
    put(tag + "_cache_retained", cache.retained_positions());
    put(tag + "_cache_info", std::vector<double>{(double)cache.capacity(), (double)cache.size(),
                                                 (double)cache.window_fill(), (double)cache.positions_seen(),
                                                 (double)cache.peak_kv()});
    put(tag + "_cache_drain", prune_cache(cache));
    put(tag + "_cache_drain2", cache.drain_evictions());
    std::vector<double> ev;
    for (size_t i = 0; i < L; ++i) ev.push_back(cache.ever_evicted(i));
    put(tag + "_cache_ever_evicted", ev);
    put1(tag + "_cache_score5", cache.frozen_score(5));
    put1(tag + "_cache_stream_tau", cache.stream().tau());
    // dense limit
    MatT<T> hc;
    MatT<T> yd = dense_causal_attention(x, P, cfg.effective_scale(D), H, &hc);
    put(tag + "_dense_y", yd.data);
    AttnGrads<T> dg = dense_causal_attention_backward(x, P, cfg.effective_scale(D), H, hc, g);
    put(tag + "_dense_dx", dg.dx.data);
    put(tag + "_dense_dwq", dg.dwq.data);
    // matmul
    put(tag + "_matmul", matmul(x, P.wq).data);
    // linear-attention mix (Appendix B.1): forward, backward with dfeat, chunked training
    LinearMixParams<T> lin;
    for (size_t h = 0; h < H; ++h) lin.feat.push_back(rnd<T>(r, D / H, D / H, 0.3));
    AttnTape<T> lt;
    MatT<T> yl = linear_mix_attention(x, P, sc, cfg, lin, &lt);
    put(tag + "_lin_y", yl.data);
    AttnGrads<T> lg = sparsek_attention_backward(lt, g, P, sc, &lin);
    put(tag + "_lin_dx", lg.dx.data);
    put(tag + "_lin_dwk", lg.dwk.data);
    put(tag + "_lin_dws", lg.dw_score);
    std::vector<double> dfe;
    for (const auto& f : lg.dfeat) dfe.insert(dfe.end(), f.data.begin(), f.data.end());
    put(tag + "_lin_dfeat", dfe);
    AttnConfig lc = cfg;
    lc.linear_mix = true;
    AttnTape<T> lct;
    MatT<T> ylc = chunked_forward(x, 32, P, sc, lc, &lct, &lin);
    put(tag + "_lin_chunked_y", ylc.data);
    AttnGrads<T> lcg = sparsek_attention_backward(lct, g, P, sc, &lin);
    put(tag + "_lin_chunked_dx", lcg.dx.data);
    // linear-mix decoding: the cache carries the prefix state
    SparseKvCache<T> lcache(lc, D, sc);
    MatT<T> lprompt(30, D);
    std::copy(x.data.begin(), x.data.begin() + 30 * D, lprompt.data.begin());
    MatT<T> lyp = lcache.forward_chunk(lprompt, P, nullptr, &lin);
    std::vector<double> ldec(lyp.data.begin(), lyp.data.end());
    for (size_t i = 30; i < L; ++i) {
        std::vector<T> row(x.row(i), x.row(i) + D);
        std::vector<T> yo = generate_step(lcache, row, P, &lin);
        ldec.insert(ldec.end(), yo.begin(), yo.end());
    }
    put(tag + "_lin_decode_y", ldec);
}

static void errors_section() {
    std::vector<double> codes;
    auto code = [&](auto fn) {
        try {
            fn();
            codes.push_back(0);
        } catch (const ShapeError&) {
            codes.push_back(1);
        } catch (const ArgumentError&) {
            codes.push_back(2);
        } catch (const NumericError&) {
            codes.push_back(3);
        } catch (const ConfigError&) {
            codes.push_back(4);
        } catch (const std::exception&) {
            codes.push_back(9);
        }
    };
    code([] { KBudget(-1.0); });
    code([] { sparsek::sparsek({}, KBudget(1.0)); });
    code([] { sparsek::sparsek({1.0, NAN}, KBudget(1.0)); });
    code([] { sparsek_partial({1.0, 2.0, 3.0}, KBudget(2.5), 2); });
    code([] { StreamState s(KBudget(2.0)); s.push(INFINITY); });
    code([] { StreamState s(KBudget(2.0)); stream_mask(s); });
    code([] {
        AttnConfig c;
        c.heads = 3;
        ScoringParams sc;
        sc.w_score.assign(8, 0.1);
        c.validate(8, sc);
    });
    code([] {
        AttnConfig c;
        c.window = 0;
        c.k = 0.5;
        ScoringParams sc;
        sc.w_score.assign(8, 0.1);
        c.validate(8, sc);
    });
    code([] {
        AttnConfig c;
        ScoringParams sc;
        sc.w_score.assign(4, 0.1);
        MatT<double> x(5, 8);
        AttnParams<double> p{MatT<double>(8, 8), MatT<double>(8, 8), MatT<double>(8, 8), MatT<double>(8, 8)};
        sparsek_attention(x, p, sc, c);
    });
    code([] {
        AttnConfig c;
        ScoringParams sc;
        sc.w_score.assign(8, 0.1);
        MatT<double> x(5, 8);
        AttnParams<double> p{MatT<double>(8, 7), MatT<double>(8, 8), MatT<double>(8, 8), MatT<double>(8, 8)};
        sparsek_attention(x, p, sc, c);
    });
    put("error_codes", codes);
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s out.txt\n", argv[0]);
        return 2;
    }
    g_out = std::fopen(argv[1], "w");
    if (!g_out) return 3;
    ops_section();
    stream_section();
    attention_section<double>("f64");
    attention_section<float>("f32");
    errors_section();
    std::fclose(g_out);
    std::printf("dropin ok\n");
    return 0;
}
