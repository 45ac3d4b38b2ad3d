// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// C-ABI shim over the UNMODIFIED reference library (/root/reference/proj).
// `oracle/Makefile` compiles this file together with the reference's own
// sources where they lie (no copies) into oracle/_ref/libsparsek_ref.so.
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg are the only callers.
//
// Every entry point forwards to the reference's public C++ API:
//   sparsek / sparsek_partial / sparsek_jvp / topk_hard  proj/include/sparsek/sparsek_op.hpp:40-66
//   StreamState::push / solution                        proj/include/sparsek/stream.hpp:26-72
//   sparsek_attention / sparsek_attention_backward      proj/include/sparsek/attention.hpp:81-91
//   SparseKvCache::forward_chunk / generate_step        proj/include/sparsek/cache.hpp:21-102
//   dense_causal_attention                              proj/include/sparsek/attention.hpp:104-106
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "sparsek/attention.hpp"
#include "sparsek/cache.hpp"
#include "sparsek/sparsek_op.hpp"
#include "sparsek/stream.hpp"

using namespace sparsek;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

#define REF_GUARD_BEGIN try {
#define REF_GUARD_END                                              \
    }                                                              \
    catch (const ShapeError& e) { return fail(e, 1); }             \
    catch (const ArgumentError& e) { return fail(e, 2); }          \
    catch (const NumericError& e) { return fail(e, 3); }           \
    catch (const ConfigError& e) { return fail(e, 4); }            \
    catch (const IoError& e) { return fail(e, 5); }                \
    catch (const std::exception& e) { return fail(e, 9); }         \
    return 0;

}  // namespace

extern "C" {

struct ref_cfg {
    double k;
    uint64_t window;
    uint64_t heads;
    double scale;
    int32_t key_mode;     // 0 hard, 1 soft
    int32_t mask_mode;    // 0 soft, 1 straight_through
    uint64_t group_size;
    double slope_eps;
    int32_t slope_enabled;
    int32_t norm_mode;    // 0 none, 1 timestep_norm
    int32_t slope_order;  // 0 slope_then_norm, 1 norm_then_slope
    int32_t pad_;
};

const char* ref_last_error() { return g_err.c_str(); }

static void fill_solution(const SparseKSolution& sol, size_t m, double* p, double* tau,
                          uint64_t* u_count, uint64_t* w_count, int32_t* degenerate,
                          int32_t* infeasible) {
    if (p) {
        if (sol.indices.empty()) {
            for (size_t i = 0; i < m; ++i) p[i] = i < sol.p.size() ? sol.p[i] : 0.0;
        } else {
            for (size_t i = 0; i < m; ++i) p[i] = 0.0;
            for (size_t s = 0; s < sol.indices.size(); ++s) p[sol.indices[s]] = sol.p[s];
        }
    }
    if (tau) *tau = sol.tau;
    if (u_count) *u_count = sol.u_count;
    if (w_count) *w_count = sol.w_count;
    if (degenerate) *degenerate = sol.degenerate ? 1 : 0;
    if (infeasible) *infeasible = sol.infeasible ? 1 : 0;
}

int ref_sparsek(const double* z, uint64_t m, double k, uint64_t sort_cap, double* p, double* tau,
                uint64_t* u_count, uint64_t* w_count, int32_t* degenerate, int32_t* infeasible) {
    REF_GUARD_BEGIN
    std::vector<double> zv(z, z + m);
    SparseKSolution sol = sort_cap > 0 ? sparsek_partial(zv, KBudget(k), sort_cap)
                                       : sparsek::sparsek(zv, KBudget(k));
    fill_solution(sol, m, p, tau, u_count, w_count, degenerate, infeasible);
    REF_GUARD_END
}

int ref_sparsek_jvp(const double* z, uint64_t m, double k, const double* v, double* out) {
    REF_GUARD_BEGIN
    std::vector<double> zv(z, z + m), vv(v, v + m);
    SparseKSolution sol = sparsek::sparsek(zv, KBudget(k));
    std::vector<double> r = sparsek_jvp(sol, vv);
    std::memcpy(out, r.data(), m * sizeof(double));
    REF_GUARD_END
}

int ref_topk_hard(const double* z, uint64_t m, uint64_t k, double* out) {
    REF_GUARD_BEGIN
    std::vector<double> zv(z, z + m);
    std::vector<double> r = topk_hard(zv, k);
    std::memcpy(out, r.data(), m * sizeof(double));
    REF_GUARD_END
}

// Push z[0..n) through one StreamState; per step: tau (−inf when infeasible),
// inserted flag, survivor count, and the solution p over the full prefix
// (only when p_last != nullptr: the final step's weights).
int ref_stream_run(const double* z, uint64_t n, double k, uint64_t heap_cap, double* tau_out,
                   uint8_t* inserted_out, uint64_t* survivors_out, double* p_last) {
    REF_GUARD_BEGIN
    StreamState st{KBudget(k), heap_cap};
    for (uint64_t t = 0; t < n; ++t) {
        StreamStepResult r = st.push(z[t]);
        if (tau_out) tau_out[t] = r.tau;
        if (inserted_out) inserted_out[t] = r.inserted ? 1 : 0;
        if (survivors_out) survivors_out[t] = st.survivor_count();
    }
    if (p_last) fill_solution(st.solution(), n, p_last, nullptr, nullptr, nullptr, nullptr, nullptr);
    REF_GUARD_END
}

// StreamState::push events: per push the StreamStepResult (tau, inserted,
// cap_forced) and its evicted indices, flattened (ev_count[t] entries each,
// in the order the reference reports them; ev_flat holds ev_cap entries).
int ref_stream_events(const double* z, uint64_t n, double k, uint64_t heap_cap, double* tau_out,
                      uint8_t* inserted_out, uint8_t* cap_forced_out, uint64_t* ev_count, uint64_t* ev_flat,
                      uint64_t ev_cap) {
    REF_GUARD_BEGIN
    StreamState st{KBudget(k), heap_cap};
    uint64_t used = 0;
    for (uint64_t t = 0; t < n; ++t) {
        StreamStepResult r = st.push(z[t]);
        tau_out[t] = r.tau;
        inserted_out[t] = r.inserted ? 1 : 0;
        cap_forced_out[t] = r.cap_forced ? 1 : 0;
        ev_count[t] = r.evicted.size();
        for (size_t e : r.evicted) {
            if (used >= ev_cap) throw ArgumentError("ref_stream_events: ev_flat too small");
            ev_flat[used++] = e;
        }
    }
    REF_GUARD_END
}

// stream_mask after pushing z[0..n) (proj/src/stream.cpp:199-222): hard/soft
// per survivor slot (ascending index; positions in pos_out), *n_out slots and
// the hard set's positions in idx_out (*n_idx of them).
int ref_stream_mask(const double* z, uint64_t n, double k, uint64_t heap_cap, uint64_t* pos_out, double* hard_out,
                    double* soft_out, uint64_t* n_out, uint64_t* idx_out, uint64_t* n_idx) {
    REF_GUARD_BEGIN
    StreamState st{KBudget(k), heap_cap};
    for (uint64_t t = 0; t < n; ++t) st.push(z[t]);
    SelectionMask m = stream_mask(st);
    const SparseKSolution sol = st.solution();
    *n_out = m.hard.size();
    for (size_t i = 0; i < m.hard.size(); ++i) {
        pos_out[i] = sol.indices[i];
        hard_out[i] = m.hard[i];
        soft_out[i] = m.soft[i];
    }
    *n_idx = m.indices.size();
    for (size_t i = 0; i < m.indices.size(); ++i) idx_out[i] = m.indices[i];
    REF_GUARD_END
}

// sparsek_st (proj/src/sparsek_op.cpp:167-172): hard forward + soft carrier p.
int ref_sparsek_st(const double* z, uint64_t m, double k, double* forward, double* p) {
    REF_GUARD_BEGIN
    std::vector<double> zv(z, z + m);
    StResult r = sparsek_st(zv, KBudget(k));
    std::memcpy(forward, r.forward.data(), m * sizeof(double));
    fill_solution(r.backward_carrier, m, p, nullptr, nullptr, nullptr, nullptr, nullptr);
    REF_GUARD_END
}

// sparsek_partial with PartialSortStats (proj/src/sparsek_op.cpp:116-139).
int ref_sparsek_partial_stats(const double* z, uint64_t m, double k, uint64_t sort_cap, double* p, double* tau,
                              uint64_t* calls, uint64_t* fallbacks) {
    REF_GUARD_BEGIN
    std::vector<double> zv(z, z + m);
    PartialSortStats st;
    SparseKSolution sol = sparsek_partial(zv, KBudget(k), sort_cap, &st);
    fill_solution(sol, m, p, tau, nullptr, nullptr, nullptr, nullptr);
    *calls = st.calls;
    *fallbacks = st.fallbacks;
    REF_GUARD_END
}

// StreamState::serialize after pushing z[0..n): *used = blob size (out may be
// null to query it; cap = out capacity).
int ref_stream_blob(const double* z, uint64_t n, double k, uint64_t heap_cap, uint8_t* out,
                    uint64_t cap, uint64_t* used) {
    REF_GUARD_BEGIN
    StreamState st{KBudget(k), heap_cap};
    for (uint64_t t = 0; t < n; ++t) st.push(z[t]);
    std::vector<std::uint8_t> blob;
    st.serialize(blob);
    *used = blob.size();
    if (out) {
        if (cap < blob.size()) throw ArgumentError("ref_stream_blob: buffer too small");
        std::memcpy(out, blob.data(), blob.size());
    }
    REF_GUARD_END
}

// StreamState::deserialize(blob), then push z[0..n) and report each tau.
int ref_stream_resume(const uint8_t* blob, uint64_t len, const double* z, uint64_t n,
                      double* tau_out) {
    REF_GUARD_BEGIN
    StreamState st = StreamState::deserialize(blob, len, nullptr);
    for (uint64_t t = 0; t < n; ++t) tau_out[t] = st.push(z[t]).tau;
    REF_GUARD_END
}

}  // extern "C"

namespace {

AttnConfig to_cfg(const ref_cfg* c) {
    AttnConfig cfg;
    cfg.k = c->k;
    cfg.window = c->window;
    cfg.heads = c->heads;
    cfg.scale = c->scale;
    cfg.key_mode = c->key_mode ? KeyMode::soft : KeyMode::hard;
    cfg.mask_mode = c->mask_mode ? MaskApply::straight_through : MaskApply::soft;
    cfg.group_size = c->group_size ? c->group_size : 128;
    return cfg;
}

ScoringParams to_scoring(const ref_cfg* c, const double* w_score, size_t D) {
    ScoringParams sp;
    sp.w_score.assign(w_score, w_score + D);
    sp.slope_eps = c->slope_eps;
    sp.slope_enabled = c->slope_enabled != 0;
    sp.norm_mode = c->norm_mode ? NormMode::timestep_norm : NormMode::none;
    sp.slope_order = c->slope_order ? SlopeOrder::norm_then_slope : SlopeOrder::slope_then_norm;
    return sp;
}

template <class T>
MatT<T> mat_in(const double* p, size_t r, size_t c) {
    MatT<T> m(r, c);
    for (size_t i = 0; i < r * c; ++i) m.data[i] = static_cast<T>(p[i]);
    return m;
}

template <class T>
void mat_out(const MatT<T>& m, double* p) {
    if (!p) return;
    for (size_t i = 0; i < m.data.size(); ++i) p[i] = static_cast<double>(m.data[i]);
}

// A forward run with its tape kept alive for inspection and backward.
struct TapeBase {
    virtual ~TapeBase() = default;
};

template <class T>
struct TapeRun : TapeBase {
    AttnParams<T> params;
    ScoringParams scoring;
    AttnTape<T> tape;
    MatT<T> y;
};

}  // namespace

extern "C" {

// Forward with tape. Returns an opaque handle in *out (free with ref_tape_free).
int ref_attention_fwd_chunked(int32_t use_float, uint64_t L, uint64_t D, const double* x,
                              const double* wq, const double* wk, const double* wv, const double* wo,
                              const double* w_score, const ref_cfg* c, uint64_t chunk_len, void** out);

int ref_attention_fwd(int32_t use_float, uint64_t L, uint64_t D, const double* x, const double* wq,
                      const double* wk, const double* wv, const double* wo,
                      const double* w_score, const ref_cfg* c, void** out) {
    return ref_attention_fwd_chunked(use_float, L, D, x, wq, wk, wv, wo, w_score, c, 0, out);
}

// chunk_len 0: sparsek_attention (attention.hpp:81-85); > 0: chunked_forward
// (cache.hpp:93-96, Algorithm 3) — same outputs, tape.chunk_starts set.
int ref_attention_fwd_chunked(int32_t use_float, uint64_t L, uint64_t D, const double* x,
                              const double* wq, const double* wk, const double* wv, const double* wo,
                              const double* w_score, const ref_cfg* c, uint64_t chunk_len, void** out) {
    REF_GUARD_BEGIN
    auto run_t = [&](auto tag) -> TapeBase* {
        using T = decltype(tag);
        auto* r = new TapeRun<T>();
        r->params = AttnParams<T>{mat_in<T>(wq, D, D), mat_in<T>(wk, D, D), mat_in<T>(wv, D, D),
                                  mat_in<T>(wo, D, D)};
        r->scoring = to_scoring(c, w_score, D);
        try {
            if (chunk_len == 0)
                r->y = sparsek_attention(mat_in<T>(x, L, D), r->params, r->scoring, to_cfg(c), &r->tape);
            else
                r->y = chunked_forward(mat_in<T>(x, L, D), chunk_len, r->params, r->scoring, to_cfg(c),
                                       &r->tape);
        } catch (...) {
            delete r;
            throw;
        }
        return r;
    };
    *out = use_float ? run_t(float{}) : run_t(double{});
    REF_GUARD_END
}

void ref_tape_free(void* h) { delete static_cast<TapeBase*>(h); }

// Sizes: n queries, total attended entries, total selected entries, tau_push length.
int ref_tape_sizes(void* h, uint64_t* n, uint64_t* total_att, uint64_t* total_sel,
                   uint64_t* n_tau) {
    REF_GUARD_BEGIN
    auto go = [&](auto* r) {
        *n = r->tape.queries.size();
        uint64_t ta = 0, ts = 0;
        for (auto& q : r->tape.queries) {
            ta += q.att.size();
            ts += q.n_sel;
        }
        *total_att = ta;
        *total_sel = ts;
        *n_tau = r->tape.tau_push.size();
    };
    if (auto* rd = dynamic_cast<TapeRun<double>*>(static_cast<TapeBase*>(h))) go(rd);
    else go(dynamic_cast<TapeRun<float>*>(static_cast<TapeBase*>(h)));
    REF_GUARD_END
}

// Copy the tape out. Any pointer may be null. att_off has n+1 entries; att is
// total_att long; gate is total_sel long (selected entries of each query in
// order); maxa/denom are n*heads; q/k/v/head_concat/y are L*D.
int ref_tape_copy(void* h, double* y, double* q, double* k, double* v, double* head_concat,
                  double* raw, double* u, double* norm_mean, double* norm_sdev, double* tau_push,
                  uint32_t* n_sel, uint64_t* att_off, uint32_t* att, double* gate, double* maxa,
                  double* denom) {
    REF_GUARD_BEGIN
    auto go = [&](auto* r) {
        auto& tp = r->tape;
        mat_out(r->y, y);
        mat_out(tp.q, q);
        mat_out(tp.k, k);
        mat_out(tp.v, v);
        mat_out(tp.head_concat, head_concat);
        auto vcopy = [](const std::vector<double>& s, double* d) {
            if (d) std::memcpy(d, s.data(), s.size() * sizeof(double));
        };
        vcopy(tp.raw, raw);
        vcopy(tp.u, u);
        vcopy(tp.norm_mean, norm_mean);
        vcopy(tp.norm_sdev, norm_sdev);
        vcopy(tp.tau_push, tau_push);
        uint64_t off = 0, soff = 0, hoff = 0;
        for (size_t i = 0; i < tp.queries.size(); ++i) {
            auto& qr = tp.queries[i];
            if (n_sel) n_sel[i] = qr.n_sel;
            if (att_off) att_off[i] = off;
            if (att) std::memcpy(att + off, qr.att.data(), qr.att.size() * sizeof(uint32_t));
            if (gate) std::memcpy(gate + soff, qr.gate.data(), qr.gate.size() * sizeof(double));
            for (size_t hh = 0; hh < qr.maxa.size(); ++hh) {
                if (maxa) maxa[hoff + hh] = static_cast<double>(qr.maxa[hh]);
                if (denom) denom[hoff + hh] = static_cast<double>(qr.denom[hh]);
            }
            hoff += qr.maxa.size();
            off += qr.att.size();
            soff += qr.gate.size();
        }
        if (att_off) att_off[tp.queries.size()] = off;
    };
    if (auto* rd = dynamic_cast<TapeRun<double>*>(static_cast<TapeBase*>(h))) go(rd);
    else go(dynamic_cast<TapeRun<float>*>(static_cast<TapeBase*>(h)));
    REF_GUARD_END
}

// Backward through the reference. Outputs are L*D (dx) and D*D (dW*), D (dw_score).
int ref_tape_backward(void* h, const double* grad_out, double* dx, double* dwq, double* dwk,
                      double* dwv, double* dwo, double* dw_score) {
    REF_GUARD_BEGIN
    auto run = [&](auto* r) {
        using T = std::remove_reference_t<decltype(r->y.data[0])>;
        MatT<T> g(r->y.rows, r->y.cols);
        for (size_t i = 0; i < g.data.size(); ++i) g.data[i] = static_cast<T>(grad_out[i]);
        AttnGrads<T> gr = sparsek_attention_backward(r->tape, g, r->params, r->scoring);
        mat_out(gr.dx, dx);
        mat_out(gr.dwq, dwq);
        mat_out(gr.dwk, dwk);
        mat_out(gr.dwv, dwv);
        mat_out(gr.dwo, dwo);
        if (dw_score) std::memcpy(dw_score, gr.dw_score.data(), gr.dw_score.size() * sizeof(double));
    };
    if (auto* rd = dynamic_cast<TapeRun<double>*>(static_cast<TapeBase*>(h))) run(rd);
    else run(dynamic_cast<TapeRun<float>*>(static_cast<TapeBase*>(h)));
    REF_GUARD_END
}

int ref_dense_attention(uint64_t L, uint64_t D, uint64_t heads, const double* x, const double* wq,
                        const double* wk, const double* wv, const double* wo, double* y) {
    REF_GUARD_BEGIN
    AttnParams<double> params{mat_in<double>(wq, D, D), mat_in<double>(wk, D, D),
                              mat_in<double>(wv, D, D), mat_in<double>(wo, D, D)};
    AttnConfig cfg;
    cfg.heads = heads;
    MatT<double> r = dense_causal_attention(mat_in<double>(x, L, D), params,
                                            cfg.effective_scale(D), heads);
    mat_out(r, y);
    REF_GUARD_END
}

// dense_causal_attention + its backward (proj/src/attention.cpp:76-205), double.
int ref_dense_attention_grads(uint64_t L, uint64_t D, uint64_t heads, const double* x, const double* wq,
                              const double* wk, const double* wv, const double* wo, const double* grad_out,
                              double* y, double* dx, double* dwq, double* dwk, double* dwv, double* dwo) {
    REF_GUARD_BEGIN
    AttnParams<double> params{mat_in<double>(wq, D, D), mat_in<double>(wk, D, D),
                              mat_in<double>(wv, D, D), mat_in<double>(wo, D, D)};
    AttnConfig cfg;
    cfg.heads = heads;
    const double scale = cfg.effective_scale(D);
    MatT<double> xm = mat_in<double>(x, L, D), hc;
    MatT<double> r = dense_causal_attention(xm, params, scale, heads, &hc);
    mat_out(r, y);
    AttnGrads<double> g = dense_causal_attention_backward(xm, params, scale, heads, hc,
                                                          mat_in<double>(grad_out, L, D));
    mat_out(g.dx, dx);
    mat_out(g.dwq, dwq);
    mat_out(g.dwk, dwk);
    mat_out(g.dwv, dwv);
    mat_out(g.dwo, dwo);
    REF_GUARD_END
}

// Prefill rows [0, prompt) with forward_chunk, then generate_step for rows
// [prompt, L). y is L*D. peak_kv receives the cache's peak retained count.
int ref_decode_run(int32_t use_float, uint64_t L, uint64_t D, uint64_t prompt, const double* x,
                   const double* wq, const double* wk, const double* wv, const double* wo,
                   const double* w_score, const ref_cfg* c, double* y, uint64_t* peak_kv) {
    REF_GUARD_BEGIN
    auto run = [&](auto tag) {
        using T = decltype(tag);
        AttnParams<T> params{mat_in<T>(wq, D, D), mat_in<T>(wk, D, D), mat_in<T>(wv, D, D),
                             mat_in<T>(wo, D, D)};
        SparseKvCache<T> cache(to_cfg(c), D, to_scoring(c, w_score, D));
        if (prompt > 0) {
            MatT<T> head = cache.forward_chunk(mat_in<T>(x, prompt, D), params);
            mat_out(head, y);
        }
        for (uint64_t i = prompt; i < L; ++i) {
            std::vector<T> row(D);
            for (size_t cc = 0; cc < D; ++cc) row[cc] = static_cast<T>(x[i * D + cc]);
            std::vector<T> o = generate_step(cache, row, params);
            for (size_t cc = 0; cc < D; ++cc) y[i * D + cc] = static_cast<double>(o[cc]);
        }
        if (peak_kv) *peak_kv = cache.peak_kv();
    };
    if (use_float) run(float{});
    else run(double{});
    REF_GUARD_END
}

// Cache snapshots (SparseKvCache::serialize / deserialize, proj/src/cache.cpp:416-545):
// run rows [0, n) (forward_chunk on [0, prompt), then generate_step), write y
// rows [0, n) and the snapshot payload.
int ref_cache_blob(int32_t use_float, uint64_t n, uint64_t D, uint64_t prompt, const double* x,
                   const double* wq, const double* wk, const double* wv, const double* wo,
                   const double* w_score, const ref_cfg* c, double* y, uint8_t* out, uint64_t cap,
                   uint64_t* used) {
    REF_GUARD_BEGIN
    auto run = [&](auto tag) {
        using T = decltype(tag);
        AttnParams<T> params{mat_in<T>(wq, D, D), mat_in<T>(wk, D, D), mat_in<T>(wv, D, D),
                             mat_in<T>(wo, D, D)};
        SparseKvCache<T> cache(to_cfg(c), D, to_scoring(c, w_score, D));
        if (prompt > 0) mat_out(cache.forward_chunk(mat_in<T>(x, prompt, D), params), y);
        for (uint64_t i = prompt; i < n; ++i) {
            std::vector<T> row(D);
            for (size_t cc = 0; cc < D; ++cc) row[cc] = static_cast<T>(x[i * D + cc]);
            std::vector<T> o = generate_step(cache, row, params);
            for (size_t cc = 0; cc < D; ++cc) y[i * D + cc] = static_cast<double>(o[cc]);
        }
        std::vector<uint8_t> blob;
        cache.serialize(blob);
        *used = blob.size();
        if (out && cap >= blob.size()) std::memcpy(out, blob.data(), blob.size());
    };
    if (use_float) run(float{});
    else run(double{});
    REF_GUARD_END
}

// deserialize a payload and generate_step rows [0, n) of x; y receives their outputs
int ref_cache_resume(int32_t use_float, const uint8_t* blob, uint64_t len, uint64_t n, uint64_t D,
                     const double* x, const double* wq, const double* wk, const double* wv,
                     const double* wo, const double* w_score, const ref_cfg* c, double* y) {
    REF_GUARD_BEGIN
    auto run = [&](auto tag) {
        using T = decltype(tag);
        AttnParams<T> params{mat_in<T>(wq, D, D), mat_in<T>(wk, D, D), mat_in<T>(wv, D, D),
                             mat_in<T>(wo, D, D)};
        SparseKvCache<T> cache =
            SparseKvCache<T>::deserialize(blob, len, to_cfg(c), D, to_scoring(c, w_score, D));
        for (uint64_t i = 0; i < n; ++i) {
            std::vector<T> row(D);
            for (size_t cc = 0; cc < D; ++cc) row[cc] = static_cast<T>(x[i * D + cc]);
            std::vector<T> o = generate_step(cache, row, params);
            for (size_t cc = 0; cc < D; ++cc) y[i * D + cc] = static_cast<double>(o[cc]);
        }
    };
    if (use_float) run(float{});
    else run(double{});
    REF_GUARD_END
}

// Linear-attention mix: linear_mix_attention (attention.hpp:93-99) with a tape,
// then sparsek_attention_backward with the same LinearMixParams (grad_out may
// be null: forward only). feat: heads x p x p row-major; dfeat likewise.
// chunk_len > 0 feeds the rows through one cache chunk by chunk (chunked_forward).
int ref_linmix(int32_t use_float, uint64_t L, uint64_t D, const double* x, const double* wq, const double* wk,
               const double* wv, const double* wo, const double* w_score, const double* feat, const ref_cfg* c,
               uint64_t chunk_len, const double* grad_out, double* y, double* dx, double* dwq, double* dwk,
               double* dwv, double* dwo, double* dws, double* dfeat) {
    REF_GUARD_BEGIN
    auto run = [&](auto tag) {
        using T = decltype(tag);
        const uint64_t H = c->heads, p = D / H;
        AttnParams<T> params{mat_in<T>(wq, D, D), mat_in<T>(wk, D, D), mat_in<T>(wv, D, D), mat_in<T>(wo, D, D)};
        ScoringParams scoring = to_scoring(c, w_score, D);
        LinearMixParams<T> lin;
        for (uint64_t h = 0; h < H; ++h) lin.feat.push_back(mat_in<T>(feat + h * p * p, p, p));
        AttnConfig cfg = to_cfg(c);
        cfg.linear_mix = true;
        AttnTape<T> tape;
        MatT<T> out;
        if (chunk_len == 0) {
            out = linear_mix_attention(mat_in<T>(x, L, D), params, scoring, cfg, lin, &tape);
        } else {
            out = chunked_forward(mat_in<T>(x, L, D), chunk_len, params, scoring, cfg, &tape, &lin);
        }
        mat_out(out, y);
        if (!grad_out) return;
        AttnGrads<T> g = sparsek_attention_backward(tape, mat_in<T>(grad_out, L, D), params, scoring, &lin);
        mat_out(g.dx, dx);
        mat_out(g.dwq, dwq);
        mat_out(g.dwk, dwk);
        mat_out(g.dwv, dwv);
        mat_out(g.dwo, dwo);
        for (uint64_t i = 0; i < g.dw_score.size(); ++i) dws[i] = g.dw_score[i];
        for (uint64_t h = 0; h < H; ++h) mat_out(g.dfeat[h], dfeat + h * p * p);
    };
    if (use_float) run(float{});
    else run(double{});
    REF_GUARD_END
}

// Linear-mix decoding: forward_chunk(prompt) then generate_step per row, with
// LinearMixParams (feat: heads x p x p).
int ref_linmix_decode(int32_t use_float, uint64_t L, uint64_t D, uint64_t prompt, const double* x, const double* wq,
                      const double* wk, const double* wv, const double* wo, const double* w_score, const double* feat,
                      const ref_cfg* c, double* y) {
    REF_GUARD_BEGIN
    auto run = [&](auto tag) {
        using T = decltype(tag);
        const uint64_t H = c->heads, p = D / H;
        AttnParams<T> params{mat_in<T>(wq, D, D), mat_in<T>(wk, D, D), mat_in<T>(wv, D, D), mat_in<T>(wo, D, D)};
        LinearMixParams<T> lin;
        for (uint64_t h = 0; h < H; ++h) lin.feat.push_back(mat_in<T>(feat + h * p * p, p, p));
        AttnConfig cfg = to_cfg(c);
        cfg.linear_mix = true;
        SparseKvCache<T> cache(cfg, D, to_scoring(c, w_score, D));
        if (prompt > 0) mat_out(cache.forward_chunk(mat_in<T>(x, prompt, D), params, nullptr, &lin), y);
        for (uint64_t i = prompt; i < L; ++i) {
            std::vector<T> row(D);
            for (size_t cc = 0; cc < D; ++cc) row[cc] = static_cast<T>(x[i * D + cc]);
            std::vector<T> o = generate_step(cache, row, params, &lin);
            for (size_t cc = 0; cc < D; ++cc) y[i * D + cc] = static_cast<double>(o[cc]);
        }
    };
    if (use_float) run(float{});
    else run(double{});
    REF_GUARD_END
}

// CPU baseline: `units` independent single-head sequences (heads=1, D=p) of
// length L, fwd (with tape) + bwd in float, one std::thread per unit with at
// most `threads` in flight, the way the reference trainer fans out batch
// workers (proj/src/trainer.cpp:555-581). Inputs are seeded reference Rng
// draws. Returns wall seconds in *secs.
int ref_bench_units(uint64_t units, uint64_t threads, uint64_t L, uint64_t p, double k,
                    uint64_t window, uint64_t seed, int32_t with_bwd, double* secs) {
    REF_GUARD_BEGIN
    struct Prob {
        MatT<float> x, g;
        AttnParams<float> params;
        ScoringParams scoring;
    };
    std::vector<Prob> probs(units);
    for (uint64_t u = 0; u < units; ++u) {
        Rng rng(seed + 7919 * u);
        Prob& pr = probs[u];
        pr.x = MatT<float>(L, p);
        for (auto& v : pr.x.data) v = static_cast<float>(rng.normal());
        pr.g = MatT<float>(L, p);
        for (auto& v : pr.g.data) v = static_cast<float>(rng.normal());
        const double s = 0.6 / std::sqrt(static_cast<double>(p));
        for (MatT<float>* m : {&pr.params.wq, &pr.params.wk, &pr.params.wv, &pr.params.wo}) {
            *m = MatT<float>(p, p);
            for (auto& v : m->data) v = static_cast<float>(s * rng.normal());
        }
        pr.scoring.w_score.resize(p);
        for (auto& v : pr.scoring.w_score) v = rng.normal() / std::sqrt(static_cast<double>(p));
    }
    AttnConfig cfg;
    cfg.k = k;
    cfg.window = window;
    cfg.heads = 1;
    std::vector<std::string> errs(units);
    auto work = [&](uint64_t u) {
        try {
            AttnTape<float> tape;
            Prob& pr = probs[u];
            MatT<float> y = sparsek_attention(pr.x, pr.params, pr.scoring, cfg, &tape);
            if (with_bwd) {
                AttnGrads<float> gr = sparsek_attention_backward(tape, pr.g, pr.params, pr.scoring);
                (void)gr;
            }
        } catch (const std::exception& e) {
            errs[u] = e.what();
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t base = 0; base < units; base += threads) {
        std::vector<std::thread> pool;
        for (uint64_t u = base; u < std::min(units, base + threads); ++u) pool.emplace_back(work, u);
        for (auto& th : pool) th.join();
    }
    const auto t1 = std::chrono::steady_clock::now();
    for (auto& e : errs)
        if (!e.empty()) throw NumericError(e);
    *secs = std::chrono::duration<double>(t1 - t0).count();
    REF_GUARD_END
}

// CPU decode baseline: `units` independent single-head caches (heads=1,
// D=p), each prefilled with forward_chunk over `prompt` rows and then timed
// over `steps` generate_step calls (proj/src/cache.cpp:570-577), float, one
// std::thread per unit with at most `threads` in flight. Once the prompt
// exceeds floor(k)+w the per-step work is O(k+w) regardless of the context.
// Returns the wall seconds of the generate_step phase in *secs.
int ref_bench_decode(uint64_t units, uint64_t threads, uint64_t prompt, uint64_t steps, uint64_t p, double k,
                     uint64_t window, uint64_t seed, double* secs) {
    REF_GUARD_BEGIN
    AttnConfig cfg;
    cfg.k = k;
    cfg.window = window;
    cfg.heads = 1;
    struct Unit {
        AttnParams<float> params;
        ScoringParams scoring;
        std::unique_ptr<SparseKvCache<float>> cache;
        std::vector<std::vector<float>> rows;
    };
    std::vector<Unit> us(units);
    std::vector<std::string> errs(units);
    auto prep = [&](uint64_t u) {
        try {
            Rng rng(seed + 104729 * u);
            Unit& un = us[u];
            const double s = 0.6 / std::sqrt(static_cast<double>(p));
            for (MatT<float>* m : {&un.params.wq, &un.params.wk, &un.params.wv, &un.params.wo}) {
                *m = MatT<float>(p, p);
                for (auto& v : m->data) v = static_cast<float>(s * rng.normal());
            }
            un.scoring.w_score.resize(p);
            for (auto& v : un.scoring.w_score) v = rng.normal() / std::sqrt(static_cast<double>(p));
            MatT<float> x(prompt, p);
            for (auto& v : x.data) v = static_cast<float>(rng.normal());
            un.cache = std::make_unique<SparseKvCache<float>>(cfg, p, un.scoring);
            (void)un.cache->forward_chunk(x, un.params);
            un.rows.assign(steps, std::vector<float>(p));
            for (auto& r : un.rows)
                for (auto& v : r) v = static_cast<float>(rng.normal());
        } catch (const std::exception& e) {
            errs[u] = e.what();
        }
    };
    auto work = [&](uint64_t u) {
        try {
            Unit& un = us[u];
            for (uint64_t i = 0; i < steps; ++i) (void)generate_step(*un.cache, un.rows[i], un.params);
        } catch (const std::exception& e) {
            errs[u] = e.what();
        }
    };
    auto fan = [&](auto fn) {
        for (uint64_t base = 0; base < units; base += threads) {
            std::vector<std::thread> pool;
            for (uint64_t u = base; u < std::min(units, base + threads); ++u) pool.emplace_back(fn, u);
            for (auto& th : pool) th.join();
        }
    };
    fan(prep);
    for (auto& e : errs)
        if (!e.empty()) throw NumericError(e);
    const auto t0 = std::chrono::steady_clock::now();
    fan(work);
    const auto t1 = std::chrono::steady_clock::now();
    for (auto& e : errs)
        if (!e.empty()) throw NumericError(e);
    *secs = std::chrono::duration<double>(t1 - t0).count();
    REF_GUARD_END
}

}  // extern "C"
