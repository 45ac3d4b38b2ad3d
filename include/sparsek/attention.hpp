// sparsek/attention.hpp — drop-in for proj/include/sparsek/attention.hpp:12-115.
//
// sparsek_attention<T> / sparsek_attention_backward<T> run on the GPU through
// skb_xattn_* (include/sparsek_b200.h): projections as library GEMMs, then K1
// scoring, K2 selection, K3 attention (K4 + JVP + K1 backward for the
// gradients). The AttnTape keeps the reference's fields (filled from the
// device after the forward) plus `device`, the device-resident state the
// backward reads; a tape without it (built by hand) is re-run from tape.x.
// Softmax statistics: the kernels keep lse = maxa + log(denom) per
// (query, head); QueryRec reports maxa = lse and denom = 1, the same softmax.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

#include "sparsek/detail/device.hpp"
#include "sparsek/numerics.hpp"
#include "sparsek/selection.hpp"

namespace sparsek {

enum class KeyMode { soft, hard };
enum class ValueMode { soft };
enum class MaskApply { soft, straight_through };

struct AttnConfig {
    double k = 8.0;
    std::size_t window = 8;
    std::size_t heads = 1;
    double scale = 0.0;
    KeyMode key_mode = KeyMode::hard;
    ValueMode value_mode = ValueMode::soft;
    MaskApply mask_mode = MaskApply::soft;
    std::size_t group_size = 128;  // blocked query execution; never changes results
    bool linear_mix = false;

    std::size_t head_dim(std::size_t d_model) const { return d_model / heads; }
    double effective_scale(std::size_t d_model) const {
        return scale > 0.0 ? scale : 1.0 / std::sqrt(static_cast<double>(head_dim(d_model)));
    }
    void validate(std::size_t d_model, const ScoringParams& scoring) const {  // attention.cpp:15-35
        if (heads == 0) throw ConfigError("attention: heads must be positive");
        if (d_model == 0 || d_model % heads != 0)
            throw ConfigError("attention: d_model must be a positive multiple of heads");
        if (!std::isfinite(k) || k < 0.0) throw ConfigError("attention: k must be finite and >= 0");
        if (!std::isfinite(scale) || scale < 0.0) throw ConfigError("attention: bad scale");
        if (group_size == 0) throw ConfigError("attention: group_size must be positive");
        if (linear_mix) {
            if (scoring.norm_mode != NormMode::timestep_norm)
                throw ConfigError(
                    "linear mix requires timestep normalization; raw scores make the linear branch blow up");
        } else if (window == 0 && std::floor(k) < 1.0) {
            throw ConfigError("attention: window + floor(k) must be >= 1 (only the linear mix can run with neither)");
        }
        if (k > 0.0 && scoring.w_score.size() != d_model)
            throw ConfigError("attention: w_score length must equal d_model");
        scoring.validate();
    }
};

template <class T>
struct AttnParams {
    MatT<T> wq, wk, wv, wo;
};

template <class T>
struct LinearMixParams {
    std::vector<MatT<T>> feat;
};

template <class T>
struct AttnTape {
    MatT<T> x, q, k, v;
    MatT<T> head_concat;
    std::vector<double> raw;
    std::vector<double> u;
    std::vector<double> norm_mean;
    std::vector<double> norm_sdev;
    std::vector<double> tau_push;
    struct QueryRec {
        std::uint32_t n_sel = 0;
        std::vector<std::uint32_t> att;
        std::vector<double> gate;
        std::vector<T> maxa;
        std::vector<T> denom;
    };
    std::vector<QueryRec> queries;
    std::vector<std::size_t> chunk_starts;
    AttnConfig cfg;
    std::size_t d_model = 0;
    // B200: the forward's device state (projections, scores, selection, lse)
    std::shared_ptr<skb_xattn> device;
};

template <class T>
struct AttnGrads {
    MatT<T> dx, dwq, dwk, dwv, dwo;
    std::vector<double> dw_score;
    std::vector<MatT<T>> dfeat;
};

namespace detail {

template <class T>
skb_x_desc x_desc(std::size_t L, std::size_t D, const AttnConfig& cfg, const ScoringParams& sc,
                  std::size_t chunk_len = 0) {
    skb_x_desc d{};
    d.batch = 1;
    d.seq_len = (int64_t)L;
    d.d_model = (int64_t)D;
    d.heads = (int64_t)cfg.heads;
    d.k = cfg.k;
    d.window = (int64_t)cfg.window;
    d.scale = cfg.scale;
    d.key_mode = cfg.key_mode == KeyMode::soft ? 1 : 0;
    d.mask_mode = cfg.mask_mode == MaskApply::straight_through ? 1 : 0;
    d.dtype = dtype_of<T>();
    d.flags = 0;
    d.chunk_len = (int64_t)chunk_len;
    d.scoring = to_c(sc);
    return d;
}

template <class T>
struct DeviceParams {
    Buf wq, wk, wv, wo, ws;
    DeviceParams(const AttnParams<T>& p, const ScoringParams& sc)
        : wq(p.wq.data), wk(p.wk.data), wv(p.wv.data), wo(p.wo.data), ws(sc.w_score) {}
};

template <class T>
void check_params(const AttnParams<T>& p, std::size_t D) {
    for (const MatT<T>* w : {&p.wq, &p.wk, &p.wv, &p.wo})
        if (w->rows != D || w->cols != D) throw ShapeError("forward_chunk: projection shapes must be d_model x d_model");
}

template <class T>
MatT<T> mat_from_device(skb_xattn* t, int field, std::size_t rows, std::size_t cols) {
    MatT<T> m(rows, cols);
    if (!m.data.empty()) check(skb_xattn_tape_get(t, field, m.data.data(), m.data.size() * sizeof(T), nullptr));
    return m;
}
inline std::vector<double> vec_from_device(skb_xattn* t, int field, std::size_t n) {
    std::vector<double> v(n);
    if (n) check(skb_xattn_tape_get(t, field, v.data(), n * 8, nullptr));
    return v;
}

// The reference tape's fields from the device state (cache.cpp:240-392's records).
template <class T>
void fill_tape(AttnTape<T>& tape, std::shared_ptr<skb_xattn> dev, std::size_t L, std::size_t D,
               const AttnConfig& cfg, std::size_t chunk_len) {
    tape.device = dev;
    tape.cfg = cfg;
    tape.d_model = D;
    skb_xattn* t = dev.get();
    tape.x = mat_from_device<T>(t, SKB_TAPE_X, L, D);
    tape.q = mat_from_device<T>(t, SKB_TAPE_Q, L, D);
    tape.k = mat_from_device<T>(t, SKB_TAPE_K, L, D);
    tape.v = mat_from_device<T>(t, SKB_TAPE_V, L, D);
    tape.head_concat = mat_from_device<T>(t, SKB_TAPE_HEAD_CONCAT, L, D);
    tape.raw = vec_from_device(t, SKB_TAPE_RAW, L);
    tape.u = vec_from_device(t, SKB_TAPE_U, L);
    tape.norm_mean = vec_from_device(t, SKB_TAPE_NORM_MEAN, L);
    tape.norm_sdev = vec_from_device(t, SKB_TAPE_NORM_SDEV, L);
    const std::size_t H = cfg.heads, w = cfg.window;
    const std::vector<double> lse = vec_from_device(t, SKB_TAPE_LSE, H * L);
    const std::size_t T_ = L > w ? L - w : 0;
    const bool sel_on = std::floor(cfg.k) >= 1.0;
    std::vector<double> tau(L, kNegInf);
    std::vector<int32_t> leave(L, 0);
    if (sel_on) {
        check(skb_xattn_tape_get(t, SKB_TAPE_TAU_PUSH, tau.data(), L * 8, nullptr));
        check(skb_xattn_tape_get(t, SKB_TAPE_LEAVE, leave.data(), L * 4, nullptr));
    }
    tape.tau_push.assign(tau.begin(), tau.begin() + (cfg.k > 0.0 ? T_ : 0));
    tape.queries.assign(L, {});
    // the reference's snapshot per query: selected ascending, then the window
    // ascending (self when w = 0 and unselected), gates of the selected
    for (std::size_t i = 0; i < L; ++i) {
        auto& q = tape.queries[i];
        if (sel_on && i >= w) {
            const std::size_t tt = i - w;
            for (std::size_t j = 0; j <= tt; ++j)
                if ((std::size_t)leave[j] > tt) {
                    q.att.push_back((std::uint32_t)j);
                    double g = tape.u[j] - tau[tt];
                    q.gate.push_back(g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g));
                }
        }
        q.n_sel = (std::uint32_t)q.att.size();
        if (w > 0) {
            for (std::size_t j = i + 1 > w ? i + 1 - w : 0; j <= i; ++j) q.att.push_back((std::uint32_t)j);
        } else if (std::find(q.att.begin(), q.att.end(), (std::uint32_t)i) == q.att.end()) {
            q.att.push_back((std::uint32_t)i);
        }
        q.maxa.resize(H);
        q.denom.assign(H, T(1));
        for (std::size_t h = 0; h < H; ++h) q.maxa[h] = static_cast<T>(lse[h * L + i]);
    }
    const std::size_t cl = chunk_len ? chunk_len : std::max<std::size_t>(L, 1);
    tape.chunk_starts.clear();
    for (std::size_t s = 0; s < L; s += cl) tape.chunk_starts.push_back(s);
}

// LinearMixParams as one float64 [H, p, p] device block (the C ABI's feat).
template <class T>
std::vector<double> pack_feat(const LinearMixParams<T>& lin, std::size_t heads, std::size_t p) {
    if (lin.feat.size() != heads) throw ShapeError("forward_chunk: one feature map per head");
    std::vector<double> out;
    out.reserve(heads * p * p);
    for (const auto& f : lin.feat) {
        if (f.rows != p || f.cols != p) throw ShapeError("forward_chunk: feature maps are head_dim x head_dim");
        for (T v : f.data) out.push_back(static_cast<double>(v));
    }
    return out;
}

template <class T>
MatT<T> run_forward(const MatT<T>& x, const AttnParams<T>& params, const ScoringParams& scoring,
                    const AttnConfig& cfg, AttnTape<T>* tape, std::size_t chunk_len,
                    const LinearMixParams<T>* lin = nullptr) {
    cfg.validate(x.cols, scoring);
    if (cfg.linear_mix && !lin) throw ConfigError("forward_chunk: linear mix needs feature parameters");
    check_params(params, x.cols);
    const std::size_t L = x.rows, D = x.cols;
    std::vector<double> feat;
    if (cfg.linear_mix) feat = pack_feat(*lin, cfg.heads, D / cfg.heads);
    MatT<T> y(L, D);
    if (L == 0) return y;
    skb_x_desc d = x_desc<T>(L, D, cfg, scoring, chunk_len);
    DeviceParams<T> dp(params, scoring);
    Buf dx(x.data), dy(y.data.size() * sizeof(T));
    skb_xattn* t = nullptr;
    if (cfg.linear_mix) {  // Appendix B.1 (proj/src/cache.cpp:322-356)
        d.flags |= SKB_FLAG_LINEAR_MIX;
        Buf df(feat);
        check(skb_xattn_forward_lin(&d, dx.get(), dp.wq.get(), dp.wk.get(), dp.wv.get(), dp.wo.get(),
                                    cfg.k > 0.0 ? dp.ws.template as<double>() : nullptr, df.template as<double>(),
                                    dy.get(), tape ? &t : nullptr, nullptr));
    } else {
        check(skb_xattn_forward(&d, dx.get(), dp.wq.get(), dp.wk.get(), dp.wv.get(), dp.wo.get(),
                                cfg.k > 0.0 ? dp.ws.template as<double>() : nullptr, dy.get(), tape ? &t : nullptr,
                                nullptr));
    }
    y.data = dy.to_host<T>(y.data.size());
    if (tape) fill_tape(*tape, std::shared_ptr<skb_xattn>(t, skb_xattn_destroy), L, D, cfg, chunk_len);
    return y;
}

}  // namespace detail

template <class T>
MatT<T> sparsek_attention(const MatT<T>& x, const AttnParams<T>& params, const ScoringParams& scoring,
                          const AttnConfig& cfg, AttnTape<T>* tape = nullptr, const LinearMixParams<T>* lin = nullptr) {
    return detail::run_forward(x, params, scoring, cfg, tape, 0, lin);
}

template <class T>
AttnGrads<T> sparsek_attention_backward(const AttnTape<T>& tape, const MatT<T>& grad_out, const AttnParams<T>& params,
                                        const ScoringParams& scoring, const LinearMixParams<T>* lin = nullptr) {
    if (tape.cfg.linear_mix && !lin) throw ConfigError("backward: linear mix needs feature parameters");
    const std::size_t L = tape.x.rows, D = tape.d_model ? tape.d_model : tape.x.cols;
    if (grad_out.rows != L || grad_out.cols != D) throw ShapeError("sparsek_attention_backward: grad_out shape");
    detail::check_params(params, D);
    std::shared_ptr<skb_xattn> dev = tape.device;
    const std::size_t chunk_len = tape.chunk_starts.size() > 1 ? tape.chunk_starts[1] - tape.chunk_starts[0] : 0;
    if (!dev) {  // a tape assembled on the host: re-run the forward from its inputs
        AttnTape<T> t2;
        detail::run_forward(tape.x, params, scoring, tape.cfg, &t2, chunk_len, tape.cfg.linear_mix ? lin : nullptr);
        dev = t2.device;
    }
    AttnGrads<T> g;
    g.dx = MatT<T>(L, D);
    g.dwq = MatT<T>(D, D);
    g.dwk = MatT<T>(D, D);
    g.dwv = MatT<T>(D, D);
    g.dwo = MatT<T>(D, D);
    g.dw_score.assign(D, 0.0);
    if (L == 0) return g;
    detail::DeviceParams<T> dp(params, scoring);
    detail::Buf dgo(grad_out.data), ddx(L * D * sizeof(T)), dq(D * D * sizeof(T)), dk(D * D * sizeof(T)),
        dv(D * D * sizeof(T)), dwo(D * D * sizeof(T)), dws(D * 8);
    const std::size_t H = tape.cfg.heads, p = D / H;
    if (tape.cfg.linear_mix) {  // attention.cpp:317-445, 519-549 (+ dfeat)
        detail::Buf df(detail::pack_feat(*lin, H, p)), ddf(H * p * p * 8);
        detail::check(skb_xattn_backward_lin(dev.get(), dgo.get(), dp.wq.get(), dp.wk.get(), dp.wv.get(),
                                             dp.wo.get(), tape.cfg.k > 0.0 ? dp.ws.template as<double>() : nullptr,
                                             df.template as<double>(), ddx.get(), dq.get(), dk.get(), dv.get(),
                                             dwo.get(), dws.as<double>(), ddf.as<double>(), nullptr));
        const std::vector<double> hf = ddf.to_host<double>(H * p * p);
        g.dfeat.assign(H, MatT<T>(p, p));
        for (std::size_t h = 0; h < H; ++h)
            for (std::size_t e = 0; e < p * p; ++e) g.dfeat[h].data[e] = static_cast<T>(hf[h * p * p + e]);
    } else {
        detail::check(skb_xattn_backward(dev.get(), dgo.get(), dp.wq.get(), dp.wk.get(), dp.wv.get(), dp.wo.get(),
                                         tape.cfg.k > 0.0 ? dp.ws.template as<double>() : nullptr, ddx.get(),
                                         dq.get(), dk.get(), dv.get(), dwo.get(), dws.as<double>(), nullptr));
    }
    g.dx.data = ddx.to_host<T>(L * D);
    g.dwq.data = dq.to_host<T>(D * D);
    g.dwk.data = dk.to_host<T>(D * D);
    g.dwv.data = dv.to_host<T>(D * D);
    g.dwo.data = dwo.to_host<T>(D * D);
    g.dw_score = dws.to_host<double>(D);
    return g;
}

template <class T>
MatT<T> linear_mix_attention(const MatT<T>& x, const AttnParams<T>& params, const ScoringParams& scoring,
                             const AttnConfig& cfg, const LinearMixParams<T>& lin, AttnTape<T>* tape = nullptr) {
    AttnConfig c = cfg;
    c.linear_mix = true;
    return sparsek_attention(x, params, scoring, c, tape, &lin);
}

template <class T>
MatT<T> multi_head(const std::vector<MatT<T>>& head_outputs, const MatT<T>& wo) {
    if (head_outputs.empty()) throw ArgumentError("multi_head: no heads");
    const std::size_t n = head_outputs[0].rows;
    std::size_t d = 0;
    for (const auto& h : head_outputs) {
        if (h.rows != n) throw ShapeError("multi_head: row count mismatch");
        d += h.cols;
    }
    if (wo.rows != d) throw ShapeError("multi_head: wo rows must equal concatenated width");
    MatT<T> concat(n, d);
    for (std::size_t i = 0; i < n; ++i) {
        std::size_t off = 0;
        for (const auto& h : head_outputs) {
            std::copy(h.row(i), h.row(i) + h.cols, concat.row(i) + off);
            off += h.cols;
        }
    }
    return matmul(concat, wo);
}

namespace detail {
// dense causal attention = the SparseK kernels with a budget above every
// prefix (tau = -inf, all gates 1) and idle scores
inline AttnConfig dense_cfg(std::size_t L, double scale, std::size_t heads) {
    AttnConfig c;
    c.k = static_cast<double>(L + 1);
    c.window = 1;
    c.heads = heads;
    c.scale = scale;
    return c;
}
inline ScoringParams dense_scoring(std::size_t D) {
    ScoringParams s;
    s.w_score.assign(D, 0.0);
    s.slope_enabled = false;
    s.norm_mode = NormMode::none;
    return s;
}
}  // namespace detail

template <class T>
MatT<T> dense_causal_attention(const MatT<T>& x, const AttnParams<T>& params, double scale, std::size_t heads = 1,
                               MatT<T>* head_concat_out = nullptr) {
    AttnTape<T> tape;
    MatT<T> y = detail::run_forward(x, params, detail::dense_scoring(x.cols), detail::dense_cfg(x.rows, scale, heads),
                                    head_concat_out ? &tape : nullptr, 0);
    if (head_concat_out) *head_concat_out = tape.head_concat;
    return y;
}

template <class T>
AttnGrads<T> dense_causal_attention_backward(const MatT<T>& x, const AttnParams<T>& params, double scale,
                                             std::size_t heads, const MatT<T>& head_concat, const MatT<T>& grad_out) {
    (void)head_concat;  // recomputed on the device with the forward's state
    const ScoringParams sc = detail::dense_scoring(x.cols);
    AttnTape<T> tape;
    detail::run_forward(x, params, sc, detail::dense_cfg(x.rows, scale, heads), &tape, 0);
    AttnGrads<T> g = sparsek_attention_backward(tape, grad_out, params, sc);
    g.dw_score.clear();
    return g;
}

}  // namespace sparsek
