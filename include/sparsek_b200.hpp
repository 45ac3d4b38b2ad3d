// sparsek_b200.hpp — the reference's C++ operator surface over the C ABI.
//
// Header-only C++17 layer above include/sparsek_b200.h that mirrors the names,
// argument meaning and error behaviour of the reference's operator API
// (proj/include/sparsek/{sparsek_op,stream,attention,cache}.hpp) for callers
// that hold device buffers:
//
//   reference (CPU, proj/include/sparsek/...)      here (B200, device buffers)
//   ---------------------------------------------  -----------------------------------------
//   ShapeError/ArgumentError/ConfigError/          same names; thrown from the C-ABI status
//     NumericError/IoError (common.hpp:9-25)         (+ CudaError for runtime failures)
//   AttnConfig, KeyMode, MaskApply                 same fields (attention.hpp:12-32)
//   sparsek(z, KBudget) (sparsek_op.hpp:47)        sparsek(z, k) -> SparseKSolution
//   sparsek_jvp (sparsek_op.hpp:60)                sparsek_jvp(z, k, v)
//   topk_hard (sparsek_op.hpp:63)                  topk_hard(z, k)
//   StreamState (stream.hpp:26-72)                 StreamState: push / tau / t / survivor_count
//   sparsek_attention fwd core (attention.hpp:81)  SparseKAttention::forward  (q,k,v,u -> o, lse)
//   sparsek_attention_backward (attention.hpp:87)  SparseKAttention::backward (-> dq,dk,dv,du)
//   SparseKvCache + generate_step (cache.hpp)      SparseKvCache::prefill / step / retained_positions
//
// The x-level projections (x*Wq etc.) are plain GEMMs left to the caller's
// BLAS; everything else runs in libsparsek_b200.so. There is no CPU fallback.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparsek_b200.h"

namespace sparsek_b200 {

// ------------------------------------------------------------------ errors
struct ShapeError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct ArgumentError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct ConfigError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct NumericError : std::domain_error {
    using std::domain_error::domain_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == SKB_OK) return;
    const std::string msg = skb_last_error();
    switch (rc) {
        case SKB_ESHAPE: throw ShapeError(msg);
        case SKB_EARG: throw ArgumentError(msg);
        case SKB_ENUMERIC: throw NumericError(msg);
        case SKB_ECONFIG: throw ConfigError(msg);
        case SKB_EIO: throw IoError(msg);
        default: throw CudaError(msg);
    }
}
inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device allocation
class DeviceBuffer {
  public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t bytes) : bytes_(bytes) {
        if (bytes) cuda_check(cudaMalloc(&p_, bytes), "cudaMalloc");
    }
    ~DeviceBuffer() {
        if (p_) cudaFree(p_);
    }
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), bytes_(o.bytes_) {
        o.p_ = nullptr;
        o.bytes_ = 0;
    }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(bytes_, o.bytes_);
        return *this;
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    void* get() const { return p_; }
    size_t size() const { return bytes_; }

  private:
    void* p_ = nullptr;
    size_t bytes_ = 0;
};

// ------------------------------------------------------------------ config
enum class KeyMode { soft, hard };                   // attention.hpp:12
enum class MaskApply { soft, straight_through };     // attention.hpp:14
enum class DType { f32 = SKB_F32, bf16 = SKB_BF16, f64 = SKB_F64 };

struct AttnConfig {  // attention.hpp:18-32 (group_size / linear_mix are CPU-only knobs)
    double k = 8.0;
    size_t window = 8;
    size_t heads = 1;
    double scale = 0.0;  // 0 -> 1/sqrt(head_dim)
    KeyMode key_mode = KeyMode::hard;
    MaskApply mask_mode = MaskApply::soft;
    size_t chunk_len = 0;  // chunked_forward (cache.hpp:93-96): backward stop-grad at chunk starts
};

inline skb_attn_desc make_desc(int64_t batch, int64_t seq_len, int64_t head_dim, const AttnConfig& c, DType dt,
                               uint32_t flags = 0) {
    skb_attn_desc d{};
    d.batch = batch;
    d.seq_len = seq_len;
    d.heads = (int64_t)c.heads;
    d.head_dim = head_dim;
    d.k = c.k;
    d.window = (int64_t)c.window;
    d.scale = c.scale;
    d.key_mode = c.key_mode == KeyMode::soft ? 1 : 0;
    d.mask_mode = c.mask_mode == MaskApply::straight_through ? 1 : 0;
    d.dtype = (int32_t)dt;
    d.flags = flags;
    d.chunk_len = (int64_t)c.chunk_len;
    return d;
}

// ------------------------------------------------------------------ operator
struct SparseKSolution {  // sparsek_op.hpp:22-38 (dense p; tau = -inf when infeasible)
    std::vector<double> p;
    double tau = -INFINITY;
    size_t u_count = 0, w_count = 0;
    bool degenerate = false, infeasible = false;
};

// Batched rows on the device; this host-vector form mirrors the reference call.
inline SparseKSolution sparsek(const std::vector<double>& z, double k, cudaStream_t st = nullptr) {
    if (z.empty()) throw ArgumentError("sparsek: empty input");
    if (!(k > 0.0) || !std::isfinite(k)) throw ArgumentError("KBudget: k must be positive and finite");
    for (double x : z)
        if (!std::isfinite(x)) throw NumericError("sparsek: non-finite input");
    const int64_t m = (int64_t)z.size();
    DeviceBuffer dz(m * 8), dp(m * 8), dt(8), du(8), dw(8), df(4);
    cuda_check(cudaMemcpyAsync(dz.get(), z.data(), m * 8, cudaMemcpyHostToDevice, st), "H2D");
    check(skb_sparsek(1, m, (const double*)dz.get(), k, (double*)dp.get(), (double*)dt.get(), (int64_t*)du.get(),
                      (int64_t*)dw.get(), (int32_t*)df.get(), st));
    SparseKSolution s;
    s.p.resize(m);
    int64_t uc = 0, wc = 0;
    int32_t fl = 0;
    cuda_check(cudaMemcpyAsync(s.p.data(), dp.get(), m * 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(&s.tau, dt.get(), 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(&uc, du.get(), 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(&wc, dw.get(), 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(&fl, df.get(), 4, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    s.u_count = (size_t)uc;
    s.w_count = (size_t)wc;
    s.degenerate = fl & 1;
    s.infeasible = (fl & 2) != 0;
    return s;
}

inline std::vector<double> sparsek_jvp(const std::vector<double>& z, double k, const std::vector<double>& v,
                                       cudaStream_t st = nullptr) {
    if (v.size() != z.size()) throw ShapeError("sparsek_jvp: v must match z");
    const int64_t m = (int64_t)z.size();
    DeviceBuffer dz(m * 8), dv(m * 8), dout(m * 8);
    cuda_check(cudaMemcpyAsync(dz.get(), z.data(), m * 8, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(dv.get(), v.data(), m * 8, cudaMemcpyHostToDevice, st), "H2D");
    check(skb_sparsek_jvp(1, m, (const double*)dz.get(), k, (const double*)dv.get(), (double*)dout.get(), st));
    std::vector<double> out(m);
    cuda_check(cudaMemcpyAsync(out.data(), dout.get(), m * 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    return out;
}

inline std::vector<double> topk_hard(const std::vector<double>& z, int64_t k, cudaStream_t st = nullptr) {
    const int64_t m = (int64_t)z.size();
    DeviceBuffer dz(m * 8), dout(m * 8);
    cuda_check(cudaMemcpyAsync(dz.get(), z.data(), m * 8, cudaMemcpyHostToDevice, st), "H2D");
    check(skb_topk_hard(1, m, (const double*)dz.get(), k, (double*)dout.get(), st));
    std::vector<double> out(m);
    cuda_check(cudaMemcpyAsync(out.data(), dout.get(), m * 8, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
    return out;
}

// ------------------------------------------------------------------ stream
class StreamState {  // stream.hpp:26-72
  public:
    explicit StreamState(double k, int64_t heap_cap = 0, int64_t capacity = 1 << 16) {
        check(skb_stream_create(k, heap_cap, capacity, &s_));
        dz_ = DeviceBuffer(8);
        dtau_ = DeviceBuffer(8);
        dins_ = DeviceBuffer(1);
    }
    ~StreamState() { skb_stream_destroy(s_); }
    StreamState(const StreamState&) = delete;
    StreamState& operator=(const StreamState&) = delete;

    struct StepResult {  // StreamStepResult (stream.hpp:12-18), evicted list omitted
        double tau;
        int64_t t;
        bool inserted;
    };
    StepResult push(double z, cudaStream_t st = nullptr) {
        if (!std::isfinite(z)) throw NumericError("stream_push: non-finite value");
        cuda_check(cudaMemcpyAsync(dz_.get(), &z, 8, cudaMemcpyHostToDevice, st), "H2D");
        check(skb_stream_push(s_, (const double*)dz_.get(), 1, (double*)dtau_.get(), (uint8_t*)dins_.get(), st));
        StepResult r{};
        uint8_t ins = 0;
        cuda_check(cudaMemcpyAsync(&r.tau, dtau_.get(), 8, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaMemcpyAsync(&ins, dins_.get(), 1, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "sync");
        r.inserted = ins != 0;
        r.t = info(st).t;
        return r;
    }
    skb_stream_info info(cudaStream_t st = nullptr) const {
        skb_stream_info i{};
        check(skb_stream_query(s_, &i, st));
        return i;
    }
    double tau() const { return info().tau; }
    int64_t t() const { return info().t; }
    int64_t survivor_count() const { return info().survivors; }

  private:
    skb_stream* s_ = nullptr;
    DeviceBuffer dz_, dtau_, dins_;
};

// ------------------------------------------------------------------ attention core
// q/k/v/o/do/dq/dk/dv: [B, L, H, p] device buffers of `dtype`; u: float64 [B, L].
class SparseKAttention {
  public:
    SparseKAttention(int64_t batch, int64_t seq_len, int64_t head_dim, const AttnConfig& cfg, DType dtype)
        : d_(make_desc(batch, seq_len, head_dim, cfg, dtype)) {
        check(skb_select_layout_of(&d_, &lay_));  // validates the config (ConfigError before compute)
        sel_ = DeviceBuffer(lay_.total_bytes);
        size_t ws = 0;
        check(skb_attn_bwd_workspace_size(&d_, &ws));
        bws_ = DeviceBuffer(ws);
    }
    // selection (K2) + forward (K3); lse: float64 [B, H, L]
    void forward(const void* q, const void* k, const void* v, const double* u, void* o, double* lse,
                 cudaStream_t st = nullptr) {
        check(skb_select(&d_, u, sel_.get(), st));
        check(skb_attn_fwd(&d_, q, k, v, u, sel_.get(), o, lse, st));
    }
    // backward (K4) + selection pullback; du: float64 [B, L]. Uses the selection of the last forward.
    void backward(const void* q, const void* k, const void* v, const void* o, const void* dout, const double* lse,
                  const double* u, void* dq, void* dk, void* dv, double* du, cudaStream_t st = nullptr) {
        check(skb_attn_bwd(&d_, q, k, v, o, dout, lse, u, sel_.get(), dq, dk, dv, du, bws_.get(), st));
    }
    const skb_select_layout& selection_layout() const { return lay_; }
    const void* selection_workspace() const { return sel_.get(); }

  private:
    skb_attn_desc d_;
    skb_select_layout lay_{};
    DeviceBuffer sel_, bws_;
};

// ------------------------------------------------------------------ scoring
// ScoringParams minus w_score (selection.hpp:19-27).
struct ScoringConfig {
    bool timestep_norm = true;
    bool norm_then_slope = true;
    bool slope_enabled = true;
    double slope_eps = 0.01;
    skb_scoring c(int32_t chunk_len = 0) const {
        skb_scoring s{};
        s.norm_mode = timestep_norm ? 1 : 0;
        s.slope_order = norm_then_slope ? 1 : 0;
        s.slope_enabled = slope_enabled ? 1 : 0;
        s.chunk_len = chunk_len;
        s.slope_eps = slope_eps;
        return s;
    }
};

// score_tokens with a carried TimestepNormState (selection.hpp:55-56,
// selection.cpp:13-31) for B sequences: the float64 state {count, mean, m2}
// per sequence lives on the device and advances with every call.
class ScoreState {
  public:
    ScoreState(int64_t batch, int64_t d_model, const ScoringConfig& sc)
        : B_(batch), D_(d_model), sc_(sc), state_(batch * 3 * sizeof(double)) {
        cuda_check(cudaMemset(state_.get(), 0, batch * 3 * sizeof(double)), "cudaMemset");
    }
    // x [B, n, D] of `dtype`, w_score float64 [D] -> raw/u float64 [B, n] (device buffers)
    void score(const void* x, DType dtype, int64_t n, const double* w_score, double* raw, double* u,
               cudaStream_t st = nullptr) {
        const skb_scoring c = sc_.c();
        check(skb_score_continue(B_, n, D_, (int32_t)dtype, x, w_score, &c, static_cast<double*>(state_.get()), raw,
                                 u, st));
    }

  private:
    int64_t B_, D_;
    ScoringConfig sc_;
    DeviceBuffer state_;
};

// ------------------------------------------------------------------ decode cache
class SparseKvCache {  // cache.hpp:21-87 + generate_step (cache.cpp:570-577)
  public:
    SparseKvCache(int64_t batch, int64_t max_positions, int64_t head_dim, const AttnConfig& cfg, DType dtype) {
        const skb_attn_desc d = make_desc(batch, max_positions, head_dim, cfg, dtype);
        check(skb_cache_create(&d, &c_));
        cap_ = (size_t)(cfg.k > 0 ? std::floor(cfg.k) : 0);
        window_ = cfg.window;
    }
    ~SparseKvCache() { skb_cache_destroy(c_); }
    SparseKvCache(const SparseKvCache&) = delete;
    SparseKvCache& operator=(const SparseKvCache&) = delete;

    // k/v [B, n, H, p], u [B, n]
    void prefill(const void* k, const void* v, const double* u, int64_t n, cudaStream_t st = nullptr) {
        check(skb_cache_prefill(c_, k, v, u, n, st));
    }
    // one decode step (generate_step): q/k/v [B, H, p], u [B] -> o [B, H, p]
    void step(const void* q, const void* k, const void* v, const double* u, void* o, cudaStream_t st = nullptr) {
        check(skb_cache_step(c_, q, k, v, u, o, st));
    }
    std::vector<int32_t> retained_positions(int64_t b, cudaStream_t st = nullptr) const {
        std::vector<int32_t> pos(cap_ + window_ + 1);
        int64_t n = 0, seen = 0, peak = 0;
        double tau = 0;
        check(skb_cache_state(c_, b, pos.data(), &n, &tau, &seen, &peak, st));
        pos.resize((size_t)n);
        return pos;
    }
    size_t capacity() const { return cap_; }
    // SparseKvCache<T>::serialize / deserialize (cache.cpp:416-545) of sequence b;
    // norm = the TimestepNormState {count, mean, m2} of the scoring feeding this cache
    std::vector<uint8_t> serialize(int64_t b, const double* norm = nullptr, cudaStream_t st = nullptr) const {
        size_t n = 0;
        check(skb_cache_snapshot(c_, b, norm, nullptr, &n, st));
        std::vector<uint8_t> out(n);
        check(skb_cache_snapshot(c_, b, norm, out.data(), &n, st));
        out.resize(n);
        return out;
    }
    void deserialize(int64_t b, const std::vector<uint8_t>& blob, double* norm_out = nullptr,
                     cudaStream_t st = nullptr) {
        check(skb_cache_restore(c_, b, blob.data(), blob.size(), norm_out, st));
    }

  private:
    skb_cache* c_ = nullptr;
    size_t cap_ = 0, window_ = 0;
};

}  // namespace sparsek_b200
