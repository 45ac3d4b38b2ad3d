// x-level SparseK attention: sparsek_attention<T> with its tape, and
// sparsek_attention_backward<T> (proj/include/sparsek/attention.hpp:47-91,
// proj/src/attention.cpp:37-43,214-575), plus the x-level recurrent cache
// (SparseKvCache<T>::forward_chunk / generate_step, proj/include/sparsek/
// cache.hpp:21-102, proj/src/cache.cpp:181-400,570-577) — the entry points the
// C++ drop-in headers (include/sparsek/*.hpp) bind.
//
// Composition (all on the caller's stream, device buffers throughout):
//   q|k|v = x Wq|Wk|Wv            library GEMMs (cuBLAS; a projection is a
//                                 plain dense GEMM)
//   raw,u,mean,sdev = K1(x, w)    skb_score_fwd (float64, bit-identical u)
//   selection, o, lse = K2, K3    skb_select + skb_attn_fwd
//   y = o Wo
// Backward: dWo = hc^T g, dhc = g Wo^T, K4 (+ JVP) -> dq dk dv du, K1 bwd
// (graw, dw_score, dx += graw w), dW* = x^T d*, dx += d* W*^T.
#include <cublas_v2.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {
void set_last_error(const char* msg);
}

namespace {

using skb::Error;

size_t esz(int dt) { return dt == SKB_F64 ? 8 : dt == SKB_F32 ? 4 : 2; }

void cublas_check(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS)
        throw Error(SKB_ECUDA, std::string("cuBLAS ") + what + " failed (" + std::to_string((int)s) + ")");
}

// one handle per (thread, device)
cublasHandle_t handle_for(cudaStream_t st) {
    thread_local cublasHandle_t h[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 63;
    if (!h[dev]) {
        cublas_check(cublasCreate(&h[dev]), "create");
        cublas_check(cublasSetMathMode(h[dev], CUBLAS_PEDANTIC_MATH), "math mode");  // true fp32, no TF32
    }
    cublas_check(cublasSetStream(h[dev], st), "set stream");
    return h[dev];
}

// A per-(thread, device) side stream forked from `st` (it sees everything
// enqueued on st so far) and joined back with an event.
class SideStream {
  public:
    SideStream(cudaStream_t st, bool on) : st_(st), on_(on) {
        if (!on_) return;
        struct Slot {
            cudaStream_t s = nullptr;
            cudaEvent_t fork = nullptr, join = nullptr;
        };
        thread_local Slot slots[64];
        int dev = 0;
        cudaGetDevice(&dev);
        Slot& sl = slots[dev & 63];
        if (!sl.s) {
            SKB_CHECK_CUDA(cudaStreamCreateWithFlags(&sl.s, cudaStreamNonBlocking));
            SKB_CHECK_CUDA(cudaEventCreateWithFlags(&sl.fork, cudaEventDisableTiming));
            SKB_CHECK_CUDA(cudaEventCreateWithFlags(&sl.join, cudaEventDisableTiming));
        }
        side_ = sl.s;
        join_ = sl.join;
        SKB_CHECK_CUDA(cudaEventRecord(sl.fork, st_));
        SKB_CHECK_CUDA(cudaStreamWaitEvent(side_, sl.fork, 0));
    }
    void* get() const { return on_ ? static_cast<void*>(side_) : static_cast<void*>(st_); }
    void join() {
        if (!on_) return;
        SKB_CHECK_CUDA(cudaEventRecord(join_, side_));
        SKB_CHECK_CUDA(cudaStreamWaitEvent(st_, join_, 0));
    }

  private:
    cudaStream_t st_, side_ = nullptr;
    cudaEvent_t join_ = nullptr;
    bool on_;
};

// Row-major C[M, N] (+)= op(A) op(B) with op(A) [M, K], op(B) [K, N]; ta/tb
// say whether the stored row-major matrix is transposed. Expressed as the
// column-major product C^T = op(B)^T op(A)^T.
void gemm(cudaStream_t st, int dt, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
          const void* B, int64_t ldb, void* C, int64_t ldc, bool accumulate) {
    if (M == 0 || N == 0) return;
    cublasHandle_t h = handle_for(st);
    const cudaDataType_t t = dt == SKB_F64 ? CUDA_R_64F : dt == SKB_F32 ? CUDA_R_32F : CUDA_R_16BF;
    const cublasComputeType_t ct = dt == SKB_F64 ? CUBLAS_COMPUTE_64F : CUBLAS_COMPUTE_32F;
    const double a64 = 1.0, b64 = accumulate ? 1.0 : 0.0;
    const float a32 = 1.f, b32 = accumulate ? 1.f : 0.f;
    const void* alpha = dt == SKB_F64 ? (const void*)&a64 : (const void*)&a32;
    const void* beta = dt == SKB_F64 ? (const void*)&b64 : (const void*)&b32;
    cublas_check(cublasGemmEx(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, (int)N, (int)M,
                              (int)K, alpha, B, t, (int)ldb, A, t, (int)lda, beta, C, t, (int)ldc, ct,
                              CUBLAS_GEMM_DEFAULT),
                 "gemm");
}

struct Allocs {
    std::vector<void*> ptrs;
    ~Allocs() {
        for (void* p : ptrs) cudaFree(p);
    }
    void* get(size_t bytes) {
        void* p = nullptr;
        SKB_CHECK_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
        ptrs.push_back(p);
        return p;
    }
};

skb_attn_desc core_desc(const skb_x_desc& d, int64_t L) {
    skb_attn_desc a{};
    a.batch = d.batch;
    a.seq_len = L;
    a.heads = d.heads;
    a.head_dim = d.d_model / d.heads;
    a.k = d.k;
    a.window = d.window;
    a.scale = d.scale;
    a.key_mode = d.key_mode;
    a.mask_mode = d.mask_mode;
    a.dtype = d.dtype;
    a.flags = d.flags;
    a.chunk_len = d.chunk_len;
    return a;
}

void validate_x(const skb_x_desc& d) {
    SKB_REQUIRE(d.batch >= 1 && d.seq_len >= 1 && d.d_model >= 1, SKB_ESHAPE,
                "attention: batch, seq_len and d_model must be positive");
    SKB_REQUIRE(d.heads >= 1, SKB_ECONFIG, "attention: heads must be positive");
    SKB_REQUIRE(d.d_model % d.heads == 0, SKB_ECONFIG, "attention: d_model must be a positive multiple of heads");
    SKB_REQUIRE(d.dtype == SKB_F32 || d.dtype == SKB_F64 || d.dtype == SKB_BF16, SKB_EARG, "attention: bad dtype");
    SKB_REQUIRE(d.window > 0 || std::floor(d.k) >= 1.0 || (d.flags & SKB_FLAG_LINEAR_MIX), SKB_ECONFIG,
                "attention: window + floor(k) must be >= 1 (only the linear mix can run with neither)");
    SKB_REQUIRE(!(d.flags & SKB_FLAG_LINEAR_MIX) || d.scoring.norm_mode == 1, SKB_ECONFIG,
                "linear mix requires timestep normalization; raw scores make the linear branch blow up");
    SKB_REQUIRE(!(d.k > 0.0) || d.scoring.slope_eps > 0.0, SKB_EARG, "ScoringParams: slope_eps must be positive");
}

void check_rc(int rc) {
    if (rc != SKB_OK) throw Error(rc, skb_last_error());
}

}  // namespace

struct skb_xattn {
    skb_x_desc d{};
    Allocs mem;
    void *x = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *o = nullptr;
    double *raw = nullptr, *u = nullptr, *mean = nullptr, *sdev = nullptr, *lse = nullptr;
    void* sel = nullptr;
    skb_select_layout lay{};
    void* lmws = nullptr;  // linear mix: the skb_linmix workspace (lse holds the mixture denominators)
    bool linear = false;
};

struct skb_xcache {
    skb_x_desc d{};
    skb_cache* cache = nullptr;
    Allocs mem;
    double* norm = nullptr;  // [B, 3] TimestepNormState {count, mean, m2}
    int64_t seen = 0;
    ~skb_xcache() {
        if (cache) skb_cache_destroy(cache);
    }
};

#define XA_BEGIN try {
#define XA_END                                       \
    }                                                \
    catch (const skb::Error& e) {                    \
        skb::set_last_error(e.what());               \
        return e.code;                               \
    }                                                \
    catch (const std::exception& e) {                \
        skb::set_last_error(e.what());               \
        return SKB_ECUDA;                            \
    }                                                \
    return SKB_OK;

extern "C" {

int skb_matmul(int32_t dtype, int64_t M, int64_t N, int64_t K, const void* a, const void* b, void* c, void* stream) {
    XA_BEGIN
    SKB_REQUIRE(M >= 0 && N >= 0 && K >= 0, SKB_ESHAPE, "matmul: negative dimension");
    SKB_REQUIRE(dtype == SKB_F32 || dtype == SKB_F64 || dtype == SKB_BF16, SKB_EARG, "matmul: bad dtype");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (K == 0) {
        SKB_CHECK_CUDA(cudaMemsetAsync(c, 0, (size_t)M * N * esz(dtype), st));
    } else {
        SKB_REQUIRE(a && b && c, SKB_EARG, "matmul: null argument");
        gemm(st, dtype, false, false, M, N, K, a, K, b, N, c, N, false);
    }
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    XA_END
}

static int xattn_forward(const skb_x_desc* d, const void* x, const void* wq, const void* wk, const void* wv,
                         const void* wo, const double* w_score, const double* feat, void* y, skb_xattn** tape,
                         void* stream) {
    XA_BEGIN
    SKB_REQUIRE(d && x && wq && wk && wv && wo && y, SKB_EARG, "sparsek_attention: null argument");
    SKB_REQUIRE(!feat == !(d->flags & SKB_FLAG_LINEAR_MIX), SKB_EARG,
                "linear mix: feature maps go with SKB_FLAG_LINEAR_MIX (and only with it)");
    validate_x(*d);
    SKB_REQUIRE(!(d->k > 0.0) || w_score != nullptr, SKB_ECONFIG, "attention: w_score length must equal d_model");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t B = d->batch, L = d->seq_len, D = d->d_model, M = B * L;
    const int dt = d->dtype;
    const size_t es = esz(dt);
    auto* t = new skb_xattn();
    try {
        t->d = *d;
        t->x = t->mem.get(M * D * es);
        t->q = t->mem.get(M * D * es);
        t->k = t->mem.get(M * D * es);
        t->v = t->mem.get(M * D * es);
        t->o = t->mem.get(M * D * es);
        t->raw = static_cast<double*>(t->mem.get(M * 8));
        t->u = static_cast<double*>(t->mem.get(M * 8));
        t->mean = static_cast<double*>(t->mem.get(M * 8));
        t->sdev = static_cast<double*>(t->mem.get(M * 8));
        t->lse = static_cast<double*>(t->mem.get(M * d->heads * 8));
        SKB_CHECK_CUDA(cudaMemcpyAsync(t->x, x, M * D * es, cudaMemcpyDefault, st));
        // K1 (a serial float64 Welford chain per sequence) runs on a side
        // stream under the three projection GEMMs: both only read x.
        SideStream side(st, d->k > 0.0);
        gemm(st, dt, false, false, M, D, D, x, D, wq, D, t->q, D, false);  // cache.cpp:204-206
        gemm(st, dt, false, false, M, D, D, x, D, wk, D, t->k, D, false);
        gemm(st, dt, false, false, M, D, D, x, D, wv, D, t->v, D, false);
        if (d->k > 0.0) {
            check_rc(skb_score_fwd(B, L, D, dt, x, w_score, &d->scoring, t->raw, t->u, t->mean, t->sdev, side.get()));
            side.join();
        } else {  // scores idle (cache.cpp:219-227)
            SKB_CHECK_CUDA(cudaMemsetAsync(t->raw, 0, M * 8, st));
            SKB_CHECK_CUDA(cudaMemsetAsync(t->u, 0, M * 8, st));
            SKB_CHECK_CUDA(cudaMemsetAsync(t->mean, 0, M * 8, st));
            SKB_CHECK_CUDA(cudaMemsetAsync(t->sdev, 0, M * 8, st));
        }
        const skb_attn_desc a = core_desc(*d, L);
        check_rc(skb_select_layout_of(&a, &t->lay));
        t->sel = t->mem.get(t->lay.total_bytes);
        check_rc(skb_select(&a, t->u, t->sel, stream));
        if (feat) {  // Appendix B.1: the mixture readout (cache.cpp:322-356); lse holds its denominators
            size_t lb = 0;
            check_rc(skb_linmix_workspace_size(&a, &lb));
            t->lmws = t->mem.get(lb);
            t->linear = true;
            check_rc(skb_linmix_fwd(&a, t->q, t->k, t->v, t->u, t->sel, feat, t->o, t->lse, t->lmws, stream));
        } else {
            check_rc(skb_attn_fwd(&a, t->q, t->k, t->v, t->u, t->sel, t->o, t->lse, stream));
        }
        gemm(st, dt, false, false, M, D, D, t->o, D, wo, D, y, D, false);  // cache.cpp:398-399
    } catch (...) {
        delete t;
        throw;
    }
    if (tape) *tape = t;
    else {
        SKB_CHECK_CUDA(cudaStreamSynchronize(st));
        delete t;
    }
    XA_END
}

static int xattn_backward(skb_xattn* t, const void* grad_out, const void* wq, const void* wk, const void* wv,
                          const void* wo, const double* w_score, const double* feat, void* dx, void* dwq, void* dwk,
                          void* dwv, void* dwo, double* dw_score, double* dfeat, void* stream) {
    XA_BEGIN
    SKB_REQUIRE(t && grad_out && wq && wk && wv && wo && dx && dwq && dwk && dwv && dwo && dw_score, SKB_EARG,
                "sparsek_attention_backward: null argument");
    SKB_REQUIRE(t->linear == (feat != nullptr), SKB_ECONFIG, "backward: linear mix needs feature parameters");
    SKB_REQUIRE(!feat || dfeat, SKB_EARG, "sparsek_attention_backward: null dfeat");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const skb_x_desc& d = t->d;
    const int64_t B = d.batch, L = d.seq_len, D = d.d_model, M = B * L;
    const int dt = d.dtype;
    const size_t es = esz(dt);
    const skb_attn_desc a = core_desc(d, L);
    Allocs tmp;
    void* dhc = tmp.get(M * D * es);
    void* dq = tmp.get(M * D * es);
    void* dk = tmp.get(M * D * es);
    void* dv = tmp.get(M * D * es);
    double* du = static_cast<double*>(tmp.get(M * 8));
    size_t wsb = 0;
    check_rc(skb_attn_bwd_workspace_size(&a, &wsb));
    void* ws = tmp.get(wsb);
    gemm(st, dt, true, false, D, D, M, t->o, D, grad_out, D, dwo, D, false);  // dWo = hc^T g (attention.cpp:236-247)
    gemm(st, dt, false, true, M, D, D, grad_out, D, wo, D, dhc, D, false);    // dhc = g Wo^T
    if (feat)  // attention.cpp:317-445, 519-549
        check_rc(skb_linmix_bwd(&a, t->q, t->k, t->v, t->u, t->sel, feat, t->lse, dhc, dq, dk, dv, du, dfeat,
                                t->lmws, stream));
    else
        check_rc(skb_attn_bwd(&a, t->q, t->k, t->v, t->o, dhc, t->lse, t->u, t->sel, dq, dk, dv, du, ws, stream));
    gemm(st, dt, true, false, D, D, M, t->x, D, dq, D, dwq, D, false);  // dW = x^T d (attention.cpp:551-573)
    gemm(st, dt, true, false, D, D, M, t->x, D, dk, D, dwk, D, false);
    gemm(st, dt, true, false, D, D, M, t->x, D, dv, D, dwv, D, false);
    gemm(st, dt, false, true, M, D, D, dq, D, wq, D, dx, D, false);     // dx = dq Wq^T + dk Wk^T + dv Wv^T
    gemm(st, dt, false, true, M, D, D, dk, D, wk, D, dx, D, true);
    gemm(st, dt, false, true, M, D, D, dv, D, wv, D, dx, D, true);
    if (d.k > 0.0) {
        SKB_REQUIRE(w_score != nullptr, SKB_EARG, "sparsek_attention_backward: null w_score");
        skb_scoring sc = d.scoring;
        if (d.chunk_len > 0) sc.chunk_len = (int32_t)d.chunk_len;
        double* graw = static_cast<double*>(tmp.get(M * 8));
        // graw, dw_score, dx += graw w (attention.cpp:482-516, 564)
        check_rc(skb_score_bwd(B, L, D, dt, t->x, w_score, &sc, du, t->raw, t->mean, t->sdev, graw, dw_score, dx,
                               stream));
    } else {
        SKB_CHECK_CUDA(cudaMemsetAsync(dw_score, 0, D * 8, st));
    }
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));  // the temporaries are freed on return
    XA_END
}

int skb_xattn_forward(const skb_x_desc* d, const void* x, const void* wq, const void* wk, const void* wv,
                      const void* wo, const double* w_score, void* y, skb_xattn** tape, void* stream) {
    return xattn_forward(d, x, wq, wk, wv, wo, w_score, nullptr, y, tape, stream);
}

int skb_xattn_forward_lin(const skb_x_desc* d, const void* x, const void* wq, const void* wk, const void* wv,
                          const void* wo, const double* w_score, const double* feat, void* y, skb_xattn** tape,
                          void* stream) {
    if (!feat) {
        skb::set_last_error("linear mix: missing feature maps");
        return SKB_EARG;
    }
    return xattn_forward(d, x, wq, wk, wv, wo, w_score, feat, y, tape, stream);
}

int skb_xattn_backward(skb_xattn* t, const void* grad_out, const void* wq, const void* wk, const void* wv,
                       const void* wo, const double* w_score, void* dx, void* dwq, void* dwk, void* dwv, void* dwo,
                       double* dw_score, void* stream) {
    return xattn_backward(t, grad_out, wq, wk, wv, wo, w_score, nullptr, dx, dwq, dwk, dwv, dwo, dw_score, nullptr,
                          stream);
}

int skb_xattn_backward_lin(skb_xattn* t, const void* grad_out, const void* wq, const void* wk, const void* wv,
                           const void* wo, const double* w_score, const double* feat, void* dx, void* dwq, void* dwk,
                           void* dwv, void* dwo, double* dw_score, double* dfeat, void* stream) {
    if (!feat) {
        skb::set_last_error("backward: linear mix needs feature parameters");
        return SKB_ECONFIG;
    }
    return xattn_backward(t, grad_out, wq, wk, wv, wo, w_score, feat, dx, dwq, dwk, dwv, dwo, dw_score, dfeat,
                          stream);
}

int skb_xattn_tape_get(skb_xattn* t, int32_t field, void* dst, size_t bytes, void* stream) {
    XA_BEGIN
    SKB_REQUIRE(t && dst, SKB_EARG, "tape_get: null argument");
    const skb_x_desc& d = t->d;
    const int64_t M = d.batch * d.seq_len, D = d.d_model;
    const size_t es = esz(d.dtype);
    const void* src = nullptr;
    size_t n = 0;
    switch (field) {
        case SKB_TAPE_X: src = t->x, n = M * D * es; break;
        case SKB_TAPE_Q: src = t->q, n = M * D * es; break;
        case SKB_TAPE_K: src = t->k, n = M * D * es; break;
        case SKB_TAPE_V: src = t->v, n = M * D * es; break;
        case SKB_TAPE_HEAD_CONCAT: src = t->o, n = M * D * es; break;
        case SKB_TAPE_RAW: src = t->raw, n = M * 8; break;
        case SKB_TAPE_U: src = t->u, n = M * 8; break;
        case SKB_TAPE_NORM_MEAN: src = t->mean, n = M * 8; break;
        case SKB_TAPE_NORM_SDEV: src = t->sdev, n = M * 8; break;
        case SKB_TAPE_LSE: src = t->lse, n = M * d.heads * 8; break;
        case SKB_TAPE_TAU_PUSH: src = static_cast<char*>(t->sel) + t->lay.tau, n = M * 8; break;
        case SKB_TAPE_LEAVE: src = static_cast<char*>(t->sel) + t->lay.leave, n = M * 4; break;
        default: throw Error(SKB_EARG, "tape_get: unknown field");
    }
    SKB_REQUIRE(bytes >= n, SKB_EARG, "tape_get: destination too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SKB_CHECK_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    XA_END
}

int skb_xattn_destroy(skb_xattn* t) {
    delete t;
    return SKB_OK;
}

// ---------------------------------------------------------------- x-level cache

int skb_xcache_create(const skb_x_desc* d, skb_xcache** out) {
    XA_BEGIN
    SKB_REQUIRE(d && out, SKB_EARG, "cache_create: null argument");
    validate_x(*d);
    auto* c = new skb_xcache();
    try {
        c->d = *d;
        const skb_attn_desc a = core_desc(*d, d->seq_len);
        check_rc(skb_cache_create(&a, &c->cache));
        c->norm = static_cast<double*>(c->mem.get(d->batch * 3 * 8));
        SKB_CHECK_CUDA(cudaMemset(c->norm, 0, d->batch * 3 * 8));
    } catch (...) {
        delete c;
        throw;
    }
    *out = c;
    XA_END
}

int skb_xcache_destroy(skb_xcache* c) {
    delete c;
    return SKB_OK;
}

skb_cache* skb_xcache_inner(skb_xcache* c) { return c ? c->cache : nullptr; }

int skb_xcache_norm_state(skb_xcache* c, double* norm_state, int32_t set, void* stream) {
    XA_BEGIN
    SKB_REQUIRE(c && norm_state, SKB_EARG, "cache_norm_state: null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (set) SKB_CHECK_CUDA(cudaMemcpyAsync(c->norm, norm_state, c->d.batch * 24, cudaMemcpyHostToDevice, st));
    else SKB_CHECK_CUDA(cudaMemcpyAsync(norm_state, c->norm, c->d.batch * 24, cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    if (set) {  // a restore: positions seen come from the device cache
        int64_t seen = 0, cnt = 0, peak = 0;
        double tau = 0;
        std::vector<int32_t> pos((size_t)(std::floor(c->d.k) + c->d.window + 2));
        check_rc(skb_cache_state(c->cache, 0, pos.data(), &cnt, &tau, &seen, &peak, stream));
        c->seen = seen;
    }
    XA_END
}

// SparseKvCache<T>::forward_chunk (proj/src/cache.cpp:181-400) for all B
// sequences: rows x [B, n, D] continue each sequence. The first chunk of a
// fresh cache runs the batch kernels over its rows and leaves the retained
// rows in the pool (skb_cache_prefill); later chunks run one generate_step
// per row (skb_cache_step: exit/admit, then the attention over the retained
// (floor(k) + w) rows), which is the reference's row order exactly.
static int xcache_forward_chunk(skb_xcache* c, const void* x, int64_t n, const void* wq, const void* wk,
                                const void* wv, const void* wo, const double* w_score, const double* feat, void* y,
                                void* stream) {
    XA_BEGIN
    SKB_REQUIRE(c && x && wq && wk && wv && wo && y, SKB_EARG, "forward_chunk: null argument");
    SKB_REQUIRE(!feat == !(c->d.flags & SKB_FLAG_LINEAR_MIX), SKB_ECONFIG,
                "forward_chunk: linear mix needs feature parameters");
    SKB_REQUIRE(n >= 1, SKB_ESHAPE, "forward_chunk: empty chunk");
    const skb_x_desc& d = c->d;
    SKB_REQUIRE(c->seen + n <= d.seq_len, SKB_ESHAPE, "forward_chunk: cache capacity (max positions) exceeded");
    SKB_REQUIRE(!(d.k > 0.0) || w_score != nullptr, SKB_ECONFIG, "attention: w_score length must equal d_model");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t B = d.batch, D = d.d_model, H = d.heads, p = D / H, M = B * n;
    const int dt = d.dtype;
    const size_t es = esz(dt);
    Allocs tmp;
    void* q = tmp.get(M * D * es);
    void* k = tmp.get(M * D * es);
    void* v = tmp.get(M * D * es);
    void* o = tmp.get(M * D * es);
    double* u = static_cast<double*>(tmp.get(M * 8));
    double* raw = static_cast<double*>(tmp.get(M * 8));
    gemm(st, dt, false, false, M, D, D, x, D, wq, D, q, D, false);
    gemm(st, dt, false, false, M, D, D, x, D, wk, D, k, D, false);
    gemm(st, dt, false, false, M, D, D, x, D, wv, D, v, D, false);
    if (d.k > 0.0)  // score_tokens with the carried TimestepNormState (selection.cpp:22-31)
        check_rc(skb_score_continue(B, n, D, dt, x, w_score, &d.scoring, c->norm, raw, u, stream));
    else
        SKB_CHECK_CUDA(cudaMemsetAsync(u, 0, M * 8, st));
    if (c->seen == 0 && n > 1) {
        skb_attn_desc a = core_desc(d, n);
        a.chunk_len = 0;
        skb_select_layout lay{};
        check_rc(skb_select_layout_of(&a, &lay));
        void* sel = tmp.get(lay.total_bytes);
        double* lse = static_cast<double*>(tmp.get(M * H * 8));
        check_rc(skb_select(&a, u, sel, stream));
        if (feat) {  // the mixture readout over the chunk, then phi(k) + the prefix state into the cache
            size_t lb = 0;
            check_rc(skb_linmix_workspace_size(&a, &lb));
            void* lws = tmp.get(lb);
            check_rc(skb_linmix_fwd(&a, q, k, v, u, sel, feat, o, lse, lws, stream));
            check_rc(skb_cache_prefill(c->cache, k, v, u, n, stream));
            double* phk = static_cast<double*>(tmp.get(M * D * 8));
            check_rc(skb_linmix_phi(M, H, p, dt, k, feat, phk, stream));
            check_rc(skb_cache_linmix_prefill(c->cache, v, phk, n, stream));
        } else {
            check_rc(skb_attn_fwd(&a, q, k, v, u, sel, o, lse, stream));
            check_rc(skb_cache_prefill(c->cache, k, v, u, n, stream));
        }
    } else {
        const size_t row = (size_t)D * es;
        void* qr = tmp.get(B * row);
        void* kr = tmp.get(B * row);
        void* vr = tmp.get(B * row);
        void* orow = tmp.get(B * row);
        double* ur = static_cast<double*>(tmp.get(B * 8));
        void* phbuf = feat ? tmp.get(2 * B * D * 8) : nullptr;
        for (int64_t r = 0; r < n; ++r) {  // generate_step per row (cache.cpp:570-577)
            SKB_CHECK_CUDA(cudaMemcpy2DAsync(qr, row, static_cast<char*>(q) + r * row, n * row, row, B,
                                             cudaMemcpyDeviceToDevice, st));
            SKB_CHECK_CUDA(cudaMemcpy2DAsync(kr, row, static_cast<char*>(k) + r * row, n * row, row, B,
                                             cudaMemcpyDeviceToDevice, st));
            SKB_CHECK_CUDA(cudaMemcpy2DAsync(vr, row, static_cast<char*>(v) + r * row, n * row, row, B,
                                             cudaMemcpyDeviceToDevice, st));
            SKB_CHECK_CUDA(cudaMemcpy2DAsync(ur, 8, u + r, n * 8, 8, B, cudaMemcpyDeviceToDevice, st));
            if (feat) {
                double* phq = static_cast<double*>(phbuf);
                double* phk = phq + B * D;
                check_rc(skb_linmix_phi(B, H, p, dt, qr, feat, phq, stream));
                check_rc(skb_linmix_phi(B, H, p, dt, kr, feat, phk, stream));
                check_rc(skb_cache_linmix_step(c->cache, qr, kr, vr, d.k > 0.0 ? ur : nullptr, phq, phk, orow,
                                               stream));
            } else {
                check_rc(skb_cache_step(c->cache, qr, kr, vr, d.k > 0.0 ? ur : nullptr, orow, stream));
            }
            SKB_CHECK_CUDA(cudaMemcpy2DAsync(static_cast<char*>(o) + r * row, n * row, orow, row, row, B,
                                             cudaMemcpyDeviceToDevice, st));
        }
    }
    (void)p;
    gemm(st, dt, false, false, M, D, D, o, D, wo, D, y, D, false);
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    c->seen += n;
    XA_END
}

int skb_xcache_forward_chunk(skb_xcache* c, const void* x, int64_t n, const void* wq, const void* wk, const void* wv,
                             const void* wo, const double* w_score, void* y, void* stream) {
    return xcache_forward_chunk(c, x, n, wq, wk, wv, wo, w_score, nullptr, y, stream);
}

int skb_xcache_forward_chunk_lin(skb_xcache* c, const void* x, int64_t n, const void* wq, const void* wk,
                                 const void* wv, const void* wo, const double* w_score, const double* feat, void* y,
                                 void* stream) {
    if (!feat) {
        skb::set_last_error("forward_chunk: linear mix needs feature parameters");
        return SKB_ECONFIG;
    }
    return xcache_forward_chunk(c, x, n, wq, wk, wv, wo, w_score, feat, y, stream);
}

}  // extern "C"
