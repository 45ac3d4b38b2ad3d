// Linear-attention mix (Appendix B.1 of the paper): linear_mix_attention
// (proj/include/sparsek/attention.hpp:93-99), forward proj/src/cache.cpp:
// 262-278 and 322-356, backward proj/src/attention.cpp:317-445 and 519-549.
//
// Per head, with phi(z) = elu(F z) + 1 (F = feat[h], p x p) and the SparseK
// snapshot of query i (selected keys with gates g, the window with weight 1):
//   m_ij = g_ij (selected), 1 (window), 0 (any other j <= i)
//   w_ij = (1 - m_ij) lambda_ij + m_ij e_ij,  lambda_ij = phi(q_i).phi(k_j),
//          e_ij = exp(scale q_i.k_j)            (no max subtraction)
//   o_i  = sum_{j<=i} w_ij v_j / sum_{j<=i} w_ij
// which is the reference's readout: exact attention over the snapshot mixed
// with positive-feature linear attention over every causal position (its
// prefix accumulators sum phi(k_j) v_j^T over j <= i).
//
// CUDA-core kernels in float64 arithmetic for the reference's float/double
// instantiations (the variant's parity path): one warp per (sequence, row,
// head), lanes over the head dimension.
//   k_phi             phi rows of Q and K (float64)
//   k_linmix_fwd      query-major: o_i and den_i
//   k_linmix_bwd_q    query-major: dq_i (attention + feature pullback),
//                     gphi_q -> dpre_q, go.o, the gate-gradient row sums
//   k_linmix_bwd_k    key-major: dv_j, dk_j (attention + feature pullback),
//                     gphi_k -> dpre_k, the gate-gradient column sums —
//                     no atomics; gradients stay inside the key's chunk
//   k_dfeat           dfeat[h] = sum_rows dpre_q q^T + dpre_k k^T
// The head-summed gate gradients then go through the O(L log L) selection
// pullback (skb_jvp.cu), exactly as for the softmax path.
#include <type_traits>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

namespace {

constexpr int kLmWarps = 8;
constexpr int kLmPer = 8;  // head_dim <= 256

template <class S>
__device__ __forceinline__ double ldd(const S* p) {
    return (double)p[0];
}

struct LmArgs {
    const void *q, *k, *v, *dout;
    void *o, *dq, *dk, *dv;
    const double* u;
    const double* feat;  // [H, p, p]
    const double *phq, *phk;
    double *den, *goo;        // [B, H, L]
    double *dpre_q, *dpre_k;  // [B, L, H, p]
    double *rowsum, *colsum;
    int* bad;
    SelView s;
    int B, L, H, p, w, T, R1, chunk_len;
    double scale;
};

__device__ __forceinline__ double clamp01(double g) { return g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g); }

// Weight m of key j for query i (t = i - w its push time) and whether j is a
// selected (gated) key: the snapshot of proj/src/cache.cpp:285-303.
__device__ __forceinline__ double mix_gate(const LmArgs& a, int64_t bl, int i, int j, bool& sel) {
    sel = false;
    if (j > i - a.w) return 1.0;  // window (empty for w = 0: the linear branch covers the query)
    const int t = i - a.w;
    if (a.R1 > 0 && j <= t && a.s.leave[bl + j] > t) {
        sel = true;
        return clamp01(a.u[bl + j] - a.s.tau[bl + t]);
    }
    return 0.0;
}

// phi rows: out[row, r] = f(sum_c F[h][r][c] z[row, c]), f(x) = x > 0 ? x + 1 : exp(x)
template <class S>
__global__ void __launch_bounds__(kLmWarps * 32) k_phi(const S* __restrict__ z, const double* __restrict__ feat,
                                                        double* __restrict__ out, int64_t rows, int H, int p) {
    __shared__ double zs[kLmWarps][32 * kLmPer];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * kLmWarps + warp;  // (b, i, h)
    if (row >= rows) return;
    const int h = (int)(row % H);
    const S* zr = z + row * p;
    for (int c = lane; c < p; c += 32) zs[warp][c] = ldd<S>(zr + c);
    __syncwarp();
    const double* F = feat + (int64_t)h * p * p;
    for (int r = lane; r < p; r += 32) {
        double acc = 0.0;
        for (int c = 0; c < p; ++c) acc += F[(int64_t)r * p + c] * zs[warp][c];
        out[row * p + r] = acc > 0.0 ? acc + 1.0 : exp(acc);
    }
}

template <class S>
struct Row {
    double x[kLmPer];
    __device__ __forceinline__ void load(const S* base, int lane, int np, int p) {
#pragma unroll
        for (int m = 0; m < kLmPer; ++m) {
            const int c = lane + 32 * m;
            x[m] = (m < np && c < p) ? ldd<S>(base + c) : 0.0;
        }
    }
};
__device__ __forceinline__ void load_d(double* x, const double* base, int lane, int np, int p) {
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) {
        const int c = lane + 32 * m;
        x[m] = (m < np && c < p) ? base[c] : 0.0;
    }
}
__device__ __forceinline__ double dot_l(const double* x, const double* y) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) s += x[m] * y[m];
    return s;
}
__device__ __forceinline__ void warp_sum2(double& a, double& b) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
}

// num/den of query i over every j <= i (the readout both passes need).
template <class S>
__device__ __forceinline__ double readout(const LmArgs& a, int b, int i, int h, const double* qv, const double* phq,
                                          double* num, int lane, int np) {
    const int64_t rs = (int64_t)a.H * a.p, bl = (int64_t)b * a.L;
    const S* K = static_cast<const S*>(a.k);
    const S* V = static_cast<const S*>(a.v);
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) num[m] = 0.0;
    double den = 0.0;
    for (int j = 0; j <= i; ++j) {
        const int64_t ro = (bl + j) * rs + (int64_t)h * a.p;
        Row<S> kr, vr;
        double pk[kLmPer];
        kr.load(K + ro, lane, np, a.p);
        load_d(pk, a.phk + ro, lane, np, a.p);
        double lam = dot_l(phq, pk), dot = dot_l(qv, kr.x);
        warp_sum2(lam, dot);
        bool sel;
        const double m = mix_gate(a, bl, i, j, sel);
        double w = (1.0 - m) * lam;
        if (m > 0.0) w += m * exp(a.scale * dot);
        vr.load(V + ro, lane, np, a.p);
#pragma unroll
        for (int e = 0; e < kLmPer; ++e) num[e] += w * vr.x[e];
        den += w;
    }
    return den;
}

template <class S>
__global__ void __launch_bounds__(kLmWarps * 32) k_linmix_fwd(LmArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = blockIdx.x * kLmWarps + warp, h = blockIdx.y, b = blockIdx.z;
    if (i >= a.L) return;
    const int np = (a.p + 31) / 32;
    const int64_t rs = (int64_t)a.H * a.p;
    const int64_t ro = ((int64_t)b * a.L + i) * rs + (int64_t)h * a.p;
    Row<S> q;
    q.load(static_cast<const S*>(a.q) + ro, lane, np, a.p);
    double phq[kLmPer], num[kLmPer];
    load_d(phq, a.phq + ro, lane, np, a.p);
    const double den = readout<S>(a, b, i, h, q.x, phq, num, lane, np);
    if (!(den > 0.0)) {  // proj/src/cache.cpp:349-350
        if (lane == 0) *a.bad = 1;
    }
    S* orow = static_cast<S*>(a.o) + ro;
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) {
        const int c = lane + 32 * m;
        if (m < np && c < a.p) orow[c] = (S)(num[m] / den);
    }
    if (lane == 0) a.den[((int64_t)b * a.H + h) * a.L + i] = den;
}

// Query pass of the backward (proj/src/attention.cpp:317-445, the per-query
// loop): dq_i, gphi_q -> dpre_q and dq_i += F^T dpre_q, go_i.o_i, and the
// head-summed gate-gradient row sum over the fractional selected keys.
template <class S>
__global__ void __launch_bounds__(kLmWarps * 32) k_linmix_bwd_q(LmArgs a) {
    __shared__ double dps[kLmWarps][32 * kLmPer];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = blockIdx.x * kLmWarps + warp, h = blockIdx.y, b = blockIdx.z;
    if (i >= a.L) return;
    const int np = (a.p + 31) / 32;
    const int64_t rs = (int64_t)a.H * a.p, bl = (int64_t)b * a.L;
    const int64_t ro = (bl + i) * rs + (int64_t)h * a.p;
    const S* K = static_cast<const S*>(a.k);
    const S* V = static_cast<const S*>(a.v);
    Row<S> q, go;
    q.load(static_cast<const S*>(a.q) + ro, lane, np, a.p);
    go.load(static_cast<const S*>(a.dout) + ro, lane, np, a.p);
    double phq[kLmPer], num[kLmPer];
    load_d(phq, a.phq + ro, lane, np, a.p);
    const double den = readout<S>(a, b, i, h, q.x, phq, num, lane, np);
    double goo = 0.0;
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) goo += go.x[m] * (num[m] / den);
    goo = warp_sum(goo);
    double dq[kLmPer], gq[kLmPer];
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) dq[m] = gq[m] = 0.0;
    double rsum = 0.0;
    for (int j = 0; j <= i; ++j) {
        const int64_t rj_o = (bl + j) * rs + (int64_t)h * a.p;
        Row<S> kr, vr;
        double pk[kLmPer];
        kr.load(K + rj_o, lane, np, a.p);
        vr.load(V + rj_o, lane, np, a.p);
        load_d(pk, a.phk + rj_o, lane, np, a.p);
        double lam = dot_l(phq, pk), dot = dot_l(q.x, kr.x);
        double bv = dot_l(go.x, vr.x);
        warp_sum2(lam, dot);
        bv = warp_sum(bv);
        bool sel;
        const double m = mix_gate(a, bl, i, j, sel);
        const double e = m > 0.0 ? exp(a.scale * dot) : 0.0;
        const double r = (bv - goo) / den;
        if (m > 0.0) {
            const double dd = r * m * e * a.scale;
#pragma unroll
            for (int x = 0; x < kLmPer; ++x) dq[x] += dd * kr.x[x];
        }
        const double glam = r * (1.0 - m);
#pragma unroll
        for (int x = 0; x < kLmPer; ++x) gq[x] += glam * pk[x];
        if (sel) {
            const double g = m;  // the gate itself
            if (g > 0.0 && g < 1.0) rsum += r * (e - lam);
        }
    }
    // query-side feature pullback: dpre = gphi_q * elu'(pre), elu'(pre) = min(phi, 1)
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) {
        const int c = lane + 32 * m;
        const double dpre = gq[m] * (phq[m] < 1.0 ? phq[m] : 1.0);
        if (m < np && c < a.p) {
            dps[warp][c] = dpre;
            a.dpre_q[ro + c] = dpre;
        }
    }
    __syncwarp();
    const double* F = a.feat + (int64_t)h * a.p * a.p;
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) {
        const int c = lane + 32 * m;
        if (m < np && c < a.p) {
            double acc = dq[m];
            for (int rr = 0; rr < a.p; ++rr) acc += dps[warp][rr] * F[(int64_t)rr * a.p + c];
            static_cast<S*>(a.dq)[ro + c] = (S)acc;
        }
    }
    if (lane == 0) {
        a.goo[((int64_t)b * a.H + h) * a.L + i] = goo;
        if (rsum != 0.0 && i >= a.w) atomicAdd(a.rowsum + bl + (i - a.w), rsum);
    }
}

// Key pass: every query i >= j of j's chunk (proj/src/attention.cpp:393-425,
// the `j >= cs` terms) — dv_j, dk_j, gphi_k -> dpre_k and dk_j += F^T dpre_k,
// and the gate-gradient column sum of j over its fractional queries.
template <class S>
__global__ void __launch_bounds__(kLmWarps * 32) k_linmix_bwd_k(LmArgs a) {
    __shared__ double dps[kLmWarps][32 * kLmPer];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = blockIdx.x * kLmWarps + warp, h = blockIdx.y, b = blockIdx.z;
    if (j >= a.L) return;
    const int np = (a.p + 31) / 32;
    const int64_t rs = (int64_t)a.H * a.p, bl = (int64_t)b * a.L;
    const int64_t ro = (bl + j) * rs + (int64_t)h * a.p;
    const S* Q = static_cast<const S*>(a.q);
    const S* G = static_cast<const S*>(a.dout);
    Row<S> kr, vr;
    kr.load(static_cast<const S*>(a.k) + ro, lane, np, a.p);
    vr.load(static_cast<const S*>(a.v) + ro, lane, np, a.p);
    double pk[kLmPer];
    load_d(pk, a.phk + ro, lane, np, a.p);
    double dk[kLmPer], dv[kLmPer], gk[kLmPer];
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) dk[m] = dv[m] = gk[m] = 0.0;
    double csum = 0.0;
    const int iend = a.chunk_len > 0 ? min(a.L, (j / a.chunk_len + 1) * a.chunk_len) : a.L;
    const double* denb = a.den + ((int64_t)b * a.H + h) * a.L;
    const double* goob = a.goo + ((int64_t)b * a.H + h) * a.L;
    for (int i = j; i < iend; ++i) {
        const int64_t ri = (bl + i) * rs + (int64_t)h * a.p;
        Row<S> q, go;
        double pq[kLmPer];
        q.load(Q + ri, lane, np, a.p);
        go.load(G + ri, lane, np, a.p);
        load_d(pq, a.phq + ri, lane, np, a.p);
        double lam = dot_l(pq, pk), dot = dot_l(q.x, kr.x);
        double bv = dot_l(go.x, vr.x);
        warp_sum2(lam, dot);
        bv = warp_sum(bv);
        bool sel;
        const double m = mix_gate(a, bl, i, j, sel);
        const double den = denb[i];
        const double e = m > 0.0 ? exp(a.scale * dot) : 0.0;
        double w = (1.0 - m) * lam;
        if (m > 0.0) w += m * e;
        const double r = (bv - goob[i]) / den;
        const double c0 = w / den;
#pragma unroll
        for (int x = 0; x < kLmPer; ++x) dv[x] += c0 * go.x[x];
        if (m > 0.0) {
            const double dd = r * m * e * a.scale;
#pragma unroll
            for (int x = 0; x < kLmPer; ++x) dk[x] += dd * q.x[x];
        }
        const double glam = r * (1.0 - m);
#pragma unroll
        for (int x = 0; x < kLmPer; ++x) gk[x] += glam * pq[x];
        if (sel && m > 0.0 && m < 1.0) csum += r * (e - lam);
    }
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) {
        const int c = lane + 32 * m;
        const double dpre = gk[m] * (pk[m] < 1.0 ? pk[m] : 1.0);
        if (m < np && c < a.p) {
            dps[warp][c] = dpre;
            a.dpre_k[ro + c] = dpre;
        }
    }
    __syncwarp();
    const double* F = a.feat + (int64_t)h * a.p * a.p;
#pragma unroll
    for (int m = 0; m < kLmPer; ++m) {
        const int c = lane + 32 * m;
        if (m < np && c < a.p) {
            double acc = dk[m];
            for (int rr = 0; rr < a.p; ++rr) acc += dps[warp][rr] * F[(int64_t)rr * a.p + c];
            static_cast<S*>(a.dk)[ro + c] = (S)acc;
            static_cast<S*>(a.dv)[ro + c] = (S)dv[m];
        }
    }
    if (lane == 0 && csum != 0.0) atomicAdd(a.colsum + bl + j, csum);
}

// dfeat[h][r][c] = sum over rows (b, i) of dpre_q[r] q[c] + dpre_k[r] k[c]:
// block (h, r) x row slab, threads over c, atomics across slabs.
template <class S>
__global__ void k_dfeat(const LmArgs a, double* __restrict__ dfeat, int rows_per) {
    const int h = blockIdx.x, r = blockIdx.y;
    const int64_t rows = (int64_t)a.B * a.L;
    const int64_t r0 = (int64_t)blockIdx.z * rows_per, r1 = min(rows, r0 + rows_per);
    const int64_t rs = (int64_t)a.H * a.p;
    const S* Q = static_cast<const S*>(a.q);
    const S* K = static_cast<const S*>(a.k);
    for (int c = threadIdx.x; c < a.p; c += blockDim.x) {
        double acc = 0.0;
        for (int64_t row = r0; row < r1; ++row) {
            const int64_t o = row * rs + (int64_t)h * a.p;
            acc += a.dpre_q[o + r] * ldd<S>(Q + o + c) + a.dpre_k[o + r] * ldd<S>(K + o + c);
        }
        atomicAdd(dfeat + ((int64_t)h * a.p + r) * a.p + c, acc);
    }
}

struct LmLayout {
    uint64_t phq, phk, dpre_q, dpre_k, goo, bwd, total;
};
LmLayout lm_layout(const skb_attn_desc& d) {
    LmLayout o{};
    const uint64_t N = (uint64_t)d.batch * d.seq_len * d.heads * d.head_dim;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t r = off;
        off = (off + bytes + 255) & ~uint64_t(255);
        return r;
    };
    o.phq = take(N * 8);
    o.phk = take(N * 8);
    o.dpre_q = take(N * 8);
    o.dpre_k = take(N * 8);
    o.goo = take((uint64_t)d.batch * d.heads * d.seq_len * 8);
    o.bwd = take(0);
    BwdLayout bl;
    bwd_layout(d, bl);  // rowsum / colsum / JVP scratch follow
    o.total = o.bwd + bl.total;
    return o;
}

LmArgs lm_args(const skb_attn_desc& d, const SelView& s) {
    LmArgs a{};
    a.s = s;
    a.B = (int)d.batch;
    a.L = (int)d.seq_len;
    a.H = (int)d.heads;
    a.p = (int)d.head_dim;
    a.w = (int)d.window;
    a.T = std::max(0, a.L - a.w);
    a.R1 = (int)floor_k(d.k);
    a.chunk_len = (int)d.chunk_len;
    a.scale = d.scale > 0.0 ? d.scale : 1.0 / std::sqrt((double)d.head_dim);
    return a;
}

template <class F>
void dispatch_lm(int32_t dt, F&& f) {
    if (dt == SKB_F64) f((const double*)nullptr);
    else if (dt == SKB_F32) f((const float*)nullptr);
    else throw Error(SKB_EARG, "linear mix: dtype must be float32 or float64 (the reference's instantiations)");
}

void check_lm(const skb_attn_desc& d) {
    validate_desc(d);
    SKB_REQUIRE(d.flags & SKB_FLAG_LINEAR_MIX, SKB_ECONFIG, "linear mix: desc must carry SKB_FLAG_LINEAR_MIX");
    SKB_REQUIRE(d.head_dim <= 32 * kLmPer, SKB_ESHAPE, "linear mix: head_dim must be <= 256");
    SKB_REQUIRE(d.dtype == SKB_F32 || d.dtype == SKB_F64, SKB_EARG,
                "linear mix: dtype must be float32 or float64 (the reference's instantiations)");
}

void run_phi(const skb_attn_desc& d, const void* q, const void* k, const double* feat, const LmLayout& lay,
             char* base, cudaStream_t st) {
    const int64_t rows = d.batch * d.seq_len * d.heads;
    dispatch_lm(d.dtype, [&](auto tag) {
        using S = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
        const unsigned g = (unsigned)cdiv(rows, kLmWarps);
        k_phi<S><<<g, kLmWarps * 32, 0, st>>>(static_cast<const S*>(q), feat,
                                               reinterpret_cast<double*>(base + lay.phq), rows, (int)d.heads,
                                               (int)d.head_dim);
        k_phi<S><<<g, kLmWarps * 32, 0, st>>>(static_cast<const S*>(k), feat,
                                               reinterpret_cast<double*>(base + lay.phk), rows, (int)d.heads,
                                               (int)d.head_dim);
    });
    SKB_CHECK_LAUNCH();
}

int* lm_bad_flag() {
    thread_local int* flags[64] = {};
    int dev = 0;
    SKB_CHECK_CUDA(cudaGetDevice(&dev));
    int*& f = flags[dev & 63];
    if (!f) SKB_CHECK_CUDA(cudaMalloc(&f, sizeof(int)));
    return f;
}

}  // namespace

void set_last_error(const char* msg);  // skb_capi.cu (thread-local skb_last_error)

}  // namespace skb

#define LM_BEGIN try {
#define LM_END                                  \
    }                                           \
    catch (const skb::Error& e) {               \
        skb::set_last_error(e.what());          \
        return e.code;                          \
    }                                           \
    catch (const std::exception& e) {           \
        skb::set_last_error(e.what());          \
        return SKB_ECUDA;                       \
    }                                           \
    return SKB_OK;

extern "C" {

int skb_linmix_phi(int64_t rows, int64_t heads, int64_t head_dim, int32_t dtype, const void* z, const double* feat,
                   double* out, void* stream) {
    LM_BEGIN
    SKB_REQUIRE(z && feat && out, SKB_EARG, "linmix_phi: null argument");
    SKB_REQUIRE(rows >= 0 && heads >= 1 && head_dim >= 1 && head_dim <= 32 * skb::kLmPer, SKB_ESHAPE,
                "linmix_phi: bad shape");
    if (rows == 0) return SKB_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n = rows * heads;
    skb::dispatch_lm(dtype, [&](auto tag) {
        using S = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
        skb::k_phi<S><<<(unsigned)skb::cdiv(n, skb::kLmWarps), skb::kLmWarps * 32, 0, st>>>(
            static_cast<const S*>(z), feat, out, n, (int)heads, (int)head_dim);
    });
    SKB_CHECK_LAUNCH();
    LM_END
}

int skb_linmix_workspace_size(const skb_attn_desc* d, size_t* bytes) {
    LM_BEGIN
    SKB_REQUIRE(d && bytes, SKB_EARG, "linmix_workspace_size: null argument");
    skb::check_lm(*d);
    *bytes = (size_t)skb::lm_layout(*d).total;
    LM_END
}

int skb_linmix_fwd(const skb_attn_desc* d, const void* q, const void* k, const void* v, const double* u,
                   const void* sel_ws, const double* feat, void* o, double* den, void* ws, void* stream) {
    LM_BEGIN
    SKB_REQUIRE(d && q && k && v && u && sel_ws && feat && o && den && ws, SKB_EARG,
                "linear_mix_attention: null argument");
    skb::check_lm(*d);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const skb::SelView s = skb::sel_view(*d, sel_ws);
    const skb::LmLayout lay = skb::lm_layout(*d);
    char* base = static_cast<char*>(ws);
    skb::run_phi(*d, q, k, feat, lay, base, st);
    skb::LmArgs a = skb::lm_args(*d, s);
    a.q = q, a.k = k, a.v = v, a.o = o, a.u = u, a.feat = feat, a.den = den;
    a.phq = reinterpret_cast<const double*>(base + lay.phq);
    a.phk = reinterpret_cast<const double*>(base + lay.phk);
    a.bad = skb::lm_bad_flag();
    SKB_CHECK_CUDA(cudaMemsetAsync(a.bad, 0, sizeof(int), st));
    const dim3 g((unsigned)skb::cdiv(d->seq_len, skb::kLmWarps), (unsigned)d->heads, (unsigned)d->batch);
    skb::dispatch_lm(d->dtype, [&](auto tag) {
        using S = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
        skb::k_linmix_fwd<S><<<g, skb::kLmWarps * 32, 0, st>>>(a);
    });
    SKB_CHECK_LAUNCH();
    int hbad = 0;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&hbad, a.bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    SKB_REQUIRE(!hbad, SKB_ENUMERIC, "linear mix: nonpositive denominator");
    LM_END
}

int skb_linmix_bwd(const skb_attn_desc* d, const void* q, const void* k, const void* v, const double* u,
                   const void* sel_ws, const double* feat, const double* den, const void* dout, void* dq, void* dk,
                   void* dv, double* du, double* dfeat, void* ws, void* stream) {
    LM_BEGIN
    SKB_REQUIRE(d && q && k && v && u && sel_ws && feat && den && dout && dq && dk && dv && du && dfeat && ws,
                SKB_EARG, "linear mix backward: null argument");
    skb::check_lm(*d);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const skb::SelView s = skb::sel_view(*d, sel_ws);
    const skb::LmLayout lay = skb::lm_layout(*d);
    skb::BwdLayout bl;
    skb::bwd_layout(*d, bl);
    char* base = static_cast<char*>(ws);
    char* bb = base + lay.bwd;
    skb::run_phi(*d, q, k, feat, lay, base, st);
    skb::LmArgs a = skb::lm_args(*d, s);
    a.q = q, a.k = k, a.v = v, a.dout = dout, a.dq = dq, a.dk = dk, a.dv = dv, a.u = u, a.feat = feat;
    a.den = const_cast<double*>(den);
    a.phq = reinterpret_cast<const double*>(base + lay.phq);
    a.phk = reinterpret_cast<const double*>(base + lay.phk);
    a.dpre_q = reinterpret_cast<double*>(base + lay.dpre_q);
    a.dpre_k = reinterpret_cast<double*>(base + lay.dpre_k);
    a.goo = reinterpret_cast<double*>(base + lay.goo);
    a.rowsum = reinterpret_cast<double*>(bb + bl.rowsum);
    a.colsum = reinterpret_cast<double*>(bb + bl.colsum);
    const size_t BL = (size_t)d->batch * d->seq_len;
    SKB_CHECK_CUDA(cudaMemsetAsync(a.rowsum, 0, BL * sizeof(double), st));
    SKB_CHECK_CUDA(cudaMemsetAsync(a.colsum, 0, BL * sizeof(double), st));
    const int p = (int)d->head_dim, H = (int)d->heads;
    SKB_CHECK_CUDA(cudaMemsetAsync(dfeat, 0, (size_t)H * p * p * sizeof(double), st));
    const dim3 g((unsigned)skb::cdiv(d->seq_len, skb::kLmWarps), (unsigned)H, (unsigned)d->batch);
    const int64_t rows = d->batch * d->seq_len;
    const int rows_per = 1024;
    const dim3 gf((unsigned)H, (unsigned)p, (unsigned)skb::cdiv(rows, rows_per));
    skb::dispatch_lm(d->dtype, [&](auto tag) {
        using S = std::remove_const_t<std::remove_pointer_t<decltype(tag)>>;
        skb::k_linmix_bwd_q<S><<<g, skb::kLmWarps * 32, 0, st>>>(a);
        skb::k_linmix_bwd_k<S><<<g, skb::kLmWarps * 32, 0, st>>>(a);
        skb::k_dfeat<S><<<gf, 128, 0, st>>>(a, dfeat, rows_per);
    });
    SKB_CHECK_LAUNCH();
    skb::run_jvp(*d, u, s, a.rowsum, a.colsum, reinterpret_cast<double*>(bb + bl.mean_prefix),
                 reinterpret_cast<double*>(bb + bl.chunk_sums), du, st);
    LM_END
}

}  // extern "C"
