// K3/K4 gather path on CUDA cores: one warp per (sequence, query, head).
//
// This is the exact-precision path (F32 computes in fp32 with fp64 gradient
// accumulation, F64 in fp64) used for parity against the reference's float and
// double instantiations, and the coalesced gather fallback for shapes the
// tensor-core kernels do not cover. Keys come from the per-block union list
// (selected, masked by j <= t < leave_j) followed by the contiguous window.
//
// Forward  = proj/src/cache.cpp:358-393 (logits, max-subtracted softmax over
//            Sel U window, value gates, no renormalisation; maxa/denom -> lse).
// Backward = proj/src/attention.cpp:265-316 (b_j, s, c_j, dq/dk/dv, gate
//            gradient gm summed over heads) — gm restricted to the fractional
//            support feeds the selection pullback (attention.cpp:447-479) via
//            per-query row sums and per-key column sums.
#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

namespace {

constexpr int kWarps = 8;
constexpr int kMaxPerLane = 8;  // head_dim <= 256

template <class S>
struct Acc {
    using C = float;
};
template <>
struct Acc<double> {
    using C = double;
};

template <class S>
__device__ __forceinline__ typename Acc<S>::C ldv(const S* p) {
    return (typename Acc<S>::C)p[0];
}
template <>
__device__ __forceinline__ float ldv<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(p[0]);
}
template <class S, class C>
__device__ __forceinline__ void stv(S* p, C v) {
    p[0] = (S)v;
}
template <>
__device__ __forceinline__ void stv<__nv_bfloat16, float>(__nv_bfloat16* p, float v) {
    p[0] = __float2bfloat16(v);
}

struct Args {
    const void *q, *k, *v, *dout;
    void *o, *dq, *dk, *dv;
    double *dk_acc, *dv_acc;
    const double* u;
    double* lse;
    SelView s;
    double *rowsum, *colsum;
    int B, L, H, p, w, T, R1;
    double scale;
    int key_soft, mask_st;
    int chunk_len;  // 0 = one chunk
};

__device__ __forceinline__ double gate_of(double uj, double tau) {
    double g = uj - tau;
    return g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g);
}

template <class S>
__global__ void __launch_bounds__(kWarps * 32) k_fwd_gather(Args a) {
    using C = typename Acc<S>::C;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = blockIdx.x * kWarps + warp, h = blockIdx.y, b = blockIdx.z;
    if (i >= a.L) return;
    const int64_t rs = (int64_t)a.H * a.p;
    const S* Q = static_cast<const S*>(a.q);
    const S* K = static_cast<const S*>(a.k);
    const S* V = static_cast<const S*>(a.v);
    const int np = (a.p + 31) / 32;
    C qv[kMaxPerLane], acc[kMaxPerLane];
    const S* qrow = Q + ((int64_t)b * a.L + i) * rs + (int64_t)h * a.p;
#pragma unroll
    for (int m = 0; m < kMaxPerLane; ++m) {
        const int c = lane + 32 * m;
        qv[m] = (m < np && c < a.p) ? ldv<S>(qrow + c) : C(0);
        acc[m] = C(0);
    }
    C mx = -INFINITY, den = C(0);
    const C scale = (C)a.scale;

    auto process = [&](int j, double g, bool sel) {
        const S* krow = K + ((int64_t)b * a.L + j) * rs + (int64_t)h * a.p;
        const S* vrow = V + ((int64_t)b * a.L + j) * rs + (int64_t)h * a.p;
        C part = C(0);
#pragma unroll
        for (int m = 0; m < kMaxPerLane; ++m) {
            const int c = lane + 32 * m;
            if (m < np && c < a.p) part += qv[m] * ldv<S>(krow + c);
        }
        const C dot = warp_sum(part);
        C aj = scale * dot;
        if (a.key_soft && sel) aj *= (C)g;
        const C wv = (sel && !a.mask_st) ? (C)g : C(1);
        if (aj > mx) {
            const C corr = exp(mx - aj);
            den *= corr;
#pragma unroll
            for (int m = 0; m < kMaxPerLane; ++m) acc[m] *= corr;
            mx = aj;
        }
        const C e = exp(aj - mx);
        den += e;
        const C ew = e * wv;
#pragma unroll
        for (int m = 0; m < kMaxPerLane; ++m) {
            const int c = lane + 32 * m;
            if (m < np && c < a.p) acc[m] += ew * ldv<S>(vrow + c);
        }
    };

    const int t = i - a.w;
    const int64_t bl = (int64_t)b * a.L;
    if (t >= 0 && a.R1 > 0) {
        const double tau = a.s.tau[bl + t];
        const int qb = i / kQBlock;
        const int cnt = a.s.qb_count[(int64_t)b * a.s.nqb + qb];
        const int* list = a.s.qb_list + ((int64_t)b * a.s.nqb + qb) * a.s.qb_cap;
        for (int e = 0; e < cnt; ++e) {
            const int j = list[e];  // the union is partitioned by tile class, not sorted
            if (j > t || a.s.leave[bl + j] <= t) continue;
            process(j, gate_of(a.u[bl + j], tau), true);
        }
    }
    if (a.w > 0) {
        for (int j = max(0, i - a.w + 1); j <= i; ++j) process(j, 1.0, false);
    } else if (a.s.leave[bl + i] <= i) {
        process(i, 1.0, false);  // w == 0: the query reads itself unless selected
    }
    S* orow = static_cast<S*>(a.o) + (bl + i) * rs + (int64_t)h * a.p;
    const C inv = C(1) / den;
#pragma unroll
    for (int m = 0; m < kMaxPerLane; ++m) {
        const int c = lane + 32 * m;
        if (m < np && c < a.p) stv<S, C>(orow + c, acc[m] * inv);
    }
    if (lane == 0) a.lse[((int64_t)b * a.H + h) * a.L + i] = (double)mx + log((double)den);
}

template <class S>
__global__ void __launch_bounds__(kWarps * 32) k_bwd_gather(Args a) {
    using C = typename Acc<S>::C;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = blockIdx.x * kWarps + warp, h = blockIdx.y, b = blockIdx.z;
    if (i >= a.L) return;
    const int64_t rs = (int64_t)a.H * a.p;
    const S* Q = static_cast<const S*>(a.q);
    const S* K = static_cast<const S*>(a.k);
    const S* V = static_cast<const S*>(a.v);
    const S* DO = static_cast<const S*>(a.dout);
    const int np = (a.p + 31) / 32;
    const int64_t bl = (int64_t)b * a.L;
    const int64_t qoff = (bl + i) * rs + (int64_t)h * a.p;
    C qv[kMaxPerLane], gv[kMaxPerLane];
    double dqa[kMaxPerLane];
#pragma unroll
    for (int m = 0; m < kMaxPerLane; ++m) {
        const int c = lane + 32 * m;
        const bool ok = m < np && c < a.p;
        qv[m] = ok ? ldv<S>(Q + qoff + c) : C(0);
        gv[m] = ok ? ldv<S>(DO + qoff + c) : C(0);
        dqa[m] = 0.0;
    }
    const double lse = a.lse[((int64_t)b * a.H + h) * a.L + i];
    const C scale = (C)a.scale;
    const int t = i - a.w;
    const double tau = (t >= 0 && a.R1 > 0) ? a.s.tau[bl + t] : -INFINITY;

    // returns (p, b, dot) for key j
    auto eval = [&](int j, double g, bool sel, double& pj, double& bj, double& dotj) {
        const int64_t ko = (bl + j) * rs + (int64_t)h * a.p;
        C pk = C(0), pv = C(0);
#pragma unroll
        for (int m = 0; m < kMaxPerLane; ++m) {
            const int c = lane + 32 * m;
            if (m < np && c < a.p) {
                pk += qv[m] * ldv<S>(K + ko + c);
                pv += gv[m] * ldv<S>(V + ko + c);
            }
        }
        const C dot = warp_sum(pk);
        const double bsum = (double)warp_sum(pv);
        C aj = scale * dot;
        if (a.key_soft && sel) aj *= (C)g;
        pj = (double)exp((C)((double)aj - lse));
        bj = bsum;
        dotj = (double)dot;
    };

    // Iterate the attended keys in a fixed order; `fn(j, g, sel)`.
    auto for_keys = [&](auto&& fn) {
        if (t >= 0 && a.R1 > 0) {
            const int qb = i / kQBlock;
            const int cnt = a.s.qb_count[(int64_t)b * a.s.nqb + qb];
            const int* list = a.s.qb_list + ((int64_t)b * a.s.nqb + qb) * a.s.qb_cap;
            for (int e = 0; e < cnt; ++e) {
                const int j = list[e];  // partitioned by tile class, not sorted
                if (j > t || a.s.leave[bl + j] <= t) continue;
                fn(j, gate_of(a.u[bl + j], tau), true);
            }
        }
        if (a.w > 0) {
            for (int j = max(0, i - a.w + 1); j <= i; ++j) fn(j, 1.0, false);
        } else if (a.s.leave[bl + i] <= i) {
            fn(i, 1.0, false);
        }
    };

    // chunk-wise training: keys left of this query's chunk start receive no
    // gradient (proj/src/attention.cpp:228-234, 284-300, 472)
    const int cs = a.chunk_len > 0 ? (i / a.chunk_len) * a.chunk_len : 0;
    // pass 1: s = sum p wv b; dv; gm (value path)
    double s = 0.0, gsum = 0.0;
    for_keys([&](int j, double g, bool sel) {
        double pj, bj, dotj;
        eval(j, g, sel, pj, bj, dotj);
        const double wv = (sel && !a.mask_st) ? g : 1.0;
        s += pj * wv * bj;
        if (j < cs) return;
        const double c0 = pj * wv;
        double* dvr = a.dv_acc + (bl + j) * rs + (int64_t)h * a.p;
#pragma unroll
        for (int m = 0; m < kMaxPerLane; ++m) {
            const int c = lane + 32 * m;
            if (m < np && c < a.p) atomicAdd(dvr + c, c0 * (double)gv[m]);
        }
    });
    // pass 2: c_j, dq, dk, gm (key path) and the fractional row/column sums
    for_keys([&](int j, double g, bool sel) {
        double pj, bj, dotj;
        eval(j, g, sel, pj, bj, dotj);
        const double wv = (sel && !a.mask_st) ? g : 1.0;
        const double cj = pj * (wv * bj - s);
        const bool gated = a.key_soft && sel;
        const double coef = a.scale * cj * (gated ? g : 1.0);
        const int64_t ko = (bl + j) * rs + (int64_t)h * a.p;
        double* dkr = a.dk_acc + ko;
#pragma unroll
        for (int m = 0; m < kMaxPerLane; ++m) {
            const int c = lane + 32 * m;
            if (m < np && c < a.p) {
                dqa[m] += coef * (double)ldv<S>(K + ko + c);
                if (j >= cs) atomicAdd(dkr + c, coef * (double)qv[m]);
            }
        }
        if (sel) {
            double gm = pj * bj;
            if (gated) gm += a.scale * cj * dotj;
            const double f = a.u[bl + j] - tau;
            if (f > 0.0 && f < 1.0) {
                gsum += gm;
                if (lane == 0 && j >= cs) atomicAdd(a.colsum + bl + j, gm);
            }
        }
    });
    if (lane == 0 && t >= 0 && a.R1 > 0) atomicAdd(a.rowsum + bl + t, gsum);
    S* dqr = static_cast<S*>(a.dq) + qoff;
#pragma unroll
    for (int m = 0; m < kMaxPerLane; ++m) {
        const int c = lane + 32 * m;
        if (m < np && c < a.p) stv<S, C>(dqr + c, (C)dqa[m]);
    }
}

template <class S>
__global__ void k_convert(const double* src, S* dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (S)src[i];
}
template <>
__global__ void k_convert<__nv_bfloat16>(const double* src, __nv_bfloat16* dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = __float2bfloat16((float)src[i]);
}

Args make_args(const skb_attn_desc& d, const SelView& s) {
    Args a{};
    a.s = s;
    a.B = (int)d.batch;
    a.L = (int)d.seq_len;
    a.H = (int)d.heads;
    a.p = (int)d.head_dim;
    a.w = (int)d.window;
    a.T = std::max(0, a.L - a.w);
    a.R1 = (int)floor_k(d.k);
    a.scale = d.scale > 0.0 ? d.scale : 1.0 / std::sqrt((double)d.head_dim);
    a.key_soft = d.key_mode;
    a.mask_st = d.mask_mode;
    a.chunk_len = (int)d.chunk_len;
    return a;
}

}  // namespace

void run_attn_fwd_gather(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                         const double* u, const SelView& s, void* o, double* lse, cudaStream_t st) {
    SKB_REQUIRE(d.head_dim <= 32 * kMaxPerLane, SKB_ESHAPE, "gather path: head_dim must be <= 256");
    Args a = make_args(d, s);
    a.q = q;
    a.k = k;
    a.v = v;
    a.o = o;
    a.u = u;
    a.lse = lse;
    dim3 g((unsigned)cdiv(d.seq_len, kWarps), (unsigned)d.heads, (unsigned)d.batch);
    if (d.dtype == SKB_F64) k_fwd_gather<double><<<g, kWarps * 32, 0, st>>>(a);
    else if (d.dtype == SKB_F32) k_fwd_gather<float><<<g, kWarps * 32, 0, st>>>(a);
    else k_fwd_gather<__nv_bfloat16><<<g, kWarps * 32, 0, st>>>(a);
    SKB_CHECK_LAUNCH();
}

void run_attn_bwd_gather(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                         const void* dout, const double* lse, const double* u, const SelView& s,
                         void* dq, void* dk, void* dv, double* rowsum, double* colsum, void* ws,
                         const BwdLayout& bl, cudaStream_t st) {
    SKB_REQUIRE(d.head_dim <= 32 * kMaxPerLane, SKB_ESHAPE, "gather path: head_dim must be <= 256");
    Args a = make_args(d, s);
    a.q = q;
    a.k = k;
    a.v = v;
    a.dout = dout;
    a.dq = dq;
    a.u = u;
    a.lse = const_cast<double*>(lse);
    a.rowsum = rowsum;
    a.colsum = colsum;
    char* base = static_cast<char*>(ws);
    a.dk_acc = reinterpret_cast<double*>(base + bl.dk_acc);
    a.dv_acc = reinterpret_cast<double*>(base + bl.dv_acc);
    const int64_t n = d.batch * d.seq_len * d.heads * d.head_dim;
    SKB_CHECK_CUDA(cudaMemsetAsync(a.dk_acc, 0, n * sizeof(double), st));
    SKB_CHECK_CUDA(cudaMemsetAsync(a.dv_acc, 0, n * sizeof(double), st));
    dim3 g((unsigned)cdiv(d.seq_len, kWarps), (unsigned)d.heads, (unsigned)d.batch);
    const unsigned cg = (unsigned)cdiv(n, 256);
    if (d.dtype == SKB_F64) {
        k_bwd_gather<double><<<g, kWarps * 32, 0, st>>>(a);
        k_convert<double><<<cg, 256, 0, st>>>(a.dk_acc, static_cast<double*>(dk), n);
        k_convert<double><<<cg, 256, 0, st>>>(a.dv_acc, static_cast<double*>(dv), n);
    } else if (d.dtype == SKB_F32) {
        k_bwd_gather<float><<<g, kWarps * 32, 0, st>>>(a);
        k_convert<float><<<cg, 256, 0, st>>>(a.dk_acc, static_cast<float*>(dk), n);
        k_convert<float><<<cg, 256, 0, st>>>(a.dv_acc, static_cast<float*>(dv), n);
    } else {
        k_bwd_gather<__nv_bfloat16><<<g, kWarps * 32, 0, st>>>(a);
        k_convert<__nv_bfloat16><<<cg, 256, 0, st>>>(a.dk_acc, static_cast<__nv_bfloat16*>(dk), n);
        k_convert<__nv_bfloat16><<<cg, 256, 0, st>>>(a.dv_acc, static_cast<__nv_bfloat16*>(dv), n);
    }
    SKB_CHECK_LAUNCH();
}

}  // namespace skb
