// Block-level building blocks of the SparseK projection solve
// (proj/src/sparsek_op.cpp:36-98): descending bitonic sort, exclusive prefix
// sums, breakpoint bracketing of F(tau) = sum clamp(z - tau, 0, 1) = k and the
// closed form tau = (sum_band z + u - k) / (w - u).
#pragma once

#include "skb_common.cuh"

namespace skb {

__device__ __forceinline__ int n_ge(const double* z, int m, double x) {
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (z[mid] >= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int n_gt(const double* z, int m, double x) {
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (z[mid] > x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
// F(b) over a descending array z with exclusive prefix sums P.
__device__ __forceinline__ double f_at(const double* z, const double* P, int m, double b) {
    const int a = n_ge(z, m, b + 1.0), c = n_gt(z, m, b);
    return (double)a + (P[c] - P[a]) - b * (double)(c - a);
}

template <class T>
__device__ T block_reduce(T v, T* sbuf, bool is_max) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const T ov = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? (ov > v ? ov : v) : (ov < v ? ov : v);
    }
    __syncthreads();
    if (lane == 0) sbuf[wid] = v;
    __syncthreads();
    T r = sbuf[0];
    for (int w = 1; w < nw; ++w) r = is_max ? (sbuf[w] > r ? sbuf[w] : r) : (sbuf[w] < r ? sbuf[w] : r);
    __syncthreads();
    return r;
}

// Descending bitonic sort of z[0..n2), n2 a power of two (pad with -inf).
__device__ inline void bitonic_desc(double* z, int n2) {
    // one thread per compare-exchange pair (n2 / 2 per stage, none idle):
    // pair p -> i = p with a zero bit inserted at jj, partner i | jj
    const int np = n2 >> 1;
    for (int kk = 2; kk <= n2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            for (int p = threadIdx.x; p < np; p += blockDim.x) {
                const int i = ((p & ~(jj - 1)) << 1) | (p & (jj - 1));
                const int ixj = i | jj;
                const double x = z[i], y = z[ixj];
                const bool desc = (i & kk) == 0;
                if (desc ? (x < y) : (x > y)) {
                    z[i] = y;
                    z[ixj] = x;
                }
            }
            __syncthreads();
        }
    }
}

// Exclusive prefix sums P[0..m] of z[0..m) (block-wide; blockDim multiple of 32, <= 1024).
__device__ inline void excl_prefix(const double* z, double* P, int m, double* sbuf32) {
    const int nt = blockDim.x;
    const int per = (m + nt - 1) / nt;
    const int lo = min(m, (int)threadIdx.x * per), hi = min(m, lo + per);
    double s = 0.0;
    for (int i = lo; i < hi; ++i) s += z[i];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) sbuf32[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const double wv = lane < (nt >> 5) ? sbuf32[lane] : 0.0;
        double wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        sbuf32[lane] = wi - wv;
    }
    __syncthreads();
    double run = sbuf32[wid] + incl - s;
    for (int i = lo; i < hi; ++i) {
        P[i] = run;
        run += z[i];
    }
    if (lo < hi && hi == m) P[m] = run;
    if (m == 0 && threadIdx.x == 0) P[0] = 0.0;
    __syncthreads();
}

// Exact tau of the projection over the sorted band (feasible: F(min-1) >= k).
// Non-degenerate: closed form on the bracketing linear piece. Degenerate (an
// all-saturated flat piece): the batch midpoint of [z_(u+1), z_(u) - 1]
// (proj/src/sparsek_op.cpp:61-72). Returns tau; *frac = |band| (0 if degenerate).
__device__ inline double solve_sorted(const double* z, const double* P, int m, double k,
                                      double* sbuf32, int* frac) {
    // Degenerate: integral k and a gap >= 1 below the k-th largest, i.e. the
    // scan's accepted pair is u == w == k (sparsek_op.cpp:61-72).
    {
        const double kr = rint(k);
        if (fabs(kr - k) <= 1e-9 && kr >= 1.0 && kr <= (double)m) {
            const int u = (int)kr;
            const double hi = z[u - 1] - 1.0;
            const double lo = u < m ? z[u] : hi - 1.0;
            if (lo <= hi) {
                *frac = 0;
                return 0.5 * (lo + hi);
            }
        }
    }
    double blo = -INFINITY, bhi = INFINITY;
    for (int i = threadIdx.x; i < 2 * m; i += blockDim.x) {
        const double bp = i < m ? z[i] : z[i - m] - 1.0;
        const double f = f_at(z, P, m, bp);
        if (f >= k) blo = fmax(blo, bp);
        else bhi = fmin(bhi, bp);
    }
    blo = block_reduce<double>(blo, sbuf32, true);
    bhi = block_reduce<double>(bhi, sbuf32, false);
    const double mid = 0.5 * (blo + bhi);
    const int us = n_ge(z, m, mid + 1.0), wsx = n_gt(z, m, mid);
    if (wsx > us) {
        *frac = wsx - us;
        return (P[wsx] - P[us] + (double)us - k) / (double)(wsx - us);
    }
    *frac = 0;
    const double hi = z[us - 1] - 1.0;
    const double lo = us < m ? z[us] : hi - 1.0;
    return 0.5 * (lo + hi);
}

// solve_sorted with the bracketing breakpoints found by a warp-wide 32-ary
// search instead of evaluating F at all 2m breakpoints: F is non-increasing in
// b, so over each descending breakpoint list ({z_i}, {z_i - 1}) the set where
// F >= k is a suffix. Warp 0 searches; the block shares the result.
__device__ inline double solve_sorted_fast(const double* z, const double* P, int m, double k, double* sbuf32,
                                           int* frac) {
    {
        const double kr = rint(k);
        if (fabs(kr - k) <= 1e-9 && kr >= 1.0 && kr <= (double)m) {
            const int u = (int)kr;
            const double hi = z[u - 1] - 1.0;
            const double lo = u < m ? z[u] : hi - 1.0;
            if (lo <= hi) {
                *frac = 0;
                return 0.5 * (lo + hi);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double blo = -INFINITY, bhi = INFINITY;
        for (int list = 0; list < 2; ++list) {
            const double off = list == 0 ? 0.0 : -1.0;
            int lo = 0, hi = m;  // first index in [lo, hi] with F(bp) >= k (m: none)
            while (hi > lo) {
                const int span = hi - lo;
                // span <= 32: lane j probes lo + j; else evenly spaced probes (lane 0: lo)
                const int p = span <= 32 ? lo + min(lane, span - 1) : lo + (int)(((int64_t)span * lane) / 32);
                const bool ge = f_at(z, P, m, z[p] + off) >= k;
                const unsigned bal = __ballot_sync(0xffffffffu, ge);
                if (span <= 32) {
                    const unsigned below = bal & ((span >= 32) ? 0xffffffffu : ((1u << span) - 1u));
                    hi = below ? lo + (__ffs(below) - 1) : hi;
                    lo = hi;
                } else {
                    if (bal & 1u) {
                        hi = lo;
                    } else {
                        const int f = bal ? __ffs(bal) - 1 : 32;  // first probe with F >= k
                        const int plo = lo + (int)(((int64_t)span * (f - 1)) / 32);
                        const int phi = f < 32 ? lo + (int)(((int64_t)span * f) / 32) : hi;
                        lo = plo + 1;
                        hi = phi;
                    }
                }
            }
            if (hi < m) blo = fmax(blo, z[hi] + off);
            if (hi > 0) bhi = fmin(bhi, z[hi - 1] + off);
        }
        if (lane == 0) {
            sbuf32[0] = blo;
            sbuf32[1] = bhi;
        }
    }
    __syncthreads();
    const double blo = sbuf32[0], bhi = sbuf32[1];
    __syncthreads();
    const double mid = 0.5 * (blo + bhi);
    const int us = n_ge(z, m, mid + 1.0), wsx = n_gt(z, m, mid);
    if (wsx > us) {
        *frac = wsx - us;
        return (P[wsx] - P[us] + (double)us - k) / (double)(wsx - us);
    }
    *frac = 0;
    const double hi = z[us - 1] - 1.0;
    const double lo = us < m ? z[us] : hi - 1.0;
    return 0.5 * (lo + hi);
}

}  // namespace skb
