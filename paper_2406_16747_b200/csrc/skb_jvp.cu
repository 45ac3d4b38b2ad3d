// Selection pullback (proj/src/attention.cpp:447-479) in O(L log L).
//
// Reference: for every query i (push time t = i - w) with S_t = {j <= t :
// 0 < u_j - tau_t < 1}, mean_t = (sum of head-summed gate gradients gm_tj over
// j in S_t n Sel_t) / |S_t|, and gu_j += gm_tj - mean_t for j in S_t — O(L)
// per query, O(L^2) overall.
//
// Here the attention backward already produced rowsum_t (the numerator) and
// colsum_j = sum_t gm_tj over the same fractional entries. Because tau_t never
// decreases, {t : j in S_t} is one interval [max(j, t_c), t_a) found by binary
// search with the reference's own predicate (u_j - tau_t > 0, u_j - tau_t < 1),
// so gu_j = colsum_j - (M[t_a] - M[t_c]) with M the prefix sums of mean_t.
#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

namespace {

__device__ __forceinline__ double mean_at(const double* rs, const int* nf, const double* tb, int t) {
    const int n = nf[t];
    return (n > 0 && tb[t] > -INFINITY) ? rs[t] / (double)n : 0.0;
}

// Sum of mean_t over every 1024-push chunk (the first level of k_mean_prefix).
__global__ void __launch_bounds__(1024)
k_mean_chunk_sums(const double* __restrict__ rowsum, const int* __restrict__ nfrac,
                  const double* __restrict__ tau, int L, int T, double* __restrict__ csum) {
    __shared__ double wsum[32];
    const int b = blockIdx.y, t = blockIdx.x * 1024 + threadIdx.x;
    const int64_t bl = (int64_t)b * L;
    double s = warp_sum(t < T ? mean_at(rowsum + bl, nfrac + bl, tau + bl, t) : 0.0);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < 32; ++w) tot += wsum[w];
        csum[(int64_t)b * gridDim.x + blockIdx.x] = tot;
    }
}

// M[t] = sum_{t' < t} mean_t' per sequence (M[T] = total): one CTA per 1024
// push times; each adds the chunk sums before it (O(T / 1024) loads) and
// scans its chunk, so no CTA waits on another.
__global__ void __launch_bounds__(1024)
k_mean_prefix(const double* __restrict__ rowsum, const int* __restrict__ nfrac,
              const double* __restrict__ tau, int L, int T, const double* __restrict__ csum,
              double* __restrict__ M) {
    __shared__ double wsum[32];
    const int b = blockIdx.y, c0 = blockIdx.x * 1024;
    const double* rs = rowsum + (int64_t)b * L;
    const int* nf = nfrac + (int64_t)b * L;
    const double* tb = tau + (int64_t)b * L;
    double* Mb = M + (int64_t)b * (L + 1);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double* cs = csum + (int64_t)b * gridDim.x;
    double pre = 0.0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += 1024) pre += cs[c];
    pre = warp_sum(pre);
    if (lane == 0) wsum[wid] = pre;
    __syncthreads();
    double before = 0.0;
    for (int w = 0; w < 32; ++w) before += wsum[w];
    __syncthreads();
    const int t = c0 + threadIdx.x;
    const double x = t < T ? mean_at(rs, nf, tb, t) : 0.0;
    double incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    for (int w = 0; w < wid; ++w) before += wsum[w];
    if (t < T) Mb[t] = before + incl - x;
    if (t == T - 1) Mb[T] = before + incl;
    if (T == 0 && blockIdx.x == 0 && threadIdx.x == 0) Mb[0] = 0.0;
}

__global__ void k_jvp(const double* __restrict__ u, const double* __restrict__ tau,
                      const double* __restrict__ colsum, const double* __restrict__ M, int L, int T,
                      int w, int chunk_len, double* __restrict__ du) {
    const int b = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= L) return;
    const int64_t bl = (int64_t)b * L;
    if (j >= T) {
        du[bl + j] = 0.0;
        return;
    }
    const double uj = u[bl + j];
    const double* tb = tau + bl;
    // t_c: first t in [j, T) with uj - tau_t < 1 (false -> true as tau grows)
    int lo = j, hi = T;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (uj - tb[mid] < 1.0) hi = mid;
        else lo = mid + 1;
    }
    const int tc = lo;
    // t_a: first t in [j, T) with !(uj - tau_t > 0)
    lo = j;
    hi = T;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (!(uj - tb[mid] > 0.0)) hi = mid;
        else lo = mid + 1;
    }
    int ta = lo;
    // chunk-wise training: only queries of j's own chunk (i < chunk end, i.e.
    // t < chunk end - w) spread gradient to j (proj/src/attention.cpp:472)
    if (chunk_len > 0) ta = min(ta, max(j, (j / chunk_len + 1) * chunk_len - w));
    const double* Mb = M + (int64_t)b * (L + 1);
    const double sub = tc < ta ? Mb[ta] - Mb[tc] : 0.0;
    du[bl + j] = colsum[bl + j] - sub;
}

}  // namespace

void bwd_layout(const skb_attn_desc& d, BwdLayout& o) {
    const uint64_t BL = (uint64_t)d.batch * d.seq_len;
    const uint64_t N = BL * d.heads * d.head_dim;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t r = off;
        off = (off + bytes + 255) & ~uint64_t(255);
        return r;
    };
    o.rowsum = take(BL * 8);
    o.colsum = take(BL * 8);
    o.mean_prefix = take((BL + d.batch) * 8);
    o.chunk_sums = take((uint64_t)d.batch * ((d.seq_len + 1023) / 1024) * 8);
    const bool tc = d.dtype == SKB_BF16 && tc_supported(d) && !(d.flags & SKB_FLAG_FORCE_GATHER);
    // gather backward: fp64 dK/dV accumulators; tensor-core backward: fp32
    // partials of the selected pass + lse2/delta rows in the dq_acc region
    // (the bf16 partials are stored in 32-key groups, skb_attn_tc_bwd.cu part_off)
    const uint64_t N32 = (uint64_t)d.batch * ((d.seq_len + 31) / 32 * 32) * d.heads * d.head_dim;
    o.dk_acc = take(tc ? N32 * 2 : N * 8);
    o.dv_acc = take(tc ? N32 * 2 : N * 8);
    o.dq_acc = take(tc ? BL * d.heads * 8 : 0);
    // per 128-entry tile of the ever-selected list: {first query tile, query tiles}
    o.sel_items = take(tc ? (uint64_t)d.batch * ((d.seq_len + 127) / 128) * 8 : 0);
    // the ever-selected keys grouped by leave time (k_sel_order)
    o.sel_order = take(tc ? BL * 4 : 0);
    // fused dQ (D = 128): the fp32 dS K accumulator the key-major passes reduce into
    o.dq32 = take(tc && d.head_dim == 128 ? N * 4 : 0);
    // unified key-major pass: the query end of every contiguous 128-key tile
    o.uni_hi = take(tc ? (uint64_t)d.batch * ((d.seq_len + 127) / 128) * 4 : 0);
    o.total = off;
}

void run_jvp(const skb_attn_desc& d, const double* u, const SelView& s, const double* rowsum,
             const double* colsum, double* mean_prefix, double* chunk_sums, double* du, cudaStream_t st) {
    const int B = (int)d.batch, L = (int)d.seq_len;
    const int T = std::max(0, L - (int)d.window);
    if (floor_k(d.k) < 1 || T == 0) {
        SKB_CHECK_CUDA(cudaMemsetAsync(du, 0, (size_t)B * L * sizeof(double), st));
        return;
    }
    const dim3 gc((unsigned)std::max<int64_t>(1, cdiv(T, 1024)), (unsigned)B);
    k_mean_chunk_sums<<<gc, 1024, 0, st>>>(rowsum, s.nfrac, s.tau, L, T, chunk_sums);
    k_mean_prefix<<<gc, 1024, 0, st>>>(rowsum, s.nfrac, s.tau, L, T, chunk_sums, mean_prefix);
    SKB_CHECK_LAUNCH();
    dim3 g((unsigned)cdiv(L, 256), B);
    k_jvp<<<g, 256, 0, st>>>(u, s.tau, colsum, mean_prefix, L, T, (int)d.window, (int)d.chunk_len, du);
    SKB_CHECK_LAUNCH();
}

}  // namespace skb
