// K2 — prefix SparseK threshold and top-floor(k) retention, fully parallel.
//
// Reference (sequential): every query i pushes position t = i - w into
// StreamState (proj/src/stream.cpp:72-152) and admits it to the min-heap cache
// (proj/src/cache.cpp:136-179); query i then reads Sel_t = the cache and
// tau_t = the stream threshold (cache.cpp:285-294).
//
// B200 restatement (same results, no sequential heap walk over L):
//   1. k_rank_leave  — Sel_t is the top-floor(k) of u_0..u_t by (value desc,
//      index asc) (brute-force oracle proj/tests/test_cache.cpp:84-97). So
//      j is in Sel_t iff j <= t < leave_j, with leave_j = the position of the
//      (R - A_j)-th later element that beats j (A_j = earlier elements that
//      beat it). One thread per j; the sequence is streamed through smem.
//   2. k_tau_chunks  — tau_t for 32 consecutive push times per CTA. Only
//      scores above theta-1 (theta = ceil(k)-th largest of the prefix) can
//      carry weight (tau_t >= theta - 1), so the CTA sorts that band, solves
//      the prefix at the chunk start exactly (breakpoint bracketing + the
//      closed form of proj/src/sparsek_op.cpp:63-98), then replays the
//      stream's own push/scan (stream.cpp:83-151) for its 32 arrivals on one
//      warp, with the sorted band standing in for the heaps.
//   3. k_union_lists — per 128-query block, the ascending union of Sel_t over
//      the block's push times (<= floor(k)+127 keys by irreversibility).
#include <cfloat>

#include <cub/block/block_radix_sort.cuh>

#include "skb_common.cuh"
#include "skb_internal.h"
#include "skb_solve.cuh"

namespace skb {

namespace {

constexpr int kRankThreads = 64;
constexpr int kRankStage = 1024;
constexpr int kTauThreads = 256;
constexpr int kOverflowSlots = 16;
#ifndef SKB_TAU_EXP
#define SKB_TAU_EXP 0
#endif
#ifdef SKB_TRACE_TAU  // phase clocks of the last chunk of sequence 0 (tools/trace_tau.py)
__device__ unsigned long long g_skb_trace_tau[16];
#define TTAU(t0_, T_, ev)                                                                     \
    do {                                                                                     \
        if (threadIdx.x == 0 && blockIdx.y == 0 && (t0_) / kChunk == ((T_) - 1) / kChunk)    \
            g_skb_trace_tau[ev] = clock64();                                                 \
    } while (0)
#else
#define TTAU(t0_, T_, ev) \
    do {                  \
    } while (0)
#endif

// ---------------------------------------------------------------- ranks
// One thread per position j. The sequence streams through shared memory in
// stages; within a stage every thread scans 8 values per step (broadcast
// reads, branch-free counts) and only drops to a per-element walk inside the
// single 8-group where a count crosses its target.
__global__ void __launch_bounds__(kRankThreads)
k_rank_leave(const double* __restrict__ u, int L, int T, int R1, int R2, int* __restrict__ leave1,
             int* __restrict__ leave2) {
    __shared__ __align__(16) double su[kRankStage];
    const int b = blockIdx.y;
    const int j = blockIdx.x * kRankThreads + threadIdx.x;
    const double* ub = u + (int64_t)b * L;
    const bool active = j < T;
    const double uj = active ? ub[j] : 0.0;
    int A = 0, cnt = 0, need1 = 0, need2 = 0;
    int l1 = T, l2 = T;
    bool done = !active, past = false;  // past: A final, counting later beaters
    for (int c0 = 0; c0 < T; c0 += kRankStage) {
        if (__syncthreads_and(done)) break;
        for (int i = threadIdx.x; i < kRankStage; i += kRankThreads) su[i] = c0 + i < T ? ub[c0 + i] : 0.0;
        __syncthreads();
        if (done) continue;
        const int n = min(kRankStage, T - c0);
        int ii = 0;
        if (!past) {
            // earlier elements: count x >= u_j up to j (exclusive)
            const int stop = min(n, j - c0);
            for (; ii + 8 <= stop; ii += 8) {
                const double2 x0 = *reinterpret_cast<const double2*>(su + ii);
                const double2 x1 = *reinterpret_cast<const double2*>(su + ii + 2);
                const double2 x2 = *reinterpret_cast<const double2*>(su + ii + 4);
                const double2 x3 = *reinterpret_cast<const double2*>(su + ii + 6);
                A += (x0.x >= uj) + (x0.y >= uj) + (x1.x >= uj) + (x1.y >= uj) + (x2.x >= uj) + (x2.y >= uj) +
                     (x3.x >= uj) + (x3.y >= uj);
            }
            for (; ii < stop; ++ii) A += su[ii] >= uj;
            if (A >= R2) {  // R2 earlier winners: never in the top R2 (nor the top R1)
                l1 = j;
                l2 = j;
                done = true;
                continue;
            }
            if (stop < n) {  // j lies in this stage
                need1 = R1 - A;
                need2 = R2 - A;
                if (need1 <= 0) l1 = j;
                past = true;
                ii = stop + 1;
            } else {
                continue;
            }
        }
        // later elements: strictly larger values beat j; find the need1-th and need2-th
        auto hit = [&](double x, int i) {
            if (x > uj) {
                ++cnt;
                if (cnt == need1) l1 = i;
                if (cnt == need2) {
                    l2 = i;
                    done = true;
                }
            }
        };
        for (; ii < n && (ii & 7); ++ii) {
            hit(su[ii], c0 + ii);
            if (done) break;
        }
        if (done) continue;
        for (; ii + 8 <= n; ii += 8) {
            const double2 x0 = *reinterpret_cast<const double2*>(su + ii);
            const double2 x1 = *reinterpret_cast<const double2*>(su + ii + 2);
            const double2 x2 = *reinterpret_cast<const double2*>(su + ii + 4);
            const double2 x3 = *reinterpret_cast<const double2*>(su + ii + 6);
            const int g = (x0.x > uj) + (x0.y > uj) + (x1.x > uj) + (x1.y > uj) + (x2.x > uj) + (x2.y > uj) +
                          (x3.x > uj) + (x3.y > uj);
            const int nxt = cnt < need1 ? need1 : need2;
            if (cnt + g >= nxt) {  // a target falls in this group: walk it
                for (int e = 0; e < 8 && !done; ++e) hit(su[ii + e], c0 + ii + e);
                if (done) break;
            } else {
                cnt += g;
            }
        }
        if (done) continue;
        for (; ii < n; ++ii) {
            hit(su[ii], c0 + ii);
            if (done) break;
        }
    }
    if (active) {
        leave1[(int64_t)b * L + j] = l1;
        leave2[(int64_t)b * L + j] = l2;
    }
}

// Two-kernel variant: (1) A_j = #{i < j : u_i >= u_j} with one CTA per
// (64-key block, 1024-score chunk) — the triangle of pairs spread over the whole
// GPU, partial counts added atomically into A; (2) one thread per key finishes
// from A_j: A_j >= R2 leaves at entry, else the later scan for the
// (R1-A_j)-th / (R2-A_j)-th strictly larger score, as in k_rank_leave.
constexpr int kRankChunk = 1024;
constexpr int kRankBeforeThreads = 256;  // keys per CTA sharing one staged score chunk
__global__ void __launch_bounds__(kRankBeforeThreads)
k_rank_before(const double* __restrict__ u, int L, int T, int* __restrict__ A, int klo, int khi) {
    __shared__ __align__(16) double su[kRankChunk];
    const int b = blockIdx.z;
    const int j0 = klo + blockIdx.x * kRankBeforeThreads, c0 = blockIdx.y * kRankChunk;
    if (c0 >= min(khi, j0 + kRankBeforeThreads)) return;  // chunk entirely after the block's keys
    const double* ub = u + (int64_t)b * L;
    const int n = min(kRankChunk, T - c0);
    for (int i = threadIdx.x; i < kRankChunk; i += kRankBeforeThreads) su[i] = i < n ? ub[c0 + i] : 0.0;
    __syncthreads();
    const int j = j0 + threadIdx.x;
    if (j >= khi) return;
    const double uj = ub[j];
    const int stop = min(n, j - c0);
    int cnt = 0, ii = 0;
    for (; ii + 8 <= stop; ii += 8) {
        const double2 x0 = *reinterpret_cast<const double2*>(su + ii);
        const double2 x1 = *reinterpret_cast<const double2*>(su + ii + 2);
        const double2 x2 = *reinterpret_cast<const double2*>(su + ii + 4);
        const double2 x3 = *reinterpret_cast<const double2*>(su + ii + 6);
        cnt += (x0.x >= uj) + (x0.y >= uj) + (x1.x >= uj) + (x1.y >= uj) + (x2.x >= uj) + (x2.y >= uj) +
               (x3.x >= uj) + (x3.y >= uj);
    }
    for (; ii < stop; ++ii) cnt += su[ii] >= uj;
    if (cnt) atomicAdd(A + (int64_t)b * L + j, cnt);
}

// (2) a warp per key: 128 later scores per step (4 coalesced loads per
// lane), ballots and popcounts for the running count of strictly larger
// scores, the target position by a rank search in the crossing ballot.
__global__ void __launch_bounds__(256)
k_rank_after_warp(const double* __restrict__ u, int L, int T, int R1, int R2, int* __restrict__ leave1,
                  int* __restrict__ leave2, int klo, int khi) {
    const int b = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int j = klo + blockIdx.x * 8 + (threadIdx.x >> 5);
    if (j >= khi) return;
    const double* ub = u + (int64_t)b * L;
    const double uj = ub[j];
    const int A = leave1[(int64_t)b * L + j];  // k_rank_before's counts
    int l1 = T, l2 = T;
    if (A >= R2) {  // R2 earlier winners: never in the top R2 (nor the top R1)
        l1 = j;
        l2 = j;
    } else {
        const int need1 = R1 - A, need2 = R2 - A;
        if (need1 <= 0) l1 = j;
        int cnt = 0;
        bool got1 = need1 <= 0;
        // the position of the r-th (1-based) set bit of m
        auto nth = [](unsigned m, int r) {
            for (int k = 1; k < r; ++k) m &= m - 1;
            return __ffs(m) - 1;
        };
        for (int i0 = j + 1; i0 < T; i0 += 128) {
            double x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = i0 + q * 32 + lane;
                x[q] = i < T ? __ldg(ub + i) : -CUDART_INF;
            }
            bool fin = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned m = __ballot_sync(0xffffffffu, x[q] > uj);
                const int c = __popc(m);
                if (!got1 && cnt + c >= need1) {
                    l1 = i0 + q * 32 + nth(m, need1 - cnt);
                    got1 = true;
                }
                if (cnt + c >= need2) {
                    l2 = i0 + q * 32 + nth(m, need2 - cnt);
                    fin = true;
                    break;
                }
                cnt += c;
            }
            if (fin) break;
        }
    }
    if (lane == 0) {
        leave1[(int64_t)b * L + j] = l1;
        leave2[(int64_t)b * L + j] = l2;
    }
}

// ---------------------------------------------------------------- tau
struct TauArgs {
    const double* u;
    const int* leave2;
    double* tau;
    int* nfrac;
    int* ovf_count;  // [1]
    int* ovf_items;  // [B * nchunks]
    int* ovf_flag;   // [B * nchunks] pass-1 overflow marks (segmented pass 2)
    double* scratch;
    int64_t scratch_stride;
    int L, T, R2;
    double k;
    int cap;  // power of two, smem capacity for the band
    int nch;  // chunks per sequence (all of them; a launch may cover a range)
    int c_off, c_end;  // this launch's chunk range [c_off, c_end)
};

__device__ void tau_chunk_tail(const TauArgs& a, int b, int chunk, const double* bz, double* P, int mcount,
                               double* red_d);

// The band of push time t0: every prefix score above theta(t0) - 1, sorted
// descending into bz. Returns its size, or -1 (nothing written) above `cap`.
// Bands of <= 2048 scores (the first pass) are sorted by a block radix sort
// (256 threads x 8 keys) whose scratch aliases the prefix-sum array P; wider
// bands (the large-cap passes) by the shared-memory bitonic sort.
constexpr int kRadixItems = 8;
#ifndef SKB_TAU_RADIX_BITS
#define SKB_TAU_RADIX_BITS 4
#endif
using BandSort = cub::BlockRadixSort<double, kTauThreads, kRadixItems, cub::NullType, SKB_TAU_RADIX_BITS>;
constexpr int kRadixMax = kTauThreads * kRadixItems;
// the segmented pass sorts bands up to 8192 keys with 32 keys per thread; its
// scratch aliases P, sized max(cap_big doubles, this)
constexpr size_t kBigSortBytes =
    sizeof(cub::BlockRadixSort<double, kTauThreads, 32, cub::NullType, SKB_TAU_RADIX_BITS>::TempStorage);
// narrower bands take a sort with fewer keys per thread (the passes cost the
// same per key slot, so an 8-slot sort of a 400-key band is mostly padding)
template <int ITEMS>
__device__ __forceinline__ void band_radix_sort(double* bz, int mcount, void* sort_tmp) {
    using Sort = cub::BlockRadixSort<double, kTauThreads, ITEMS, cub::NullType, SKB_TAU_RADIX_BITS>;
    // (callers: ITEMS <= 8 alias the first pass's P (>= cap + 1 doubles), 32 the
    // segmented pass's P (kRadixBig doubles))
    static_assert(ITEMS > 8 || sizeof(typename Sort::TempStorage) <= sizeof(BandSort::TempStorage), "scratch");
    double keys[ITEMS];
#pragma unroll
    for (int e = 0; e < ITEMS; ++e) {
        const int idx = threadIdx.x * ITEMS + e;
        keys[e] = idx < mcount ? bz[idx] : -CUDART_INF;
    }
    Sort(*static_cast<typename Sort::TempStorage*>(sort_tmp)).SortDescending(keys);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < ITEMS; ++e) {
        const int idx = threadIdx.x * ITEMS + e;
        if (idx < mcount) bz[idx] = keys[e];
    }
    __syncthreads();
}

#ifndef SKB_TAU_SCAN_ILP  // prefix loads in flight per thread in the band scans
#define SKB_TAU_SCAN_ILP 8
#endif
constexpr int kScanILP = SKB_TAU_SCAN_ILP;
template <bool BIG = false>
__device__ int tau_band(const TauArgs& a, int b, int t0, double* bz, int cap, double* red_d,
                        void* sort_tmp = nullptr) {
    __shared__ int s_m;
    const double* ub = a.u + (int64_t)b * a.L;
    const int* lv = a.leave2 + (int64_t)b * a.L;

    TTAU(t0, a.T, 0);
    // theta = R2-th largest of prefix [0, t0): min over j < t0 still in the top R2 at t0-1.
    double theta = -CUDART_INF;
    if (t0 >= a.R2 && a.R2 > 0) {
        double mn = CUDART_INF;
        // 4 independent load pairs in flight per thread (the pass is latency-bound)
        for (int j0 = threadIdx.x; j0 < t0; j0 += kScanILP * blockDim.x) {
            int lvv[kScanILP];
            double uv[kScanILP];
#pragma unroll
            for (int q = 0; q < kScanILP; ++q) {
                const int j = j0 + q * blockDim.x;
                lvv[q] = j < t0 ? lv[j] : -1;
                uv[q] = j < t0 ? ub[j] : CUDART_INF;
            }
#pragma unroll
            for (int q = 0; q < kScanILP; ++q)
                if (lvv[q] >= t0) mn = fmin(mn, uv[q]);
        }
        theta = block_reduce<double>(mn, red_d, false);
    }
    const double cut = theta - 1.0;
    TTAU(t0, a.T, 1);
    if (threadIdx.x == 0) s_m = 0;
    __syncthreads();
    // one pass: warp-aggregated slots, stores only below the cap (an oversized
    // band is reported after the pass; the order is irrelevant, bz is sorted next)
    const int lane = threadIdx.x & 31;
    for (int j0 = 0; j0 < t0; j0 += kScanILP * blockDim.x) {
        double xv[kScanILP];
#pragma unroll
        for (int q = 0; q < kScanILP; ++q) {
            const int j = j0 + q * blockDim.x + threadIdx.x;
            xv[q] = j < t0 ? ub[j] : -CUDART_INF;
        }
#pragma unroll
        for (int q = 0; q < kScanILP; ++q) {
            const double x = xv[q];
            const bool p = x > cut;
            const unsigned m = __ballot_sync(0xffffffffu, p);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(&s_m, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            const int slot = base + __popc(m & ((1u << lane) - 1u));
            if (p && slot < cap) bz[slot] = x;
        }
    }
    __syncthreads();
    const int mcount = s_m;
    __syncthreads();
    TTAU(t0, a.T, 2);
    if (mcount > cap) return -1;
    if (sort_tmp != nullptr && mcount <= kRadixMax && blockDim.x == kTauThreads) {
        if (mcount <= kTauThreads * 2) band_radix_sort<2>(bz, mcount, sort_tmp);
        else if (mcount <= kTauThreads * 3) band_radix_sort<3>(bz, mcount, sort_tmp);
        else if (mcount <= kTauThreads * 4) band_radix_sort<4>(bz, mcount, sort_tmp);
        else if (mcount <= kTauThreads * 5) band_radix_sort<5>(bz, mcount, sort_tmp);
        else if (mcount <= kTauThreads * 6) band_radix_sort<6>(bz, mcount, sort_tmp);
        else band_radix_sort<kRadixItems>(bz, mcount, sort_tmp);
        TTAU(t0, a.T, 3);
        return mcount;
    }
    if constexpr (BIG) {
        if (sort_tmp != nullptr && mcount <= kTauThreads * 32 && blockDim.x == kTauThreads) {
            band_radix_sort<32>(bz, mcount, sort_tmp);  // wide bands (the segmented pass)
            TTAU(t0, a.T, 3);
            return mcount;
        }
    }
    int n2 = 1;
    while (n2 < mcount) n2 <<= 1;
    __syncthreads();
    for (int i = mcount + threadIdx.x; i < n2; i += blockDim.x) bz[i] = -CUDART_INF;
    __syncthreads();
    bitonic_desc(bz, n2);
    TTAU(t0, a.T, 3);
    return mcount;
}

// One chunk: band collection, sort, exact solve at the chunk start, stream replay.
// Returns false (without writing outputs) when the band exceeds `cap`.
__device__ bool tau_chunk(const TauArgs& a, int b, int chunk, double* bz, double* P, int cap,
                          bool probe_only_if_overflow) {
    __shared__ double red_d[32];
    (void)probe_only_if_overflow;
    // the radix sort's scratch aliases P (written only after the sort)
    const int mcount = tau_band(a, b, chunk * kChunk, bz, cap, red_d, probe_only_if_overflow ? nullptr : P);
    if (mcount < 0) return false;
    tau_chunk_tail(a, b, chunk, bz, P, mcount, red_d);
    return true;
}

// Exact state at the chunk start from the sorted band bz[0, mcount), then the
// stream's own push/scan for the chunk's arrivals.
__device__ void tau_chunk_tail(const TauArgs& a, int b, int chunk, const double* bz, double* P, int mcount,
                               double* red_d) {
    const int t0 = chunk * kChunk;
    const double* ub = a.u + (int64_t)b * a.L;
    excl_prefix(bz, P, mcount, red_d);
    TTAU(t0, a.T, 4);

    // exact state after pushes [0, t0)
    double tau0 = -CUDART_INF;
    int ws = mcount, uf = mcount;
    if ((double)t0 >= a.k && mcount > 0) {
        int frac0;
#if SKB_TAU_EXP == 2
        tau0 = bz[0] - 1.0;  // experiment: no exact solve
        frac0 = 0;
#else
        tau0 = solve_sorted_fast(bz, P, mcount, a.k, red_d, &frac0);
#endif
        ws = n_gt(bz, mcount, tau0);
        uf = n_ge(bz, mcount, tau0 + 1.0);
    }
    TTAU(t0, a.T, 5);

    // stream replay (proj/src/stream.cpp:72-152) for the chunk's arrivals. The
    // survivors are the sorted band prefix bz[0, ws) plus chunk entries; the
    // chunk's <= 32 values are ranked once (value desc, earlier arrival first,
    // i.e. heap order reversed) so set membership is a bitmask and the minima
    // are bit scans — one thread, no shuffles per pop.
    __shared__ double s_cv[kChunk];
    __shared__ int s_rank[kChunk];
    const int nvalid = min(kChunk, a.T - t0);
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const double cz = lane < nvalid ? ub[t0 + lane] : -CUDART_INF;
        int rank = 0;
        for (int e = 0; e < nvalid; ++e) {
            const double y = __shfl_sync(0xffffffffu, cz, e);
            rank += (y > cz) || (y == cz && e < lane);
        }
        if (lane < nvalid) {
            s_cv[rank] = cz;
            s_rank[lane] = rank;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && SKB_TAU_EXP != 1) {  // (experiment 1: no replay)
        uint32_t smask = 0, fmask = 0;
        double tau = tau0;
        double sum_s = P[ws], sum_f = P[uf];
        int frac = (tau0 > -CUDART_INF) ? ws - uf : 0;
        for (int e = 0; e < nvalid; ++e) {
            const int t = t0 + e;
            const int rk = s_rank[e];
            const double z = s_cv[rk];
            const double count = (double)(t + 1);
            if (z > tau) {
                smask |= 1u << rk;
                sum_s += z;
                if (z >= tau + 1.0) {
                    fmask |= 1u << rk;
                    sum_f += z;
                }
                if (count < a.k) {
                    tau = -CUDART_INF;
                    frac = 0;
                } else {
                    bool popped = false;
                    double last = 0.0;
                    // every iteration pops one entry; the guard only bounds a
                    // numerically broken input (NaN sums) so the GPU never hangs
                    for (int guard = 2 * (mcount + kChunk) + 8; guard > 0; --guard) {
                        const int cu = uf + __popc(fmask);
                        const int cw = ws + __popc(smask);
                        // minima: chunk entries (later indices) pop first on value ties
                        const int sr = smask ? 31 - __clz(smask) : -1;
                        const int fr = fmask ? 31 - __clz(fmask) : -1;
                        bool s_chunk = sr >= 0 && (ws == 0 || s_cv[sr] <= bz[ws - 1]);
                        bool f_chunk = fr >= 0 && (uf == 0 || s_cv[fr] <= bz[uf - 1]);
                        const double smin = s_chunk ? s_cv[sr] : (ws > 0 ? bz[ws - 1] : CUDART_INF);
                        const double fmn = f_chunk ? s_cv[fr] : (uf > 0 ? bz[uf - 1] : CUDART_INF);
                        if (cu == cw) {
                            const double hi = fmn - 1.0;
                            const double lo = popped ? last : fmax(tau, hi - 1.0);
                            if (fabs((double)cu - a.k) <= 1e-9) {
                                tau = fmax(tau, 0.5 * (lo + hi));
                                frac = 0;
                                break;
                            }
                            sum_f -= fmn;
                            if (f_chunk) fmask &= ~(1u << fr);
                            else --uf;
                            continue;
                        }
                        const double cand = (sum_s - sum_f + (double)cu - a.k) / (double)(cw - cu);
                        if (smin > cand && (cu == 0 || fmn >= cand + 1.0)) {
                            tau = cand;
                            frac = cw - cu;
                            break;
                        }
                        if (cu == 0 || smin <= fmn - 1.0) {
                            last = smin;
                            popped = true;
                            sum_s -= smin;
                            if (s_chunk) smask &= ~(1u << sr);
                            else --ws;
                            if (cw - 1 == 0) break;  // internal guard (reference throws)
                        } else {
                            sum_f -= fmn;
                            if (f_chunk) fmask &= ~(1u << fr);
                            else --uf;
                        }
                    }
                }
            }
            a.tau[(int64_t)b * a.L + t] = tau;
            a.nfrac[(int64_t)b * a.L + t] = frac;
        }
    }
    __syncthreads();
    TTAU(t0, a.T, 6);
}

#ifndef SKB_TAU_MINB  // resident CTAs per SM asked of ptxas for the first tau pass
#define SKB_TAU_MINB 4
#endif
__global__ void __launch_bounds__(kTauThreads, SKB_TAU_MINB) k_tau_chunks(TauArgs a) {
    extern __shared__ double smem[];
    // latest chunks first: their prefixes are the longest (the scans and the
    // band grow with t0), so they must not be left to a trailing partial wave
    const int b = blockIdx.y, chunk = a.c_end - 1 - blockIdx.x;
    double* bz = smem;
    double* P = smem + a.cap;
    if (!tau_chunk(a, b, chunk, bz, P, a.cap, false)) {
        if (threadIdx.x == 0) {
            const int slot = atomicAdd(a.ovf_count, 1);
            a.ovf_items[slot] = b * a.nch + chunk;
            a.ovf_flag[b * a.nch + chunk] = 1;
        }
    }
}

// Pass 2, segmented: a CTA owns kSegChunks consecutive chunks and handles its
// flagged ones from the first to the last. The band is sorted once, at the
// first; each later chunk start merges the previous chunk's <= 32 arrivals in
// (ranked on one warp, placed by binary search), takes theta = the R2-th band
// entry (every top-R2 score exceeds the previous cut, theta never decreases)
// and trims at theta - 1: the same band, hence the same tau, as a fresh sort.
// P1 (the first pass, small cap): every chunk of the segment; past the cap the
// remaining chunks are flagged for pass 2 (large cap, flagged chunks only).
constexpr int kSegChunks = 8;
template <bool P1>
__global__ void __launch_bounds__(kTauThreads) k_tau_segments(TauArgs a, int nchunks, int seg_chunks, int* q2_count,
                                                              int* q2_items) {
    extern __shared__ double smem[];
    __shared__ double red_d[32];
    __shared__ double s_new[kChunk];
    __shared__ int s_lim[2];
    const int b = blockIdx.y, seg = a.c_off / seg_chunks + blockIdx.x;
    const int c_lo = seg * seg_chunks, c_hi = min(min(nchunks, a.c_end), c_lo + seg_chunks);
    int* fl = a.ovf_flag + (int64_t)b * nchunks;
    if (threadIdx.x == 0) {
        int f = -1, l = -1;
        for (int c = c_lo; c < c_hi; ++c)
            if (P1 || fl[c]) {
                if (f < 0) f = c;
                l = c;
            }
        s_lim[0] = f;
        s_lim[1] = l;
    }
    __syncthreads();
    const int cf = s_lim[0], cl = s_lim[1];
    if (cf < 0) return;
    // phase clocks of the segment holding sequence 0's last chunk (tools/trace_tau.py)
    const bool trs = blockIdx.y == 0 && c_lo <= (a.T - 1) / kChunk && (a.T - 1) / kChunk < c_hi;
#define TSEG(ev)                                                      \
    do {                                                              \
        if (trs) TTAU((a.T - 1) / kChunk * kChunk, a.T, ev);          \
    } while (0)
    TSEG(7);
    double* bz = smem;
    double* bz2 = smem + a.cap;
    double* P = smem + 2 * a.cap;
    const double* ub = a.u + (int64_t)b * a.L;
    // the radix scratch aliases P (cap_big doubles), written only after the sort
    int m = tau_band<true>(a, b, cf * kChunk, bz, a.cap, red_d, a.cap >= 8192 ? P : nullptr);
    TSEG(8);
    for (int c = cf; c <= cl; ++c) {
        if (c == cl) TSEG(9);
        if (c > cf) {
            const int tp = (c - 1) * kChunk;
            const int nv = min(kChunk, a.T - tp);
            if (m < 0 || m + nv > a.cap) {
                m = -1;
            } else {
                if (threadIdx.x < 32) {  // the previous chunk's arrivals, descending
                    const int lane = threadIdx.x;
                    const double cz = lane < nv ? ub[tp + lane] : -CUDART_INF;
                    int rank = 0;
                    for (int e = 0; e < nv; ++e) {
                        const double y = __shfl_sync(0xffffffffu, cz, e);
                        rank += (y > cz) || (y == cz && e < lane);
                    }
                    if (lane < nv) s_new[rank] = cz;
                }
                __syncthreads();
                for (int i = threadIdx.x; i < m; i += blockDim.x) bz2[i + n_gt(s_new, nv, bz[i])] = bz[i];
                for (int e = threadIdx.x; e < nv; e += blockDim.x) bz2[e + n_ge(bz, m, s_new[e])] = s_new[e];
                __syncthreads();
                double* t = bz;
                bz = bz2;
                bz2 = t;
                m += nv;
                const int t0 = c * kChunk;
                const double theta = (t0 >= a.R2 && a.R2 > 0) ? bz[a.R2 - 1] : -CUDART_INF;
                m = n_gt(bz, m, theta - 1.0);
            }
        }
        if (c == cl) TSEG(10);
        if (m < 0) {  // beyond the cap: the next pass takes the rest
            if (threadIdx.x == 0)
                for (int cc = c; cc <= cl; ++cc) {
                    if (P1) {  // flag (segmented pass 2) and queue (the global-scratch pass)
                        fl[cc] = 1;
                        a.ovf_items[atomicAdd(a.ovf_count, 1)] = b * nchunks + cc;
                    } else if (fl[cc]) {
                        q2_items[atomicAdd(q2_count, 1)] = b * nchunks + cc;
                    }
                }
            return;
        }
        if (P1 || fl[c]) tau_chunk_tail(a, b, c, bz, P, m, red_d);
    }
}
#undef TSEG

// Second pass over the chunks whose band exceeded the first pass's small
// shared-memory cap, with the large cap; its own overflows go to queue 2.
__global__ void __launch_bounds__(kTauThreads) k_tau_chunks_big(TauArgs a, int nchunks, int* q2_count, int* q2_items) {
    extern __shared__ double smem[];
    const int n = *a.ovf_count;
    double* bz = smem;
    double* P = smem + a.cap;
    for (int it = blockIdx.x; it < n; it += gridDim.x) {
        const int item = a.ovf_items[it];
        if (!tau_chunk(a, item / nchunks, item % nchunks, bz, P, a.cap, false)) {
            if (threadIdx.x == 0) q2_items[atomicAdd(q2_count, 1)] = item;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kTauThreads) k_tau_overflow(TauArgs a, int nchunks, int cap2) {
    const int n = *a.ovf_count;
    double* bz = a.scratch + (int64_t)blockIdx.x * a.scratch_stride;
    double* P = bz + cap2;
    for (int it = blockIdx.x; it < n; it += gridDim.x) {
        const int item = a.ovf_items[it];
        tau_chunk(a, item / nchunks, item % nchunks, bz, P, cap2, true);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- unions
// Ordered block compaction of keys j in [0, t_hi] with leave_j > max(j, t_lo),
// 4 x blockDim keys per step (4 sub-chunks in order; two barriers per step).
__global__ void __launch_bounds__(1024)
k_union_lists(const int* __restrict__ leave1, int L, int T, int window, int nqb, int cap,
              int* __restrict__ qb_count, int* __restrict__ qb_list) {
    __shared__ int wsum[4][32];
    const int b = blockIdx.y, qb = blockIdx.x;
    const int t_lo = qb * kQBlock - window;
    const int t_hi = min(qb * kQBlock + kQBlock - 1 - window, T - 1);
    const int* lv = leave1 + (int64_t)b * L;
    int* out = qb_list + ((int64_t)b * nqb + qb) * cap;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int base = 0;
    const int nt = blockDim.x, nw = nt >> 5;
    for (int j0 = 0; j0 <= t_hi; j0 += 4 * nt) {
        unsigned bal[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = j0 + q * nt + threadIdx.x;
            bool keep = false;
            if (j <= t_hi) {
                const int l = lv[j];
                keep = l > j && l > t_lo;
            }
            bal[q] = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) wsum[q][wid] = __popc(bal[q]);
        }
        __syncthreads();
        int off = base;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int before = 0, tot = 0;
            for (int w = 0; w < nw; ++w) {
                before += w < wid ? wsum[q][w] : 0;
                tot += wsum[q][w];
            }
            if ((bal[q] >> lane) & 1u) {
                const int pos = off + before + __popc(bal[q] & ((1u << lane) - 1u));
                if (pos < cap) out[pos] = j0 + q * nt + threadIdx.x;
            }
            off += tot;
        }
        base = off;
        __syncthreads();
    }
    if (threadIdx.x == 0) qb_count[(int64_t)b * nqb + qb] = min(base, cap);
}

// Kept-key count of every 1024-key chunk (the first level of k_ever_list's scan).
__global__ void __launch_bounds__(1024)
k_ever_chunk_counts(const int* __restrict__ leave1, int L, int T, int* __restrict__ cnt) {
    __shared__ int wsum[32];
    const int b = blockIdx.y, j = blockIdx.x * 1024 + threadIdx.x;
    const int* lv = leave1 + (int64_t)b * L;
    const int c = __syncthreads_count(j < T && lv[j] > j);
    if (threadIdx.x == 0) cnt[(int64_t)b * gridDim.x + blockIdx.x] = c;
    (void)wsum;
}

// Ever-selected keys per sequence, ascending: one CTA per 1024 keys; each
// adds the chunk counts before it (k_ever_chunk_counts: O(T / 1024) loads,
// so the whole scan is O(T + (T / 1024)^2)) and compacts its chunk.
__global__ void __launch_bounds__(1024)
k_ever_list(const int* __restrict__ leave1, int L, int T, const int* __restrict__ chunk_cnt,
            int* __restrict__ ever_count, int* __restrict__ ever_list) {
    __shared__ int wsum[32];
    const int b = blockIdx.y, c0 = blockIdx.x * 1024;
    const int* lv = leave1 + (int64_t)b * L;
    int* out = ever_list + (int64_t)b * L;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int* cc = chunk_cnt + (int64_t)b * gridDim.x;
    int pre = 0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += 1024) pre += cc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    if (lane == 0) wsum[wid] = pre;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < 32; ++w) base += wsum[w];
    __syncthreads();
    const int j = c0 + threadIdx.x;
    const bool keep = j < T && lv[j] > j;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wsum[wid] = __popc(bal);
    __syncthreads();
    int off = base;
    for (int w = 0; w < wid; ++w) off += wsum[w];
    if (keep) out[off + __popc(bal & ((1u << lane) - 1u))] = j;
    if (c0 + 1024 >= T && threadIdx.x == 0) {  // the last chunk: the total
        int tot = base;
        for (int w = 0; w < 32; ++w) tot += wsum[w];
        ever_count[b] = tot;
    }
}

// Per-block metadata for the tensor-core kernels, so their producers issue no
// dependent loads: for every union entry (padded to whole 128-entry tiles with
// key -1) its leave and u, and per tile the fast-path flags.
__global__ void __launch_bounds__(128)
k_union_meta(const int* __restrict__ leave1, const float* __restrict__ uf, const float* __restrict__ tauf,
             int L, int T, int window, int nqb, int cap, const int* __restrict__ qb_count, int* __restrict__ qb_list,
             int* __restrict__ qb_leave, float* __restrict__ qb_uf, int* __restrict__ qb_flags, int part) {
    extern __shared__ int um_keys[];  // [cap] the block's union, partitioned (dynamic; 0 = keep the order)
    __shared__ int cls_tot[4], cls_run[4];
    const int b = blockIdx.y, qb = blockIdx.x;
    const int64_t bl = (int64_t)b * L;
    const int64_t row = (int64_t)b * nqb + qb;
    const int cnt = qb_count[row];
    const int t_lo = qb * kQBlock - window;
    const int t_hi = min(qb * kQBlock + kQBlock - 1 - window, T - 1);
    const float tau_hi = t_hi >= 0 ? tauf[bl + t_hi] : -INFINITY;
    const int ntiles = (cnt + 127) / 128;
    int* list = qb_list + row * cap;
    // Class of an entry: bit 0 = it is valid for every push time of the
    // block (no interval mask), bit 1 = its gate saturates for every query of
    // the block (tau is nondecreasing, so u >= tau_hi + 1 suffices). Entries
    // are stably partitioned by class (both, mask-free, gate-free, neither)
    // so that as many 128-entry tiles as possible take the kernels' fast
    // paths; attention is order-independent over the union.
    auto cls_of = [&](int key) {
        const int lv = leave1[bl + key];
        const bool ok = key <= t_lo && lv > t_hi;
        const bool sat = uf[bl + key] >= tau_hi + 1.f;
        return ok && sat ? 0 : ok ? 1 : sat ? 2 : 3;
    };
    // part: launched with cap ints of dynamic shared memory
    if (part && cnt > 0) {
        if (threadIdx.x < 4) cls_tot[threadIdx.x] = 0, cls_run[threadIdx.x] = 0;
        __syncthreads();
        int mine[4] = {0, 0, 0, 0};
        for (int idx = threadIdx.x; idx < cnt; idx += 128) ++mine[cls_of(list[idx])];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int v = mine[c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((threadIdx.x & 31) == 0 && v) atomicAdd(&cls_tot[c], v);
        }
        __syncthreads();
        const int base[4] = {0, cls_tot[0], cls_tot[0] + cls_tot[1], cls_tot[0] + cls_tot[1] + cls_tot[2]};
        __shared__ int wcnt[4][4];
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int i0 = 0; i0 < cnt; i0 += 128) {
            const int idx = i0 + threadIdx.x;
            const int key = idx < cnt ? list[idx] : -1;
            const int c = key >= 0 ? cls_of(key) : -1;
            unsigned bal[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                bal[q] = __ballot_sync(0xffffffffu, c == q);
                if (lane == 0) wcnt[q][wid] = __popc(bal[q]);
            }
            __syncthreads();
            if (c >= 0) {
                int before = 0;
                for (int w2 = 0; w2 < wid; ++w2) before += wcnt[c][w2];
                um_keys[base[c] + cls_run[c] + before + __popc(bal[c] & ((1u << lane) - 1u))] = key;
            }
            __syncthreads();
            if (threadIdx.x < 4) cls_run[threadIdx.x] += wcnt[threadIdx.x][0] + wcnt[threadIdx.x][1] +
                                                         wcnt[threadIdx.x][2] + wcnt[threadIdx.x][3];
            __syncthreads();
        }
        for (int idx = threadIdx.x; idx < cnt; idx += 128) list[idx] = um_keys[idx];
        __syncthreads();
    }
    for (int t = 0; t < ntiles; ++t) {
        const int idx = t * 128 + threadIdx.x;
        int key = -1, lv = 0;
        float u = 0.f;
        const bool real = idx < cnt;
        if (real) {
            key = list[idx];
            lv = leave1[bl + key];
            u = uf[bl + key];
        } else {
            // padding re-reads the block's first key (a valid row, so the
            // gathers need no bounds check); ext = 0 masks it everywhere
            list[idx] = list[0];
        }
        // the interval mask in one unsigned compare:
        // valid(t) <=> (unsigned)(t - key) < (unsigned)(leave - key); padding: 0
        qb_leave[row * cap + idx] = real ? lv - key : 0;
        qb_uf[row * cap + idx] = u;
        const bool ok = real && key <= t_lo && lv > t_hi;
        const bool sat = !real || u >= tau_hi + 1.f;
        const int all_ok = __syncthreads_and(ok);
        const int all_sat = __syncthreads_and(sat);
        if (threadIdx.x == 0) qb_flags[(row * (cap / 128) + t) * 4] = (all_ok ? 1 : 0) | (all_sat ? 2 : 0);
    }
}

__global__ void k_to_float(const double* __restrict__ u, const double* __restrict__ tau,
                           float* __restrict__ uf, float* __restrict__ tauf, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        uf[i] = (float)u[i];
        tauf[i] = (float)tau[i];
    }
}

__global__ void k_fill_int(int* p, int64_t n, int v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_leave_identity(int* leave, int L) {
    const int b = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < L) leave[(int64_t)b * L + j] = j;
}

__global__ void k_fill_tau(double* tau, int* nfrac, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        tau[i] = -CUDART_INF;
        nfrac[i] = 0;
    }
}

// Maximum of every 1024-push chunk (the first level of k_tau_monotone_chunks).
__global__ void __launch_bounds__(1024) k_tau_chunk_max(const double* __restrict__ tau_in, int L, int T,
                                                        double* __restrict__ cmax) {
    __shared__ double wmax[32];
    const int b = blockIdx.y, t = blockIdx.x * 1024 + threadIdx.x;
    double m = warp_max(t < T ? tau_in[(int64_t)b * L + t] : -CUDART_INF);
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 32; ++w) m = fmax(m, wmax[w]);
        cmax[(int64_t)b * gridDim.x + blockIdx.x] = fmax(m, wmax[0]);
    }
}

// The same running maximum with one CTA per 1024 push times: each CTA reduces
// the chunk maxima before it (O(T / 1024) loads) and scans its chunk, so no
// CTA waits on another. Reads tau_in, writes tau_out (distinct).
__global__ void __launch_bounds__(1024) k_tau_monotone_chunks(const double* __restrict__ tau_in,
                                                              double* __restrict__ tau_out, int L, int T,
                                                              const double* __restrict__ cmax) {
    __shared__ double wmax[32];
    const int b = blockIdx.y, c0 = blockIdx.x * 1024;
    const double* ti = tau_in + (int64_t)b * L;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double* cm = cmax + (int64_t)b * gridDim.x;
    double pre = -CUDART_INF;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += 1024) pre = fmax(pre, cm[c]);
    pre = warp_max(pre);
    if (lane == 0) wmax[wid] = pre;
    __syncthreads();
    double before = -CUDART_INF;
    for (int w = 0; w < 32; ++w) before = fmax(before, wmax[w]);
    __syncthreads();
    const int t = c0 + threadIdx.x;
    const double v = t < T ? ti[t] : -CUDART_INF;
    double incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = fmax(incl, y);
    }
    if (lane == 31) wmax[wid] = incl;
    __syncthreads();
    for (int w = 0; w < wid; ++w) before = fmax(before, wmax[w]);
    if (t < T) tau_out[(int64_t)b * L + t] = fmax(before, incl);
}

// tau_t := max over t' <= t (the stream's tau never decreases, stream.cpp:128;
// chunk-start solves and replays can differ from it by rounding only).
__global__ void __launch_bounds__(1024) k_tau_monotone(double* tau, int L, int T) {
    __shared__ double wmax[32];
    double* tb = tau + (int64_t)blockIdx.x * L;
    const int per = (T + blockDim.x - 1) / blockDim.x;
    const int lo = min(T, (int)threadIdx.x * per), hi = min(T, lo + per);
    double m = -CUDART_INF;
    for (int i0 = lo; i0 < hi; i0 += 8) {  // 8 independent loads in flight
        double x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = i0 + q < hi ? tb[i0 + q] : -CUDART_INF;
#pragma unroll
        for (int q = 0; q < 8; ++q) m = fmax(m, x[q]);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double incl = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = fmax(incl, y);
    }
    if (lane == 31) wmax[wid] = incl;
    __syncthreads();
    double pre = -CUDART_INF;
    for (int w = 0; w < wid; ++w) pre = fmax(pre, wmax[w]);
    double excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = -CUDART_INF;
    double run = fmax(pre, excl);
    for (int i0 = lo; i0 < hi; i0 += 8) {
        double x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = i0 + q < hi ? tb[i0 + q] : -CUDART_INF;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            run = fmax(run, x[q]);
            if (i0 + q < hi) tb[i0 + q] = run;
        }
    }
}

int next_pow2(int x) {
    int n = 1;
    while (n < x) n <<= 1;
    return n;
}

}  // namespace

static uint64_t align256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

void select_layout(const skb_attn_desc& d, skb_select_layout& o) {
    const int64_t B = d.batch, L = d.seq_len;
    const int64_t nqb = cdiv(L, kQBlock);
    const int64_t cap = cdiv(floor_k(d.k) + kQBlock, 128) * 128;
    const int64_t nch = cdiv(L, kChunk);
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t r = off;
        off = align256(off + bytes);
        return r;
    };
    o.leave = take(B * L * 4);
    o.leave_ceil = take(B * L * 4);
    o.tau = take(B * L * 8);
    o.nfrac = take(B * L * 4);
    o.qb_count = take(B * nqb * 4);
    o.qb_list = take(B * nqb * cap * 4);
    o.ever_count = take(B * 4);
    o.ever_list = take(B * L * 4);
    o.misc = take((2 + 3 * B * nch) * 4);  // two overflow queues [count, items...] + pass-1 flags
    const int64_t cap2 = next_pow2((int)std::max<int64_t>(L, 1));
    // the overflow pass's global bands; afterwards the running-max staging of tau [B, L]
    // (+ per-1024 chunk aggregates of the two-level scans after the staging area)
    o.scratch = take(std::max<uint64_t>((uint64_t)kOverflowSlots * (cap2 + L + 1),
                                        (uint64_t)B * L + (uint64_t)B * cdiv(L, 1024)) * 8);
    o.uf = take(B * L * 4);
    o.tauf = take(B * L * 4);
    o.qb_leave = take(B * nqb * cap * 4);
    o.qb_uf = take(B * nqb * cap * 4);
    o.qb_flags = take(B * nqb * (cap / 128) * 16);  // one 16-byte record per tile (bulk-copyable)
    o.total_bytes = off;
    o.qblock = kQBlock;
    o.nqb = nqb;
    o.qb_cap = cap;
}

void validate_desc(const skb_attn_desc& d) {
    SKB_REQUIRE(d.batch >= 1 && d.seq_len >= 1 && d.heads >= 1 && d.head_dim >= 1, SKB_ESHAPE,
                "attention: batch, seq_len, heads and head_dim must be positive");
    SKB_REQUIRE(d.seq_len < (int64_t(1) << 30), SKB_ESHAPE, "attention: seq_len too large");
    SKB_REQUIRE(std::isfinite(d.k) && d.k >= 0.0, SKB_ECONFIG, "attention: k must be finite and >= 0");
    SKB_REQUIRE(std::isfinite(d.scale) && d.scale >= 0.0, SKB_ECONFIG, "attention: bad scale");
    SKB_REQUIRE(d.window >= 0, SKB_ECONFIG, "attention: window must be >= 0");
    SKB_REQUIRE(!(d.window == 0 && std::floor(d.k) < 1.0) || (d.flags & SKB_FLAG_LINEAR_MIX), SKB_ECONFIG,
                "attention: window + floor(k) must be >= 1 (only the linear mix can run with neither)");
    SKB_REQUIRE(d.key_mode == 0 || d.key_mode == 1, SKB_EARG, "key_mode must be 'soft' or 'hard'");
    SKB_REQUIRE(d.mask_mode == 0 || d.mask_mode == 1, SKB_EARG,
                "mask_mode must be 'soft' or 'straight_through'");
    SKB_REQUIRE(d.dtype == SKB_F32 || d.dtype == SKB_BF16 || d.dtype == SKB_F64, SKB_EARG,
                "attention: unsupported dtype");
    SKB_REQUIRE(d.chunk_len >= 0, SKB_EARG, "chunked_forward: chunk_len must be positive");
}

void run_select(const skb_attn_desc& d, const double* u, void* ws, cudaStream_t st) {
    validate_desc(d);
    skb_select_layout lay;
    select_layout(d, lay);
    char* base = static_cast<char*>(ws);
    int* leave1 = reinterpret_cast<int*>(base + lay.leave);
    int* leave2 = reinterpret_cast<int*>(base + lay.leave_ceil);
    double* tau = reinterpret_cast<double*>(base + lay.tau);
    int* nfrac = reinterpret_cast<int*>(base + lay.nfrac);
    int* qb_count = reinterpret_cast<int*>(base + lay.qb_count);
    int* qb_list = reinterpret_cast<int*>(base + lay.qb_list);
    int* ever_count = reinterpret_cast<int*>(base + lay.ever_count);
    int* ever_list = reinterpret_cast<int*>(base + lay.ever_list);
    int* misc = reinterpret_cast<int*>(base + lay.misc);
    double* scratch = reinterpret_cast<double*>(base + lay.scratch);

    const int B = (int)d.batch, L = (int)d.seq_len, w = (int)d.window;
    const int T = std::max(0, L - w);
    const int R1 = (int)floor_k(d.k), R2 = (int)ceil_k(d.k);
    const int64_t BL = (int64_t)B * L;

    k_fill_tau<<<(unsigned)cdiv(BL, 256), 256, 0, st>>>(tau, nfrac, BL);
    SKB_CHECK_LAUNCH();
    if (R2 == 0 || T == 0) {
        // no budget: every position leaves at entry
        dim3 g((unsigned)cdiv(L, 256), B);
        k_leave_identity<<<g, 256, 0, st>>>(leave1, L);
        k_leave_identity<<<g, 256, 0, st>>>(leave2, L);
        SKB_CHECK_LAUNCH();
    } else {
        static const int rank2 = getenv("SKB_RANK2") ? atoi(getenv("SKB_RANK2")) : 1;
        dim3 g((unsigned)cdiv(T, kRankThreads), B);
        if (rank2) {
            SKB_CHECK_CUDA(cudaMemsetAsync(leave1, 0, (size_t)B * L * sizeof(int), st));
            dim3 g1((unsigned)cdiv(T, kRankBeforeThreads), (unsigned)cdiv(T, kRankChunk), B);
            k_rank_before<<<g1, kRankBeforeThreads, 0, st>>>(u, L, T, leave1, 0, T);
            SKB_CHECK_LAUNCH();
            k_rank_after_warp<<<dim3((unsigned)cdiv(T, 8), B), 256, 0, st>>>(u, L, T, R1, R2, leave1, leave2, 0, T);
        } else {
            k_rank_leave<<<g, kRankThreads, 0, st>>>(u, L, T, R1, R2, leave1, leave2);
        }
        SKB_CHECK_LAUNCH();
    }
    if (d.k > 0.0 && T > 0) {
        const int nch = (int)cdiv(T, kChunk);
        SKB_CHECK_CUDA(cudaMemsetAsync(misc, 0, (2 + 3 * (size_t)B * nch) * 4, st));
        int* q2 = misc + 1 + B * nch;  // second queue: [count, items...]
        TauArgs a;
        a.u = u;
        a.leave2 = leave2;
        a.tau = tau;
        a.nfrac = nfrac;
        a.ovf_count = misc;
        a.ovf_items = misc + 1;
        a.ovf_flag = misc + 2 + 2 * B * nch;
        a.L = L;
        a.T = T;
        a.R2 = R2;
        a.k = d.k;
        a.nch = nch;
        a.c_off = 0;
        a.c_end = nch;
        const int cap_big = std::min(8192, next_pow2(std::max(T, 32)));
        // pass 1: a small band cap (many CTAs per SM) serves slope-dominated
        // scores, whose band is ~ceil(k) wide; wider bands spill to pass 2
        a.cap = std::min(cap_big, std::max(256, next_pow2(2 * R2)));
        const int cap2 = next_pow2(std::max(L, 1));
        a.scratch = scratch;
        a.scratch_stride = cap2 + L + 1;
        static uint64_t attr_set = 0;
        if (first_on_device(&attr_set)) {
            SKB_CHECK_CUDA(cudaFuncSetAttribute(k_tau_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(8192 * 2 * sizeof(double) + 8 + 16)));  // bz + P[cap + 1]
            SKB_CHECK_CUDA(cudaFuncSetAttribute(k_tau_chunks_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(8192 * 2 * sizeof(double) + 16)));
            SKB_CHECK_CUDA(cudaFuncSetAttribute(k_tau_segments<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(8192 * 2 * sizeof(double) +
                                                      std::max(8192 * sizeof(double), kBigSortBytes) + 16)));
            SKB_CHECK_CUDA(cudaFuncSetAttribute(k_tau_segments<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(8192 * 3 * sizeof(double) + 16)));
        }
        static const int p1seg = getenv("SKB_TAU_P1SEG") ? atoi(getenv("SKB_TAU_P1SEG")) : 0;  // per-chunk pass 1 measured faster
        if (p1seg > 0) {
            dim3 g1((unsigned)cdiv(nch, p1seg), (unsigned)B);
            k_tau_segments<true><<<g1, kTauThreads, (size_t)a.cap * 3 * sizeof(double) + 16, st>>>(a, nch, p1seg,
                                                                                                   nullptr, nullptr);
        } else {
            dim3 g(nch, B);
            // bz + P; P also holds the block radix sort's scratch
        const size_t p1smem = (size_t)a.cap * sizeof(double) +
                              std::max((size_t)(a.cap + 1) * sizeof(double), sizeof(BandSort::TempStorage)) + 16;
        k_tau_chunks<<<g, kTauThreads, p1smem, st>>>(a);
        }
        SKB_CHECK_LAUNCH();
        if (cap_big > a.cap) {
            TauArgs a2 = a;
            a2.cap = cap_big;
            // segments sized so the flagged chunks spread over every SM: a segment's
            // CTA walks its chunks serially (one sort, then per-chunk merges), so
            // at B = 1 (a strong-scaling rank) 4-chunk segments halve the latency
            const int seg = (int)std::min<int64_t>(kSegChunks, std::max<int64_t>(1, cdiv((int64_t)nch * B, num_sms())));
            dim3 gs((unsigned)cdiv(nch, seg), (unsigned)B);
            const size_t seg_smem = (size_t)cap_big * 2 * sizeof(double) +
                                    std::max((size_t)cap_big * sizeof(double), cap_big >= 8192 ? kBigSortBytes : 0) + 16;
            k_tau_segments<false><<<gs, kTauThreads, seg_smem, st>>>(a2, nch, seg, q2, q2 + 1);
            SKB_CHECK_LAUNCH();
            a.ovf_count = q2;  // the global-scratch pass serves what is left
            a.ovf_items = q2 + 1;
        }
        k_tau_overflow<<<kOverflowSlots, kTauThreads, 0, st>>>(a, nch, cap2);
        SKB_CHECK_LAUNCH();
        // running max into the uf/tauf scratch (rewritten by k_to_float below), then back
        {
            double* tmp = reinterpret_cast<double*>(base + lay.scratch);
            double* cmax = tmp + BL;
            const dim3 gc((unsigned)cdiv(T, 1024), (unsigned)B);
            k_tau_chunk_max<<<gc, 1024, 0, st>>>(tau, L, T, cmax);
            k_tau_monotone_chunks<<<gc, 1024, 0, st>>>(tau, tmp, L, T, cmax);
            SKB_CHECK_LAUNCH();
            SKB_CHECK_CUDA(cudaMemcpy2DAsync(tau, (size_t)L * 8, tmp, (size_t)L * 8, (size_t)T * 8, B,
                                             cudaMemcpyDeviceToDevice, st));
        }
    }
    k_to_float<<<(unsigned)cdiv(BL, 256), 256, 0, st>>>(u, tau, reinterpret_cast<float*>(base + lay.uf),
                                                          reinterpret_cast<float*>(base + lay.tauf), BL);
    SKB_CHECK_LAUNCH();
    const int nqb = (int)lay.nqb;
    if (R1 > 0 && T > 0) {
        dim3 g(nqb, B);
        k_union_lists<<<g, 512, 0, st>>>(leave1, L, T, w, nqb, (int)lay.qb_cap, qb_count, qb_list);
        {
            int* ccnt = reinterpret_cast<int*>(reinterpret_cast<double*>(base + lay.scratch) + BL);
            const dim3 gc((unsigned)cdiv(T, 1024), (unsigned)B);
            k_ever_chunk_counts<<<gc, 1024, 0, st>>>(leave1, L, T, ccnt);
            k_ever_list<<<gc, 1024, 0, st>>>(leave1, L, T, ccnt, ever_count, ever_list);
        }
        SKB_CHECK_LAUNCH();
        // partitioned by class when the union fits in shared memory, in key order otherwise
        const size_t um_smem = (size_t)lay.qb_cap * sizeof(int);
        const bool um_part = um_smem <= 160 * 1024;
        static uint64_t um_attr = 0;
        if (um_part && first_on_device(&um_attr))
            SKB_CHECK_CUDA(cudaFuncSetAttribute(k_union_meta, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        k_union_meta<<<g, 128, um_part ? um_smem : 0, st>>>(leave1, reinterpret_cast<const float*>(base + lay.uf),
                                        reinterpret_cast<const float*>(base + lay.tauf), L, T, w, nqb,
                                        (int)lay.qb_cap, qb_count, qb_list, reinterpret_cast<int*>(base + lay.qb_leave),
                                        reinterpret_cast<float*>(base + lay.qb_uf),
                                        reinterpret_cast<int*>(base + lay.qb_flags), um_part ? 1 : 0);
        SKB_CHECK_LAUNCH();
    } else {
        const int64_t n = (int64_t)B * nqb;
        k_fill_int<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(qb_count, n, 0);
        k_fill_int<<<1, 256, 0, st>>>(ever_count, B, 0);
        SKB_CHECK_LAUNCH();
    }
}

SelView sel_view(const skb_attn_desc& d, const void* ws) {
    skb_select_layout lay;
    select_layout(d, lay);
    const char* base = static_cast<const char*>(ws);
    SelView s;
    s.leave = reinterpret_cast<const int*>(base + lay.leave);
    s.tau = reinterpret_cast<const double*>(base + lay.tau);
    s.nfrac = reinterpret_cast<const int*>(base + lay.nfrac);
    s.qb_count = reinterpret_cast<const int*>(base + lay.qb_count);
    s.qb_list = reinterpret_cast<const int*>(base + lay.qb_list);
    s.ever_count = reinterpret_cast<const int*>(base + lay.ever_count);
    s.ever_list = reinterpret_cast<const int*>(base + lay.ever_list);
    s.uf = reinterpret_cast<const float*>(base + lay.uf);
    s.tauf = reinterpret_cast<const float*>(base + lay.tauf);
    s.qb_leave = reinterpret_cast<const int*>(base + lay.qb_leave);
    s.qb_uf = reinterpret_cast<const float*>(base + lay.qb_uf);
    s.qb_flags = reinterpret_cast<const int*>(base + lay.qb_flags);
    s.nqb = (int)lay.nqb;
    s.qb_cap = (int)lay.qb_cap;
    return s;
}

}  // namespace skb

#ifdef SKB_TRACE_TAU
extern "C" int skb_debug_trace_tau(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, skb::g_skb_trace_tau, sizeof(unsigned long long) * (n < 16 ? n : 16));
}
#endif
