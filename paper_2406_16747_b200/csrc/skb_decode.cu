// K5 — the constant-(floor(k)+w) KV cache for decoding, and the device-resident
// incremental SparseK stream (Algorithm 2) it is built on.
//
// Reference: SparseKvCache (proj/include/sparsek/cache.hpp:21-87) driven by
// generate_step (proj/src/cache.cpp:570-577) = forward_chunk on one row: the
// new position enters the window ring, the position leaving the window is
// pushed into StreamState (proj/src/stream.cpp:72-152) and admitted to the
// top-floor(k) min-heap or dropped (exit_window/admit_to_cache,
// proj/src/cache.cpp:136-179); the query then reads the retained rows with
// gates clamp(u_j - tau, 0, 1) (cache.cpp:285-311, 358-393).
//
// B200 layout (per sequence b):
//   * slot pool: K and V as [B, S, H, p] with S = floor(k) + w + 1 slots (the
//     reference's peak_kv bound, proj/tests/test_cache.cpp:124,148); a row
//     is written once into a free slot when its position arrives and never
//     moves — leaving the window for the selected set is a table update.
//   * stream state: survivors and saturated entries as two arrays sorted by
//     (value desc, index asc), so the heaps' minima (HeapCmp, stream.cpp:14-18)
//     are the array tails and the selected set is the survivors' head
//     [0, floor(k)): a top-floor(k) position is never below tau, so the stream
//     order and the cache heap (SlotCmp, cache.cpp:53-60) agree. One warp
//     per sequence does the push: count (parallel), shift (parallel), scan
//     (uniform scalar control flow, identical arithmetic to the reference:
//     running sums with the same += / -= order, so tau is bit-identical).
//   * per step three launches: k_cache_control (one warp per sequence:
//     append, exit/admit/evict, attended slot list with gates), k_cache_attn
//     (split over the attended slots, all heads per CTA: each slot's H*p row
//     is one contiguous read), k_cache_combine (merge the split softmaxes).
//     HBM-bound: 2 * S * H * p * sizeof(T) bytes per sequence per step.
//
// Deviation (documented in DESIGN.md): the reference re-sums its heaps every
// 2^16 pushes (stream.cpp:78-81, refresh_sums) in heap-array order; here the
// re-sum runs in sorted order, so after 65536 pushes tau may differ from the
// reference by rounding (never the selected set).
#include <algorithm>
#include <cfloat>
#include <cstring>
#include <type_traits>
#include <vector>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {
namespace {

struct StreamCtl {
    double k, tau, sum_s, sum_f;
    long long t;            // elements pushed
    long long heap_cap;     // 0 = unbounded (StreamState heap_cap)
    unsigned long long heap_ops, cap_drops;
    int nS, nF;
    int since_refresh;
    int cap;                // array capacity (maximum pushes)
    int error;              // 1 = scan exhausted (reference throws NumericError), 2 = overflow
    int pad;
};

struct StreamArr {
    double* sv;
    int* si;
    double* fv;
    int* fi;
    uint8_t* evicted;  // [cap] or null
    int* evlog;        // indices popped from the survivors, in pop order (or null)
    int* evcount;      // entries in evlog (lane 0 owns both)
};

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// number of entries with value >= z in a (value desc) array: the slot a new,
// later-indexed z takes (ties keep the earlier index first).
__device__ int warp_count_ge(const double* v, int n, double z) {
    const int lane = threadIdx.x & 31;
    int c = 0;
    for (int i = lane; i < n; i += 32) c += v[i] >= z;
    return warp_sum_i(c);
}

// Shift [pos, n) up by one and put (z, zi) at pos. Blocks of 32 x 8 elements
// from the top: all loads of a block are issued before any store, so a block
// costs two memory round trips instead of one per 32 elements.
__device__ void warp_insert(double* v, int* ix, int n, int pos, double z, int zi) {
    const int lane = threadIdx.x & 31;
    constexpr int U = 8;
    for (int top = n - 1; top >= pos; top -= 32 * U) {
        double a[U];
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = top - u * 32 - lane;
            if (i >= pos) {
                a[u] = v[i];
                c[u] = ix[i];
            }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = top - u * 32 - lane;
            if (i >= pos) {
                v[i + 1] = a[u];
                ix[i + 1] = c[u];
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        v[pos] = z;
        ix[pos] = zi;
    }
    __syncwarp();
}

// StreamState::push (proj/src/stream.cpp:72-152), executed uniformly by all 32
// lanes of one warp (c is a per-lane copy; lane 0 owns the stores). Returns
// whether z entered the survivors; *rank = its position in the survivor array.
__device__ bool warp_stream_push(StreamCtl& c, const StreamArr& a, double z, int* rank) {
    const int lane = threadIdx.x & 31;
    const int index = (int)c.t;
    c.t += 1;
    *rank = -1;
    if (++c.since_refresh >= (1 << 16)) {  // refresh_sums (see header note)
        double ss = 0.0, sf = 0.0;
        for (int i = 0; i < c.nS; ++i) ss += a.sv[i];
        for (int i = 0; i < c.nF; ++i) sf += a.fv[i];
        c.sum_s = ss;
        c.sum_f = sf;
        c.since_refresh = 0;
    }
    if (!(z > c.tau)) {  // at or below the threshold: zero mass now and forever
        if (a.evicted && lane == 0) a.evicted[index] = 1;
        return false;
    }
    if (c.nS >= c.cap) {
        c.error = 2;
        return false;
    }
    const int ps = warp_count_ge(a.sv, c.nS, z);
    warp_insert(a.sv, a.si, c.nS, ps, z, index);
    c.nS += 1;
    c.sum_s += z;
    c.heap_ops += 1;
    *rank = ps;
    if (z >= c.tau + 1.0) {
        const int pf = warp_count_ge(a.fv, c.nF, z);
        warp_insert(a.fv, a.fi, c.nF, pf, z, index);
        c.nF += 1;
        c.sum_f += z;
        c.heap_ops += 1;
    }
    auto pop_s = [&]() {
        const double v = a.sv[c.nS - 1];
        const int ix = a.si[c.nS - 1];
        c.nS -= 1;
        c.sum_s -= v;
        if (a.evicted && lane == 0) a.evicted[ix] = 1;
        if (a.evlog && lane == 0) a.evlog[(*a.evcount)++] = ix;
        c.heap_ops += 1;
    };
    auto pop_f = [&]() {
        c.sum_f -= a.fv[c.nF - 1];
        c.nF -= 1;
        c.heap_ops += 1;
    };
    if (c.heap_cap > 0) {
        while ((long long)c.nS > c.heap_cap) {
            if (c.nF > 0 && a.fi[c.nF - 1] == a.si[c.nS - 1]) pop_f();
            pop_s();
            c.cap_drops += 1;
        }
    }
    if ((double)c.t < c.k) {  // budget not binding yet
        c.tau = -CUDART_INF;
        __syncwarp();
        return true;
    }
    bool popped = false;
    double last = 0.0;
    for (;;) {
        const int u = c.nF, w = c.nS;
        if (u == w) {
            if (u == 0) {
                c.error = 1;
                break;
            }
            const double hi = a.fv[u - 1] - 1.0;
            const double lo = popped ? last : fmax(c.tau, hi - 1.0);
            if (fabs((double)u - c.k) <= 1e-9) {
                c.tau = fmax(c.tau, 0.5 * (lo + hi));
                break;
            }
            pop_f();
            continue;
        }
        const double cand = (c.sum_s - c.sum_f + (double)u - c.k) / (double)(w - u);
        const double smin = a.sv[w - 1];
        if (smin > cand && (u == 0 || a.fv[u - 1] >= cand + 1.0)) {
            c.tau = cand;
            break;
        }
        if (u == 0 || smin <= a.fv[u - 1] - 1.0) {
            last = smin;
            popped = true;
            pop_s();
            if (c.nS == 0) {
                c.error = 1;
                break;
            }
        } else {
            pop_f();
        }
    }
    __syncwarp();
    return true;
}

// ------------------------------------------------------------------ stream API
__global__ void k_stream_push(StreamCtl* ctl, StreamArr a, const double* __restrict__ z, int n,
                              double* __restrict__ tau_out, uint8_t* __restrict__ ins_out) {
    StreamCtl c = *ctl;
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < n; ++i) {
        int rank;
        const bool ins = warp_stream_push(c, a, z[i], &rank);
        if (lane == 0) {
            if (tau_out) tau_out[i] = c.tau;
            if (ins_out) ins_out[i] = ins ? 1 : 0;
        }
        if (c.error) break;
    }
    if (lane == 0) *ctl = c;
}

// One push with the reference's StreamStepResult (proj/include/sparsek/stream.hpp:12-18):
// tau, t, inserted, cap_forced and the survivors popped by this push (evlog).
struct StreamStepRes {
    double tau;
    long long t;
    int inserted, cap_forced, n_evicted, error;
};
__global__ void k_stream_push_step(StreamCtl* ctl, StreamArr a, double z, StreamStepRes* res) {
    StreamCtl c = *ctl;
    const int lane = threadIdx.x & 31;
    if (lane == 0) *a.evcount = 0;
    __syncwarp();
    const unsigned long long drops0 = c.cap_drops;
    int rank;
    const bool ins = c.t < c.cap ? warp_stream_push(c, a, z, &rank) : (c.error = 2, false);
    if (lane == 0) {
        *ctl = c;
        StreamStepRes r;
        r.tau = c.tau;
        r.t = c.t;
        r.inserted = ins ? 1 : 0;
        r.cap_forced = c.cap_drops != drops0 ? 1 : 0;
        r.n_evicted = *a.evcount;
        r.error = c.error;
        *res = r;
    }
}

// StreamState::solution + stream_mask (proj/src/stream.cpp:154-222) on the
// device: survivors in ascending index order with p = clamp(z - tau, 0, 1)
// (all ones while t < k), and the hard top-floor(k) flag — the survivors
// array is sorted by (value desc, index asc), so its first floor(k) entries
// are the mask's (p desc, index asc) top (saturated entries are at most k).
// One CTA: scatter each survivor's rank to its index, compact in index order.
struct StreamSolRes {
    int n, u_count, w_count, pad;
};
__global__ void __launch_bounds__(1024) k_stream_solution(const StreamCtl* ctl, StreamArr a, int* rank_of,
                                                          double* p_out, long long* idx_out, uint8_t* hard_out,
                                                          StreamSolRes* res) {
    __shared__ int wsum[32];
    __shared__ int s_u, s_w;
    const StreamCtl c = *ctl;
    const int T = (int)c.t, nS = c.nS;
    const int kk = (int)floor(c.k);
    const bool infeasible = (double)c.t < c.k;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_u = s_w = 0;
    for (int j = threadIdx.x; j < T; j += 1024) rank_of[j] = -1;
    __syncthreads();
    for (int r = threadIdx.x; r < nS; r += 1024) rank_of[a.si[r]] = r;
    __syncthreads();
    int base = 0, nu = 0, nw = 0;
    for (int j0 = 0; j0 < T; j0 += 1024) {
        const int j = j0 + threadIdx.x;
        const int r = j < T ? rank_of[j] : -1;
        const bool keep = r >= 0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        int off = base, tot = 0;
        for (int w = 0; w < 32; ++w) {
            if (w < wid) off += wsum[w];
            tot += wsum[w];
        }
        if (keep) {
            const int o = off + __popc(bal & ((1u << lane) - 1u));
            double pj = 1.0;
            if (!infeasible) {
                pj = a.sv[r] - c.tau;
                pj = pj < 0.0 ? 0.0 : (pj > 1.0 ? 1.0 : pj);
            }
            p_out[o] = pj;
            idx_out[o] = j;
            if (hard_out) hard_out[o] = r < kk ? 1 : 0;
            nu += pj == 1.0;
            nw += pj > 0.0;
        }
        base += tot;
        __syncthreads();
    }
    atomicAdd(&s_u, nu);
    atomicAdd(&s_w, nw);
    __syncthreads();
    if (threadIdx.x == 0) {
        StreamSolRes r;
        r.n = base;
        r.u_count = s_u;
        r.w_count = s_w;
        r.pad = 0;
        *res = r;
    }
}

// ------------------------------------------------------------------ cache
struct CacheCtl {
    StreamCtl st;
    long long t;     // positions seen
    long long peak;  // peak retained rows (cache + ring + in-flight)
    int free_top;    // free-slot stack height
    int nsel;        // |selected set|
    int error;
    int pad;
};

struct CacheArgs {
    CacheCtl* ctl;      // [B]
    double* sv;         // [B, Lmax] survivors (value desc, index asc)
    int* si;
    double* fv;         // [B, Lmax] saturated
    int* fi;
    double* u_hist;     // [B, Lmax] frozen scores
    uint8_t* ins_hist;  // [B, Lmax] the exit push of each position inserted it (z > tau); snapshots
    int* slot_of;       // [B, Lmax] position -> slot (-1 = dropped)
    int* pos_of;        // [B, S]    slot -> position (-1 = free)
    int* free_stack;    // [B, S]
    int* att_slot;      // [B, S]    attended slots of the current step
    double* att_kg;     // [B, S]    logit multiplier (gate under soft keys, else 1)
    double* att_vg;     // [B, S]    value weight (gate under soft mask, else 1)
    int* att_n;         // [B]
    uint8_t* kpool;     // [B, S, H, p] dtype
    uint8_t* vpool;
    int Lmax, S, cap, w, key_soft, mask_st;
    int lin;            // linear mix (Appendix B.1): no self entry when w = 0 (the linear branch covers it)
    int64_t row_bytes;  // H * p * esize
};

// threads [tid, nthr) of the caller copy one row
__device__ __forceinline__ void copy_row(uint8_t* dst, const uint8_t* src, int64_t bytes, int tid, int nthr) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | (uintptr_t)bytes) & 15) == 0) {
        const uint4* s = reinterpret_cast<const uint4*>(src);
        uint4* d = reinterpret_cast<uint4*>(dst);
        for (int64_t i = tid; i < bytes / 16; i += nthr) d[i] = s[i];
    } else {
        const uint16_t* s = reinterpret_cast<const uint16_t*>(src);
        uint16_t* d = reinterpret_cast<uint16_t*>(dst);
        for (int64_t i = tid; i < bytes / 2; i += nthr) d[i] = s[i];
    }
}
__device__ __forceinline__ void warp_copy_row(uint8_t* dst, const uint8_t* src, int64_t bytes) {
    copy_row(dst, src, bytes, threadIdx.x & 31, 32);
}

// One position of forward_chunk's pass 1 (proj/src/cache.cpp:259-311) for one
// sequence, uniformly on one warp. kv_src: this position's K/V rows (null in
// a prefill replay: the rows are copied once at the end). Builds the
// attended list when `emit` is set.
// One position through the cache, phase 1 (one warp): the row enters the
// window ring, the exiting position's stream push (selection, tau), the
// retained-row peak. freed[] receives the positions whose slots phase 3 frees.
__device__ bool warp_cache_push(const CacheArgs& A, int b, CacheCtl& c, double u_new, const uint8_t* k_src,
                                const uint8_t* v_src, int* slot_out, int freed[2], const StreamArr* arr = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t bL = (int64_t)b * A.Lmax, bS = (int64_t)b * A.S;
    if (c.t >= A.Lmax) {
        c.error = 2;
        return false;
    }
    const int pos = (int)c.t;
    const StreamArr sa = arr ? *arr : StreamArr{A.sv + bL, A.si + bL, A.fv + bL, A.fi + bL, nullptr, nullptr, nullptr};
    if (lane == 0) A.u_hist[bL + pos] = u_new;
    // the new row enters the window ring (kv_.emplace + ring_.push_back)
    const int slot = A.free_stack[bS + c.free_top - 1];
    c.free_top -= 1;
    if (lane == 0) {
        A.slot_of[bL + pos] = slot;
        A.pos_of[bS + slot] = pos;
    }
    if (k_src) {
        warp_copy_row(A.kpool + (bS + slot) * A.row_bytes, k_src, A.row_bytes);
        warp_copy_row(A.vpool + (bS + slot) * A.row_bytes, v_src, A.row_bytes);
    }
    const long long ring_before = c.t < A.w ? c.t : A.w;
    c.peak = max(c.peak, ring_before + 1 + c.nsel);  // note_peak after ring push
    freed[0] = freed[1] = -1;
    *slot_out = slot;
    __syncwarp();
    if (c.t + 1 > A.w) {  // ring_.size() > window: exit_window(ring_.front())
        const int e = pos - A.w;
        const double ue = (e == pos) ? u_new : A.u_hist[bL + e];
        bool admitted = false;
        if (A.cap > 0) {
            const int nS_before = c.st.nS;
            int rank;
            const bool ins = warp_stream_push(c.st, sa, ue, &rank);
            if (lane == 0) A.ins_hist[bL + e] = ins ? 1 : 0;
            if (ins && rank >= 0 && rank < A.cap) {
                admitted = true;
                // the previous rank floor(k)-1 entry is pushed out of the top floor(k)
                // (pops only shorten the array, so index cap still holds it)
                if (nS_before >= A.cap) freed[1] = sa.si[A.cap];
                c.nsel = min(c.nsel + 1, A.cap);
            }
        } else if (c.st.k > 0.0) {
            int rank;
            const bool ins = warp_stream_push(c.st, sa, ue, &rank);  // tau still advances (floor(k) = 0)
            if (lane == 0) A.ins_hist[bL + e] = ins ? 1 : 0;
        }
        if (!admitted) freed[0] = e;
    }
    const long long ring_after = (c.t + 1) < A.w ? (c.t + 1) : A.w;
    c.peak = max(c.peak, ring_after + c.nsel);
    return true;
}

// Phase 2: the attended list (snapshot): selected (survivor order), then the
// window ring. Threads [tid, nthr) of the caller stride over the entries; the
// w = 0 self-read test is a warp vote (callers with nthr > 32 run it on warp 0).
__device__ void cache_emit(const CacheArgs& A, int b, const CacheCtl& c, int slot, int tid, int nthr,
                           const StreamArr* arr = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t bL = (int64_t)b * A.Lmax, bS = (int64_t)b * A.S;
    const int pos = (int)c.t;
    const StreamArr sa = arr ? *arr : StreamArr{A.sv + bL, A.si + bL, A.fv + bL, A.fi + bL, nullptr, nullptr, nullptr};
    const double tau = c.st.tau;
    const int ns = c.nsel;
    for (int r = tid; r < ns; r += nthr) {
        const int jp = sa.si[r];
        const double g = fmin(1.0, fmax(0.0, sa.sv[r] - tau));
        A.att_slot[bS + r] = A.slot_of[bL + jp];
        A.att_kg[bS + r] = A.key_soft ? g : 1.0;
        A.att_vg[bS + r] = A.mask_st ? 1.0 : g;
    }
    int n = ns;
    if (A.w > 0) {
        const int r0 = max(0, pos - A.w + 1);
        for (int jp = r0 + tid; jp <= pos; jp += nthr) {
            const int r = ns + (jp - r0);
            A.att_slot[bS + r] = A.slot_of[bL + jp];
            A.att_kg[bS + r] = 1.0;
            A.att_vg[bS + r] = 1.0;
        }
        n += pos - r0 + 1;
    }
    if (tid >= 32) return;  // warp 0: the self-read test and the count
    if (A.w == 0 && !A.lin) {
        // nothing window-resident: the query reads itself unless selected
        bool selected = false;
        for (int r = lane; r < ns; r += 32) selected |= sa.si[r] == pos;
        selected = __any_sync(0xffffffffu, selected);
        if (!selected) {
            if (lane == 0) {
                A.att_slot[bS + n] = slot;
                A.att_kg[bS + n] = 1.0;
                A.att_vg[bS + n] = 1.0;
            }
            n += 1;
        }
    }
    if (lane == 0) A.att_n[b] = n;
}

// Phase 3 (one warp): drop_kv frees the slots now (the attention of this step
// reads only the attended list; slots are reallocated by the next control).
__device__ void warp_cache_drop(const CacheArgs& A, int b, CacheCtl& c, const int freed[2]) {
    const int lane = threadIdx.x & 31;
    const int64_t bL = (int64_t)b * A.Lmax, bS = (int64_t)b * A.S;
    __syncwarp();
    for (int f = 0; f < 2; ++f) {
        const int fp = freed[f];
        if (fp < 0) continue;
        const int fs = A.slot_of[bL + fp];
        __syncwarp();
        if (lane == 0) {
            A.free_stack[bS + c.free_top] = fs;
            A.slot_of[bL + fp] = -1;
            A.pos_of[bS + fs] = -1;
        }
        c.free_top += 1;
        __syncwarp();
    }
    c.t += 1;
    if (c.st.error) c.error = 1;
}


__device__ void warp_cache_advance(const CacheArgs& A, int b, CacheCtl& c, double u_new,
                                   const uint8_t* k_src, const uint8_t* v_src, bool emit) {
    int slot, freed[2];
    if (!warp_cache_push(A, b, c, u_new, k_src, v_src, &slot, freed)) return;
    if (emit) cache_emit(A, b, c, slot, threadIdx.x & 31, 32);
    warp_cache_drop(A, b, c, freed);
}

__global__ void k_cache_init(CacheArgs A, double k) {
    const int b = blockIdx.x;
    const int64_t bS = (int64_t)b * A.S;
    for (int s = threadIdx.x; s < A.S; s += blockDim.x) {
        A.free_stack[bS + s] = A.S - 1 - s;  // slot 0 on top
        A.pos_of[bS + s] = -1;
    }
    if (threadIdx.x == 0) {
        CacheCtl c{};
        c.st.k = k;
        c.st.tau = -CUDART_INF;
        c.st.cap = A.Lmax;
        c.free_top = A.S;
        A.ctl[b] = c;
        A.att_n[b] = 0;
    }
}

// one decode step: a warp per sequence
// One step's control, a CTA per sequence: the sequence's survivor and
// saturated arrays (sorted, ~floor(k) entries) are staged in shared memory,
// warp 0 runs the stream push on them (the reference's serial arithmetic;
// the insert shifts and the pop loop's dependent reads were global round
// trips), then all kControlThreads threads write the new K/V rows, the
// attended list and the arrays back, and warp 0 frees the dropped slots.
// Sequences whose arrays outgrow kCtlSmemEntries keep them in global memory.
constexpr int kControlThreads = 256;
constexpr int kCtlSmemEntries = 4096;
constexpr size_t kCtlSmemBytes = (size_t)kCtlSmemEntries * 2 * (sizeof(double) + sizeof(int));
__global__ void __launch_bounds__(kControlThreads) k_cache_control(CacheArgs A, int B, const uint8_t* __restrict__ k_new,
                                                                   const uint8_t* __restrict__ v_new,
                                                                   const double* __restrict__ u_new) {
    extern __shared__ __align__(16) uint8_t ctl_smem[];
    double* s_sv = reinterpret_cast<double*>(ctl_smem);
    double* s_fv = s_sv + kCtlSmemEntries;
    int* s_si = reinterpret_cast<int*>(s_fv + kCtlSmemEntries);
    int* s_fi = s_si + kCtlSmemEntries;
    const int b = blockIdx.x;
    const int64_t bL = (int64_t)b * A.Lmax;
    __shared__ CacheCtl cs;
    __shared__ int s_slot, s_freed[2], s_ok;
    const CacheCtl c0 = A.ctl[b];
    // one push adds at most one entry to each array
    const bool staged = c0.error == 0 && c0.st.nS + 1 <= kCtlSmemEntries && c0.st.nF + 1 <= kCtlSmemEntries;
    if (staged) {
        for (int i = threadIdx.x; i < c0.st.nS; i += blockDim.x) {
            s_sv[i] = A.sv[bL + i];
            s_si[i] = A.si[bL + i];
        }
        for (int i = threadIdx.x; i < c0.st.nF; i += blockDim.x) {
            s_fv[i] = A.fv[bL + i];
            s_fi[i] = A.fi[bL + i];
        }
    }
    __syncthreads();
    const StreamArr glob{A.sv + bL, A.si + bL, A.fv + bL, A.fi + bL, nullptr, nullptr, nullptr};
    const StreamArr shar{s_sv, s_si, s_fv, s_fi, nullptr, nullptr, nullptr};
    const StreamArr* arr = staged ? &shar : &glob;
    if (threadIdx.x < 32) {
        CacheCtl c = c0;
        int slot = -1, freed[2] = {-1, -1};
        bool ok = false;
        if (c.error == 0) ok = warp_cache_push(A, b, c, u_new[b], nullptr, nullptr, &slot, freed, arr);
        if (threadIdx.x == 0) {
            cs = c;
            s_slot = slot;
            s_freed[0] = freed[0];
            s_freed[1] = freed[1];
            s_ok = ok ? 1 : 0;
        }
    }
    __syncthreads();
    if (s_ok) {  // the new K/V rows into their slot (the attention of this step reads them), the attended list
        const int64_t dst = ((int64_t)b * A.S + s_slot) * A.row_bytes;
        copy_row(A.kpool + dst, k_new + (int64_t)b * A.row_bytes, A.row_bytes, threadIdx.x, blockDim.x);
        copy_row(A.vpool + dst, v_new + (int64_t)b * A.row_bytes, A.row_bytes, threadIdx.x, blockDim.x);
        cache_emit(A, b, cs, s_slot, threadIdx.x, blockDim.x, arr);
    }
    if (staged) {  // the arrays back (entries past the new lengths were popped)
        for (int i = threadIdx.x; i < cs.st.nS; i += blockDim.x) {
            A.sv[bL + i] = s_sv[i];
            A.si[bL + i] = s_si[i];
        }
        for (int i = threadIdx.x; i < cs.st.nF; i += blockDim.x) {
            A.fv[bL + i] = s_fv[i];
            A.fi[bL + i] = s_fi[i];
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        CacheCtl c = cs;
        if (s_ok) {
            const int freed[2] = {s_freed[0], s_freed[1]};
            warp_cache_drop(A, b, c, freed);
        }
        if (threadIdx.x == 0) A.ctl[b] = c;
    }
}

// prefill replay: n positions per sequence, no attention; rows copied after.
__global__ void k_cache_prefill(CacheArgs A, int B, const double* __restrict__ u_hist, int n) {
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= B) return;
    CacheCtl c = A.ctl[b];
    for (int i = 0; i < n && c.error == 0; ++i)
        warp_cache_advance(A, b, c, u_hist[(int64_t)b * n + i], nullptr, nullptr, false);
    if ((threadIdx.x & 31) == 0) A.ctl[b] = c;
}

// rows of the live slots that arrived during a prefill of n positions starting at p0
__global__ void k_cache_fill_rows(CacheArgs A, const uint8_t* __restrict__ k_hist,
                                  const uint8_t* __restrict__ v_hist, int p0, int n) {
    const int b = blockIdx.y;
    const int slot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (slot >= A.S) return;
    const int pos = A.pos_of[(int64_t)b * A.S + slot];
    if (pos < p0 || pos >= p0 + n) return;
    const int64_t src = ((int64_t)b * n + (pos - p0)) * A.row_bytes;
    const int64_t dst = ((int64_t)b * A.S + slot) * A.row_bytes;
    warp_copy_row(A.kpool + dst, k_hist + src, A.row_bytes);
    warp_copy_row(A.vpool + dst, v_hist + src, A.row_bytes);
}

// ------------------------------------------------------------------ attention
constexpr int kAttnThreads = 256;
#ifndef SKB_DEC_SLOTS
#define SKB_DEC_SLOTS 48  // measured best of 48/64/96/128 at cfg4 (0.299 vs 0.308 ms)
#endif
constexpr int kSlotsPerCta = SKB_DEC_SLOTS;  // attended entries per attention CTA

template <int VEC>
__device__ __forceinline__ void ldv(const __nv_bfloat16* p, float* o) {
    if constexpr (VEC == 4) {
        const uint2 r = *reinterpret_cast<const uint2*>(p);
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
        const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
        o[0] = a.x, o[1] = a.y, o[2] = c.x, o[3] = c.y;
    } else if constexpr (VEC == 2) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
        o[0] = a.x, o[1] = a.y;
    } else {
        o[0] = __bfloat162float(*p);
    }
}
template <int VEC>
__device__ __forceinline__ void ldv(const float* p, float* o) {
    if constexpr (VEC == 4) {
        const float4 r = *reinterpret_cast<const float4*>(p);
        o[0] = r.x, o[1] = r.y, o[2] = r.z, o[3] = r.w;
    } else if constexpr (VEC == 2) {
        const float2 r = *reinterpret_cast<const float2*>(p);
        o[0] = r.x, o[1] = r.y;
    } else {
        o[0] = *p;
    }
}
template <int VEC>
__device__ __forceinline__ void ldv(const double* p, double* o) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) o[e] = p[e];
}
// float64 pools accumulate in float64 (the reference's double build), the
// others in float32
template <class T>
using AccOf = typename std::conditional<std::is_same<T, double>::value, double, float>::type;
__device__ __forceinline__ float exp_acc(float x) { return expf(x); }
__device__ __forceinline__ double exp_acc(double x) { return exp(x); }

// CTA = (chunk of kSlotsPerCta attended entries, sequence), all heads. Each
// (entry, head) row is p contiguous elements; a warp covers it with lanes
// owning VEC consecutive elements per 32*VEC stride.
template <class T, int VEC>
__global__ void __launch_bounds__(kAttnThreads)
k_cache_attn(CacheArgs A, const T* __restrict__ q, int H, int p, double scale_d, void* po_,
             void* pm_, void* pl_, int nsplit) {
    using Acc = AccOf<T>;
    Acc* po = static_cast<Acc*>(po_);
    Acc* pm = static_cast<Acc*>(pm_);
    Acc* pl = static_cast<Acc*>(pl_);
    const Acc scale = (Acc)scale_d;
    extern __shared__ __align__(16) unsigned char smraw[];
    Acc* sq = reinterpret_cast<Acc*>(smraw);  // [H * p] query
    Acc* sp = sq + H * p;                     // [H][kSlotsPerCta] logits -> probabilities
    Acc* svg = sp + H * kSlotsPerCta;         // [kSlotsPerCta] value weights
    int* ss = reinterpret_cast<int*>(svg + kSlotsPerCta);  // [kSlotsPerCta] slots
    const int b = blockIdx.y, chunk = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kAttnThreads / 32;
    const int n = A.att_n[b];
    const int e0 = chunk * kSlotsPerCta;
    const int ne = max(0, min(kSlotsPerCta, n - e0));
    const int64_t bS = (int64_t)b * A.S;
    const int hp = H * p;
    for (int i = threadIdx.x; i < hp; i += kAttnThreads) sq[i] = (Acc)q[(int64_t)b * hp + i];
    for (int e = threadIdx.x; e < ne; e += kAttnThreads) {
        ss[e] = A.att_slot[bS + e0 + e];
        svg[e] = (Acc)A.att_vg[bS + e0 + e];
    }
    __syncthreads();
    const T* kp = reinterpret_cast<const T*>(A.kpool);
    const T* vp = reinterpret_cast<const T*>(A.vpool);
    // logits: unit = (entry, head), consecutive warps take consecutive heads
    const int units = ne * H;
    constexpr int U = 4;
    for (int u0 = warp * U; u0 < units; u0 += nw * U) {
        Acc acc[U];
#pragma unroll
        for (int x = 0; x < U; ++x) acc[x] = 0;
#pragma unroll
        for (int x = 0; x < U; ++x) {
            const int un = u0 + x;
            if (un < units) {
                const int e = un / H, h = un % H;
                const T* kr = kp + ((bS + ss[e]) * H + h) * (int64_t)p;
                const Acc* qr = sq + h * p;
                for (int c = lane * VEC; c < p; c += 32 * VEC) {
                    Acc kv[VEC];
                    ldv<VEC>(kr + c, kv);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[x] = fma(qr[c + v], kv[v], acc[x]);
                }
            }
        }
#pragma unroll
        for (int x = 0; x < U; ++x) {
            const Acc s = warp_sum(acc[x]);
            const int un = u0 + x;
            if (lane == 0 && un < units) {
                const int e = un / H, h = un % H;
                sp[h * kSlotsPerCta + e] = s * scale * (Acc)A.att_kg[bS + e0 + e];
            }
        }
    }
    __syncthreads();
    // per-head softmax over this chunk (partial: max m, sum l of exp(a - m))
    for (int h = warp; h < H; h += nw) {
        Acc m = -INFINITY;
        for (int e = lane; e < ne; e += 32) m = fmax(m, sp[h * kSlotsPerCta + e]);
        m = warp_max(m);
        Acc l = 0;
        for (int e = lane; e < ne; e += 32) {
            const Acc pe = ne > 0 ? exp_acc(sp[h * kSlotsPerCta + e] - m) : Acc(0);
            sp[h * kSlotsPerCta + e] = pe;
            l += pe;
        }
        l = warp_sum(l);
        if (lane == 0) {
            const int64_t o = ((int64_t)b * nsplit + chunk) * H + h;
            pm[o] = ne > 0 ? m : -INFINITY;
            pl[o] = l;
        }
    }
    __syncthreads();
    // o_partial[h] = sum_e p_e * vg_e * v_e
    for (int h = warp; h < H; h += nw) {
        for (int c0 = lane * VEC; c0 < p; c0 += 32 * VEC) {
            Acc acc[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] = 0;
            int e = 0;
            for (; e + 4 <= ne; e += 4) {
                Acc vv[4][VEC];
#pragma unroll
                for (int x = 0; x < 4; ++x) ldv<VEC>(vp + ((bS + ss[e + x]) * H + h) * (int64_t)p + c0, vv[x]);
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const Acc w = sp[h * kSlotsPerCta + e + x] * svg[e + x];
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = fma(w, vv[x][v], acc[v]);
                }
            }
            for (; e < ne; ++e) {
                Acc vv[VEC];
                ldv<VEC>(vp + ((bS + ss[e]) * H + h) * (int64_t)p + c0, vv);
                const Acc w = sp[h * kSlotsPerCta + e] * svg[e];
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[v] = fma(w, vv[v], acc[v]);
            }
            Acc* out = po + (((int64_t)b * nsplit + chunk) * H + h) * p + c0;
#pragma unroll
            for (int v = 0; v < VEC; ++v) out[v] = acc[v];
        }
    }
}

// bf16 fast path (head_dim 64/128, H a multiple of 32/(D/8)): every load is a
// 16-byte chunk and a warp instruction covers 512 contiguous bytes of a slot
// row (HPL heads); warp w owns head groups j = w, w+8, ... for all entries of
// the chunk, so the K and V streams are fully coalesced with many loads in
// flight per lane.
#ifndef SKB_DEC_MINB  // resident CTAs per SM asked of ptxas (2 at 104 registers)
#define SKB_DEC_MINB 3
#endif
template <int D, int JMAX = 4>
__global__ void __launch_bounds__(kAttnThreads, SKB_DEC_MINB)
k_cache_attn_bf16(CacheArgs A, const __nv_bfloat16* __restrict__ q, int H, float scale, float* __restrict__ po,
                  float* __restrict__ pm, float* __restrict__ pl, int nsplit, int hs, int* __restrict__ done,
                  __nv_bfloat16* __restrict__ o) {
    // CTA = (chunk of kSlotsPerCta attended entries, sequence, group of hs
    // heads): the head groups multiply the CTA count, so the grid runs in
    // whole-ish waves. The last CTA of a (sequence, head group) to finish
    // merges the split softmax of every chunk (no separate combine launch).
    constexpr int LPH = D / 8;     // lanes per head row (16 B each)
    constexpr int HPL = 32 / LPH;  // heads per warp load
    // JMAX: head groups per warp (hs <= 8 warps * HPL * JMAX)
    extern __shared__ float sm[];
    float* sp = sm;                                           // [hs][kSlotsPerCta]
    int* ss = reinterpret_cast<int*>(sp + hs * kSlotsPerCta);  // [kSlotsPerCta]
    float* svg = reinterpret_cast<float*>(ss + kSlotsPerCta);
    float* skg = svg + kSlotsPerCta;
    __shared__ int s_last;
    const int b = blockIdx.y, chunk = blockIdx.x, h0 = blockIdx.z * hs;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kAttnThreads / 32;
    const int n = A.att_n[b];
    const int e0 = chunk * kSlotsPerCta;
    const int ne = max(0, min(kSlotsPerCta, n - e0));
    const int64_t bS = (int64_t)b * A.S;
    for (int e = threadIdx.x; e < ne; e += kAttnThreads) {
        ss[e] = A.att_slot[bS + e0 + e];
        svg[e] = (float)A.att_vg[bS + e0 + e];
        skg[e] = (float)A.att_kg[bS + e0 + e] * scale;
    }
    const int nj = hs / HPL;
    const int hsub = lane / LPH, dch = (lane % LPH) * 8;
    float qv[JMAX][8];
#pragma unroll
    for (int jj = 0; jj < JMAX; ++jj) {
        const int j = warp + jj * nw;
        if (j < nj) {
            const uint4 r = *reinterpret_cast<const uint4*>(q + ((int64_t)b * H + h0 + j * HPL + hsub) * D + dch);
            const uint32_t w4[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[x]));
                qv[jj][2 * x] = f.x;
                qv[jj][2 * x + 1] = f.y;
            }
        }
    }
    __syncthreads();
    const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(A.kpool);
    const __nv_bfloat16* vp = reinterpret_cast<const __nv_bfloat16*>(A.vpool);
    auto dot8 = [](const uint4& r, const float* qq) {
        const uint32_t w4[4] = {r.x, r.y, r.z, r.w};
        float acc = 0.f;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[x]));
            acc = fmaf(qq[2 * x], f.x, fmaf(qq[2 * x + 1], f.y, acc));
        }
        return acc;
    };
    // logits
#pragma unroll
    for (int jj = 0; jj < JMAX; ++jj) {
        const int j = warp + jj * nw;
        if (j >= nj) break;
        const int hl = j * HPL + hsub, h = h0 + hl;
        for (int eb = 0; eb < ne; eb += 8) {
            uint4 r[8];
#pragma unroll
            for (int x = 0; x < 8; ++x)
                if (eb + x < ne) r[x] = *reinterpret_cast<const uint4*>(kp + ((bS + ss[eb + x]) * H + h) * D + dch);
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                float d = eb + x < ne ? dot8(r[x], qv[jj]) : 0.f;
#pragma unroll
                for (int o2 = LPH / 2; o2 > 0; o2 >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o2);
                if ((lane % LPH) == 0 && eb + x < ne) sp[hl * kSlotsPerCta + eb + x] = d * skg[eb + x];
            }
        }
    }
    __syncthreads();
    for (int hl = warp; hl < hs; hl += nw) {
        const int h = h0 + hl;
        float m = -INFINITY;
        for (int e = lane; e < ne; e += 32) m = fmaxf(m, sp[hl * kSlotsPerCta + e]);
        m = warp_max(m);
        float l = 0.f;
        for (int e = lane; e < ne; e += 32) {
            const float pe = expf(sp[hl * kSlotsPerCta + e] - m);
            sp[hl * kSlotsPerCta + e] = pe * svg[e];  // value-gated weight; l keeps the ungated sum
            l += pe;
        }
        l = warp_sum(l);
        if (lane == 0) {
            const int64_t oi = ((int64_t)b * nsplit + chunk) * H + h;
            pm[oi] = ne > 0 ? m : -INFINITY;
            pl[oi] = l;
        }
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < JMAX; ++jj) {
        const int j = warp + jj * nw;
        if (j >= nj) break;
        const int hl = j * HPL + hsub, h = h0 + hl;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int eb = 0; eb < ne; eb += 8) {
            uint4 r[8];
#pragma unroll
            for (int x = 0; x < 8; ++x)
                if (eb + x < ne) r[x] = *reinterpret_cast<const uint4*>(vp + ((bS + ss[eb + x]) * H + h) * D + dch);
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                if (eb + x >= ne) break;
                const float w = sp[hl * kSlotsPerCta + eb + x];
                const uint32_t w4[4] = {r[x].x, r[x].y, r[x].z, r[x].w};
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[y]));
                    acc[2 * y] = fmaf(w, f.x, acc[2 * y]);
                    acc[2 * y + 1] = fmaf(w, f.y, acc[2 * y + 1]);
                }
            }
        }
        float* out = po + (((int64_t)b * nsplit + chunk) * H + h) * D + dch;
        *reinterpret_cast<float4*>(out) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        *reinterpret_cast<float4*>(out + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
    if (o == nullptr) return;  // the separate combine kernel merges the chunks
    // the last chunk CTA of (b, head group) merges every chunk's partials
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        int* cnt = done + (int64_t)b * gridDim.z + blockIdx.z;
        const int t = atomicAdd(cnt, 1);
        s_last = t == (int)gridDim.x - 1;
        if (s_last) *cnt = 0;  // every chunk of this step has arrived: rearm for the next step
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int used = min(nsplit, (n + kSlotsPerCta - 1) / kSlotsPerCta);
    float* sM = sp;            // [hs] reuse the logit tile
    float* sL = sp + hs;       // [hs]
    for (int hl = warp; hl < hs; hl += nw) {
        const int h = h0 + hl;
        float M = -INFINITY;
        for (int sidx = lane; sidx < used; sidx += 32) M = fmaxf(M, __ldcg(pm + ((int64_t)b * nsplit + sidx) * H + h));
        M = warp_max(M);
        float Ls = 0.f;
        for (int sidx = lane; sidx < used; sidx += 32) {
            const int64_t i = ((int64_t)b * nsplit + sidx) * H + h;
            const float mi = __ldcg(pm + i);
            if (mi > -INFINITY) Ls += __ldcg(pl + i) * __expf(mi - M);
        }
        Ls = warp_sum(Ls);
        if (lane == 0) sM[hl] = M, sL[hl] = Ls;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < hs * D; idx += kAttnThreads) {
        const int hl = idx / D, c = idx % D, h = h0 + hl;
        const float M = sM[hl], inv = sL[hl] > 0.f ? 1.f / sL[hl] : 0.f;
        float acc = 0.f;
        for (int sidx = 0; sidx < used; ++sidx) {
            const int64_t i = ((int64_t)b * nsplit + sidx) * H + h;
            const float mi = __ldcg(pm + i);
            if (mi > -INFINITY) acc += __ldcg(po + i * D + c) * __expf(mi - M);
        }
        o[((int64_t)b * H + h) * D + c] = __float2bfloat16(acc * inv);
    }
}

template <class T>
__global__ void __launch_bounds__(128) k_cache_combine(const void* po_, const void* pm_, const void* pl_,
                                                       const int* __restrict__ att_n, int H, int p, int nsplit,
                                                       T* __restrict__ o) {
    // the chunks' weights exp(m_s - M) once per (sequence, head) in shared
    // memory, then every output element's sum over the chunks with its loads
    // in flight together (the per-element loop was latency-bound)
    using Acc = AccOf<T>;
    extern __shared__ __align__(16) uint8_t csm[];
    Acc* wsp = reinterpret_cast<Acc*>(csm);  // [nsplit]
    __shared__ Acc red[4];
    const Acc* po = static_cast<const Acc*>(po_);
    const Acc* pm = static_cast<const Acc*>(pm_);
    const Acc* pl = static_cast<const Acc*>(pl_);
    const int h = blockIdx.x, b = blockIdx.y;
    const int used = min(nsplit, (att_n[b] + kSlotsPerCta - 1) / kSlotsPerCta);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Acc M = -INFINITY;
    for (int s = threadIdx.x; s < used; s += blockDim.x) M = fmax(M, pm[((int64_t)b * nsplit + s) * H + h]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, off));
    if (lane == 0) red[warp] = M;
    __syncthreads();
    M = fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
    __syncthreads();
    Acc ls = 0;
    for (int s = threadIdx.x; s < used; s += blockDim.x) {
        const int64_t i = ((int64_t)b * nsplit + s) * H + h;
        const Acc w = pm[i] > -INFINITY ? exp_acc(pm[i] - M) : Acc(0);
        wsp[s] = w;
        ls += pl[i] * w;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
    if (lane == 0) red[warp] = ls;
    __syncthreads();
    const Acc Lsum = (red[0] + red[1]) + (red[2] + red[3]);
    const Acc inv = Lsum > 0 ? Acc(1) / Lsum : Acc(0);
    for (int c = threadIdx.x; c < p; c += blockDim.x) {
        const Acc* src = po + ((int64_t)b * nsplit * H + h) * p + c;  // + s * H * p
        const int64_t step = (int64_t)H * p;
        Acc a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        int s = 0;
        for (; s + 4 <= used; s += 4) {
            a0 += src[(s + 0) * step] * wsp[s + 0];
            a1 += src[(s + 1) * step] * wsp[s + 1];
            a2 += src[(s + 2) * step] * wsp[s + 2];
            a3 += src[(s + 3) * step] * wsp[s + 3];
        }
        for (; s < used; ++s) a0 += src[s * step] * wsp[s];
        o[((int64_t)b * H + h) * p + c] = (T)(((a0 + a1) + (a2 + a3)) * inv);
    }
}

// ------------------------------------------------------------------ linear mix
// Linear-attention mix decode (Appendix B.1; forward_chunk with linear_mix,
// proj/src/cache.cpp:262-278,322-356): the cache keeps phi(k) of every slot
// row and the prefix state M = sum_j phi(k_j) v_j^T, b = sum_j phi(k_j) over
// every position seen (not only the retained ones).

// M += phi(k_j) v_j^T and b += phi(k_j) over positions [0, n) of a chunk
// (phk float64 [B, n, H, p], v [B, n, H, p]); one CTA per (sequence, head).
template <class S>
__global__ void k_lin_state_add(const double* __restrict__ phk, const S* __restrict__ v, int n, int H, int p,
                                double* __restrict__ M, double* __restrict__ bv) {
    const int b = blockIdx.y, h = blockIdx.x;
    double* Mh = M + ((int64_t)b * H + h) * p * p;
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
        const int r = e / p, c = e % p;
        double acc = 0.0;
        for (int j = 0; j < n; ++j) {
            const int64_t row = (((int64_t)b * n + j) * H + h) * p;
            acc += phk[row + r] * (double)v[row + c];
        }
        Mh[e] += acc;
    }
    for (int r = threadIdx.x; r < p; r += blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += phk[(((int64_t)b * n + j) * H + h) * p + r];
        bv[((int64_t)b * H + h) * p + r] += acc;
    }
}

// phi(k) rows of the positions [t - n, t) that hold a slot -> the phi pool
__global__ void k_lin_fill_phi(CacheArgs A, const double* __restrict__ phk, int n, int H, int p,
                               double* __restrict__ pool) {
    const int b = blockIdx.y, slot = blockIdx.x;
    const int t = A.ctl[b].t;
    const int pos = A.pos_of[(int64_t)b * A.S + slot];
    if (pos < t - n || pos >= t) return;
    const double* src = phk + ((int64_t)b * n + (pos - (t - n))) * H * p;
    double* dst = pool + ((int64_t)b * A.S + slot) * H * p;
    for (int e = threadIdx.x; e < H * p; e += blockDim.x) dst[e] = src[e];
}

// o_i = [sum_att m (e - lambda) v + phi(q)^T M] / [sum_att m (e - lambda) + phi(q).b]; warp per (sequence, head)
template <class S>
__global__ void __launch_bounds__(128) k_lin_decode(CacheArgs A, const S* __restrict__ q, const double* __restrict__ phq,
                                                    const double* __restrict__ pool, const double* __restrict__ M,
                                                    const double* __restrict__ bv, int B, int H, int p, double scale,
                                                    S* __restrict__ o, int* __restrict__ bad) {
    constexpr int kPer = 8;  // head_dim <= 256
    __shared__ double s_pq[4][32 * kPer];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t wid = (int64_t)blockIdx.x * 4 + warp;
    if (wid >= (int64_t)B * H) return;
    const int b = (int)(wid / H), h = (int)(wid % H);
    const int np = (p + 31) / 32;
    double qv[kPer], pq[kPer], num[kPer];
#pragma unroll
    for (int m = 0; m < kPer; ++m) {
        const int c = lane + 32 * m;
        const bool ok = m < np && c < p;
        qv[m] = ok ? (double)q[((int64_t)b * H + h) * p + c] : 0.0;
        pq[m] = ok ? phq[((int64_t)b * H + h) * p + c] : 0.0;
        if (ok) s_pq[warp][c] = pq[m];
        num[m] = 0.0;
    }
    __syncwarp();
    double den = 0.0;
    const int n = A.att_n[b];
    const int64_t bS = (int64_t)b * A.S;
    const S* kp = reinterpret_cast<const S*>(A.kpool);
    const S* vp = reinterpret_cast<const S*>(A.vpool);
    for (int e = 0; e < n; ++e) {
        const int slot = A.att_slot[bS + e];
        const double m = A.att_vg[bS + e];  // the gate (selected) or 1 (window)
        const int64_t ro = ((bS + slot) * H + h) * p;
        double dot = 0.0, lam = 0.0;
#pragma unroll
        for (int x = 0; x < kPer; ++x) {
            const int c = lane + 32 * x;
            if (x < np && c < p) {
                dot += qv[x] * (double)kp[ro + c];
                lam += pq[x] * pool[ro + c];
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            dot += __shfl_xor_sync(0xffffffffu, dot, off);
            lam += __shfl_xor_sync(0xffffffffu, lam, off);
        }
        const double wexact = m * exp(scale * dot), wlin = m * lam;
#pragma unroll
        for (int x = 0; x < kPer; ++x) {
            const int c = lane + 32 * x;
            if (x < np && c < p) num[x] += (wexact - wlin) * (double)vp[ro + c];
        }
        den += wexact - wlin;
    }
    // + phi(q)^T M and phi(q) . b (the prefix accumulators)
    const double* Mh = M + ((int64_t)b * H + h) * p * p;
    const double* bh = bv + ((int64_t)b * H + h) * p;
    double pb = 0.0;
    for (int r = 0; r < p; ++r) {
        const double pr = s_pq[warp][r];
#pragma unroll
        for (int x = 0; x < kPer; ++x) {
            const int c = lane + 32 * x;
            if (x < np && c < p) num[x] += pr * Mh[(int64_t)r * p + c];
        }
        pb += pr * bh[r];
    }
    den += pb;
    if (!(den > 0.0) && lane == 0) *bad = 1;  // proj/src/cache.cpp:349-350
#pragma unroll
    for (int x = 0; x < kPer; ++x) {
        const int c = lane + 32 * x;
        if (x < np && c < p) o[((int64_t)b * H + h) * p + c] = (S)(num[x] / den);
    }
}

}  // namespace
}  // namespace skb

// ====================================================================== C ABI
using namespace skb;

struct skb_stream {
    StreamCtl* ctl = nullptr;
    StreamArr arr{};
    int64_t capacity = 0;
    int* rank_of = nullptr;          // [capacity] solution scratch
    StreamStepRes* dres = nullptr;   // device result of the last push_step
    StreamSolRes* dsol = nullptr;
    uint8_t* hres = nullptr;         // pinned: StreamStepRes + the first kLogInline evicted indices
    static constexpr int kLogInline = 64;
};

// Host-side state of a SparseKvCache snapshot that the device arrays do not
// hold: the cache min-heap in the reference's array order, the evicted bitmap
// and the pending-eviction list (proj/src/cache.cpp:115-179). Replayed from
// the recorded exit pushes (ins_hist) starting at `t0` (0, or a restore point).
struct SnapBase {
    long long t0 = 0;
    std::vector<std::pair<double, long long>> heap;  // (score, pos)
    std::vector<long long> cache_pos;                // ascending
    std::vector<uint8_t> evicted;
    std::vector<long long> pending;
};

struct skb_cache {
    skb_attn_desc d{};
    CacheArgs A{};
    std::vector<SnapBase> base;
    int nsplit = 0;
    int vec = 1;
    double* po = nullptr;  // split partials: float64 for float64 pools, else float32
    int* done = nullptr;   // [B, head groups] chunk CTAs finished this step (bf16 fast path; self-rearming)
    double* pm = nullptr;
    double* pl = nullptr;
    double* zeros = nullptr;  // [B] idle scores for k = 0 (on the cache's device)
    // linear mix: phi(k) of every slot row [B, S, H, p], the prefix state
    // M = sum phi(k_j) v_j^T [B, H, p, p] and b = sum phi(k_j) [B, H, p] (float64)
    double *lphk = nullptr, *lm = nullptr, *lb = nullptr;
    int* flag = nullptr;  // device word for kernel-side errors (linear mix)
    int* zeros_flag() {
        if (!flag) flag = alloc<int>(1);
        return flag;
    }
    std::vector<void*> allocs;
    ~skb_cache() {
        for (void* p : allocs) cudaFree(p);
    }
    template <class P>
    P* alloc(size_t count) {
        void* p = nullptr;
        SKB_CHECK_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(P)));
        allocs.push_back(p);
        return static_cast<P*>(p);
    }
};

namespace skb {
void set_last_error(const char* msg);  // skb_capi.cu (thread-local skb_last_error)
}

#define K5_BEGIN try {
#define K5_END                                                              \
    }                                                                       \
    catch (const skb::Error& e) {                                           \
        skb::set_last_error(e.what());                                      \
        return e.code;                                                      \
    }                                                                       \
    catch (const std::exception& e) {                                       \
        skb::set_last_error(e.what());                                      \
        return SKB_ECUDA;                                                   \
    }                                                                       \
    return SKB_OK;

static size_t esize_of(int dt) { return dt == SKB_F64 ? 8 : dt == SKB_F32 ? 4 : 2; }

extern "C" {

int skb_stream_create(double k, int64_t heap_cap, int64_t capacity, skb_stream** out) {
    K5_BEGIN
    SKB_REQUIRE(out != nullptr, SKB_EARG, "stream_create: null out");
    SKB_REQUIRE(std::isfinite(k) && k > 0.0, SKB_EARG, "KBudget: k must be positive and finite");
    SKB_REQUIRE(heap_cap >= 0, SKB_EARG, "stream_create: heap_cap must be >= 0");
    SKB_REQUIRE(heap_cap == 0 || (double)heap_cap >= std::ceil(k), SKB_EARG,
                "stream: heap_cap below ceil(k)");
    SKB_REQUIRE(capacity >= 1 && capacity < (int64_t(1) << 30), SKB_EARG, "stream_create: bad capacity");
    skb_stream* s = new skb_stream();
    s->capacity = capacity;
    void* p = nullptr;
    // ctl | sv fv | si fi | evlog rank_of | step/solution results | evcount | evicted bits
    const size_t ctl_b = (sizeof(StreamCtl) + 15) & ~size_t(15);
    cudaError_t e = cudaMalloc(&p, ctl_b + (size_t)capacity * (8 + 8 + 4 + 4 + 4 + 4 + 1) + 256);
    if (e != cudaSuccess) {
        delete s;
        throw skb::Error(SKB_ECUDA, std::string("stream_create: ") + cudaGetErrorString(e));
    }
    char* base = static_cast<char*>(p);
    s->ctl = reinterpret_cast<StreamCtl*>(base);
    char* q = base + ctl_b;
    s->arr.sv = reinterpret_cast<double*>(q);
    s->arr.fv = s->arr.sv + capacity;
    s->arr.si = reinterpret_cast<int*>(s->arr.fv + capacity);
    s->arr.fi = s->arr.si + capacity;
    s->arr.evlog = s->arr.fi + capacity;
    s->rank_of = s->arr.evlog + capacity;
    char* r8 = reinterpret_cast<char*>(s->rank_of + capacity);
    r8 = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(r8) + 15) & ~uintptr_t(15));
    s->dres = reinterpret_cast<StreamStepRes*>(r8);
    s->dsol = reinterpret_cast<StreamSolRes*>(r8 + 64);
    s->arr.evcount = reinterpret_cast<int*>(r8 + 96);
    s->arr.evicted = reinterpret_cast<uint8_t*>(r8 + 128);
    e = cudaMallocHost(&s->hres, 64 + sizeof(int) * skb_stream::kLogInline);
    if (e != cudaSuccess) {
        cudaFree(p);
        delete s;
        throw skb::Error(SKB_ECUDA, std::string("stream_create: ") + cudaGetErrorString(e));
    }
    StreamCtl c{};
    c.k = k;
    c.tau = -INFINITY;
    c.heap_cap = heap_cap;
    c.cap = (int)capacity;
    SKB_CHECK_CUDA(cudaMemcpy(s->ctl, &c, sizeof(c), cudaMemcpyHostToDevice));
    SKB_CHECK_CUDA(cudaMemset(s->arr.evicted, 0, capacity));
    *out = s;
    K5_END
}

int skb_stream_destroy(skb_stream* s) {
    if (s) {
        cudaFreeHost(s->hres);
        cudaFree(s->ctl);
        delete s;
    }
    return SKB_OK;
}

int skb_stream_push(skb_stream* s, const double* z, int64_t n, double* tau_out, uint8_t* inserted_out,
                    void* stream) {
    K5_BEGIN
    SKB_REQUIRE(s != nullptr, SKB_EARG, "stream_push: null stream");
    SKB_REQUIRE(n >= 0, SKB_EARG, "stream_push: n must be >= 0");
    if (n == 0) return SKB_OK;
    SKB_REQUIRE(z != nullptr, SKB_EARG, "stream_push: null z");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamCtl c;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    SKB_REQUIRE(c.t + n <= s->capacity, SKB_ESHAPE, "stream_push: capacity exceeded");
    StreamArr arr = s->arr;
    arr.evlog = nullptr;  // batched pushes report through tau/inserted only
    k_stream_push<<<1, 32, 0, st>>>(s->ctl, arr, z, (int)n, tau_out, inserted_out);
    SKB_CHECK_LAUNCH();
    SKB_CHECK_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    SKB_REQUIRE(c.error == 0, SKB_ENUMERIC, "stream scan exhausted (internal)");
    K5_END
}

int skb_stream_push_step(skb_stream* s, double z, skb_stream_step* out, int64_t* evicted, int64_t max_evicted,
                         void* stream) {
    K5_BEGIN
    SKB_REQUIRE(s != nullptr && out != nullptr, SKB_EARG, "stream_push: null argument");
    SKB_REQUIRE(std::isfinite(z), SKB_ENUMERIC, "stream_push: non-finite value");
    SKB_REQUIRE(max_evicted >= 0 && (max_evicted == 0 || evicted != nullptr), SKB_EARG,
                "stream_push: bad evicted buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_stream_push_step<<<1, 32, 0, st>>>(s->ctl, s->arr, z, s->dres);
    SKB_CHECK_LAUNCH();
    // one round trip: the result and the first kLogInline popped indices
    SKB_CHECK_CUDA(cudaMemcpyAsync(s->hres, s->dres, sizeof(StreamStepRes), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaMemcpyAsync(s->hres + 64, s->arr.evlog, sizeof(int) * skb_stream::kLogInline,
                                   cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    StreamStepRes r;
    std::memcpy(&r, s->hres, sizeof(r));
    SKB_REQUIRE(r.error != 2, SKB_ESHAPE, "stream_push: capacity exceeded");
    SKB_REQUIRE(r.error == 0, SKB_ENUMERIC, "stream scan exhausted (internal)");
    out->tau = r.tau;
    out->t = r.t;
    out->inserted = r.inserted;
    out->cap_forced = r.cap_forced;
    out->n_evicted = r.n_evicted;
    const int64_t ncopy = std::min<int64_t>(r.n_evicted, max_evicted);
    const int* inl = reinterpret_cast<const int*>(s->hres + 64);
    std::vector<int> tail;
    if (ncopy > skb_stream::kLogInline) {
        tail.resize((size_t)ncopy);
        SKB_CHECK_CUDA(cudaMemcpy(tail.data(), s->arr.evlog, sizeof(int) * ncopy, cudaMemcpyDeviceToHost));
        inl = tail.data();
    }
    for (int64_t i = 0; i < ncopy; ++i) evicted[i] = inl[i];
    K5_END
}

int skb_stream_solution(skb_stream* s, double* p, int64_t* indices, uint8_t* hard, skb_stream_solution_info* out,
                        void* stream) {
    K5_BEGIN
    SKB_REQUIRE(s != nullptr && out != nullptr && p != nullptr && indices != nullptr, SKB_EARG,
                "stream_solution: null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_stream_solution<<<1, 1024, 0, st>>>(s->ctl, s->arr, s->rank_of, p, reinterpret_cast<long long*>(indices),
                                          hard, s->dsol);
    SKB_CHECK_LAUNCH();
    StreamCtl c;
    StreamSolRes r;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaMemcpyAsync(&r, s->dsol, sizeof(r), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    const bool infeasible = (double)c.t < c.k;
    out->tau = infeasible ? -INFINITY : c.tau;
    out->t = c.t;
    out->n = r.n;
    out->u_count = r.u_count;
    out->w_count = r.w_count;
    out->infeasible = infeasible ? 1 : 0;
    out->degenerate = (infeasible || r.u_count == r.w_count) ? 1 : 0;
    K5_END
}

int skb_stream_query(skb_stream* s, skb_stream_info* out, void* stream) {
    K5_BEGIN
    SKB_REQUIRE(s != nullptr && out != nullptr, SKB_EARG, "stream_query: null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamCtl c;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    out->tau = c.tau;
    out->t = c.t;
    out->survivors = c.nS;
    out->saturated = c.nF;
    out->cap_drops = c.cap_drops;
    out->heap_ops = c.heap_ops;
    out->k = c.k;
    K5_END
}

int skb_stream_serialize(skb_stream* s, uint8_t* out, size_t* bytes, void* stream) {
    K5_BEGIN
    SKB_REQUIRE(s != nullptr && bytes != nullptr, SKB_EARG, "stream_serialize: null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamCtl c;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    const size_t need = 8 * 9 + 8 + (size_t)c.nS * 16 + 8 + (size_t)c.nF * 16 + 8 + (size_t)(c.t + 7) / 8;
    if (!out) {
        *bytes = need;
        return SKB_OK;
    }
    SKB_REQUIRE(*bytes >= need, SKB_EARG, "stream_serialize: buffer too small");
    std::vector<double> sv(c.nS), fv(c.nF);
    std::vector<int> si(c.nS), fi(c.nF);
    std::vector<uint8_t> ev(c.t);
    if (c.nS) {
        SKB_CHECK_CUDA(cudaMemcpyAsync(sv.data(), s->arr.sv, c.nS * 8, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaMemcpyAsync(si.data(), s->arr.si, c.nS * 4, cudaMemcpyDeviceToHost, st));
    }
    if (c.nF) {
        SKB_CHECK_CUDA(cudaMemcpyAsync(fv.data(), s->arr.fv, c.nF * 8, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaMemcpyAsync(fi.data(), s->arr.fi, c.nF * 4, cudaMemcpyDeviceToHost, st));
    }
    if (c.t) SKB_CHECK_CUDA(cudaMemcpyAsync(ev.data(), s->arr.evicted, c.t, cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    size_t off = 0;
    auto put = [&](const void* p, size_t n) {
        std::memcpy(out + off, p, n);
        off += n;
    };
    const uint64_t hc = (uint64_t)c.heap_cap, tt = (uint64_t)c.t, psr = (uint64_t)c.since_refresh;
    put(&c.k, 8);
    put(&hc, 8);
    put(&c.tau, 8);
    put(&tt, 8);
    put(&c.sum_s, 8);
    put(&c.sum_f, 8);
    put(&c.cap_drops, 8);
    put(&c.heap_ops, 8);
    put(&psr, 8);
    auto put_heap = [&](const std::vector<double>& v, const std::vector<int>& ix) {
        const uint64_t n = v.size();
        put(&n, 8);
        for (size_t r = v.size(); r-- > 0;) {  // (value asc, index desc): a valid HeapCmp heap
            const uint64_t i64 = (uint64_t)ix[r];
            put(&v[r], 8);
            put(&i64, 8);
        }
    };
    put_heap(sv, si);
    put_heap(fv, fi);
    put(&tt, 8);
    for (int64_t i = 0; i < c.t; i += 8) {
        uint8_t byte = 0;
        for (int b = 0; b < 8 && i + b < c.t; ++b)
            if (ev[i + b]) byte |= (uint8_t)(1u << b);
        put(&byte, 1);
    }
    *bytes = off;
    K5_END
}

int skb_stream_deserialize(const uint8_t* data, size_t bytes, int64_t capacity, skb_stream** out) {
    K5_BEGIN
    SKB_REQUIRE(data != nullptr && out != nullptr, SKB_EARG, "stream_deserialize: null argument");
    size_t off = 0;
    auto get = [&](void* p, size_t n) {
        SKB_REQUIRE(off + n <= bytes, SKB_EIO, "stream state: truncated buffer");
        std::memcpy(p, data + off, n);
        off += n;
    };
    double k, tau, sum_s, sum_f;
    uint64_t heap_cap, t, cap_drops, heap_ops, psr;
    get(&k, 8);
    get(&heap_cap, 8);
    get(&tau, 8);
    get(&t, 8);
    get(&sum_s, 8);
    get(&sum_f, 8);
    get(&cap_drops, 8);
    get(&heap_ops, 8);
    get(&psr, 8);
    auto get_heap = [&](std::vector<std::pair<double, int64_t>>& h) {
        uint64_t n;
        get(&n, 8);
        SKB_REQUIRE(n <= bytes / 16, SKB_EIO, "stream state: truncated buffer");
        h.resize(n);
        for (auto& e : h) {
            uint64_t ix;
            get(&e.first, 8);
            get(&ix, 8);
            e.second = (int64_t)ix;
        }
        // device layout: (value desc, index asc)
        std::sort(h.begin(), h.end(), [](const auto& a, const auto& b) {
            return a.first > b.first || (a.first == b.first && a.second < b.second);
        });
    };
    std::vector<std::pair<double, int64_t>> hs, hf;
    get_heap(hs);
    get_heap(hf);
    uint64_t nbits;
    get(&nbits, 8);
    SKB_REQUIRE(nbits == t, SKB_EIO, "stream state: evicted bits do not cover the pushes");
    std::vector<uint8_t> ev(nbits);
    for (uint64_t i = 0; i < nbits; i += 8) {
        uint8_t byte;
        get(&byte, 1);
        for (uint64_t b = 0; b < 8 && i + b < nbits; ++b) ev[i + b] = (byte >> b) & 1u;
    }
    SKB_REQUIRE(capacity >= (int64_t)t, SKB_EARG, "stream_deserialize: capacity below the pushes so far");
    skb_stream* s = nullptr;
    int rc = skb_stream_create(k, (int64_t)heap_cap, std::max<int64_t>(capacity, 1), &s);
    if (rc != SKB_OK) return rc;
    StreamCtl c{};
    c.k = k;
    c.tau = tau;
    c.sum_s = sum_s;
    c.sum_f = sum_f;
    c.t = (long long)t;
    c.heap_cap = (long long)heap_cap;
    c.heap_ops = heap_ops;
    c.cap_drops = cap_drops;
    c.nS = (int)hs.size();
    c.nF = (int)hf.size();
    c.since_refresh = (int)psr;
    c.cap = (int)s->capacity;
    std::vector<double> v(std::max(hs.size(), hf.size()));
    std::vector<int> ix(v.size());
    auto upload = [&](const std::vector<std::pair<double, int64_t>>& h, double* dv, int* di) {
        for (size_t i = 0; i < h.size(); ++i) {
            v[i] = h[i].first;
            ix[i] = (int)h[i].second;
        }
        if (!h.empty()) {
            SKB_CHECK_CUDA(cudaMemcpy(dv, v.data(), h.size() * 8, cudaMemcpyHostToDevice));
            SKB_CHECK_CUDA(cudaMemcpy(di, ix.data(), h.size() * 4, cudaMemcpyHostToDevice));
        }
    };
    upload(hs, s->arr.sv, s->arr.si);
    upload(hf, s->arr.fv, s->arr.fi);
    if (t) SKB_CHECK_CUDA(cudaMemcpy(s->arr.evicted, ev.data(), t, cudaMemcpyHostToDevice));
    SKB_CHECK_CUDA(cudaMemcpy(s->ctl, &c, sizeof(c), cudaMemcpyHostToDevice));
    *out = s;
    K5_END
}

int skb_stream_survivors(skb_stream* s, double* values, int64_t* indices, uint8_t* evicted, void* stream) {
    K5_BEGIN
    SKB_REQUIRE(s != nullptr, SKB_EARG, "stream_survivors: null stream");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamCtl c;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof(c), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    std::vector<double> v(c.nS);
    std::vector<int> ix(c.nS);
    if (c.nS) {
        SKB_CHECK_CUDA(cudaMemcpyAsync(v.data(), s->arr.sv, c.nS * 8, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaMemcpyAsync(ix.data(), s->arr.si, c.nS * 4, cudaMemcpyDeviceToHost, st));
    }
    if (evicted && c.t)
        SKB_CHECK_CUDA(cudaMemcpyAsync(evicted, s->arr.evicted, (size_t)c.t, cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    // ascending index order (StreamState::solution, proj/src/stream.cpp:157-158)
    std::vector<int> order(c.nS);
    for (int i = 0; i < c.nS; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return ix[a] < ix[b]; });
    for (int i = 0; i < c.nS; ++i) {
        if (values) values[i] = v[order[i]];
        if (indices) indices[i] = ix[order[i]];
    }
    K5_END
}

int skb_cache_create(const skb_attn_desc* d, skb_cache** out) {
    K5_BEGIN
    SKB_REQUIRE(d != nullptr && out != nullptr, SKB_EARG, "cache_create: null argument");
    skb::validate_desc(*d);
    const int64_t B = d->batch, Lmax = d->seq_len, H = d->heads, p = d->head_dim;
    const int cap = (int)floor_k(d->k);
    const int64_t S = cap + d->window + 1;
    SKB_REQUIRE(S < (int64_t(1) << 24), SKB_ECONFIG, "cache: floor(k) + window too large");
    auto* c = new skb_cache();
    try {
        c->d = *d;
        CacheArgs& A = c->A;
        A.Lmax = (int)Lmax;
        A.S = (int)S;
        A.cap = cap;
        A.w = (int)d->window;
        A.lin = (d->flags & SKB_FLAG_LINEAR_MIX) ? 1 : 0;
        // the mixture weight of a selected key is its gate whatever the key/mask modes (cache.cpp:330)
        A.key_soft = A.lin ? 0 : d->key_mode;
        A.mask_st = A.lin ? 0 : d->mask_mode;
        A.row_bytes = H * p * (int64_t)esize_of(d->dtype);
        A.ctl = c->alloc<CacheCtl>(B);
        A.sv = c->alloc<double>(B * Lmax);
        A.si = c->alloc<int>(B * Lmax);
        A.fv = c->alloc<double>(B * Lmax);
        A.fi = c->alloc<int>(B * Lmax);
        A.u_hist = c->alloc<double>(B * Lmax);
        A.slot_of = c->alloc<int>(B * Lmax);
        A.ins_hist = c->alloc<uint8_t>(B * Lmax);
        c->base.assign((size_t)B, SnapBase{});
        A.pos_of = c->alloc<int>(B * S);
        A.free_stack = c->alloc<int>(B * S);
        A.att_slot = c->alloc<int>(B * S);
        A.att_kg = c->alloc<double>(B * S);
        A.att_vg = c->alloc<double>(B * S);
        A.att_n = c->alloc<int>(B);
        A.kpool = c->alloc<uint8_t>((size_t)(B * S) * A.row_bytes);
        A.vpool = c->alloc<uint8_t>((size_t)(B * S) * A.row_bytes);
        SKB_CHECK_CUDA(cudaMemset(A.kpool, 0, (size_t)(B * S) * A.row_bytes));
        SKB_CHECK_CUDA(cudaMemset(A.vpool, 0, (size_t)(B * S) * A.row_bytes));
        c->nsplit = (int)cdiv(S, kSlotsPerCta);
        c->po = c->alloc<double>(B * c->nsplit * H * p);  // sized for float64 partials
        c->pm = c->alloc<double>(B * c->nsplit * H);
        c->pl = c->alloc<double>(B * c->nsplit * H);
        c->done = c->alloc<int>(B * H);  // >= one counter per (sequence, head group)
        SKB_CHECK_CUDA(cudaMemset(c->done, 0, (size_t)B * H * sizeof(int)));
        c->vec = (p % 128 == 0) ? 4 : (p % 64 == 0) ? 2 : 1;
        c->zeros = c->alloc<double>(B);
        SKB_CHECK_CUDA(cudaMemset(c->zeros, 0, B * sizeof(double)));
        if (A.lin) {
            SKB_REQUIRE(d->dtype == SKB_F32 || d->dtype == SKB_F64, SKB_EARG,
                        "linear mix: dtype must be float32 or float64 (the reference's instantiations)");
            c->lphk = c->alloc<double>(B * S * H * p);
            c->lm = c->alloc<double>(B * H * p * p);
            c->lb = c->alloc<double>(B * H * p);
            SKB_CHECK_CUDA(cudaMemset(c->lm, 0, (size_t)B * H * p * p * 8));
            SKB_CHECK_CUDA(cudaMemset(c->lb, 0, (size_t)B * H * p * 8));
        }
        k_cache_init<<<(unsigned)B, 256>>>(A, d->k);
        SKB_CHECK_LAUNCH();
        SKB_CHECK_CUDA(cudaDeviceSynchronize());
    } catch (...) {
        delete c;
        throw;
    }
    *out = c;
    K5_END
}

int skb_cache_destroy(skb_cache* c) {
    delete c;
    return SKB_OK;
}

}  // extern "C"

template <class T>
static void cache_attend(skb_cache* c, const void* q, void* o, cudaStream_t st) {
    const skb_attn_desc& d = c->d;
    const int H = (int)d.heads, p = (int)d.head_dim;
    const double scale_d = d.scale > 0.0 ? d.scale : 1.0 / std::sqrt((double)p);
    const float scale = (float)scale_d;
    const size_t asz = sizeof(AccOf<T>);
    const size_t smem = (size_t)H * p * asz + (size_t)H * kSlotsPerCta * asz + kSlotsPerCta * (asz + 4);
    SKB_REQUIRE(smem <= 200 * 1024, SKB_ECONFIG, "cache: heads * head_dim too large for the decode kernel");
    dim3 g((unsigned)c->nsplit, (unsigned)d.batch);
    auto launch = [&](auto kern) {
        if (smem > 48 * 1024)
            SKB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<g, kAttnThreads, smem, st>>>(c->A, static_cast<const T*>(q), H, p, scale_d, c->po, c->pm, c->pl,
                                            c->nsplit);
    };
    constexpr bool kBf16 = std::is_same<T, __nv_bfloat16>::value;
    const bool fast = kBf16 && (p == 128 || p == 64) && (H % (256 / p)) == 0 && H / (256 / p) <= 4 * 8;
    if (fast) {
        // head groups of 16 (or 8 at head_dim 64): 2-4x the CTAs of one group per
        // (chunk, sequence), so the grid runs in several waves instead of 1.35
        const int hpl = 256 / p;  // heads per warp load
        static const int hs_env = getenv("SKB_DEC_HS") ? atoi(getenv("SKB_DEC_HS")) : 16;  // heads per CTA (cfg4: 16 vs 32 measured -1.1 %)
        static const int fuse = getenv("SKB_DEC_FUSE") ? atoi(getenv("SKB_DEC_FUSE")) : 0;
        int hs = std::min(H, hs_env > 0 ? hs_env : H);
        hs = std::max(hpl, hs - hs % hpl);
        while (H % hs) hs -= hpl;  // a divisor of H, a multiple of hpl (H % hpl == 0 on this path)
        const size_t fsmem = (size_t)hs * kSlotsPerCta * 4 + kSlotsPerCta * 12;
        const dim3 gh((unsigned)c->nsplit, (unsigned)d.batch, (unsigned)(H / hs));
        auto run = [&](auto kern) {
            if (fsmem > 48 * 1024)
                SKB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
            kern<<<gh, kAttnThreads, fsmem, st>>>(c->A, reinterpret_cast<const __nv_bfloat16*>(q), H, scale,
                                                  reinterpret_cast<float*>(c->po), reinterpret_cast<float*>(c->pm),
                                                  reinterpret_cast<float*>(c->pl), c->nsplit, hs, c->done,
                                                  fuse ? static_cast<__nv_bfloat16*>(o) : nullptr);
        };
        SKB_REQUIRE(H % hs == 0, SKB_ECONFIG, "cache: heads must be a multiple of the decode head group");
        // the head groups a warp covers: hs / hpl over 8 warps
        const bool j2 = hs / hpl <= 2 * (kAttnThreads / 32);
        if (p == 128) {
            if (j2) run(k_cache_attn_bf16<128, 2>);
            else run(k_cache_attn_bf16<128, 4>);
        } else {
            if (j2) run(k_cache_attn_bf16<64, 2>);
            else run(k_cache_attn_bf16<64, 4>);
        }
        SKB_CHECK_LAUNCH();
        if (fuse) return;  // the last chunk CTA of each (sequence, head group) wrote o
    } else if (c->vec == 4) launch(k_cache_attn<T, 4>);
    else if (c->vec == 2) launch(k_cache_attn<T, 2>);
    else launch(k_cache_attn<T, 1>);
    SKB_CHECK_LAUNCH();
    k_cache_combine<T><<<dim3((unsigned)H, (unsigned)d.batch), 128, (size_t)c->nsplit * sizeof(AccOf<T>), st>>>(
        c->po, c->pm, c->pl, c->A.att_n, H, p, c->nsplit, static_cast<T*>(o));
    SKB_CHECK_LAUNCH();
}
// the control launch (dynamic shared memory above 48 KB is a per-device attribute)
static void launch_control(skb_cache* c, int B, const void* k, const void* v, const double* uu, cudaStream_t st) {
    static uint64_t attr = 0;
    if (first_on_device(&attr))
        SKB_CHECK_CUDA(cudaFuncSetAttribute(k_cache_control, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kCtlSmemBytes));
    k_cache_control<<<(unsigned)B, kControlThreads, kCtlSmemBytes, st>>>(c->A, B, static_cast<const uint8_t*>(k),
                                                                         static_cast<const uint8_t*>(v), uu);
}


extern "C" {

int skb_cache_step(skb_cache* c, const void* q, const void* k, const void* v, const double* u, void* o,
                   void* stream) {
    K5_BEGIN
    SKB_REQUIRE(c != nullptr, SKB_EARG, "cache_step: null cache");
    SKB_REQUIRE(q && k && v && o, SKB_EARG, "cache_step: null tensor");
    SKB_REQUIRE(u != nullptr || c->d.k == 0.0, SKB_EARG, "cache_step: null scores");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = (int)c->d.batch;
    const double* uu = u;
    if (!uu) uu = c->zeros;  // k = 0: scores idle (proj/src/cache.cpp:219-227)
    launch_control(c, B, k, v, uu, st);
    SKB_CHECK_LAUNCH();
    if (c->d.dtype == SKB_BF16) cache_attend<__nv_bfloat16>(c, q, o, st);
    else if (c->d.dtype == SKB_F32) cache_attend<float>(c, q, o, st);
    else cache_attend<double>(c, q, o, st);
    K5_END
}

// Linear-attention mix (Appendix B.1) on a cache created with
// SKB_FLAG_LINEAR_MIX (float32/float64): after skb_cache_prefill(k, v, u, n),
// skb_cache_linmix_prefill(v, phk, n) records phi(k) of the retained rows and
// adds the n positions to the prefix state; a step is
// skb_cache_linmix_step(q, k, v, u, phq, phk) -> the mixture readout o.
// phq / phk: float64 phi rows (skb_linmix_phi) [B, H, p] (step) or [B, n, H, p].
int skb_cache_linmix_prefill(skb_cache* c, const void* v, const double* phk, int64_t n, void* stream) {
    K5_BEGIN
    SKB_REQUIRE(c != nullptr && v && phk, SKB_EARG, "cache_linmix_prefill: null argument");
    SKB_REQUIRE(c->A.lin, SKB_ECONFIG, "forward_chunk: linear mix needs feature parameters");
    if (n == 0) return SKB_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = (int)c->d.batch, H = (int)c->d.heads, p = (int)c->d.head_dim;
    k_lin_fill_phi<<<dim3((unsigned)c->A.S, (unsigned)B), 128, 0, st>>>(c->A, phk, (int)n, H, p, c->lphk);
    SKB_CHECK_LAUNCH();
    if (c->d.dtype == SKB_F64)
        k_lin_state_add<double><<<dim3((unsigned)H, (unsigned)B), 256, 0, st>>>(
            phk, static_cast<const double*>(v), (int)n, H, p, c->lm, c->lb);
    else
        k_lin_state_add<float><<<dim3((unsigned)H, (unsigned)B), 256, 0, st>>>(
            phk, static_cast<const float*>(v), (int)n, H, p, c->lm, c->lb);
    SKB_CHECK_LAUNCH();
    K5_END
}

int skb_cache_linmix_step(skb_cache* c, const void* q, const void* k, const void* v, const double* u,
                          const double* phq, const double* phk, void* o, void* stream) {
    K5_BEGIN
    SKB_REQUIRE(c != nullptr && q && k && v && phq && phk && o, SKB_EARG, "cache_linmix_step: null argument");
    SKB_REQUIRE(c->A.lin, SKB_ECONFIG, "forward_chunk: linear mix needs feature parameters");
    SKB_REQUIRE(u != nullptr || c->d.k == 0.0, SKB_EARG, "cache_step: null scores");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = (int)c->d.batch, H = (int)c->d.heads, p = (int)c->d.head_dim;
    SKB_REQUIRE(p <= 256, SKB_ESHAPE, "linear mix: head_dim must be <= 256");
    const double* uu = u ? u : c->zeros;
    launch_control(c, B, k, v, uu, st);
    SKB_CHECK_LAUNCH();
    // pass 1 of the position: its phi(k) row and the prefix state include it (cache.cpp:267-278)
    k_lin_fill_phi<<<dim3((unsigned)c->A.S, (unsigned)B), 128, 0, st>>>(c->A, phk, 1, H, p, c->lphk);
    const double scale = c->d.scale > 0.0 ? c->d.scale : 1.0 / std::sqrt((double)p);
    int* bad = c->zeros_flag();
    SKB_CHECK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    const unsigned g = (unsigned)cdiv((int64_t)B * H, 4);
    if (c->d.dtype == SKB_F64) {
        k_lin_state_add<double><<<dim3((unsigned)H, (unsigned)B), 256, 0, st>>>(
            phk, static_cast<const double*>(v), 1, H, p, c->lm, c->lb);
        k_lin_decode<double><<<dim3(g), 128, 0, st>>>(c->A, static_cast<const double*>(q), phq, c->lphk, c->lm, c->lb,
                                                      B, H, p, scale, static_cast<double*>(o), bad);
    } else {
        k_lin_state_add<float><<<dim3((unsigned)H, (unsigned)B), 256, 0, st>>>(
            phk, static_cast<const float*>(v), 1, H, p, c->lm, c->lb);
        k_lin_decode<float><<<dim3(g), 128, 0, st>>>(c->A, static_cast<const float*>(q), phq, c->lphk, c->lm, c->lb,
                                                     B, H, p, scale, static_cast<float*>(o), bad);
    }
    SKB_CHECK_LAUNCH();
    int hbad = 0;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    SKB_REQUIRE(!hbad, SKB_ENUMERIC, "linear mix: nonpositive denominator");
    K5_END
}

int skb_cache_prefill(skb_cache* c, const void* k, const void* v, const double* u, int64_t n, void* stream) {
    K5_BEGIN
    SKB_REQUIRE(c != nullptr, SKB_EARG, "cache_prefill: null cache");
    SKB_REQUIRE(n >= 0, SKB_EARG, "cache_prefill: n must be >= 0");
    if (n == 0) return SKB_OK;
    SKB_REQUIRE(k && v, SKB_EARG, "cache_prefill: null tensor");
    SKB_REQUIRE(u != nullptr, SKB_EARG, "cache_prefill: null scores");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = (int)c->d.batch;
    CacheCtl c0;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&c0, c->A.ctl, sizeof(c0), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    SKB_REQUIRE(c0.t + n <= c->A.Lmax, SKB_ESHAPE, "cache_prefill: more positions than seq_len");
    k_cache_prefill<<<(unsigned)cdiv(B, 4), 128, 0, st>>>(c->A, B, u, (int)n);
    SKB_CHECK_LAUNCH();
    dim3 g((unsigned)cdiv(c->A.S, 8), (unsigned)B);
    k_cache_fill_rows<<<g, 256, 0, st>>>(c->A, static_cast<const uint8_t*>(k), static_cast<const uint8_t*>(v),
                                         (int)c0.t, (int)n);
    SKB_CHECK_LAUNCH();
    K5_END
}

int skb_cache_state(skb_cache* c, int64_t b, int32_t* positions, int64_t* count, double* tau, int64_t* seen,
                    int64_t* peak, void* stream) {
    K5_BEGIN
    SKB_REQUIRE(c != nullptr, SKB_EARG, "cache_state: null cache");
    SKB_REQUIRE(b >= 0 && b < c->d.batch, SKB_EARG, "cache_state: batch index out of range");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const CacheArgs& A = c->A;
    CacheCtl cc;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&cc, A.ctl + b, sizeof(cc), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    SKB_REQUIRE(cc.error == 0, cc.error == 2 ? SKB_ESHAPE : SKB_ENUMERIC,
                cc.error == 2 ? "cache: more positions than seq_len" : "stream scan exhausted (internal)");
    std::vector<int> sel(cc.nsel);
    if (cc.nsel)
        SKB_CHECK_CUDA(cudaMemcpyAsync(sel.data(), A.si + b * A.Lmax, cc.nsel * 4, cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    std::sort(sel.begin(), sel.end());
    // retained_positions: cache (ascending) then the window ring (proj/src/cache.cpp:585-589)
    std::vector<int> out(sel.begin(), sel.end());
    const long long r0 = std::max<long long>(0, cc.t - A.w);
    for (long long jp = r0; jp < cc.t; ++jp) out.push_back((int)jp);
    if (positions)
        for (size_t i = 0; i < out.size(); ++i) positions[i] = out[i];
    if (count) *count = (int64_t)out.size();
    if (tau) *tau = cc.st.tau;
    if (seen) *seen = cc.t;
    if (peak) *peak = cc.peak;
    K5_END
}

}  // extern "C"

// ------------------------------------------------------------------ snapshots
namespace {

// the reference's cache heap order (SlotCmp, proj/src/cache.cpp:55-60):
// std heaps with this comparator keep the lowest (score, then latest pos) in front
struct SnapSlotCmp {
    bool operator()(const std::pair<double, long long>& a, const std::pair<double, long long>& b) const {
        return a.first > b.first || (a.first == b.first && a.second < b.second);
    }
};

struct Bytes {
    std::vector<uint8_t> v;
    void raw(const void* p, size_t n) {
        const uint8_t* q = static_cast<const uint8_t*>(p);
        v.insert(v.end(), q, q + n);
    }
    void u64(uint64_t x) { raw(&x, 8); }
    void f64(double x) { raw(&x, 8); }
    void u8(uint8_t x) { v.push_back(x); }
};

struct Reader {
    const uint8_t* p;
    size_t n, off = 0;
    void raw(void* dst, size_t k) {
        SKB_REQUIRE(off + k <= n, SKB_EIO, "cache snapshot: truncated");
        std::memcpy(dst, p + off, k);
        off += k;
    }
    uint64_t u64() {
        uint64_t x;
        raw(&x, 8);
        return x;
    }
    double f64() {
        double x;
        raw(&x, 8);
        return x;
    }
    uint8_t u8() {
        uint8_t x;
        raw(&x, 1);
        return x;
    }
    // an element count, bounded by the bytes left (each element >= elem bytes)
    uint64_t count(size_t elem) {
        const uint64_t c = u64();
        SKB_REQUIRE(c <= (n - off) / elem, SKB_EIO, "cache snapshot: truncated");
        return c;
    }
};

void evict_mark(SnapBase& sb, long long pos) {  // drop_kv (proj/src/cache.cpp:115-125)
    if ((long long)sb.evicted.size() <= pos) sb.evicted.resize((size_t)pos + 1, 0);
    sb.evicted[(size_t)pos] = 1;
    sb.pending.push_back(pos);
}

// exit_window + admit_to_cache (proj/src/cache.cpp:136-179) for one departing position
void replay_exit(SnapBase& sb, long long e, double score, bool has_stream, bool inserted, size_t cap) {
    if (!has_stream || !inserted || cap == 0) {
        evict_mark(sb, e);
        return;
    }
    if (sb.heap.size() < cap) {
        sb.heap.push_back({score, e});
        std::push_heap(sb.heap.begin(), sb.heap.end(), SnapSlotCmp{});
        sb.cache_pos.push_back(e);
        return;
    }
    const auto worst = sb.heap.front();
    if (score < worst.first || score == worst.first) {
        evict_mark(sb, e);
        return;
    }
    std::pop_heap(sb.heap.begin(), sb.heap.end(), SnapSlotCmp{});
    sb.heap.back() = {score, e};
    std::push_heap(sb.heap.begin(), sb.heap.end(), SnapSlotCmp{});
    evict_mark(sb, worst.second);
    sb.cache_pos.erase(std::lower_bound(sb.cache_pos.begin(), sb.cache_pos.end(), worst.second));
    sb.cache_pos.push_back(e);
}

double to_f64(const uint8_t* p, int dt) {
    if (dt == SKB_F64) {
        double x;
        std::memcpy(&x, p, 8);
        return x;
    }
    if (dt == SKB_F32) {
        float x;
        std::memcpy(&x, p, 4);
        return (double)x;
    }
    uint16_t h;
    std::memcpy(&h, p, 2);
    const uint32_t w = (uint32_t)h << 16;
    float x;
    std::memcpy(&x, &w, 4);
    return (double)x;
}

void from_f64(double x, uint8_t* p, int dt) {
    if (dt == SKB_F64) {
        std::memcpy(p, &x, 8);
    } else if (dt == SKB_F32) {
        const float f = (float)x;
        std::memcpy(p, &f, 4);
    } else {
        const __nv_bfloat16 h = __double2bfloat16(x);
        std::memcpy(p, &h, 2);
    }
}

}  // namespace

extern "C" {

// SparseKvCache<T>::serialize (proj/src/cache.cpp:416-475) of sequence b; the
// reference's TimestepNormState {count, mean, m2} comes from the caller (the
// cache works at the q/k/v/u level; null = a fresh state).
// The eviction ledger of sequence b (SparseKvCache::drain_evictions /
// ever_evicted, proj/src/cache.cpp:115-125, proj/include/sparsek/cache.hpp:38-45):
// the host replay advances to the current position (its base moves forward),
// then reports the pending evictions (cleared when drain != 0), the evicted
// flag of the first evicted_cap positions and the frozen scores.
int skb_cache_ledger(skb_cache* c, int64_t b, int32_t drain, int64_t* pending, int64_t pending_cap,
                     int64_t* n_pending, uint8_t* evicted, int64_t evicted_cap, double* scores, int64_t scores_cap,
                     void* stream) {
    K5_BEGIN
    SKB_REQUIRE(c != nullptr && n_pending != nullptr, SKB_EARG, "cache_ledger: null argument");
    SKB_REQUIRE(b >= 0 && b < c->d.batch, SKB_EARG, "cache_ledger: sequence out of range");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const CacheArgs& A = c->A;
    const int64_t bL = b * A.Lmax;
    CacheCtl cc;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&cc, A.ctl + b, sizeof(cc), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    const long long t = cc.t, w = A.w;
    SnapBase& sb = c->base[(size_t)b];
    const long long e0 = std::max(0LL, sb.t0 - w), e1 = std::max(0LL, t - w);
    std::vector<double> u((size_t)std::max<long long>(t, 1));
    std::vector<uint8_t> ins((size_t)std::max<long long>(t, 1));
    if (t) {
        SKB_CHECK_CUDA(cudaMemcpyAsync(u.data(), A.u_hist + bL, t * 8, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaMemcpyAsync(ins.data(), A.ins_hist + bL, t, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    }
    for (long long e = e0; e < e1; ++e)
        replay_exit(sb, e, u[(size_t)e], c->d.k > 0.0, ins[(size_t)e] != 0, (size_t)A.cap);
    sb.t0 = t;
    *n_pending = (int64_t)sb.pending.size();
    if (pending)
        for (size_t i = 0; i < sb.pending.size() && (int64_t)i < pending_cap; ++i) pending[i] = sb.pending[i];
    if (drain) sb.pending.clear();
    if (evicted)
        for (int64_t i = 0; i < evicted_cap; ++i)
            evicted[i] = (i < (int64_t)sb.evicted.size() && sb.evicted[(size_t)i]) ? 1 : 0;
    if (scores)
        for (int64_t i = 0; i < scores_cap && i < t; ++i) scores[i] = u[(size_t)i];
    K5_END
}

int skb_cache_snapshot(skb_cache* c, int64_t b, const double* norm_state, uint8_t* out, size_t* bytes,
                       void* stream) {
    K5_BEGIN
    SKB_REQUIRE(c == nullptr || !c->A.lin, SKB_ECONFIG,
                "cache snapshot: the linear mix's prefix state is not serialised by this backend");
    SKB_REQUIRE(c != nullptr && bytes != nullptr, SKB_EARG, "cache_snapshot: null argument");
    SKB_REQUIRE(b >= 0 && b < c->d.batch, SKB_EARG, "cache_snapshot: sequence out of range");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const CacheArgs& A = c->A;
    const int dt = (int)c->d.dtype;
    const int64_t bL = b * A.Lmax, bS = b * A.S;
    CacheCtl cc;
    SKB_CHECK_CUDA(cudaMemcpyAsync(&cc, A.ctl + b, sizeof(cc), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    SKB_REQUIRE(cc.error == 0, SKB_ESHAPE, "cache_snapshot: the cache is in an error state");
    const long long t = cc.t;
    std::vector<double> u(t), sv(cc.st.nS), fv(cc.st.nF);
    std::vector<uint8_t> ins(t);
    std::vector<int> si(cc.st.nS), fi(cc.st.nF), slot_of(t);
    if (t) {
        SKB_CHECK_CUDA(cudaMemcpyAsync(u.data(), A.u_hist + bL, t * 8, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaMemcpyAsync(ins.data(), A.ins_hist + bL, t, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaMemcpyAsync(slot_of.data(), A.slot_of + bL, t * 4, cudaMemcpyDeviceToHost, st));
    }
    if (cc.st.nS) {
        SKB_CHECK_CUDA(cudaMemcpyAsync(sv.data(), A.sv + bL, cc.st.nS * 8, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaMemcpyAsync(si.data(), A.si + bL, cc.st.nS * 4, cudaMemcpyDeviceToHost, st));
    }
    if (cc.st.nF) {
        SKB_CHECK_CUDA(cudaMemcpyAsync(fv.data(), A.fv + bL, cc.st.nF * 8, cudaMemcpyDeviceToHost, st));
        SKB_CHECK_CUDA(cudaMemcpyAsync(fi.data(), A.fi + bL, cc.st.nF * 4, cudaMemcpyDeviceToHost, st));
    }
    std::vector<uint8_t> kp((size_t)A.S * A.row_bytes), vp((size_t)A.S * A.row_bytes);
    SKB_CHECK_CUDA(cudaMemcpyAsync(kp.data(), A.kpool + bS * A.row_bytes, kp.size(), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaMemcpyAsync(vp.data(), A.vpool + bS * A.row_bytes, vp.size(), cudaMemcpyDeviceToHost, st));
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));

    const bool has_stream = c->d.k > 0.0;
    const size_t cap = (size_t)A.cap;
    const long long w = A.w;
    SnapBase sb = c->base[(size_t)b];  // replay the exits since the base point
    for (long long e = std::max(0LL, sb.t0 - w); e < std::max(0LL, t - w); ++e)
        replay_exit(sb, e, u[(size_t)e], has_stream, ins[(size_t)e] != 0, cap);
    const long long d_model = c->d.heads * c->d.head_dim;
    Bytes o;
    o.u64((uint64_t)d_model);
    o.u64((uint64_t)c->d.heads);
    o.u64((uint64_t)w);
    o.u64((uint64_t)cap);
    o.f64(c->d.k);
    o.u8(0);  // linear mix: not on the B200 path
    o.u8(has_stream ? 1 : 0);
    o.u64((uint64_t)t);
    o.u64((uint64_t)t);
    for (long long i = 0; i < t; ++i) o.f64(u[(size_t)i]);
    o.u64(norm_state ? (uint64_t)norm_state[0] : 0);
    o.f64(norm_state ? norm_state[1] : 0.0);
    o.f64(norm_state ? norm_state[2] : 0.0);
    o.f64(1e-5);  // TimestepNormState::eps (proj/include/sparsek/selection.hpp:35)
    if (has_stream) {  // StreamState::serialize (proj/src/stream.cpp:224-252)
        Bytes sbl;
        const long long pushes = cc.st.t;
        sbl.f64(cc.st.k);
        sbl.u64((uint64_t)cc.st.heap_cap);
        sbl.f64(cc.st.tau);
        sbl.u64((uint64_t)pushes);
        sbl.f64(cc.st.sum_s);
        sbl.f64(cc.st.sum_f);
        sbl.u64(cc.st.cap_drops);
        sbl.u64(cc.st.heap_ops);
        sbl.u64((uint64_t)cc.st.since_refresh);
        auto heap = [&](const std::vector<double>& v, const std::vector<int>& ix) {
            sbl.u64(v.size());
            for (size_t r2 = v.size(); r2-- > 0;) {  // (value asc, index desc): a valid heap
                sbl.f64(v[r2]);
                sbl.u64((uint64_t)ix[r2]);
            }
        };
        heap(sv, si);
        heap(fv, fi);
        // evicted = every push not in the survivor set (rejected at entry or popped)
        std::vector<uint8_t> ev((size_t)pushes, 1);
        for (int x : si)
            if (x >= 0 && x < pushes) ev[(size_t)x] = 0;
        sbl.u64((uint64_t)pushes);
        for (long long i = 0; i < pushes; i += 8) {
            uint8_t byte = 0;
            for (int q = 0; q < 8 && i + q < pushes; ++q)
                if (ev[(size_t)(i + q)]) byte |= (uint8_t)(1u << q);
            sbl.u8(byte);
        }
        o.u64(sbl.v.size());
        o.raw(sbl.v.data(), sbl.v.size());
    }
    const long long r0 = std::max(0LL, t - w);  // the window ring, oldest first
    o.u64((uint64_t)(t - r0));
    for (long long ppos = r0; ppos < t; ++ppos) o.u64((uint64_t)ppos);
    o.u64(sb.heap.size());
    for (const auto& hs : sb.heap) {
        o.f64(hs.first);
        o.u64((uint64_t)hs.second);
    }
    o.u64(sb.cache_pos.size());
    for (long long cp : sb.cache_pos) o.u64((uint64_t)cp);
    o.u64((uint64_t)((t - r0) + (long long)sb.cache_pos.size()));
    const size_t es = dt == SKB_F64 ? 8 : dt == SKB_F32 ? 4 : 2;
    auto put_kv = [&](long long ppos) {
        const int slot = slot_of[(size_t)ppos];
        SKB_REQUIRE(slot >= 0 && slot < A.S, SKB_ENUMERIC, "cache_snapshot: retained position without a row");
        o.u64((uint64_t)ppos);
        for (long long x = 0; x < d_model; ++x) o.f64(to_f64(kp.data() + (size_t)slot * A.row_bytes + x * es, dt));
        for (long long x = 0; x < d_model; ++x) o.f64(to_f64(vp.data() + (size_t)slot * A.row_bytes + x * es, dt));
    };
    for (long long ppos = r0; ppos < t; ++ppos) put_kv(ppos);
    for (long long cp : sb.cache_pos) put_kv(cp);
    o.u64(sb.evicted.size());
    for (size_t i = 0; i < sb.evicted.size(); i += 8) {
        uint8_t byte = 0;
        for (size_t q = 0; q < 8 && i + q < sb.evicted.size(); ++q)
            if (sb.evicted[i + q]) byte |= (uint8_t)(1u << q);
        o.u8(byte);
    }
    o.u64(sb.pending.size());
    for (long long pe : sb.pending) o.u64((uint64_t)pe);
    o.u64((uint64_t)cc.peak);
    if (!out) {
        *bytes = o.v.size();
        return SKB_OK;
    }
    SKB_REQUIRE(*bytes >= o.v.size(), SKB_EARG, "cache_snapshot: buffer too small");
    std::memcpy(out, o.v.data(), o.v.size());
    *bytes = o.v.size();
    K5_END
}

// SparseKvCache<T>::deserialize (proj/src/cache.cpp:477-545) into sequence b of
// an existing cache of the same configuration; norm_state receives the
// TimestepNormState {count, mean, m2} for the caller's scoring.
int skb_cache_restore(skb_cache* c, int64_t b, const uint8_t* data, size_t bytes, double* norm_state,
                      void* stream) {
    K5_BEGIN
    SKB_REQUIRE(c != nullptr && data != nullptr, SKB_EARG, "cache_restore: null argument");
    SKB_REQUIRE(b >= 0 && b < c->d.batch, SKB_EARG, "cache_restore: sequence out of range");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const CacheArgs& A = c->A;
    const int dt = (int)c->d.dtype;
    const int64_t bL = b * A.Lmax, bS = b * A.S;
    const long long d_model = c->d.heads * c->d.head_dim;
    const bool has_stream_cfg = c->d.k > 0.0;
    Reader r{data, bytes};
    if (r.u64() != (uint64_t)d_model || r.u64() != (uint64_t)c->d.heads || r.u64() != (uint64_t)A.w ||
        r.u64() != (uint64_t)A.cap)
        throw skb::Error(SKB_EIO, "cache snapshot: configuration mismatch");
    if (r.f64() != c->d.k) throw skb::Error(SKB_EIO, "cache snapshot: budget mismatch");
    if (r.u8() != 0) throw skb::Error(SKB_EIO, "cache snapshot: mode mismatch");
    const bool has_stream = r.u8() != 0;
    if (has_stream != has_stream_cfg) throw skb::Error(SKB_EIO, "cache snapshot: stream mismatch");
    const long long t = (long long)r.u64();
    SKB_REQUIRE(t <= A.Lmax, SKB_ESHAPE, "cache_restore: snapshot longer than the cache's max positions");
    const uint64_t ns = r.count(8);
    SKB_REQUIRE(ns == (uint64_t)t, SKB_EIO, "cache snapshot: score count != positions");
    std::vector<double> u((size_t)t);
    for (auto& x : u) x = r.f64();
    double norm[3];
    norm[0] = (double)r.u64();
    norm[1] = r.f64();
    norm[2] = r.f64();
    (void)r.f64();  // eps
    CacheCtl cc{};
    std::vector<std::pair<double, long long>> hs, hf;
    std::vector<uint8_t> sev;
    cc.st.k = c->d.k;
    cc.st.tau = -INFINITY;
    cc.st.cap = A.Lmax;
    if (has_stream) {
        const uint64_t blen = r.u64();
        const size_t end = r.off + blen;
        cc.st.k = r.f64();
        cc.st.heap_cap = (long long)r.u64();
        cc.st.tau = r.f64();
        cc.st.t = (long long)r.u64();
        cc.st.sum_s = r.f64();
        cc.st.sum_f = r.f64();
        cc.st.cap_drops = r.u64();
        cc.st.heap_ops = r.u64();
        cc.st.since_refresh = (int)r.u64();
        auto heap = [&](std::vector<std::pair<double, long long>>& h) {
            const uint64_t n = r.count(16);
            h.resize(n);
            for (auto& e : h) {
                e.first = r.f64();
                e.second = (long long)r.u64();
                SKB_REQUIRE(e.second >= 0 && e.second < t, SKB_EIO, "cache snapshot: stream entry out of range");
            }
            std::sort(h.begin(), h.end(), [](const auto& a, const auto& b2) {  // device: (value desc, index asc)
                return a.first > b2.first || (a.first == b2.first && a.second < b2.second);
            });
        };
        heap(hs);
        heap(hf);
        const uint64_t nb = r.u64();
        SKB_REQUIRE(nb <= 8 * (uint64_t)(bytes - r.off), SKB_EIO, "cache snapshot: truncated");
        for (uint64_t i = 0; i < nb; i += 8) (void)r.u8();
        SKB_REQUIRE(r.off == end, SKB_EIO, "cache snapshot: stream blob length mismatch");
        cc.st.nS = (int)hs.size();
        cc.st.nF = (int)hf.size();
    }
    std::vector<long long> ring(r.count(8));
    for (auto& x : ring) x = (long long)r.u64();
    SnapBase sb;
    sb.t0 = t;
    sb.heap.resize(r.count(16));
    for (auto& e : sb.heap) {
        e.first = r.f64();
        e.second = (long long)r.u64();
    }
    sb.cache_pos.resize(r.count(8));
    for (auto& x : sb.cache_pos) x = (long long)r.u64();
    const uint64_t nkv = r.u64();
    SKB_REQUIRE(nkv == ring.size() + sb.cache_pos.size() && nkv <= (uint64_t)A.S, SKB_EIO,
                "cache snapshot: row count does not match the retained positions");
    const size_t es = dt == SKB_F64 ? 8 : dt == SKB_F32 ? 4 : 2;
    std::vector<uint8_t> kp((size_t)A.S * A.row_bytes, 0), vp((size_t)A.S * A.row_bytes, 0);
    std::vector<int> slot_of((size_t)std::max<long long>(t, 1), -1), pos_of((size_t)A.S, -1);
    for (uint64_t i = 0; i < nkv; ++i) {
        const long long ppos = (long long)r.u64();
        SKB_REQUIRE(ppos >= 0 && ppos < t, SKB_EIO, "cache snapshot: row position out of range");
        for (long long x = 0; x < d_model; ++x) from_f64(r.f64(), kp.data() + i * A.row_bytes + x * es, dt);
        for (long long x = 0; x < d_model; ++x) from_f64(r.f64(), vp.data() + i * A.row_bytes + x * es, dt);
        slot_of[(size_t)ppos] = (int)i;
        pos_of[i] = (int)ppos;
    }
    const uint64_t nbits = r.u64();
    SKB_REQUIRE(nbits <= 8 * (uint64_t)(bytes - r.off), SKB_EIO, "cache snapshot: truncated");
    sb.evicted.assign(nbits, 0);
    for (uint64_t i = 0; i < nbits; i += 8) {
        const uint8_t byte = r.u8();
        for (uint64_t q = 0; q < 8 && i + q < nbits; ++q) sb.evicted[i + q] = (byte >> q) & 1u;
    }
    sb.pending.resize(r.count(8));
    for (auto& x : sb.pending) x = (long long)r.u64();
    cc.peak = (long long)r.u64();
    SKB_REQUIRE(r.off == bytes, SKB_EIO, "cache snapshot: trailing bytes");
    SKB_REQUIRE((long long)ring.size() == t - std::max(0LL, t - (long long)A.w), SKB_EIO,
                "cache snapshot: window ring does not hold the last w positions");
    for (size_t i = 0; i < ring.size(); ++i)
        SKB_REQUIRE(ring[i] == t - (long long)ring.size() + (long long)i, SKB_EIO,
                    "cache snapshot: window ring does not hold the last w positions");
    // the retained cache positions must be the stream's top floor(k) survivors
    SKB_REQUIRE(sb.cache_pos.size() <= (size_t)A.cap, SKB_EIO, "cache snapshot: cache larger than floor(k)");
    // the device attends slot_of[survivor] for the first nsel survivors: each
    // must be a stored row, and together they must be exactly cache_pos
    // (the reference throws NumericError on an attended position with no row)
    SKB_REQUIRE(hs.size() >= sb.cache_pos.size(), SKB_EIO, "cache snapshot: fewer survivors than cached rows");
    {
        std::vector<long long> head;
        for (size_t i = 0; i < sb.cache_pos.size(); ++i) {
            const long long pp = hs[i].second;
            SKB_REQUIRE(pp >= 0 && pp < t && slot_of[(size_t)pp] >= 0, SKB_ENUMERIC,
                        "attended position has no stored row");
            head.push_back(pp);
        }
        std::sort(head.begin(), head.end());
        std::vector<long long> cp(sb.cache_pos);
        std::sort(cp.begin(), cp.end());
        SKB_REQUIRE(head == cp, SKB_EIO, "cache snapshot: cached positions are not the stream's top floor(k)");
        for (long long pp : ring)
            SKB_REQUIRE(pp >= 0 && pp < t && slot_of[(size_t)pp] >= 0, SKB_ENUMERIC,
                        "attended position has no stored row");
    }
    cc.t = t;
    cc.nsel = (int)sb.cache_pos.size();
    cc.free_top = A.S - (int)nkv;
    std::vector<int> free_stack((size_t)A.S);
    for (int i = 0; i < cc.free_top; ++i) free_stack[(size_t)i] = A.S - 1 - i;  // the unused slots
    // device upload
    std::vector<double> sv(hs.size()), fv(hf.size());
    std::vector<int> si(hs.size()), fi(hf.size());
    for (size_t i = 0; i < hs.size(); ++i) sv[i] = hs[i].first, si[i] = (int)hs[i].second;
    for (size_t i = 0; i < hf.size(); ++i) fv[i] = hf[i].first, fi[i] = (int)hf[i].second;
    std::vector<uint8_t> ins((size_t)std::max<long long>(t, 1), 0);
    SKB_CHECK_CUDA(cudaStreamSynchronize(st));
    if (t) {
        SKB_CHECK_CUDA(cudaMemcpy(A.u_hist + bL, u.data(), t * 8, cudaMemcpyHostToDevice));
        SKB_CHECK_CUDA(cudaMemcpy(A.slot_of + bL, slot_of.data(), t * 4, cudaMemcpyHostToDevice));
        SKB_CHECK_CUDA(cudaMemcpy(A.ins_hist + bL, ins.data(), t, cudaMemcpyHostToDevice));
    }
    if (!sv.empty()) {
        SKB_CHECK_CUDA(cudaMemcpy(A.sv + bL, sv.data(), sv.size() * 8, cudaMemcpyHostToDevice));
        SKB_CHECK_CUDA(cudaMemcpy(A.si + bL, si.data(), si.size() * 4, cudaMemcpyHostToDevice));
    }
    if (!fv.empty()) {
        SKB_CHECK_CUDA(cudaMemcpy(A.fv + bL, fv.data(), fv.size() * 8, cudaMemcpyHostToDevice));
        SKB_CHECK_CUDA(cudaMemcpy(A.fi + bL, fi.data(), fi.size() * 4, cudaMemcpyHostToDevice));
    }
    SKB_CHECK_CUDA(cudaMemcpy(A.pos_of + bS, pos_of.data(), A.S * 4, cudaMemcpyHostToDevice));
    SKB_CHECK_CUDA(cudaMemcpy(A.free_stack + bS, free_stack.data(), A.S * 4, cudaMemcpyHostToDevice));
    SKB_CHECK_CUDA(cudaMemcpy(A.kpool + bS * A.row_bytes, kp.data(), kp.size(), cudaMemcpyHostToDevice));
    SKB_CHECK_CUDA(cudaMemcpy(A.vpool + bS * A.row_bytes, vp.data(), vp.size(), cudaMemcpyHostToDevice));
    SKB_CHECK_CUDA(cudaMemcpy(A.ctl + b, &cc, sizeof(cc), cudaMemcpyHostToDevice));
    c->base[(size_t)b] = std::move(sb);
    if (norm_state)
        for (int i = 0; i < 3; ++i) norm_state[i] = norm[i];
    K5_END
}

}  // extern "C"
