// K4 tensor-core backward (tcgen05 + TMEM), BF16, head_dim 64 or 128.
//
// sparsek_attention_backward's core (proj/src/attention.cpp:265-316) as three
// kernels over the same selection products as the forward:
//   k_bwd_prep     lse in log2 units and delta_i = dO_i . O_i (the reference's
//                  s = sum_j P_ij wv_ij b_ij equals dO_i . O_i).
//   k_bwd_dkdv_tc  key-major: a CTA owns 128 keys — a contiguous window tile
//                  or 128 entries of the ever-selected list — and walks the
//                  64-query tiles that read them (window: [j, j+w); selected:
//                  [j+w, leave_j+w)). S^T = K Q^T and dP^T = V dO^T in TMEM
//                  (double-buffered), elementwise P~^T / dS^T to smem, then
//                  dV += P~^T dO and dK += dS^T Q accumulate in TMEM. The
//                  selected pass stores fp32 partials, the window pass adds
//                  them and writes bf16. colsum_j (gate gradient over the
//                  fractional support, summed over heads) is per thread.
//   k_bwd_dq_tc    query-major over 64-key tiles: dQ = dS K accumulates in
//                  TMEM; rowsum_t (the pullback numerator) is per thread.
// rowsum/colsum feed the O(L log L) selection pullback (skb_jvp.cu).
#include <climits>
#include <type_traits>

#include "skb_common.cuh"
#include "skb_internal.h"
#include "skb_tc.cuh"
#include "skb_tmap.h"

// experiment builds only: 1 = the selected pass's math warps skip the
// elementwise work (tensor pipe alone), 2 = no S/dP MMAs, 3 = no dV/dK MMAs
#ifndef SKB_BWD_EXP
#define SKB_BWD_EXP 0
#endif


#ifdef SKB_TRACE
// CTAs 100 and 101 (a pair of the pair pass) at offsets 0 and 4096
__device__ unsigned long long g_skb_trace_bwd[8192];
#define SKB_TRB(role, jt, ev)                                                                        \
    do {                                                                                              \
        if ((blockIdx.x == 100 || blockIdx.x == 101) && blockIdx.y == 0 && blockIdx.z == 0 && (jt) < 32 && \
            (role) < 8)                                                                               \
            g_skb_trace_bwd[(blockIdx.x - 100) * 4096 + (((role) * 512 + (jt) * 16 + (ev)) & 4095)] = clock64(); \
    } while (0)
extern "C" int skb_debug_trace_bwd(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_skb_trace_bwd, sizeof(unsigned long long) * (n < 8192 ? n : 8192));
}
#else
#define SKB_TRB(role, jt, ev) \
    do {                      \
    } while (0)
#endif

namespace skb {

namespace {

using namespace tc;

struct BwdArgs {
    CUtensorMap tm_q128, tm_do128;  // 3-D row tiles (box 64 x rows)
    CUtensorMap tm_k64, tm_v64;
    CUtensorMap tm_q64, tm_do64;
    CUtensorMap tm_q32, tm_do32;  // 32-row boxes (the pair pass's per-CTA query halves)
    CUtensorMap tm_q96, tm_do96;  // 96-row boxes (the unified pass's query tiles)
    CUtensorMap tm_k128, tm_v128;
    CUtensorMap tm_dk_st, tm_dv_st;  // 32-key group stores (tmap_groups4d)
    const __nv_bfloat16 *q, *k, *v, *dout;
    __nv_bfloat16 *dq, *dk, *dv;
    __nv_bfloat16 *dk_acc, *dv_acc;  // partials of the selected pass, 32-key groups (part_off)
    const float* lse2;       // [B, H, L] lse * log2(e)
    const float* delta;      // [B, H, L] rowsum(dO * O)
    const float* uf;
    const float* tauf;
    const int* leave;
    const int* qb_count;
    const int* qb_list;
    const int* qb_leave;  // leave - key per union entry (0 = padding)
    const float* qb_uf;
    const int* qb_flags;  // 16-byte record per 128-entry tile
    const int* ever_count;
    const int* ever_list;
    double *rowsum, *colsum;
    float* dq32;      // fused dQ: fp32 [B, L, H, D] accumulator of dS K (unscaled), reduced into by the key-major passes
    int2* sel_items;  // [B][cdiv(L,128)] {q_lo, nq} of the selected pass's key tiles
    int* sel_order;   // [B][L] ever-selected keys grouped by leave time (the selected pass's order)
    int* uni_hi;      // [B][cdiv(L,128)] query end of each contiguous key tile (unified pass)
    int uni;          // 1: dense sequences take the unified key-major pass (k_bwd_dkdv_win_tc<.., UNI>)
    int nqb, qb_cap;
    int B, L, H, w, T, R1;
    float scale, scale_log2;
    int mask_st;
    int chunk_len;  // 0 = one chunk
};

// dK/dV partials of the selected pass (bf16; the window pass adds them to its
// fp32 accumulators), [B][H][ceil(L/32)][D/8][32 keys][8]: the 32 consecutive
// keys of a warp write one 8-column group as 512 contiguous bytes, and a
// 128-key window tile's partials are one contiguous block (one bulk copy).
template <int D>
__device__ __forceinline__ int64_t part_off(const BwdArgs& a, int b, int h, int key, int c8) {
    const int ng = (a.L + 31) >> 5;
    return ((((int64_t)(b * a.H + h) * ng + (key >> 5)) * (D / 8) + c8) * 32 + (key & 31)) * 8;
}

// One (b, i, h) row per D/(8 VPT) threads: VPT 16-byte loads of O and dO per
// thread (cfg3: 84 us = 6.4 TB/s with two in flight per tensor, 115 us with one), a
// shuffle-reduced dot product, lse converted to log2 units. HBM-bound.
template <int D, int VPT = 2>
__global__ void __launch_bounds__(256) k_bwd_prep(const __nv_bfloat16* __restrict__ o,
                                                  const __nv_bfloat16* __restrict__ dout,
                                                  const double* __restrict__ lse, float* __restrict__ lse2,
                                                  float* __restrict__ delta, int B, int L, int H) {
    constexpr int kTpr = D / (8 * VPT);  // threads per row
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = gt / kTpr;  // (b, i, h)
    const int sub = (int)(gt % kTpr);
    const bool ok = row < (int64_t)B * L * H;
    float acc = 0.f;
    if (ok) {
        uint4 x[VPT], g[VPT];
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            x[v] = *reinterpret_cast<const uint4*>(o + row * D + (sub * VPT + v) * 8);
            g[v] = *reinterpret_cast<const uint4*>(dout + row * D + (sub * VPT + v) * 8);
        }
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            const uint32_t xs[4] = {x[v].x, x[v].y, x[v].z, x[v].w}, gs[4] = {g[v].x, g[v].y, g[v].z, g[v].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 a2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[e]));
                const float2 b2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gs[e]));
                acc = fmaf(a2.x, b2.x, fmaf(a2.y, b2.y, acc));
            }
        }
    }
#pragma unroll
    for (int off = kTpr / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (ok && sub == 0) {
        const int h = (int)(row % H);
        const int64_t bi = row / H;
        const int i = (int)(bi % L), b = (int)(bi / L);
        const int64_t o2 = ((int64_t)b * H + h) * L + i;
        delta[o2] = acc;
        lse2[o2] = (float)(lse[o2] * 1.4426950408889634);
    }
}

// ------------------------------------------------------------------ dK / dV
// Key-major: a CTA owns 128 keys (a contiguous window tile, or 128 entries of
// the ever-selected list) and walks the 64-query tiles that read them. Per
// tile: S^T = K Q^T and dP^T = V dO^T (M=128, N=64) in TMEM; two math
// warpgroups (32 queries each) write P~^T and dS^T back into TMEM as bf16
// over their consumed columns — the A operands of the TS-MMAs dV += P~^T dO
// and dK += dS^T Q. Q/dO tiles arrive by 3-D TMA (contiguous queries), the
// per-query lse/delta/tau by cp.async; a stage is released by the MMA commit.
constexpr int kQS = 3;  // Q/dO ring depth

// The selected pass without fused dQ holds 4 Q/dO stages: a stage is busy
// from its TMA issue (~2.5k cycles to land under load) to the commit of the
// tile's dV/dK MMAs, and with 3 stages that loop, not the tensor pipe, set the
// tile period (tools/trace_selp.py; SKB_BWD_EXP decomposition in DESIGN.md).
constexpr int kSelQS = 4;

template <int D, int QS = kQS, bool FQ = false>
struct KSmem {
    static constexpr int kKV = 128 * D * 2;  // 128-key tile
    static constexpr int kQT = 64 * D * 2;   // 64-query tile
    static constexpr int kK = 0;
    static constexpr int kV = kK + kKV;
    static constexpr int kQ = kV + kKV;          // [QS]
    static constexpr int kDO = kQ + QS * kQT;    // [QS]
    static constexpr int kDS = kDO + QS * kQT;   // dS^T of the tile (fused dQ): 128 keys x 64 queries bf16
    static constexpr int kStage = kDS + (FQ ? 128 * 64 * 2 : 0);  // fused dQ: per-warp 16 x 32 fp32 transpose
    static constexpr int kMeta = kStage + (FQ ? 8 * 2048 : 0);      // [QS][lse2|delta|tau][64] f32
    static constexpr int kBar = kMeta + QS * 3 * 64 * 4;
    static constexpr int kNumBars = 24;
    static constexpr int kTmemSlot = kBar + kNumBars * 8;
    static constexpr int kAlloc = kTmemSlot + 16 + 1024;
};
enum { KB_KVFULL = 0, KB_QDFULL = 1, KB_QDEMPTY = 4, KB_SFULL = 7, KB_SEMPTY = 9, KB_PDSFULL = 11,
       KB_ACCDONE = 13 };  // 14 barriers

template <int D, bool SEL, bool KEY_SOFT>
__global__ void __launch_bounds__(kThreads, 1) k_bwd_dkdv_tc(const __grid_constant__ BwdArgs a) {
    using SM = KSmem<D>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    float* qmeta = reinterpret_cast<float*>(smem + SM::kMeta);  // [stage][lse2|delta|tau][64]
    __shared__ int s_range[2];

    const int kt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bl = (int64_t)b * a.L;
    const int* elist = a.ever_list + bl;
    int nkeys, j0 = 0;
    if (SEL) {
        const int ec = a.ever_count[b];
        if (kt * 128 >= ec) return;
        nkeys = min(128, ec - kt * 128);
    } else {
        j0 = kt * 128;
        if (j0 >= a.L) return;
        nkeys = min(128, a.L - j0);
    }
    auto key_of = [&](int r) -> int {
        if (r >= nkeys) return -1;
        return SEL ? __ldg(elist + kt * 128 + r) : j0 + r;
    };
    if (threadIdx.x == 0) SKB_TRB(6, 31, 7);
    if (threadIdx.x == 0) {
        s_range[0] = SEL ? __ldg(elist + kt * 128) + a.w : j0;  // the list is ascending
        s_range[1] = 0;
    }
    __syncthreads();
    if (threadIdx.x < 128) {  // warps 0-3 cover the 128 keys
        const int key = key_of(threadIdx.x);
        int hi = 0;
        if (key >= 0) {
            hi = SEL ? __ldg(a.leave + bl + key) + a.w : key + a.w;  // exclusive
            if (a.chunk_len > 0) hi = min(hi, (key / a.chunk_len + 1) * a.chunk_len);
        }
        hi = warp_max_i(hi);
        if (lane == 0) atomicMax(&s_range[1], hi);
    }
    if (threadIdx.x == 0) {
        mbar_init(&bars[KB_KVFULL], kProducers + 1);
        for (int s = 0; s < kQS; ++s) {
            mbar_init(&bars[KB_QDFULL + s], kProducers + 1);
            mbar_init(&bars[KB_QDEMPTY + s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[KB_SFULL + s], 1);
            mbar_init(&bars[KB_SEMPTY + s], kMath);
            mbar_init(&bars[KB_PDSFULL + s], kMath);
        }
        mbar_init(&bars[KB_ACCDONE], 1);
        mbar_fence_init();
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;
    const int q_lo = (s_range[0] / 64) * 64;
    const int q_hi = min(a.L, s_range[1]);
    const int nq = q_hi > q_lo ? (q_hi - q_lo + 63) / 64 : 0;

    if (warp >= kProdWarp0 && warp < kMmaWarp) {
        constexpr int kAtoms = D / 64;
        const int pw = warp - kProdWarp0, ptid = threadIdx.x - kProdWarp0 * 32;
        if (SEL) {  // the ever-selected rows: one gather per CTA
            RowKeys<D, 128> kk;
            kk.fetch(pw, lane, key_of);
            kk.issue(sbase + SM::kK, a.k, b, h, a.L, a.H, pw, lane);
            kk.issue(sbase + SM::kV, a.v, b, h, a.L, a.H, pw, lane);
            cp_async_arrive_noinc(&bars[KB_KVFULL]);
            if (ptid == 0) mbar_arrive(&bars[KB_KVFULL]);
        } else {
            if (ptid == 0) {
                mbar_expect_tx(&bars[KB_KVFULL], 2 * 128 * D * 2);
#pragma unroll
                for (int at = 0; at < kAtoms; ++at) {
                    tma_load_3d(sbase + SM::kK + at * 128 * 128, &a.tm_k128, h * D + at * 64, j0, b, &bars[KB_KVFULL]);
                    tma_load_3d(sbase + SM::kV + at * 128 * 128, &a.tm_v128, h * D + at * 64, j0, b, &bars[KB_KVFULL]);
                }
            }
            mbar_arrive(&bars[KB_KVFULL]);
        }
        const float* lse2 = a.lse2 + ((int64_t)b * a.H + h) * a.L;
        const float* dlt = a.delta + ((int64_t)b * a.H + h) * a.L;
        for (int qt = 0; qt < nq; ++qt) {
            const int s = qt % kQS;
            if (ptid == 0) SKB_TRB(4 + 2, qt, 0);
            if (qt >= kQS) mbar_wait(&bars[KB_QDEMPTY + s], ((qt - kQS) / kQS) & 1);
            if (ptid == 0) SKB_TRB(4 + 2, qt, 1);
            const int qs = q_lo + qt * 64;
            for (int c = ptid; c < 64; c += kProducers) {
                const int i = qs + c;
                const bool ok = i < a.L;
                const int t = i - a.w;
                const uint32_t mb = smem_u32(qmeta + (s * 3) * 64 + c);
                cp_async4(mb, lse2 + (ok ? i : 0), ok);
                cp_async4(mb + 64 * 4, dlt + (ok ? i : 0), ok);
                cp_async4(mb + 128 * 4, a.tauf + bl + (ok && t >= 0 ? t : 0), ok && t >= 0);
            }
            cp_async_arrive_noinc(&bars[KB_QDFULL + s]);
            if (ptid == 0) {
                mbar_expect_tx(&bars[KB_QDFULL + s], 2 * 64 * D * 2);
#pragma unroll
                for (int at = 0; at < kAtoms; ++at) {
                    tma_load_3d(sbase + SM::kQ + s * SM::kQT + at * 64 * 128, &a.tm_q64, h * D + at * 64, qs, b,
                                &bars[KB_QDFULL + s]);
                    tma_load_3d(sbase + SM::kDO + s * SM::kQT + at * 64 * 128, &a.tm_do64, h * D + at * 64, qs, b,
                                &bars[KB_QDFULL + s]);
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0 && nq > 0) {
            constexpr uint32_t id_s = umma_idesc(128, 64, false, false);
            constexpr uint32_t id_acc = umma_idesc(128, D, false, true);
            mbar_wait(&bars[KB_KVFULL], 0);
            fence_proxy_async();
            auto acc = [&](int j) {
                const int s = j & 1, qs = j % kQS;
                mbar_wait(&bars[KB_PDSFULL + s], (j >> 1) & 1);
                SKB_TRB(4 + 3, j, 2);
                tc_after_sync();
                const uint32_t dob = sbase + SM::kDO + qs * SM::kQT, qb = sbase + SM::kQ + qs * SM::kQT;
                // P~^T / dS^T of query half hf (32 queries) sit in TMEM columns [hf*32, hf*32+16)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint32_t co = s * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
                    umma_f16_ts(tDV, tS + co, desc_mnmajor(dob, 64, kk), id_acc, (j > 0 || kk > 0) ? 1u : 0u);
                    umma_f16_ts(tDK, tP + co, desc_mnmajor(qb, 64, kk), id_acc, (j > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&bars[KB_QDEMPTY + qs]);
            };
            for (int qt = 0; qt < nq; ++qt) {
                const int s = qt & 1, qs = qt % kQS;
                SKB_TRB(4 + 3, qt, 8);
                mbar_wait(&bars[KB_QDFULL + qs], (qt / kQS) & 1);
                SKB_TRB(4 + 3, qt, 0);
                if (qt >= 2) mbar_wait(&bars[KB_SEMPTY + s], ((qt - 2) >> 1) & 1);
                tc_after_sync();
                const uint32_t qb = sbase + SM::kQ + qs * SM::kQT, dob = sbase + SM::kDO + qs * SM::kQT;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    umma_f16(tS + s * 64, desc_kmajor(sbase + SM::kK, 128, kk), desc_kmajor(qb, 64, kk), id_s,
                             kk > 0 ? 1u : 0u);
                    umma_f16(tP + s * 64, desc_kmajor(sbase + SM::kV, 128, kk), desc_kmajor(dob, 64, kk), id_s,
                             kk > 0 ? 1u : 0u);
                }
                umma_commit(&bars[KB_SFULL + s]);
                SKB_TRB(4 + 3, qt, 1);
                if (qt >= 1) acc(qt - 1);
            }
            acc(nq - 1);
            umma_commit(&bars[KB_ACCDONE]);
        }
        __syncwarp();
    } else if (warp < kProdWarp0) {
        // key rows: two math warpgroups, each owning 32 of the 64 query columns
        const int hf = warp >> 2;
        const int r = ((warp & 3) << 5) | lane;
        const int key = key_of(r);
        const int leave = (SEL && key >= 0) ? __ldg(a.leave + bl + key) : 0;
        const float uj = (SEL && key >= 0) ? __ldg(a.uf + bl + key) : 0.f;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sl2 = a.scale_log2;
        const float2 sl22 = make_float2(sl2, sl2);
        // queries reading this key form one interval: window [j, j+w), selected
        // [j+w, leave_j+w) (proj/src/cache.cpp:259-311)
        const int lo_i = SEL ? key + a.w : key;
        int hi_i = min(a.L, SEL ? leave + a.w : key + a.w);  // exclusive
        // chunk-wise training: gradients never cross to the left of a chunk
        // start, so a key only hears from queries of its own chunk
        // (proj/src/attention.cpp:228-234, 284-300)
        if (a.chunk_len > 0 && key >= 0) hi_i = min(hi_i, (key / a.chunk_len + 1) * a.chunk_len);
        float colsum = 0.f;
        for (int qt = 0; qt < nq; ++qt) {
            const int s = qt & 1, qs3 = qt % kQS;
            const int qs = q_lo + qt * 64 + hf * 32;  // first query of this thread's columns
            if (lane == 0 && (warp & 3) == 0) SKB_TRB(4 + hf, qt, 9);
            mbar_wait(&bars[KB_SFULL + s], (qt >> 1) & 1);
            mbar_wait(&bars[KB_QDFULL + qs3], (qt / kQS) & 1);
            if (lane == 0 && (warp & 3) == 0) SKB_TRB(4 + hf, qt, 0);
            tc_after_sync();
            float sv[32], dp[32];
            tmem_ld32(tS + lane_off + s * 64 + hf * 32, sv);
            tmem_ld32(tP + lane_off + s * 64 + hf * 32, dp);
            tmem_wait_ld();
            tc_before_sync();
            mbar_arrive(&bars[KB_SEMPTY + s]);
            const float* ml = qmeta + (qs3 * 3) * 64 + hf * 32;
            const float* md = ml + 64;
            const float* mt = ml + 128;
            const int cmin = key >= 0 ? lo_i - qs : 32;
            const int cmax = key >= 0 ? hi_i - 1 - qs : -1;
            const bool full = __all_sync(0xffffffffu, cmin <= 0 && cmax >= 31);
            bool sat = true;  // all gates of this key saturated over these columns (tau nondecreasing)
            if (SEL) {
                const int clast = max(0, min(31, a.L - 1 - qs));
                sat = __all_sync(0xffffffffu, key < 0 || uj >= mt[clast] + 1.f);
            }
            if (!full) {
#pragma unroll
                for (int c = 0; c < 32; ++c) sv[c] = (c >= cmin && c <= cmax) ? sv[c] : -INFINITY;
            }
            if (!SEL || sat) {  // all gates 1 on these columns: plain softmax backward, packed fp32x2
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 l4 = *reinterpret_cast<const float4*>(ml + c);
                    const float4 d4 = *reinterpret_cast<const float4*>(md + c);
                    float2 x0 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, make_float2(-l4.x, -l4.y));
                    float2 x1 = __ffma2_rn(make_float2(sv[c + 2], sv[c + 3]), sl22, make_float2(-l4.z, -l4.w));
                    x0.x = ex2(x0.x);
                    x0.y = ex2(x0.y);
                    x1.x = ex2(x1.x);
                    x1.y = ex2(x1.y);
                    const float2 c0 = __fmul2_rn(x0, __fadd2_rn(make_float2(dp[c], dp[c + 1]), make_float2(-d4.x, -d4.y)));
                    const float2 c1 = __fmul2_rn(x1, __fadd2_rn(make_float2(dp[c + 2], dp[c + 3]), make_float2(-d4.z, -d4.w)));
                    sv[c] = x0.x, sv[c + 1] = x0.y, sv[c + 2] = x1.x, sv[c + 3] = x1.y;  // P~^T
                    dp[c] = c0.x, dp[c + 1] = c0.y, dp[c + 2] = c1.x, dp[c + 3] = c1.y;  // dS^T (unscaled)
                }
            } else {
                float csum = 0.f;
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 l4 = *reinterpret_cast<const float4*>(ml + c);
                    const float4 d4 = *reinterpret_cast<const float4*>(md + c);
                    const float4 t4 = *reinterpret_cast<const float4*>(mt + c);
                    const float la[4] = {l4.x, l4.y, l4.z, l4.w};
                    const float da[4] = {d4.x, d4.y, d4.z, d4.w};
                    const float ta[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int cc_ = c + e;
                        const float g = __saturatef(uj - ta[e]);
                        const float kap = KEY_SOFT ? g : 1.f;
                        const float raw = sv[cc_];
                        const float x = (KEY_SOFT && raw == -INFINITY) ? raw : raw * kap;
                        const float p = ex2(fmaf(x, sl2, -la[e]));  // masked: 0
                        const float wv = a.mask_st ? 1.f : g;
                        const float cc = p * fmaf(wv, dp[cc_], -da[e]);
                        float gm = p * dp[cc_];
                        if (KEY_SOFT) gm += a.scale * cc * (raw == -INFINITY ? 0.f : raw);
                        csum += (g > 0.f && g < 1.f) ? gm : 0.f;
                        sv[cc_] = p * wv;    // P~^T
                        dp[cc_] = cc * kap;  // dS^T (scale applied in the epilogue)
                    }
                }
                colsum += csum;
            }
            {  // P~^T and dS^T -> TMEM over this half's consumed columns (packed bf16x2)
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[2 * e], sv[2 * e + 1]);
                tmem_st16u(tS + lane_off + s * 64 + hf * 32, pk);
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(dp[2 * e], dp[2 * e + 1]);
                tmem_st16u(tP + lane_off + s * 64 + hf * 32, pk);
                tmem_wait_st();
            }
            tc_before_sync();
            if (lane == 0 && (warp & 3) == 0) SKB_TRB(4 + hf, qt, 4);
            mbar_arrive(&bars[KB_PDSFULL + s]);
        }
        if (SEL && key >= 0 && colsum != 0.f) atomicAdd(a.colsum + bl + key, (double)colsum);
        if (nq > 0) {
            mbar_wait(&bars[KB_ACCDONE], 0);
            tc_after_sync();
        }
        if (lane == 0 && (warp & 3) == 0) SKB_TRB(4 + hf, 31, 5);
        const bool has_sel = !SEL && key >= 0 && a.R1 > 0 && key < a.T && __ldg(a.leave + bl + key) > key;
        const int64_t rowoff = ((bl + (key >= 0 ? key : 0)) * a.H + h) * D + hf * (D / 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
            float dv[32], dk[32];
            const int col = hf * (D / 2) + c * 32;
            if (nq > 0) {
                tmem_ld32(tDV + lane_off + col, dv);
                tmem_ld32(tDK + lane_off + col, dk);
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) dv[e] = dk[e] = 0.f;
            }
            if (key < 0) continue;
#pragma unroll
            for (int e = 0; e < 32; ++e) dk[e] *= a.scale;
            if (SEL) {
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    const int64_t po = part_off<D>(a, b, h, key, (col + e) >> 3);
                    uint4 x, y;
                    x.x = pack_bf16(dk[e], dk[e + 1]);
                    x.y = pack_bf16(dk[e + 2], dk[e + 3]);
                    x.z = pack_bf16(dk[e + 4], dk[e + 5]);
                    x.w = pack_bf16(dk[e + 6], dk[e + 7]);
                    y.x = pack_bf16(dv[e], dv[e + 1]);
                    y.y = pack_bf16(dv[e + 2], dv[e + 3]);
                    y.z = pack_bf16(dv[e + 4], dv[e + 5]);
                    y.w = pack_bf16(dv[e + 6], dv[e + 7]);
                    *reinterpret_cast<uint4*>(a.dk_acc + po) = x;
                    *reinterpret_cast<uint4*>(a.dv_acc + po) = y;
                }
            } else {
                static_assert(SEL, "the window pass is k_bwd_dkdv_win_tc");
                __nv_bfloat16* gk = a.dk + rowoff + c * 32;
                __nv_bfloat16* gv = a.dv + rowoff + c * 32;
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    uint4 x, y;
                    x.x = pack_bf16(dk[e], dk[e + 1]);
                    x.y = pack_bf16(dk[e + 2], dk[e + 3]);
                    x.z = pack_bf16(dk[e + 4], dk[e + 5]);
                    x.w = pack_bf16(dk[e + 6], dk[e + 7]);
                    y.x = pack_bf16(dv[e], dv[e + 1]);
                    y.y = pack_bf16(dv[e + 2], dv[e + 3]);
                    y.z = pack_bf16(dv[e + 4], dv[e + 5]);
                    y.w = pack_bf16(dv[e + 6], dv[e + 7]);
                    *reinterpret_cast<uint4*>(gk + e) = x;
                    *reinterpret_cast<uint4*>(gv + e) = y;
                }
            }
        }
    }
    if (lane == 0 && (warp & 3) == 0 && warp < kProdWarp0) SKB_TRB(4 + (warp >> 2), 31, 6);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

// Window pass, persistent: one CTA per SM walks key tiles wi = blockIdx.x,
// blockIdx.x + gridDim.x, ... (key tile fastest, so the CTAs in flight share
// their query tiles in L2). Every ring (Q/dO stages, S buffers) runs on a
// global counter across work items, so the next item's K/V and first query
// tiles load while the current item finishes its last dV/dK MMAs and its
// epilogue; K/V are released by the commit of an item's last S/dP MMA, the
// dV/dK accumulators by the math warps once they are read out.
template <int D, int QS = kQS, bool FQ = false, bool UNI = false>
struct KWSmem {
    static constexpr int kKV = 128 * D * 2;
    static constexpr int kQT = 64 * D * 2;
    static constexpr int kK = 0;
    static constexpr int kV = kK + kKV;
    static constexpr int kQ = kV + kKV;           // [QS]
    static constexpr int kDO = kQ + QS * kQT;     // [QS]
    static constexpr int kPart = kDO + QS * kQT;  // dK then dV partials of the tile (part_off order);
    static constexpr int kPartB = UNI ? 0 : 128 * D * 2;  //   the epilogue stages its bf16 rows in place
    static constexpr int kDS = kPart + 2 * kPartB;         // fused dQ: dS^T of the tile, 128 keys x 64 queries
    static constexpr int kStage = kDS + (FQ ? 128 * 64 * 2 : 0);  // fused dQ: per-warp 16 x 32 fp32 transpose
    static constexpr int kMeta = kStage + (FQ ? 8 * 2048 : 0);       // [QS][lse2|delta(|tau)][64] f32
    static constexpr int kBar = kMeta + QS * (UNI ? 3 : 2) * 64 * 4;
    static constexpr int kTmemSlot = kBar + 24 * 8;
    static constexpr int kAlloc = kTmemSlot + 16 + 1024;
    static_assert(kAlloc <= 232448, "smem");
};
enum { KW_KVFULL = 0, KW_KVEMPTY = 1, KW_QDFULL = 2, KW_QDEMPTY = 6, KW_SFULL = 10, KW_SEMPTY = 12,
       KW_PDSFULL = 14, KW_ACCDONE = 16, KW_ACCEMPTY = 17, KW_PARTFULL = 18, KW_STGFULL = 19,
       KW_DQFULL = 20, KW_DQEMPTY = 22 };  // 24 barriers (Q/dO rings up to 4 stages) (fused dQ: DQFULL x2 = a tile's dQ^T is complete
                                           // in TMEM, DQEMPTY x2 = it has been read back)

// Fused dQ (D = 128): the key-major passes also form dQ^T = K^T dS^T per
// 64-query tile (M = 128 head dims, N = 64 queries, K = 128 keys) in the
// consumed dP^T columns of the tile's TMEM buffer; the math warps read it
// back during the next tile (or at the item's end) and add it into the fp32
// accumulator with coalesced reductions (a warp covers 32 consecutive head
// dims of one query). The separate query-major dQ pass, which recomputed S
// and dP, disappears: 5 GEMM-units per attended pair instead of 7 (opt-in,
// SKB_BWD_FUSEDQ=1; fused_dq below says why it is not the default).
template <int D>
__device__ __forceinline__ void dq_reduce(const BwdArgs& a, int b, int h, int q0, int drow, const float* v,
                                          float* stage) {
#if defined(SKB_FQ_EXP) && SKB_FQ_EXP == 1
    return;  // experiment: no reductions (timing only)
#endif
    // this warp holds head dims [d0, d0 + 32) (one per lane) of queries
    // [q0, q0 + 32): transposed through a 16-query shared-memory tile so each
    // lane adds 4 consecutive head dims of one query (red.global.add.v4.f32;
    // 8 lanes cover one query's 128 contiguous bytes)
    const int lane = threadIdx.x & 31, d0 = drow - lane;
    const int64_t st = (int64_t)a.H * D;
    float* gbase = a.dq32 + (((int64_t)b * a.L + q0) * a.H + h) * D + d0 + (lane & 7) * 4;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 16; ++c) stage[c * 32 + lane] = v[half * 16 + c];
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int qq = it * 4 + (lane >> 3);  // query within the half
            const int q = half * 16 + qq;
            if (q0 + q < a.L) {
                const float4 x = *reinterpret_cast<const float4*>(stage + qq * 32 + (lane & 7) * 4);
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gbase + q * st), "f"(x.x),
                             "f"(x.y), "f"(x.z), "f"(x.w)
                             : "memory");
            }
        }
    }
}
// Row (key) r's 32 dS^T values of query half hf -> the SW128 dS^T tile
// (row r = 128 B = 64 queries; the K-major A operand of dK += dS^T Q and the
// MN-major B operand of dQ^T = K^T dS^T).
__device__ __forceinline__ void ds_store(uint32_t ds_base, int r, int hf, const float* dp) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const int chunk = hf * 4 + cc;
        st_shared_v4(ds_base + r * 128 + ((chunk ^ (r & 7)) << 4), pack_bf16(dp[8 * cc], dp[8 * cc + 1]),
                     pack_bf16(dp[8 * cc + 2], dp[8 * cc + 3]), pack_bf16(dp[8 * cc + 4], dp[8 * cc + 5]),
                     pack_bf16(dp[8 * cc + 6], dp[8 * cc + 7]));
    }
}
// producer threads (warps 8-9) on the Q/dO ring; warp 10 moves the partials in
// and the finished dK/dV rows out
constexpr int kWinQProd = 64;

// Under the unified pass the selected/window passes serve the sparse
// sequences only: nothing to do (return before any setup) when none is sparse.
__device__ __forceinline__ bool no_sparse_sequence(const BwdArgs& a) {
    if (!a.uni) return false;
    for (int b = 0; b < a.B; ++b)
        if (2 * __ldg(a.ever_count + b) <= a.T) return false;
    return true;
}

// The unified pass's elementwise step where some columns are gated: the
// selected pass's arithmetic with gate 1 on the window columns c < cwc (which
// makes them plain softmax-backward columns with no gate-gradient term).
__device__ __forceinline__ float uni_frac_math(const BwdArgs& a, float uj, int cwc, const float* ml, const float* md,
                                               const float* mt, float2 sl22, float* sv, float* dp) {
    float2 csum2 = make_float2(0.f, 0.f);
    const bool mst = a.mask_st != 0;
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
        const float2 l2 = *reinterpret_cast<const float2*>(ml + c);
        const float2 d2 = *reinterpret_cast<const float2*>(md + c);
        const float2 t2 = *reinterpret_cast<const float2*>(mt + c);
        const float g0 = c < cwc ? 1.f : __saturatef(uj - t2.x);
        const float g1 = c + 1 < cwc ? 1.f : __saturatef(uj - t2.y);
        float2 p2 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, make_float2(-l2.x, -l2.y));
        p2.x = ex2(p2.x);  // masked: 0
        p2.y = ex2(p2.y);
        const float2 dp2 = make_float2(dp[c], dp[c + 1]);
        const float2 nd2 = make_float2(-d2.x, -d2.y);
        const float2 g2 = mst ? make_float2(1.f, 1.f) : make_float2(g0, g1);
        const float2 cc2 = __fmul2_rn(p2, __ffma2_rn(g2, dp2, nd2));
        const float2 fr2 = make_float2((__float_as_uint(g0) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f,
                                       (__float_as_uint(g1) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f);
        csum2 = __fadd2_rn(csum2, __fmul2_rn(__fmul2_rn(p2, dp2), fr2));
        const float2 pw2 = __fmul2_rn(p2, g2);
        sv[c] = pw2.x, sv[c + 1] = pw2.y;  // P~^T
        dp[c] = cc2.x, dp[c + 1] = cc2.y;  // dS^T (scale applied in the epilogue)
    }
    return csum2.x + csum2.y;
}

template <int D, bool FQ, bool UNI = false>
__global__ void __launch_bounds__(kThreads, 1) k_bwd_dkdv_win_tc(const __grid_constant__ BwdArgs a) {
    if (!UNI && no_sparse_sequence(a)) return;
    // the fused-dQ build gives one Q/dO stage to the dS^T tile; the unified
    // pass has no partial buffer and spends it on a fourth stage
    constexpr int QS = FQ ? 2 : (UNI ? 4 : kQS);
    constexpr int kMN = UNI ? 3 : 2;  // per-query metadata arrays: lse2, delta (, tau)
    using SM = KWSmem<D, QS, FQ, UNI>;
    static_assert(!(UNI && FQ), "unified pass: no fused dQ");
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    float* qmeta = reinterpret_cast<float*>(smem + SM::kMeta);  // [stage][lse2|delta][64]
    // the selected pass touched keys of this tile (its partials must be added)
    auto tile_sel = [&](int j0) { return a.R1 > 0 && j0 < a.T; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SKB_TRACE_WIN  // items 20.. of the CTA (tools/trace_win.py)
#define TRW(role, gg, ev) \
    if ((gg) >= tr0) SKB_TRB(role, (gg) - tr0, ev)
#else
#define TRW(role, gg, ev) \
    do {                  \
    } while (0)
#endif
    const int ntk = (a.L + 127) / 128;
    const int nitems = ntk * a.H * a.B;
    // the queries reading key tile kt: [j0, hi) with hi = max over its keys of
    // min(key + w, chunk end) — both nondecreasing in key, so the last key's
    // (unified pass: the window and the selection of every key of the tile,
    // [j0, uni_hi) — dense sequences only; the window pass then skips them)
    auto item = [&](int wi, int& b, int& h, int& j0, int& nkeys, int& nq) -> bool {
        const int kt = wi % ntk;
        const int bh = wi / ntk;
        h = bh % a.H;
        b = bh / a.H;
        j0 = kt * 128;
        nkeys = min(128, a.L - j0);
        if (UNI || a.uni) {
            const bool dense = 2 * __ldg(a.ever_count + b) > a.T;
            if (dense != UNI) return false;
            if (UNI) {
                nq = (__ldg(a.uni_hi + b * ntk + kt) - j0 + 63) / 64;
                return true;
            }
        }
        const int jl = j0 + nkeys - 1;
        int hi = jl + a.w;
        if (a.chunk_len > 0) hi = min(hi, (jl / a.chunk_len + 1) * a.chunk_len);
        hi = min(a.L, max(hi, jl + 1));
        nq = (hi - j0 + 63) / 64;
        return true;
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars[KW_KVFULL], 1);
        mbar_init(&bars[KW_KVEMPTY], 1);
        for (int s = 0; s < QS; ++s) {
            mbar_init(&bars[KW_QDFULL + s], kWinQProd + 1);
            mbar_init(&bars[KW_QDEMPTY + s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[KW_SFULL + s], 1);
            mbar_init(&bars[KW_SEMPTY + s], kMath);
            mbar_init(&bars[KW_PDSFULL + s], kMath);
        }
        mbar_init(&bars[KW_ACCDONE], 1);
        mbar_init(&bars[KW_ACCEMPTY], kMath);
        mbar_init(&bars[KW_PARTFULL], 1);
        mbar_init(&bars[KW_STGFULL], kMath);
        mbar_init(&bars[KW_DQFULL], 1);
        mbar_init(&bars[KW_DQFULL + 1], 1);
        mbar_init(&bars[KW_DQEMPTY], kMath);
        mbar_init(&bars[KW_DQEMPTY + 1], kMath);
        mbar_fence_init();
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

    if (warp == kMmaWarp - 1) {
        if (UNI) {  // no partials, the math warps store their rows
        } else
        // the math warps stage tile n's bf16 rows (part_off order) in the
        // partial buffer; this lane stores them (one TMA store per 32-key
        // group and half), waits for the reads, then loads tile n+1's partials
        // — all while tile n+1 computes
        if (lane == 0) {
            int it = 0, pb_ = 0, pj0 = 0, pnk = 0, ph = 0;
            auto store_prev = [&](int itp) {
                mbar_wait(&bars[KW_STGFULL], itp & 1);
                for (int t2 = 0; t2 < 2; ++t2) {
                    const CUtensorMap* tm = t2 == 0 ? &a.tm_dk_st : &a.tm_dv_st;
                    const uint32_t pbuf = sbase + SM::kPart + t2 * SM::kPartB;
                    for (int gq = 0; gq < (pnk + 31) / 32; ++gq)
                        for (int hf = 0; hf < 2; ++hf)
                            tma_store_4d(tm, pbuf + gq * (32 * D * 2) + hf * (D / 16) * 512, 0, pj0 + gq * 32,
                                         ph * (D / 8) + hf * (D / 16), pb_);
                }
                bulk_commit();
                bulk_wait_read0();
            };
            for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
                int b, h, j0, nkeys, nq;
                if (!item(wi, b, h, j0, nkeys, nq)) {
                    --it;
                    continue;
                }
                if (it > 0) store_prev(it - 1);
                pb_ = b, pj0 = j0, pnk = nkeys, ph = h;
                if (tile_sel(j0)) {
                    const uint32_t pb = (uint32_t)(((nkeys + 31) >> 5) * 32 * D * 2);
                    mbar_expect_tx(&bars[KW_PARTFULL], 2 * pb);
                    bulk_load(sbase + SM::kPart, a.dk_acc + part_off<D>(a, b, h, j0, 0), pb, &bars[KW_PARTFULL]);
                    bulk_load(sbase + SM::kPart + SM::kPartB, a.dv_acc + part_off<D>(a, b, h, j0, 0), pb,
                              &bars[KW_PARTFULL]);
                } else {
                    mbar_arrive(&bars[KW_PARTFULL]);
                }
            }
            if (it > 0) store_prev(it - 1);
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes complete before exit
        }
        __syncwarp();
    } else if (warp >= kProdWarp0 && warp < kMmaWarp - 1) {
        constexpr int kAtoms = D / 64;
        const int ptid = threadIdx.x - kProdWarp0 * 32;
        int g = 0, it = 0, tr0 = 1 << 20;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
            int b, h, j0, nkeys, nq;
            if (!item(wi, b, h, j0, nkeys, nq)) {
                --it;
                continue;
            }
            if (it == 20) tr0 = g;
            if (ptid == 0) {
                if (it > 0) mbar_wait(&bars[KW_KVEMPTY], (it - 1) & 1);
                TRW(6, g, 2);
                mbar_expect_tx(&bars[KW_KVFULL], 2 * 128 * D * 2);
#pragma unroll
                for (int at = 0; at < kAtoms; ++at) {
                    tma_load_3d(sbase + SM::kK + at * 128 * 128, &a.tm_k128, h * D + at * 64, j0, b, &bars[KW_KVFULL]);
                    tma_load_3d(sbase + SM::kV + at * 128 * 128, &a.tm_v128, h * D + at * 64, j0, b, &bars[KW_KVFULL]);
                }
            }
            const float* lse2 = a.lse2 + ((int64_t)b * a.H + h) * a.L;
            const float* dlt = a.delta + ((int64_t)b * a.H + h) * a.L;
            const int64_t bl = (int64_t)b * a.L;
            for (int qt = 0; qt < nq; ++qt, ++g) {
                const int s = g % QS;
                if (ptid == 0) TRW(6, g, 0);
                if (g >= QS) mbar_wait(&bars[KW_QDEMPTY + s], ((g - QS) / QS) & 1);
                if (ptid == 0) TRW(6, g, 1);
                const int qs = j0 + qt * 64;
                {
                    const int c = ptid;
                    const int i = qs + c;
                    const bool ok = i < a.L;
                    const uint32_t mb = smem_u32(qmeta + (s * kMN) * 64 + c);
                    cp_async4(mb, lse2 + (ok ? i : 0), ok);
                    cp_async4(mb + 64 * 4, dlt + (ok ? i : 0), ok);
                    if (UNI) {
                        const int t = i - a.w;
                        cp_async4(mb + 128 * 4, a.tauf + bl + (ok && t >= 0 ? t : 0), ok && t >= 0);
                    }
                }
                cp_async_arrive_noinc(&bars[KW_QDFULL + s]);
                if (ptid == 0) {
                    mbar_expect_tx(&bars[KW_QDFULL + s], 2 * 64 * D * 2);
#pragma unroll
                    for (int at = 0; at < kAtoms; ++at) {
                        tma_load_3d(sbase + SM::kQ + s * SM::kQT + at * 64 * 128, &a.tm_q64, h * D + at * 64, qs, b,
                                    &bars[KW_QDFULL + s]);
                        tma_load_3d(sbase + SM::kDO + s * SM::kQT + at * 64 * 128, &a.tm_do64, h * D + at * 64, qs, b,
                                    &bars[KW_QDFULL + s]);
                    }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0) {
            constexpr uint32_t id_s = umma_idesc(128, 64, false, false);
            constexpr uint32_t id_acc = umma_idesc(128, D, false, true);
            int g = 0, it = 0, tr0 = 1 << 20;
            // dV += P~^T dO, dK += dS^T Q for the tile at global index gj (item
            // tile qt); the first tile of an item waits for the accumulators
            auto acc = [&](int gj, int qt, int itn) {
                const int s = gj & 1, qs = gj % QS;
                mbar_wait_fast(&bars[KW_PDSFULL + s], (gj >> 1) & 1);
                TRW(7, gj, 2);
                if (qt == 0 && itn > 0) mbar_wait_fast(&bars[KW_ACCEMPTY], (itn - 1) & 1);
                TRW(7, gj, 3);
                tc_after_sync();
                const uint32_t dob = sbase + SM::kDO + qs * SM::kQT, qb = sbase + SM::kQ + qs * SM::kQT;
                if constexpr (FQ) {
                    fence_proxy_async();  // the dS^T tile (st.shared) -> the MMAs
                    constexpr uint32_t id_dq = umma_idesc(128, 64, true, true);
                    const uint32_t dsb = sbase + SM::kDS;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t co = s * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
                        umma_f16_ts(tDV, tS + co, desc_mnmajor(dob, 64, kk), id_acc, (qt > 0 || kk > 0) ? 1u : 0u);
                        umma_f16(tDK, desc_kmajor(dsb, 128, kk), desc_mnmajor(qb, 64, kk), id_acc,
                                 (qt > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&bars[KW_QDEMPTY + qs]);
                    // dQ^T = K^T dS^T into the tile's consumed dP^T columns
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tP + s * 64, desc_mnmajor(sbase + SM::kK, 128, kk), desc_mnmajor(dsb, 128, kk), id_dq,
                                 kk > 0 ? 1u : 0u);
                    umma_commit(&bars[KW_DQFULL + s]);
                } else {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t co = s * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
                        umma_f16_ts(tDV, tS + co, desc_mnmajor(dob, 64, kk), id_acc, (qt > 0 || kk > 0) ? 1u : 0u);
                        umma_f16_ts(tDK, tP + co, desc_mnmajor(qb, 64, kk), id_acc, (qt > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&bars[KW_QDEMPTY + qs]);
                }
            };
            for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
                int b, h, j0, nkeys, nq;
                if (!item(wi, b, h, j0, nkeys, nq)) {
                    --it;
                    continue;
                }
                if (it == 20) tr0 = g;
                mbar_wait_fast(&bars[KW_KVFULL], it & 1);
                TRW(7, g, 4);
                tc_after_sync();
                for (int qt = 0; qt < nq; ++qt, ++g) {
                    const int s = g & 1, qs = g % QS;
                    TRW(7, g, 8);
                    mbar_wait_fast(&bars[KW_QDFULL + qs], (g / QS) & 1);
                    TRW(7, g, 0);
                    if (FQ && g >= 2) mbar_wait_fast(&bars[KW_SEMPTY + s], ((g - 2) >> 1) & 1);  // (non-fused: implied by PDSFULL(g - 2))
                    TRW(7, g, 5);
                    tc_after_sync();
                    const uint32_t qb = sbase + SM::kQ + qs * SM::kQT, dob = sbase + SM::kDO + qs * SM::kQT;
                    if constexpr (FQ) {  // S^T first: dP^T's columns may still hold dQ^T(g-2) being read back
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            umma_f16(tS + s * 64, desc_kmajor(sbase + SM::kK, 128, kk), desc_kmajor(qb, 64, kk), id_s,
                                     kk > 0 ? 1u : 0u);
                        if (g >= 2) mbar_wait_fast(&bars[KW_DQEMPTY + s], ((g - 2) >> 1) & 1);
                        tc_after_sync();
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            umma_f16(tP + s * 64, desc_kmajor(sbase + SM::kV, 128, kk), desc_kmajor(dob, 64, kk), id_s,
                                     kk > 0 ? 1u : 0u);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            umma_f16(tS + s * 64, desc_kmajor(sbase + SM::kK, 128, kk), desc_kmajor(qb, 64, kk), id_s,
                                     kk > 0 ? 1u : 0u);
                            umma_f16(tP + s * 64, desc_kmajor(sbase + SM::kV, 128, kk), desc_kmajor(dob, 64, kk), id_s,
                                     kk > 0 ? 1u : 0u);
                        }
                    }
                    umma_commit(&bars[KW_SFULL + s]);
                    TRW(7, g, 1);
                    if (!FQ && qt == nq - 1) umma_commit(&bars[KW_KVEMPTY]);
                    if (qt >= 1) acc(g - 1, qt - 1, it);
                }
                acc(g - 1, nq - 1, it);
                if (FQ) umma_commit(&bars[KW_KVEMPTY]);  // the last dQ^T MMA has read K
                umma_commit(&bars[KW_ACCDONE]);
            }
        }
        __syncwarp();
    } else if (warp < kProdWarp0) {
        const int hf = warp >> 2;
        const int r = ((warp & 3) << 5) | lane;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sl2 = a.scale_log2;
        const float2 sl22 = make_float2(sl2, sl2);
        int g = 0, it = 0, tr0 = 1 << 20;
        const bool trl = lane == 0 && (warp & 3) == 0;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
            int b, h, j0, nkeys, nq;
            if (!item(wi, b, h, j0, nkeys, nq)) {
                --it;
                continue;
            }
            if (it == 20) tr0 = g;
            const int64_t bl = (int64_t)b * a.L;
            const int key = r < nkeys ? j0 + r : -1;
            // queries [key, key + w) read this key from the window
            // (proj/src/cache.cpp:259-311); chunk-wise training clips them to
            // the key's chunk (proj/src/attention.cpp:228-234, 284-300)
            int hi_i = min(a.L, key + a.w);
            if (a.chunk_len > 0 && key >= 0) hi_i = min(hi_i, (key / a.chunk_len + 1) * a.chunk_len);
            const bool has_sel = !UNI && key >= 0 && key < a.T && tile_sel(j0) && __ldg(a.leave + bl + key) > key;
            // unified pass: the key's selection follows its window, queries
            // [key + w, leave + w) (proj/src/cache.cpp:259-311), gated
            bool sel_u = false;
            float uj = 0.f, colsum = 0.f;
            if (UNI && key >= 0 && key < a.T && a.R1 > 0) {
                const int lv = __ldg(a.leave + bl + key);
                sel_u = lv > key;
                if (sel_u) {
                    hi_i = min(a.L, lv + a.w);
                    uj = __ldg(a.uf + bl + key);
                }
            }
            for (int qt = 0; qt < nq; ++qt, ++g) {
                const int s = g & 1, qs3 = g % QS;
                const int qs = j0 + qt * 64 + hf * 32;
                if (trl) TRW(4 + hf, g, 9);
                mbar_wait(&bars[KW_SFULL + s], (g >> 1) & 1);
                mbar_wait(&bars[KW_QDFULL + qs3], (g / QS) & 1);
                if (trl) TRW(4 + hf, g, 0);
                tc_after_sync();
                float sv[32], dp[32];
                tmem_ld32(tS + lane_off + s * 64 + hf * 32, sv);
                tmem_ld32(tP + lane_off + s * 64 + hf * 32, dp);
                tmem_wait_ld();
                tc_before_sync();
                mbar_arrive(&bars[KW_SEMPTY + s]);  // fused dQ: the dP^T half is released after its dQ^T is read
                const float* ml = qmeta + (qs3 * kMN) * 64 + hf * 32;
                const float* md = ml + 64;
                const int cmin = key >= 0 ? key - qs : 32;
                const int cmax = key >= 0 ? hi_i - 1 - qs : -1;
                if (!__all_sync(0xffffffffu, cmin <= 0 && cmax >= 31)) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) sv[c] = (c >= cmin && c <= cmax) ? sv[c] : -INFINITY;
                }
                bool plain = true;
                if constexpr (UNI) {
                    // columns c < cwc read the key from the window (gate 1); the
                    // rest from the selection, all gates 1 once u_j >= tau + 1
                    // over the tile's last query (tau nondecreasing)
                    const float* mt = ml + 128;
                    const int cwc = key + a.w - qs;
                    const int clast = max(0, min(31, a.L - 1 - qs));
                    plain = __all_sync(0xffffffffu, !sel_u || cwc > 31 || uj >= mt[clast] + 1.f);
                    if (!plain) colsum += uni_frac_math(a, uj, cwc, ml, md, mt, sl22, sv, dp);
                }
                if (plain)
#pragma unroll
                for (int c = 0; c < 32; c += 4) {  // gates 1: plain softmax backward, packed fp32x2
                    const float4 l4 = *reinterpret_cast<const float4*>(ml + c);
                    const float4 d4 = *reinterpret_cast<const float4*>(md + c);
                    float2 x0 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, make_float2(-l4.x, -l4.y));
                    float2 x1 = __ffma2_rn(make_float2(sv[c + 2], sv[c + 3]), sl22, make_float2(-l4.z, -l4.w));
                    x0.x = ex2(x0.x);
                    x0.y = ex2(x0.y);
                    x1.x = ex2(x1.x);
                    x1.y = ex2(x1.y);
                    const float2 c0 = __fmul2_rn(x0, __fadd2_rn(make_float2(dp[c], dp[c + 1]), make_float2(-d4.x, -d4.y)));
                    const float2 c1 = __fmul2_rn(x1, __fadd2_rn(make_float2(dp[c + 2], dp[c + 3]), make_float2(-d4.z, -d4.w)));
                    sv[c] = x0.x, sv[c + 1] = x0.y, sv[c + 2] = x1.x, sv[c + 3] = x1.y;
                    dp[c] = c0.x, dp[c + 1] = c0.y, dp[c + 2] = c1.x, dp[c + 3] = c1.y;
                }
                if constexpr (FQ) {
                    {
                        uint32_t pk[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[2 * e], sv[2 * e + 1]);
                        tmem_st16u(tS + lane_off + s * 64 + hf * 32, pk);
                    }
                    const int sp = (g - 1) & 1;
                    // the single dS^T tile is free once the previous tile's dK / dQ^T MMAs completed
                    if (qt > 0) mbar_wait(&bars[KW_DQFULL + sp], ((g - 1) >> 1) & 1);
                    ds_store(sbase + SM::kDS, r, hf, dp);
                    fence_async_smem();
                    tmem_wait_st();
                    tc_before_sync();
                    if (trl) TRW(4 + hf, g, 4);
                    mbar_arrive(&bars[KW_PDSFULL + s]);
                    if (qt > 0) {  // the previous tile's dQ^T -> the fp32 accumulator
                        tc_after_sync();
                        float qv[32];
                        tmem_ld32(tP + lane_off + sp * 64 + hf * 32, qv);
                        tmem_wait_ld();
                        tc_before_sync();
                        mbar_arrive(&bars[KW_DQEMPTY + sp]);
                        dq_reduce<D>(a, b, h, qs - 64, r, qv, reinterpret_cast<float*>(smem + SM::kStage) + warp * 512);
                    }
                } else {
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[2 * e], sv[2 * e + 1]);
                    tmem_st16u(tS + lane_off + s * 64 + hf * 32, pk);
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(dp[2 * e], dp[2 * e + 1]);
                    tmem_st16u(tP + lane_off + s * 64 + hf * 32, pk);
                    tmem_wait_st();
                    tc_before_sync();
                    if (trl) TRW(4 + hf, g, 4);
                    mbar_arrive(&bars[KW_PDSFULL + s]);
                }
            }
            if constexpr (FQ) {  // the item's last tile: its dQ^T
                const int sp = (g - 1) & 1;
                mbar_wait(&bars[KW_DQFULL + sp], ((g - 1) >> 1) & 1);
                tc_after_sync();
                float qv[32];
                tmem_ld32(tP + lane_off + sp * 64 + hf * 32, qv);
                tmem_wait_ld();
                tc_before_sync();
                mbar_arrive(&bars[KW_DQEMPTY + sp]);
                dq_reduce<D>(a, b, h, j0 + (nq - 1) * 64 + hf * 32, r, qv, reinterpret_cast<float*>(smem + SM::kStage) + warp * 512);
            }
            mbar_wait(&bars[KW_ACCDONE], it & 1);
            if (trl) TRW(4 + hf, g, 5);
            tc_after_sync();
            float dv[D / 2], dk[D / 2];
#pragma unroll
            for (int c = 0; c < D / 64; ++c) {
                tmem_ld32(tDV + lane_off + hf * (D / 2) + c * 32, dv + c * 32);
                tmem_ld32(tDK + lane_off + hf * (D / 2) + c * 32, dk + c * 32);
            }
            tmem_wait_ld();
            tc_before_sync();
            if (trl) TRW(4 + hf, g, 6);
            mbar_arrive(&bars[KW_ACCEMPTY]);
#pragma unroll
            for (int e = 0; e < D / 2; ++e) dk[e] *= a.scale;
            if constexpr (UNI) {  // final rows, straight from registers (no partials)
                if (key < 0) continue;
                if (colsum != 0.f) atomicAdd(a.colsum + bl + key, (double)colsum);
                const int64_t ro = (((int64_t)b * a.L + key) * a.H + h) * D + hf * (D / 2);
#pragma unroll
                for (int e = 0; e < D / 2; e += 8) {
                    uint4 x, y;
                    x.x = pack_bf16(dk[e], dk[e + 1]);
                    x.y = pack_bf16(dk[e + 2], dk[e + 3]);
                    x.z = pack_bf16(dk[e + 4], dk[e + 5]);
                    x.w = pack_bf16(dk[e + 6], dk[e + 7]);
                    y.x = pack_bf16(dv[e], dv[e + 1]);
                    y.y = pack_bf16(dv[e + 2], dv[e + 3]);
                    y.z = pack_bf16(dv[e + 4], dv[e + 5]);
                    y.w = pack_bf16(dv[e + 6], dv[e + 7]);
                    *reinterpret_cast<uint4*>(a.dk + ro + e) = x;
                    *reinterpret_cast<uint4*>(a.dv + ro + e) = y;
                }
                continue;
            }
            // + the selected pass's partials (bulk-copied to smem in part_off
            // order: 32-key groups of [D/8][32][8]); the bf16 result is staged in
            // place and stored by the warpgroup as contiguous 16-byte row chunks
            mbar_wait(&bars[KW_PARTFULL], it & 1);
            constexpr int kGrp = 32 * D * 2;  // bytes per 32-key group
#pragma unroll
            for (int t2 = 0; t2 < 2; ++t2) {
                float* x = t2 == 0 ? dk : dv;
                uint8_t* pbuf = smem + SM::kPart + t2 * SM::kPartB;
                uint8_t* prow = pbuf + (r >> 5) * kGrp + (r & 31) * 16;  // + c8 * 512
#pragma unroll
                for (int e = 0; e < D / 2; e += 8) {
                    uint4* cell = reinterpret_cast<uint4*>(prow + ((hf * (D / 2) + e) >> 3) * 512);
                    if (has_sel) {
                        const uint4 pp = *cell;
                        const uint32_t pw[4] = {pp.x, pp.y, pp.z, pp.w};
#pragma unroll
                        for (int q2 = 0; q2 < 4; ++q2) {
                            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pw[q2]));
                            x[e + 2 * q2] += f.x;
                            x[e + 2 * q2 + 1] += f.y;
                        }
                    }
                    uint4 v4;
                    v4.x = pack_bf16(x[e], x[e + 1]);
                    v4.y = pack_bf16(x[e + 2], x[e + 3]);
                    v4.z = pack_bf16(x[e + 4], x[e + 5]);
                    v4.w = pack_bf16(x[e + 6], x[e + 7]);
                    *cell = v4;
                }
                if (trl) TRW(4 + hf, g, 10 + 3 * t2);
            }
            fence_async_smem();  // the staged rows -> the TMA stores (async proxy)
            mbar_arrive(&bars[KW_STGFULL]);
            if (trl) TRW(4 + hf, g, 7);
        }
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
#undef TRW
}

// The selected pass's key order. Sparse ever-selected sets (e.g. iid scores,
// ~25 % of the keys): the keys (ascending) stably bucketed by leave time, so a
// 128-key tile holds keys whose retention intervals end together and its query
// range [min key + w, max leave + w) wastes little (45 % fewer 64-query tiles
// than key order, bwd 6.8 -> 4.7 ms at cfg3). Dense sets (recency scores: every
// key is selected once): key order — the bucketed order saves only ~3 % of the
// tiles there but scatters the row gathers and the partial stores (+8 % time).
// One CTA per sequence: per-thread chunk histograms, a bucket-major scan, an
// in-order scatter.
constexpr int kOrdThreads = 256, kOrdBuckets = 64;  // bucket width 256 at cfg3 (measured best of 64..512)
constexpr int kOrdCntBytes = (kOrdBuckets + 1) * kOrdThreads * 4;  // 65 KB of dynamic smem
constexpr int kOrdMaxBk = 128 * 1024;  // bucket ids staged in smem (1 B each) up to this many keys
__global__ void __launch_bounds__(kOrdThreads) k_sel_order(BwdArgs a) {
    extern __shared__ __align__(16) uint8_t osm[];
    int* cnt = reinterpret_cast<int*>(osm);  // [bucket][thread]
    uint8_t* bks = osm + kOrdCntBytes;      // [key index] bucket id
    __shared__ int wtot[kOrdThreads / 32];
    const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int n = a.ever_count[b];
    const int* el = a.ever_list + (int64_t)b * a.L;
    const int* lv = a.leave + (int64_t)b * a.L;
    int* out = a.sel_order + (int64_t)b * a.L;
    if (2 * n > a.T) {  // dense (most keys are selected at some point): key order keeps the
        // gathers and the 32-key partial groups contiguous, which measured faster
        if (a.uni) return;  // (the unified key-major pass covers dense sequences)
        for (int e = t; e < n; e += kOrdThreads) out[e] = el[e];
        return;
    }
    const int bw = max(256, (a.T + kOrdBuckets) / kOrdBuckets);  // <= kOrdBuckets + 1 buckets
    const bool staged = n <= kOrdMaxBk;
    if (staged)  // coalesced: every gather of leave in flight at once
        for (int e = t; e < n; e += kOrdThreads) bks[e] = (uint8_t)min(kOrdBuckets, lv[el[e]] / bw);
    auto bucket = [&](int e) { return staged ? (int)bks[e] : min(kOrdBuckets, lv[el[e]] / bw); };
    const int c = (n + kOrdThreads - 1) / kOrdThreads;
    const int lo = min(n, t * c), hi = min(n, lo + c);
    for (int k = 0; k <= kOrdBuckets; ++k) cnt[k * kOrdThreads + t] = 0;
    __syncthreads();
    for (int e = lo; e < hi; ++e) ++cnt[bucket(e) * kOrdThreads + t];
    __syncthreads();
    int base = 0;
    for (int k = 0; k <= kOrdBuckets; ++k) {  // exclusive scan in (bucket, thread) order
        const int x = cnt[k * kOrdThreads + t];
        int incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wtot[wid] = incl;
        __syncthreads();
        int pre = base, tot = 0;
        for (int w2 = 0; w2 < kOrdThreads / 32; ++w2) {
            if (w2 < wid) pre += wtot[w2];
            tot += wtot[w2];
        }
        cnt[k * kOrdThreads + t] = pre + incl - x;
        base += tot;
        __syncthreads();
    }
    for (int e = lo; e < hi; ++e) out[cnt[bucket(e) * kOrdThreads + t]++] = el[e];
}

// The query range of each 128-entry tile of the selected pass's order (shared
// by all heads): one warp per tile, [min key + w, max(leave + w)) clipped to the
// keys' chunks, in 64-query tiles.
__global__ void k_sel_items(BwdArgs a, int ntk) {
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (wid >= a.B * ntk) return;
    const int b = wid / ntk, kt = wid % ntk;
    const int ec = a.ever_count[b];
    int2 res = make_int2(0, 0);
    if (kt * 128 < ec && !(a.uni && 2 * ec > a.T)) {  // (dense + unified: no selected pass, no order)
        const int* el = a.sel_order + (int64_t)b * a.L + kt * 128;
        const int n = min(128, ec - kt * 128);
        int hi = 0, kmin = INT_MAX;
        for (int r = lane; r < n; r += 32) {
            const int key = el[r];
            int x = a.leave[(int64_t)b * a.L + key] + a.w;
            if (a.chunk_len > 0) x = min(x, (key / a.chunk_len + 1) * a.chunk_len);
            hi = max(hi, x);
            kmin = min(kmin, key);
        }
        hi = min(a.L, warp_max_i(hi));
        kmin = -warp_max_i(-kmin);
        const int q_lo = ((kmin + a.w) / 64) * 64;
        res = make_int2(q_lo, hi > q_lo ? (hi - q_lo + 63) / 64 : 0);
    }
    if (lane == 0) a.sel_items[wid] = res;
}

// The unified pass's query end per contiguous 128-key tile: max over its keys
// of max(key, leave) + w (window, then selection), at least one query tile.
__global__ void __launch_bounds__(128) k_uni_items(BwdArgs a, int ntk) {
    __shared__ int wmax[4];
    const int kt = blockIdx.x, b = blockIdx.y, j0 = kt * 128, j = j0 + threadIdx.x;
    int hi = 0;
    if (j < a.L) {
        int lv = j;
        if (j < a.T && a.R1 > 0) lv = max(j, __ldg(a.leave + (int64_t)b * a.L + j));
        hi = min(a.L, lv + a.w);
    }
    hi = warp_max_i(hi);
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = hi;
    __syncthreads();
    if (threadIdx.x == 0)
        a.uni_hi[b * ntk + kt] = max(max(max(wmax[0], wmax[1]), max(wmax[2], wmax[3])), j0 + 1);
}

// Selected pass, persistent: work item = (128-entry tile of the ever-selected
// list, head); the rings run across items as in the window pass, so the next
// tile's row gathers and first query tiles load under the current tile's last
// MMAs and epilogue. K/V rows are gathered (cp.async) after the commit of the
// item's last S/dP MMA releases the buffer.
template <int D, bool KEY_SOFT, bool FQ>
__global__ void __launch_bounds__(kThreads, 1) k_bwd_dkdv_sel_tc(const __grid_constant__ BwdArgs a) {
    if (no_sparse_sequence(a)) return;
    constexpr int QS = FQ ? kQS : kSelQS;
    using SM = KSmem<D, QS, FQ>;
    static_assert(KW_DQFULL + 1 < SM::kNumBars, "barrier slots");
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    float* qmeta = reinterpret_cast<float*>(smem + SM::kMeta);  // [stage][lse2|delta|tau][64]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SKB_TRACE_SEL  // items 6.. of the CTA (tools/trace_selp.py)
#define TRS(role, gg, ev) \
    if ((gg) >= tr0) SKB_TRB(role, (gg) - tr0, ev)
#else
#define TRS(role, gg, ev) \
    do {                  \
    } while (0)
#endif
    const int ntk = (a.L + 127) / 128;
    const int nitems = ntk * a.H * a.B;
    // item wi -> (kt fastest, h, b); invalid tiles (beyond the list) are skipped
    // by every role alike; nq == 0 tiles only write zero partials
    auto item = [&](int wi, int& b, int& h, int& kt, int& nkeys, int& q_lo, int& nq) -> bool {
        kt = wi % ntk;
        const int bh = wi / ntk;
        h = bh % a.H;
        b = bh / a.H;
        const int ec = __ldg(a.ever_count + b);
        if (kt * 128 >= ec) return false;
        if (a.uni && 2 * ec > a.T) return false;  // the unified pass has it
        nkeys = min(128, ec - kt * 128);
        const int2 info = a.sel_items[b * ntk + kt];
        q_lo = info.x;
        nq = info.y;
        return true;
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars[KW_KVFULL], kProducers + 1);
        mbar_init(&bars[KW_KVEMPTY], 1);
        for (int s = 0; s < QS; ++s) {
            mbar_init(&bars[KW_QDFULL + s], kProducers + 1);
            mbar_init(&bars[KW_QDEMPTY + s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[KW_SFULL + s], 1);
            mbar_init(&bars[KW_SEMPTY + s], kMathArrivals);
            mbar_init(&bars[KW_PDSFULL + s], kMathArrivals);
        }
        mbar_init(&bars[KW_ACCDONE], 1);
        mbar_init(&bars[KW_ACCEMPTY], kMathArrivals);
        mbar_init(&bars[KW_DQFULL], 1);
        mbar_init(&bars[KW_DQFULL + 1], 1);
        mbar_init(&bars[KW_DQEMPTY], kMathArrivals);
        mbar_init(&bars[KW_DQEMPTY + 1], kMathArrivals);
        mbar_fence_init();
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

    if (warp >= kProdWarp0 && warp < kMmaWarp) {
        constexpr int kAtoms = D / 64;
        const int pw = warp - kProdWarp0, ptid = threadIdx.x - kProdWarp0 * 32;
        int g = 0, kit = 0, tr0 = 1 << 28;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x) {
            int b, h, kt, nkeys, q_lo, nq;
            if (!item(wi, b, h, kt, nkeys, q_lo, nq) || nq == 0) continue;
            if (kit == 6) tr0 = g;
            const int64_t bl = (int64_t)b * a.L;
            const int* elist = a.sel_order + bl + kt * 128;
            RowKeys<D, 128> kk;
            kk.fetch(pw, lane, [&](int r) { return r < nkeys ? __ldg(elist + r) : -1; });
            if (ptid == 0) TRS(6, g, 3);
            if (kit > 0) mbar_wait(&bars[KW_KVEMPTY], (kit - 1) & 1);
            if (ptid == 0) TRS(6, g, 2);
            kk.issue(sbase + SM::kK, a.k, b, h, a.L, a.H, pw, lane);
            kk.issue(sbase + SM::kV, a.v, b, h, a.L, a.H, pw, lane);
            cp_async_arrive_noinc(&bars[KW_KVFULL]);
            if (ptid == 0) mbar_arrive(&bars[KW_KVFULL]);
            ++kit;
            const float* lse2 = a.lse2 + ((int64_t)b * a.H + h) * a.L;
            const float* dlt = a.delta + ((int64_t)b * a.H + h) * a.L;
            for (int qt = 0; qt < nq; ++qt, ++g) {
                const int s = g % QS;
                if (g >= QS) mbar_wait(&bars[KW_QDEMPTY + s], ((g - QS) / QS) & 1);
                if (ptid == 0) TRS(6, g, 1);
                const int qs = q_lo + qt * 64;
                for (int c = ptid; c < 64; c += kProducers) {
                    const int i = qs + c;
                    const bool ok = i < a.L;
                    const int t = i - a.w;
                    const uint32_t mb = smem_u32(qmeta + (s * 3) * 64 + c);
                    cp_async4(mb, lse2 + (ok ? i : 0), ok);
                    cp_async4(mb + 64 * 4, dlt + (ok ? i : 0), ok);
                    cp_async4(mb + 128 * 4, a.tauf + bl + (ok && t >= 0 ? t : 0), ok && t >= 0);
                }
                cp_async_arrive_noinc(&bars[KW_QDFULL + s]);
                if (ptid == 0) {
                    mbar_expect_tx(&bars[KW_QDFULL + s], 2 * 64 * D * 2);
#pragma unroll
                    for (int at = 0; at < kAtoms; ++at) {
                        tma_load_3d(sbase + SM::kQ + s * SM::kQT + at * 64 * 128, &a.tm_q64, h * D + at * 64, qs, b,
                                    &bars[KW_QDFULL + s]);
                        tma_load_3d(sbase + SM::kDO + s * SM::kQT + at * 64 * 128, &a.tm_do64, h * D + at * 64, qs, b,
                                    &bars[KW_QDFULL + s]);
                    }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0) {
            constexpr uint32_t id_s = umma_idesc(128, 64, false, false);
            constexpr uint32_t id_acc = umma_idesc(128, D, false, true);
            int g = 0, kit = 0, tr0 = 1 << 28;
            auto acc = [&](int gj, int qt, int kitn) {
                const int s = gj & 1, qs = gj % QS;
                mbar_wait_fast(&bars[KW_PDSFULL + s], (gj >> 1) & 1);
                TRS(7, gj, 2);
                if (qt == 0 && kitn > 0) mbar_wait_fast(&bars[KW_ACCEMPTY], (kitn - 1) & 1);
                tc_after_sync();
                const uint32_t dob = sbase + SM::kDO + qs * SM::kQT, qb = sbase + SM::kQ + qs * SM::kQT;
                if constexpr (FQ) {
                    fence_proxy_async();  // the dS^T tile (st.shared) -> the MMAs
                    constexpr uint32_t id_dq = umma_idesc(128, 64, true, true);
                    const uint32_t dsb = sbase + SM::kDS;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t co = s * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
                        umma_f16_ts(tDV, tS + co, desc_mnmajor(dob, 64, kk), id_acc, (qt > 0 || kk > 0) ? 1u : 0u);
                        umma_f16(tDK, desc_kmajor(dsb, 128, kk), desc_mnmajor(qb, 64, kk), id_acc,
                                 (qt > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&bars[KW_QDEMPTY + qs]);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tP + s * 64, desc_mnmajor(sbase + SM::kK, 128, kk), desc_mnmajor(dsb, 128, kk), id_dq,
                                 kk > 0 ? 1u : 0u);
                    umma_commit(&bars[KW_DQFULL + s]);
                } else {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if (SKB_BWD_EXP == 3) break;
                        const uint32_t co = s * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
                        umma_f16_ts(tDV, tS + co, desc_mnmajor(dob, 64, kk), id_acc, (qt > 0 || kk > 0) ? 1u : 0u);
                        umma_f16_ts(tDK, tP + co, desc_mnmajor(qb, 64, kk), id_acc, (qt > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&bars[KW_QDEMPTY + qs]);
                }
            };
            for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x) {
                int b, h, kt, nkeys, q_lo, nq;
                if (!item(wi, b, h, kt, nkeys, q_lo, nq) || nq == 0) continue;
                if (kit == 6) tr0 = g;
                mbar_wait_fast(&bars[KW_KVFULL], kit & 1);
                TRS(7, g, 4);
                fence_proxy_async();  // cp.async rows -> the MMA (async proxy)
                tc_after_sync();
                for (int qt = 0; qt < nq; ++qt, ++g) {
                    const int s = g & 1, qs = g % QS;
                    mbar_wait_fast(&bars[KW_QDFULL + qs], (g / QS) & 1);
                    TRS(7, g, 0);
                    if (FQ && g >= 2) mbar_wait_fast(&bars[KW_SEMPTY + s], ((g - 2) >> 1) & 1);  // (non-fused: implied by PDSFULL(g - 2))
                    tc_after_sync();
                    const uint32_t qb = sbase + SM::kQ + qs * SM::kQT, dob = sbase + SM::kDO + qs * SM::kQT;
                    if constexpr (FQ) {  // S^T first: dP^T's columns may still hold dQ^T(g-2) being read back
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            umma_f16(tS + s * 64, desc_kmajor(sbase + SM::kK, 128, kk), desc_kmajor(qb, 64, kk), id_s,
                                     kk > 0 ? 1u : 0u);
                        if (g >= 2) mbar_wait_fast(&bars[KW_DQEMPTY + s], ((g - 2) >> 1) & 1);
                        tc_after_sync();
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk)
                            umma_f16(tP + s * 64, desc_kmajor(sbase + SM::kV, 128, kk), desc_kmajor(dob, 64, kk), id_s,
                                     kk > 0 ? 1u : 0u);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            if (SKB_BWD_EXP == 2) break;
                            umma_f16(tS + s * 64, desc_kmajor(sbase + SM::kK, 128, kk), desc_kmajor(qb, 64, kk), id_s,
                                     kk > 0 ? 1u : 0u);
                            umma_f16(tP + s * 64, desc_kmajor(sbase + SM::kV, 128, kk), desc_kmajor(dob, 64, kk), id_s,
                                     kk > 0 ? 1u : 0u);
                        }
                    }
                    umma_commit(&bars[KW_SFULL + s]);
                    TRS(7, g, 1);
                    if (!FQ && qt == nq - 1) umma_commit(&bars[KW_KVEMPTY]);
                    if (qt >= 1) acc(g - 1, qt - 1, kit);
                }
                acc(g - 1, nq - 1, kit);
                if (FQ) umma_commit(&bars[KW_KVEMPTY]);  // the last dQ^T MMA has read K
                umma_commit(&bars[KW_ACCDONE]);
                ++kit;
            }
        }
        __syncwarp();
    } else if (warp < kProdWarp0) {
        const int hf = warp >> 2;
        const int r = ((warp & 3) << 5) | lane;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sl2 = a.scale_log2;
        const float2 sl22 = make_float2(sl2, sl2);
        int g = 0, kit = 0, tr0 = 1 << 28;
        const bool trl = lane == 0 && (warp & 3) == 0;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x) {
            int b, h, kt, nkeys, q_lo, nq;
            if (!item(wi, b, h, kt, nkeys, q_lo, nq)) continue;
            if (kit == 6 && nq > 0) tr0 = g;
            const int64_t bl = (int64_t)b * a.L;
            const int key = r < nkeys ? __ldg(a.sel_order + bl + kt * 128 + r) : -1;
            const int leave = key >= 0 ? __ldg(a.leave + bl + key) : 0;
            const float uj = key >= 0 ? __ldg(a.uf + bl + key) : 0.f;
            // queries [key + w, leave + w) read this key from the selection
            // (proj/src/cache.cpp:259-311), clipped to the key's chunk
            const int lo_i = key + a.w;
            int hi_i = min(a.L, leave + a.w);
            if (a.chunk_len > 0 && key >= 0) hi_i = min(hi_i, (key / a.chunk_len + 1) * a.chunk_len);
            float colsum = 0.f;
            for (int qt = 0; qt < nq; ++qt, ++g) {
                const int s = g & 1, qs3 = g % QS;
                const int qs = q_lo + qt * 64 + hf * 32;
                if (trl) TRS(4 + hf, g, 9);
                mbar_wait(&bars[KW_SFULL + s], (g >> 1) & 1);
                mbar_wait(&bars[KW_QDFULL + qs3], (g / QS) & 1);
                if (trl) TRS(4 + hf, g, 0);
                tc_after_sync();
                float sv[32], dp[32];
                tmem_ld32(tS + lane_off + s * 64 + hf * 32, sv);
                tmem_ld32(tP + lane_off + s * 64 + hf * 32, dp);
                tmem_wait_ld();
                tc_before_sync();
                if (FQ) warp_arrive(&bars[KW_SEMPTY + s]);  // fused dQ: the dP^T half is released after its dQ^T is read
                if (SKB_BWD_EXP == 1 && !FQ) {
                    warp_arrive(&bars[KW_PDSFULL + s]);
                    continue;
                }
                const float* ml = qmeta + (qs3 * 3) * 64 + hf * 32;
                const float* md = ml + 64;
                const float* mt = ml + 128;
                const int cmin = key >= 0 ? lo_i - qs : 32;
                const int cmax = key >= 0 ? hi_i - 1 - qs : -1;
                const bool full = __all_sync(0xffffffffu, cmin <= 0 && cmax >= 31);
                // all gates of this key saturated over these columns (tau nondecreasing)
                const int clast = max(0, min(31, a.L - 1 - qs));
                const bool sat = __all_sync(0xffffffffu, key < 0 || uj >= mt[clast] + 1.f);
                if (!full) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) sv[c] = (c >= cmin && c <= cmax) ? sv[c] : -INFINITY;
                }
                float rg[FQ ? 32 : 1];  // fused dQ: this key's fractional gate gradients per query (row sums)
                if (sat) {  // gates 1 on these columns: plain softmax backward, packed fp32x2
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const float4 l4 = *reinterpret_cast<const float4*>(ml + c);
                        const float4 d4 = *reinterpret_cast<const float4*>(md + c);
                        float2 x0 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, make_float2(-l4.x, -l4.y));
                        float2 x1 = __ffma2_rn(make_float2(sv[c + 2], sv[c + 3]), sl22, make_float2(-l4.z, -l4.w));
                        x0.x = ex2(x0.x);
                        x0.y = ex2(x0.y);
                        x1.x = ex2(x1.x);
                        x1.y = ex2(x1.y);
                        const float2 c0 =
                            __fmul2_rn(x0, __fadd2_rn(make_float2(dp[c], dp[c + 1]), make_float2(-d4.x, -d4.y)));
                        const float2 c1 =
                            __fmul2_rn(x1, __fadd2_rn(make_float2(dp[c + 2], dp[c + 3]), make_float2(-d4.z, -d4.w)));
                        sv[c] = x0.x, sv[c + 1] = x0.y, sv[c + 2] = x1.x, sv[c + 3] = x1.y;
                        dp[c] = c0.x, dp[c + 1] = c0.y, dp[c + 2] = c1.x, dp[c + 3] = c1.y;
                    }
                } else if constexpr (!KEY_SOFT) {
                    // hard keys, fractional gates: packed fp32x2 except the gate
                    // saturation and the fractional-support test; one loop per
                    // (uniform) mask mode
                    auto frac_loop = [&](auto mst_c) {
                        constexpr bool kMst = decltype(mst_c)::value;
                        float2 csum2 = make_float2(0.f, 0.f);
#pragma unroll
                        for (int c = 0; c < 32; c += 2) {
                            const float2 l2 = *reinterpret_cast<const float2*>(ml + c);
                            const float2 d2 = *reinterpret_cast<const float2*>(md + c);
                            const float2 t2 = *reinterpret_cast<const float2*>(mt + c);
                            const float g0 = __saturatef(uj - t2.x), g1 = __saturatef(uj - t2.y);
                            float2 p2 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, make_float2(-l2.x, -l2.y));
                            p2.x = ex2(p2.x);  // masked: 0
                            p2.y = ex2(p2.y);
                            const float2 dp2 = make_float2(dp[c], dp[c + 1]);
                            const float2 nd2 = make_float2(-d2.x, -d2.y);
                            const float2 g2 = make_float2(g0, g1);
                            const float2 cc2 = kMst ? __fmul2_rn(p2, __fadd2_rn(dp2, nd2))
                                                    : __fmul2_rn(p2, __ffma2_rn(g2, dp2, nd2));
                            // 0 < g < 1 <=> (bits(g) - 1) < bits(1.0) - 1 (g in [0, 1])
                            const float2 fr2 = make_float2((__float_as_uint(g0) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f,
                                                           (__float_as_uint(g1) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f);
                            const float2 gf2 = __fmul2_rn(__fmul2_rn(p2, dp2), fr2);
                            csum2 = __fadd2_rn(csum2, gf2);
                            if constexpr (FQ) rg[c] = gf2.x, rg[c + 1] = gf2.y;
                            const float2 pw2 = kMst ? p2 : __fmul2_rn(p2, g2);
                            sv[c] = pw2.x, sv[c + 1] = pw2.y;  // P~^T
                            dp[c] = cc2.x, dp[c + 1] = cc2.y;  // dS^T (scale applied in the epilogue)
                        }
                        colsum += csum2.x + csum2.y;
                    };
                    if (a.mask_st) frac_loop(std::true_type{});
                    else frac_loop(std::false_type{});
                } else {
                    float csum = 0.f;
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const float4 l4 = *reinterpret_cast<const float4*>(ml + c);
                        const float4 d4 = *reinterpret_cast<const float4*>(md + c);
                        const float4 t4 = *reinterpret_cast<const float4*>(mt + c);
                        const float la[4] = {l4.x, l4.y, l4.z, l4.w};
                        const float da[4] = {d4.x, d4.y, d4.z, d4.w};
                        const float ta[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int cc_ = c + e;
                            const float gt = __saturatef(uj - ta[e]);
                            const float kap = KEY_SOFT ? gt : 1.f;
                            const float raw = sv[cc_];
                            const float x = (KEY_SOFT && raw == -INFINITY) ? raw : raw * kap;
                            const float p = ex2(fmaf(x, sl2, -la[e]));  // masked: 0
                            const float wv = a.mask_st ? 1.f : gt;
                            const float cc = p * fmaf(wv, dp[cc_], -da[e]);
                            float gm = p * dp[cc_];
                            if (KEY_SOFT) gm += a.scale * cc * (raw == -INFINITY ? 0.f : raw);
                            const float gf = (gt > 0.f && gt < 1.f) ? gm : 0.f;
                            csum += gf;
                            if constexpr (FQ) rg[cc_] = gf;
                            sv[cc_] = p * wv;    // P~^T
                            dp[cc_] = cc * kap;  // dS^T (scale applied in the epilogue)
                        }
                    }
                    colsum += csum;
                }
                if constexpr (FQ) {
                    if (!sat) {  // the query-side sums of the gate gradients (the dQ pass's rowsum):
                        // reduce-scatter over the warp's 32 keys, lane c ends with query column c
#pragma unroll
                        for (int off = 16; off >= 1; off >>= 1) {
                            const bool up = (lane & off) != 0;
#pragma unroll
                            for (int q2 = 0; q2 < off; ++q2) {
                                const float keep = up ? rg[q2 + off] : rg[q2];
                                const float send = up ? rg[q2] : rg[q2 + off];
                                rg[q2] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                            }
                        }
                        const int i = qs + lane, t = i - a.w;
                        if (rg[0] != 0.f && i < a.L && t >= 0) atomicAdd(a.rowsum + bl + t, (double)rg[0]);
                    }
                    {
                        uint32_t pk[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[2 * e], sv[2 * e + 1]);
                        tmem_st16u(tS + lane_off + s * 64 + hf * 32, pk);
                    }
                    const int sp = (g - 1) & 1;
                    // the single dS^T tile is free once the previous tile's dK / dQ^T MMAs completed
                    if (qt > 0) mbar_wait(&bars[KW_DQFULL + sp], ((g - 1) >> 1) & 1);
                    ds_store(sbase + SM::kDS, r, hf, dp);
                    fence_async_smem();
                    tmem_wait_st();
                    tc_before_sync();
                    if (trl) TRS(4 + hf, g, 4);
                    warp_arrive(&bars[KW_PDSFULL + s]);
                    if (qt > 0) {  // the previous tile's dQ^T -> the fp32 accumulator
                        tc_after_sync();
                        float qv[32];
                        tmem_ld32(tP + lane_off + sp * 64 + hf * 32, qv);
                        tmem_wait_ld();
                        tc_before_sync();
                        warp_arrive(&bars[KW_DQEMPTY + sp]);
                        dq_reduce<D>(a, b, h, qs - 64, r, qv, reinterpret_cast<float*>(smem + SM::kStage) + warp * 512);
                    }
                } else {
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[2 * e], sv[2 * e + 1]);
                    tmem_st16u(tS + lane_off + s * 64 + hf * 32, pk);
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(dp[2 * e], dp[2 * e + 1]);
                    tmem_st16u(tP + lane_off + s * 64 + hf * 32, pk);
                    tmem_wait_st();
                    tc_before_sync();
                    if (trl) TRS(4 + hf, g, 4);
                    warp_arrive(&bars[KW_PDSFULL + s]);
                }
            }
            if constexpr (FQ) {
                if (nq > 0) {  // the item's last tile: its dQ^T
                    const int sp = (g - 1) & 1;
                    mbar_wait(&bars[KW_DQFULL + sp], ((g - 1) >> 1) & 1);
                    tc_after_sync();
                    float qv[32];
                    tmem_ld32(tP + lane_off + sp * 64 + hf * 32, qv);
                    tmem_wait_ld();
                    tc_before_sync();
                    warp_arrive(&bars[KW_DQEMPTY + sp]);
                    dq_reduce<D>(a, b, h, q_lo + (nq - 1) * 64 + hf * 32, r, qv, reinterpret_cast<float*>(smem + SM::kStage) + warp * 512);
                }
            }
            if (key >= 0 && colsum != 0.f) atomicAdd(a.colsum + bl + key, (double)colsum);
            float dv[D / 2], dk[D / 2];
            if (nq > 0) {
                mbar_wait(&bars[KW_ACCDONE], kit & 1);
                if (trl) TRS(4 + hf, g, 5);
                tc_after_sync();
#pragma unroll
                for (int c = 0; c < D / 64; ++c) {
                    tmem_ld32(tDV + lane_off + hf * (D / 2) + c * 32, dv + c * 32);
                    tmem_ld32(tDK + lane_off + hf * (D / 2) + c * 32, dk + c * 32);
                }
                tmem_wait_ld();
                tc_before_sync();
                warp_arrive(&bars[KW_ACCEMPTY]);
                ++kit;
            } else {
#pragma unroll
                for (int e = 0; e < D / 2; ++e) dv[e] = dk[e] = 0.f;
            }
            if (key < 0) continue;
#pragma unroll
            for (int e = 0; e < D / 2; e += 8) {
                const int64_t po = part_off<D>(a, b, h, key, (hf * (D / 2) + e) >> 3);
                uint4 x, y;
                x.x = pack_bf16(dk[e] * a.scale, dk[e + 1] * a.scale);
                x.y = pack_bf16(dk[e + 2] * a.scale, dk[e + 3] * a.scale);
                x.z = pack_bf16(dk[e + 4] * a.scale, dk[e + 5] * a.scale);
                x.w = pack_bf16(dk[e + 6] * a.scale, dk[e + 7] * a.scale);
                y.x = pack_bf16(dv[e], dv[e + 1]);
                y.y = pack_bf16(dv[e + 2], dv[e + 3]);
                y.z = pack_bf16(dv[e + 4], dv[e + 5]);
                y.w = pack_bf16(dv[e + 6], dv[e + 7]);
                *reinterpret_cast<uint4*>(a.dk_acc + po) = x;
                *reinterpret_cast<uint4*>(a.dv_acc + po) = y;
            }
            if (trl) TRS(4 + hf, g, 6);
        }
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
#undef TRS
}

// The selected pass's elementwise step for one thread's 32 query columns of a
// key row (the single-CTA pass inlines the same arithmetic next to its fused-dQ
// variant): P~^T into sv, dS^T (unscaled) into dp; returns the colsum term.
template <bool KEY_SOFT>
__device__ __forceinline__ float sel_tile_math(const BwdArgs& a, bool sat, float uj, const float* ml, const float* md,
                                               const float* mt, float sl2, float2 sl22, float* sv, float* dp) {
    float colsum = 0.f;
    if (sat) {  // gates 1 on these columns: plain softmax backward, packed fp32x2
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
            const float4 l4 = *reinterpret_cast<const float4*>(ml + c);
            const float4 d4 = *reinterpret_cast<const float4*>(md + c);
            float2 x0 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, make_float2(-l4.x, -l4.y));
            float2 x1 = __ffma2_rn(make_float2(sv[c + 2], sv[c + 3]), sl22, make_float2(-l4.z, -l4.w));
            x0.x = ex2(x0.x);
            x0.y = ex2(x0.y);
            x1.x = ex2(x1.x);
            x1.y = ex2(x1.y);
            const float2 c0 = __fmul2_rn(x0, __fadd2_rn(make_float2(dp[c], dp[c + 1]), make_float2(-d4.x, -d4.y)));
            const float2 c1 = __fmul2_rn(x1, __fadd2_rn(make_float2(dp[c + 2], dp[c + 3]), make_float2(-d4.z, -d4.w)));
            sv[c] = x0.x, sv[c + 1] = x0.y, sv[c + 2] = x1.x, sv[c + 3] = x1.y;
            dp[c] = c0.x, dp[c + 1] = c0.y, dp[c + 2] = c1.x, dp[c + 3] = c1.y;
        }
    } else if constexpr (!KEY_SOFT) {
        auto frac_loop = [&](auto mst_c) {
            constexpr bool kMst = decltype(mst_c)::value;
            float2 csum2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
                const float2 l2 = *reinterpret_cast<const float2*>(ml + c);
                const float2 d2 = *reinterpret_cast<const float2*>(md + c);
                const float2 t2 = *reinterpret_cast<const float2*>(mt + c);
                const float g0 = __saturatef(uj - t2.x), g1 = __saturatef(uj - t2.y);
                float2 p2 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, make_float2(-l2.x, -l2.y));
                p2.x = ex2(p2.x);  // masked: 0
                p2.y = ex2(p2.y);
                const float2 dp2 = make_float2(dp[c], dp[c + 1]);
                const float2 nd2 = make_float2(-d2.x, -d2.y);
                const float2 g2 = make_float2(g0, g1);
                const float2 cc2 = kMst ? __fmul2_rn(p2, __fadd2_rn(dp2, nd2)) : __fmul2_rn(p2, __ffma2_rn(g2, dp2, nd2));
                // 0 < g < 1 <=> (bits(g) - 1) < bits(1.0) - 1 (g in [0, 1])
                const float2 fr2 = make_float2((__float_as_uint(g0) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f,
                                               (__float_as_uint(g1) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f);
                const float2 gf2 = __fmul2_rn(__fmul2_rn(p2, dp2), fr2);
                csum2 = __fadd2_rn(csum2, gf2);
                const float2 pw2 = kMst ? p2 : __fmul2_rn(p2, g2);
                sv[c] = pw2.x, sv[c + 1] = pw2.y;  // P~^T
                dp[c] = cc2.x, dp[c + 1] = cc2.y;  // dS^T (scale applied in the epilogue)
            }
            colsum += csum2.x + csum2.y;
        };
        if (a.mask_st) frac_loop(std::true_type{});
        else frac_loop(std::false_type{});
    } else {
        float csum = 0.f;
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
            const float4 l4 = *reinterpret_cast<const float4*>(ml + c);
            const float4 d4 = *reinterpret_cast<const float4*>(md + c);
            const float4 t4 = *reinterpret_cast<const float4*>(mt + c);
            const float la[4] = {l4.x, l4.y, l4.z, l4.w};
            const float da[4] = {d4.x, d4.y, d4.z, d4.w};
            const float ta[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int cc_ = c + e;
                const float gt = __saturatef(uj - ta[e]);
                const float kap = gt;
                const float raw = sv[cc_];
                const float x = raw == -INFINITY ? raw : raw * kap;
                const float p = ex2(fmaf(x, sl2, -la[e]));  // masked: 0
                const float wv = a.mask_st ? 1.f : gt;
                const float cc = p * fmaf(wv, dp[cc_], -da[e]);
                float gm = p * dp[cc_];
                gm += a.scale * cc * (raw == -INFINITY ? 0.f : raw);
                const float gf = (gt > 0.f && gt < 1.f) ? gm : 0.f;
                csum += gf;
                sv[cc_] = p * wv;    // P~^T
                dp[cc_] = cc * kap;  // dS^T (scale applied in the epilogue)
            }
        }
        colsum += csum;
    }
    return colsum;
}

// ------------------------------------------------------------ unified pass, 128-query tiles
// The unified key-major pass (dense sequences, D = 128) with N = 128 query
// tiles. A tcgen05.mma with N <= 128 costs the same ~64-75 cycles
// (tools/probes/mma_rate.cu), so the 64-query tiles of the passes above run
// their S^T/dP^T at half rate. Here one 128-column TMEM region R holds S^T and
// then dP^T of a tile in turn (each read into registers by the math warps and
// released at once), P~^T and dS^T (bf16) sit in a second 128-column region,
// and dV/dK take the other 256 — 32 MMAs per 128 queries instead of 48:
//   MMA:  S^T(g) -> R | dV,dK(g-1) | [R free] dP^T(g) -> R | [R free] S^T(g+1) ...
//   math: [S(g)] P = exp2(S - lse), P~ = P g -> TMEM | [dP(g)] dS = P (g dP - delta) -> TMEM
// The dV/dK MMAs of tile g-1 run while the math warps load S(g); P is kept in
// registers (64 columns per thread) until dP arrives.
// NQT = 128: two Q/dO stages (64 KB each) — a stage is busy from its load to
// the tile's dV/dK, which follow the next tile's S^T, so two stages leave the
// loads ~one tile of lead and the ring, not the MMAs, sets the period
// (tools/trace_kmaj.py). NQT = 96: three 48 KB stages.
template <int NQT>
struct KQSmem {
    static constexpr int kStages = NQT == 128 ? 2 : 3;
    static constexpr int kKV = 128 * 128 * 2;  // 128 keys x 128 columns
    static constexpr int kT = NQT * 128 * 2;   // NQT queries x 128 columns
    static constexpr int kK = 0;
    static constexpr int kV = kK + kKV;
    static constexpr int kQ = kV + kKV;                  // [kStages]
    static constexpr int kDO = kQ + kStages * kT;        // [kStages]
    static constexpr int kMeta = kDO + kStages * kT;     // [kStages][lse2|delta|tau][NQT] f32
    static constexpr int kBar = kMeta + kStages * 3 * NQT * 4;
    static constexpr int kNumBars = 18;
    static constexpr int kTmemSlot = kBar + kNumBars * 8;
    static constexpr int kAlloc = kTmemSlot + 16 + 1024;
    static_assert(kAlloc <= 232448, "smem");
};
enum { KQ_KVFULL = 0, KQ_KVEMPTY = 1, KQ_QDFULL = 2, KQ_QDEMPTY = 5, KQ_MFULL = 8, KQ_SFULL = 11, KQ_DPFULL = 12,
       KQ_REMPTY = 13, KQ_PDEMPTY = 14, KQ_PDSFULL = 15, KQ_ACCDONE = 16, KQ_ACCEMPTY = 17 };  // 18 (<= 3 stages)

// Per math thread: CT = NQT / 2 query columns of every tile. NQT = 128: warp-
// group hf owns columns [64 hf, 64 hf + 64); NQT = 96: [32 hf, 32 hf + 32) and
// [64 + 16 hf, 80 + 16 hf) (TMEM loads of 32 and 16 columns at aligned
// offsets). qc(c) maps the thread's column index to the tile's.
template <int NQT>
__global__ void __launch_bounds__(kThreads, 1) k_bwd_kmaj_q(const __grid_constant__ BwdArgs a) {
    using SM = KQSmem<NQT>;
    constexpr int D = 128;
    constexpr int QS = SM::kStages;
    constexpr int CT = NQT / 2;
    static_assert(NQT == 128 || NQT == 96, "query tile");
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    float* qmeta = reinterpret_cast<float*>(smem + SM::kMeta);  // [stage][lse2|delta|tau][128]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SKB_TRACE_KMAJ  // tiles 12.. of CTA 100 (tools/trace_kmaj.py)
#define TRK(role, gg, ev) \
    if ((gg) >= 12) SKB_TRB(role, (gg) - 12, ev)
#else
#define TRK(role, gg, ev) \
    do {                  \
    } while (0)
#endif
    const int ntk = (a.L + 127) / 128;
    const int nitems = ntk * a.H * a.B;
    // item wi -> (key tile fastest, h, b); dense sequences only, queries [j0, uni_hi)
    auto item = [&](int wi, int& b, int& h, int& j0, int& nq) -> bool {
        const int kt = wi % ntk;
        const int bh = wi / ntk;
        h = bh % a.H;
        b = bh / a.H;
        j0 = kt * 128;
        if (2 * __ldg(a.ever_count + b) <= a.T) return false;
        nq = (__ldg(a.uni_hi + b * ntk + kt) - j0 + NQT - 1) / NQT;
        return true;
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars[KQ_KVFULL], 1);
        mbar_init(&bars[KQ_KVEMPTY], 1);
        for (int s = 0; s < QS; ++s) {
            mbar_init(&bars[KQ_QDFULL + s], 1);
            mbar_init(&bars[KQ_QDEMPTY + s], 1);
            mbar_init(&bars[KQ_MFULL + s], kProducers + 1);
        }
        mbar_init(&bars[KQ_SFULL], 1);
        mbar_init(&bars[KQ_DPFULL], 1);
        mbar_init(&bars[KQ_REMPTY], kMath / 32);
        mbar_init(&bars[KQ_PDEMPTY], 1);
        mbar_init(&bars[KQ_PDSFULL], kMath / 32);
        mbar_init(&bars[KQ_ACCDONE], 1);
        mbar_init(&bars[KQ_ACCEMPTY], kMath / 32);
        mbar_fence_init();
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tR = tmem, tPS = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

    if (warp >= kProdWarp0 && warp < kMmaWarp) {
        const int ptid = threadIdx.x - kProdWarp0 * 32;
        int g = 0, it = 0;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x) {
            int b, h, j0, nq;
            if (!item(wi, b, h, j0, nq)) continue;
            if (ptid == 0) {
                if (it > 0) mbar_wait(&bars[KQ_KVEMPTY], (it - 1) & 1);
                mbar_expect_tx(&bars[KQ_KVFULL], 2 * SM::kKV);
#pragma unroll
                for (int at = 0; at < 2; ++at) {
                    tma_load_3d(sbase + SM::kK + at * 128 * 128, &a.tm_k128, h * D + at * 64, j0, b, &bars[KQ_KVFULL]);
                    tma_load_3d(sbase + SM::kV + at * 128 * 128, &a.tm_v128, h * D + at * 64, j0, b, &bars[KQ_KVFULL]);
                }
            }
            ++it;
            if (ptid == 32) {  // the next item's K/V rows into L2 while this item runs
                int nb, nh, nj0, nnq;
                for (int nw = wi + gridDim.x; nw < nitems; nw += gridDim.x)
                    if (item(nw, nb, nh, nj0, nnq)) {
#pragma unroll
                        for (int at = 0; at < 2; ++at) {
                            tma_prefetch_3d(&a.tm_k128, nh * D + at * 64, nj0, nb);
                            tma_prefetch_3d(&a.tm_v128, nh * D + at * 64, nj0, nb);
                        }
                        break;
                    }
            }
            const float* lse2 = a.lse2 + ((int64_t)b * a.H + h) * a.L;
            const float* dlt = a.delta + ((int64_t)b * a.H + h) * a.L;
            const int64_t bl = (int64_t)b * a.L;
            const CUtensorMap* tmq = NQT == 128 ? &a.tm_q128 : &a.tm_q96;
            const CUtensorMap* tmo = NQT == 128 ? &a.tm_do128 : &a.tm_do96;
            for (int qt = 0; qt < nq; ++qt, ++g) {
                const int s = g % QS;
                const int qs = j0 + qt * NQT;
                if (ptid == 32 && qt + QS < nq) {  // this item's tile QS ahead into L2
#pragma unroll
                    for (int at = 0; at < 2; ++at) {
                        tma_prefetch_3d(tmq, h * D + at * 64, qs + QS * NQT, b);
                        tma_prefetch_3d(tmo, h * D + at * 64, qs + QS * NQT, b);
                    }
                }
                if (g >= QS) mbar_wait(&bars[KQ_QDEMPTY + s], ((g - QS) / QS) & 1);
                for (int c = ptid; c < NQT; c += kProducers) {
                    const int i = qs + c;
                    const bool ok = i < a.L;
                    const int t = i - a.w;
                    const uint32_t mb = smem_u32(qmeta + (s * 3) * NQT + c);
                    cp_async4(mb, lse2 + (ok ? i : 0), ok);
                    cp_async4(mb + NQT * 4, dlt + (ok ? i : 0), ok);
                    cp_async4(mb + 2 * NQT * 4, a.tauf + bl + (ok && t >= 0 ? t : 0), ok && t >= 0);
                }
                cp_async_arrive_noinc(&bars[KQ_MFULL + s]);
                if (ptid == 0) {
                    mbar_arrive(&bars[KQ_MFULL + s]);
                    mbar_expect_tx(&bars[KQ_QDFULL + s], 2 * SM::kT);
#pragma unroll
                    for (int at = 0; at < 2; ++at) {
                        tma_load_3d(sbase + SM::kQ + s * SM::kT + at * NQT * 128, tmq, h * D + at * 64, qs, b,
                                    &bars[KQ_QDFULL + s]);
                        tma_load_3d(sbase + SM::kDO + s * SM::kT + at * NQT * 128, tmo, h * D + at * 64, qs, b,
                                    &bars[KQ_QDFULL + s]);
                    }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0) {
            constexpr uint32_t id_s = umma_idesc(128, NQT, false, false);
            constexpr uint32_t id_acc = umma_idesc(128, D, false, true);
            int g = 0, it = 0, rp = 0;  // rp: REMPTY phases consumed
            // dV += P~^T dO, dK += dS^T Q for global tile gj (item tile qj)
            auto acc = [&](int gj, int qj, int itn) {
                const int s = gj % QS;
                mbar_wait_fast(&bars[KQ_PDSFULL], gj & 1);
                TRK(7, gj, 2);
                if (qj == 0 && itn > 0) mbar_wait_fast(&bars[KQ_ACCEMPTY], (itn - 1) & 1);
                tc_after_sync();
                const uint32_t qb = sbase + SM::kQ + s * SM::kT, dob = sbase + SM::kDO + s * SM::kT;
#pragma unroll
                for (int kk = 0; kk < NQT / 16; ++kk) {
                    umma_f16_ts(tDV, tPS + kk * 8, desc_mnmajor(dob, NQT, kk), id_acc, (qj > 0 || kk > 0) ? 1u : 0u);
                    umma_f16_ts(tDK, tPS + NQT / 2 + kk * 8, desc_mnmajor(qb, NQT, kk), id_acc,
                                (qj > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&bars[KQ_PDEMPTY]);
                umma_commit(&bars[KQ_QDEMPTY + s]);
            };
            for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x) {
                int b, h, j0, nq;
                if (!item(wi, b, h, j0, nq)) continue;
                mbar_wait_fast(&bars[KQ_KVFULL], it & 1);
                tc_after_sync();
                for (int qt = 0; qt < nq; ++qt, ++g) {
                    const int s = g % QS;
                    mbar_wait_fast(&bars[KQ_QDFULL + s], (g / QS) & 1);
                    TRK(7, g, 0);
                    if (g > 0) mbar_wait_fast(&bars[KQ_REMPTY], (rp++) & 1);  // dP(g-1) read out of R
                    TRK(7, g, 5);
                    tc_after_sync();
                    const uint32_t qb = sbase + SM::kQ + s * SM::kT, dob = sbase + SM::kDO + s * SM::kT;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        umma_f16(tR, desc_kmajor(sbase + SM::kK, 128, kk), desc_kmajor(qb, NQT, kk), id_s,
                                 kk > 0 ? 1u : 0u);
                    umma_commit(&bars[KQ_SFULL]);
                    TRK(7, g, 1);
                    if (qt >= 1) acc(g - 1, qt - 1, it);
                    TRK(7, g, 6);
                    mbar_wait_fast(&bars[KQ_REMPTY], (rp++) & 1);  // S(g) read out of R
                    TRK(7, g, 7);
                    tc_after_sync();
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        umma_f16(tR, desc_kmajor(sbase + SM::kV, 128, kk), desc_kmajor(dob, NQT, kk), id_s,
                                 kk > 0 ? 1u : 0u);
                    umma_commit(&bars[KQ_DPFULL]);
                    TRK(7, g, 3);
                    if (qt == nq - 1) umma_commit(&bars[KQ_KVEMPTY]);
                }
                acc(g - 1, nq - 1, it);
                umma_commit(&bars[KQ_ACCDONE]);
                ++it;
            }
        }
        __syncwarp();
    } else if (warp < kProdWarp0) {
        const int hf = warp >> 2;
        // tile column of the thread's column c (c even pairs stay in one group)
        auto qc = [&](int c) { return NQT == 128 ? 64 * hf + c : (c < 32 ? 32 * hf + c : 32 + 16 * hf + c); };
        const int r = ((warp & 3) << 5) | lane;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sl2 = a.scale_log2;
        const float2 sl22 = make_float2(sl2, sl2);
        const bool mst = a.mask_st != 0;
        int g = 0, it = 0;
        const bool trl = lane == 0 && (warp & 3) == 0;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x) {
            int b, h, j0, nq;
            if (!item(wi, b, h, j0, nq)) continue;
            const int64_t bl = (int64_t)b * a.L;
            const int key = j0 + r < a.L ? j0 + r : -1;
            // queries [key, key + w) read the key from the window, [key + w,
            // leave + w) from the selection (proj/src/cache.cpp:259-311)
            int hi_i = key >= 0 ? min(a.L, key + a.w) : 0;
            bool sel_u = false;
            float uj = 0.f, colsum = 0.f;
            if (key >= 0 && key < a.T && a.R1 > 0) {
                const int lv = __ldg(a.leave + bl + key);
                sel_u = lv > key;
                if (sel_u) {
                    hi_i = min(a.L, lv + a.w);
                    uj = __ldg(a.uf + bl + key);
                }
            }
            for (int qt = 0; qt < nq; ++qt, ++g) {
                const int s = g % QS;
                const int qs = j0 + qt * NQT;  // the tile's first query
                if (trl) TRK(4 + hf, g, 9);
                mbar_wait(&bars[KQ_SFULL], g & 1);
                mbar_wait(&bars[KQ_MFULL + s], (g / QS) & 1);
                tc_after_sync();
                float sv[CT], dp[CT];
                auto ld_r = [&](float* v) {
                    if constexpr (NQT == 128) {
                        tmem_ld32(tR + lane_off + hf * 64, v);
                        tmem_ld32(tR + lane_off + hf * 64 + 32, v + 32);
                    } else {
                        tmem_ld32(tR + lane_off + hf * 32, v);
                        tmem_ld16(tR + lane_off + 64 + hf * 16, v + 32);
                    }
                };
                ld_r(sv);
                tmem_wait_ld();
                tc_before_sync();
                warp_arrive(&bars[KQ_REMPTY]);
                if (trl) TRK(4 + hf, g, 0);
                const float* ml = qmeta + (s * 3) * NQT;  // indexed by tile column
                const float* md = ml + NQT;
                const float* mt = ml + 2 * NQT;
                const int cmin = key >= 0 ? key - qs : NQT;
                const int cmax = key >= 0 ? hi_i - 1 - qs : -1;
                if (!__all_sync(0xffffffffu, cmin <= 0 && cmax >= NQT - 1)) {
#pragma unroll
                    for (int c = 0; c < CT; ++c) sv[c] = (qc(c) >= cmin && qc(c) <= cmax) ? sv[c] : -INFINITY;
                }
                const int cwc = key + a.w - qs;  // tile columns < cwc: window, gate 1
                const int clast = max(0, min(NQT - 1, a.L - 1 - qs));
                const bool plain = __all_sync(0xffffffffu, !sel_u || cwc > NQT - 1 || uj >= mt[clast] + 1.f);
                uint32_t pk[CT / 2];
                // P (ungated, kept for dS) and P~ = P g -> TMEM
#pragma unroll
                for (int c = 0; c < CT; c += 2) {
                    const float2 l2 = *reinterpret_cast<const float2*>(ml + qc(c));
                    float2 p2 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, make_float2(-l2.x, -l2.y));
                    p2.x = ex2(p2.x);  // masked: 0
                    p2.y = ex2(p2.y);
                    sv[c] = p2.x, sv[c + 1] = p2.y;
                    float2 pw = p2;
                    if (!plain && !mst) {
                        const float2 t2 = *reinterpret_cast<const float2*>(mt + qc(c));
                        const float g0 = qc(c) < cwc ? 1.f : __saturatef(uj - t2.x);
                        const float g1 = qc(c) + 1 < cwc ? 1.f : __saturatef(uj - t2.y);
                        pw = __fmul2_rn(p2, make_float2(g0, g1));
                    }
                    pk[c >> 1] = pack_bf16(pw.x, pw.y);
                }
                if (trl) TRK(4 + hf, g, 1);
                if (g >= 1) mbar_wait(&bars[KQ_PDEMPTY], (g - 1) & 1);  // dV/dK(g-1) have read P~/dS
                if (trl) TRK(4 + hf, g, 2);
                tc_after_sync();
                // packed column = tile column / 2
                auto st_ps = [&](uint32_t base) {
                    if constexpr (NQT == 128) {
                        tmem_st16u(base + lane_off + hf * 32, pk);
                        tmem_st16u(base + lane_off + hf * 32 + 16, pk + 16);
                    } else {
                        tmem_st16u(base + lane_off + hf * 16, pk);
                        tmem_st8u(base + lane_off + 32 + hf * 8, pk + 16);
                    }
                };
                st_ps(tPS);
                mbar_wait(&bars[KQ_DPFULL], g & 1);
                if (trl) TRK(4 + hf, g, 3);
                tc_after_sync();
                ld_r(dp);
                tmem_wait_ld();
                tc_before_sync();
                warp_arrive(&bars[KQ_REMPTY]);
                // dS = P (g dP - delta) (unscaled); colsum: the gate gradient on the fractional support
                if (plain) {
#pragma unroll
                    for (int c = 0; c < CT; c += 2) {
                        const float2 d2 = *reinterpret_cast<const float2*>(md + qc(c));
                        const float2 cc = __fmul2_rn(make_float2(sv[c], sv[c + 1]),
                                                     __fadd2_rn(make_float2(dp[c], dp[c + 1]), make_float2(-d2.x, -d2.y)));
                        pk[c >> 1] = pack_bf16(cc.x, cc.y);
                    }
                } else {
                    float2 csum2 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int c = 0; c < CT; c += 2) {
                        const float2 d2 = *reinterpret_cast<const float2*>(md + qc(c));
                        const float2 t2 = *reinterpret_cast<const float2*>(mt + qc(c));
                        const float g0 = qc(c) < cwc ? 1.f : __saturatef(uj - t2.x);
                        const float g1 = qc(c) + 1 < cwc ? 1.f : __saturatef(uj - t2.y);
                        const float2 p2 = make_float2(sv[c], sv[c + 1]);
                        const float2 dp2 = make_float2(dp[c], dp[c + 1]);
                        const float2 g2 = mst ? make_float2(1.f, 1.f) : make_float2(g0, g1);
                        const float2 cc = __fmul2_rn(p2, __ffma2_rn(g2, dp2, make_float2(-d2.x, -d2.y)));
                        // 0 < g < 1 <=> (bits(g) - 1) < bits(1.0) - 1 (g in [0, 1])
                        const float2 fr2 = make_float2((__float_as_uint(g0) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f,
                                                       (__float_as_uint(g1) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f);
                        csum2 = __ffma2_rn(__fmul2_rn(p2, dp2), fr2, csum2);
                        pk[c >> 1] = pack_bf16(cc.x, cc.y);
                    }
                    colsum += csum2.x + csum2.y;
                }
                st_ps(tPS + NQT / 2);
                tmem_wait_st();
                tc_before_sync();
                warp_arrive(&bars[KQ_PDSFULL]);
                if (trl) TRK(4 + hf, g, 4);
            }
            mbar_wait(&bars[KQ_ACCDONE], it & 1);
            tc_after_sync();
            float dv[64], dk[64];
            tmem_ld32(tDV + lane_off + hf * 64, dv);
            tmem_ld32(tDV + lane_off + hf * 64 + 32, dv + 32);
            tmem_ld32(tDK + lane_off + hf * 64, dk);
            tmem_ld32(tDK + lane_off + hf * 64 + 32, dk + 32);
            tmem_wait_ld();
            tc_before_sync();
            warp_arrive(&bars[KQ_ACCEMPTY]);
            ++it;
            if (key < 0) continue;
            if (colsum != 0.f) atomicAdd(a.colsum + bl + key, (double)colsum);
            const int64_t ro = (((int64_t)b * a.L + key) * a.H + h) * D + hf * 64;
#pragma unroll
            for (int e = 0; e < 64; e += 8) {
                uint4 x, y;
                x.x = pack_bf16(dk[e] * a.scale, dk[e + 1] * a.scale);
                x.y = pack_bf16(dk[e + 2] * a.scale, dk[e + 3] * a.scale);
                x.z = pack_bf16(dk[e + 4] * a.scale, dk[e + 5] * a.scale);
                x.w = pack_bf16(dk[e + 6] * a.scale, dk[e + 7] * a.scale);
                y.x = pack_bf16(dv[e], dv[e + 1]);
                y.y = pack_bf16(dv[e + 2], dv[e + 3]);
                y.z = pack_bf16(dv[e + 4], dv[e + 5]);
                y.w = pack_bf16(dv[e + 6], dv[e + 7]);
                *reinterpret_cast<uint4*>(a.dk + ro + e) = x;
                *reinterpret_cast<uint4*>(a.dv + ro + e) = y;
            }
        }
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
#undef TRK
}

// ------------------------------------------------------------ selected pass on CTA pairs
// The selected pass (D = 128) as cta_group::2 MMAs on a cluster of two CTAs:
// a work item is 256 entries of the ever-selected order (128 per CTA) and the
// 64-query tiles that read any of them; the even CTA issues M = 256 MMAs.
// A tcgen05.mma with M = 128 costs ~72 cycles for any N <= 128
// (tools/probes/mma_rate.cu: N = 64 runs at half rate), and the single-CTA
// pass's S^T / dP^T are N = 64; a pair instruction moves twice the keys in
// the same time. Each CTA's TMEM, math warps and epilogue are those of the
// single-CTA pass; what the pair changes is the B operands, split in halves:
//   S^T = K Q^T, dP^T = V dO^T   (N = 64 queries): each CTA stages its 32
//                                 query rows x 128 columns       ("X", 8 KB)
//   dV += P~^T dO, dK += dS^T Q  (N = 128 columns): each CTA stages all 64
//                                 query rows x its 64 columns     ("Y", 8 KB)
// so a stage is 16 KB of Q + 16 KB of dO per CTA, as before, for twice the keys.
// Barriers: the even CTA's QDFULL collects both CTAs' TMA bytes, its PDSFULL /
// ACCEMPTY / KVFULL one arrival per warp (or relay) from each CTA; the MMA
// commits multicast SFULL / QDEMPTY / KVEMPTY / ACCDONE to both CTAs.
constexpr int kPairQS = 4;

template <int D>
struct PSmem {
    static_assert(D == 128, "pair pass: D = 128");
    static constexpr int kKV = 128 * D * 2;
    static constexpr int kHalf = 32 * D * 2;  // X: 32 query rows x D (2 atom columns)
    static constexpr int kQT = 2 * kHalf;     // X + Y (Y: 64 query rows x 64 columns)
    static constexpr int kK = 0;
    static constexpr int kV = kK + kKV;
    static constexpr int kQ = kV + kKV;             // [kPairQS]
    static constexpr int kDO = kQ + kPairQS * kQT;  // [kPairQS]
    static constexpr int kMeta = kDO + kPairQS * kQT;  // [kPairQS][lse2|delta|tau][64] f32
    static constexpr int kBar = kMeta + kPairQS * 3 * 64 * 4;
    static constexpr int kNumBars = 24;
    static constexpr int kTmemSlot = kBar + kNumBars * 8;
    static constexpr int kAlloc = kTmemSlot + 16 + 1024;
    static_assert(kAlloc <= 232448, "smem");
};
enum { PB_KVFULL = 0, PB_KVLOC = 1, PB_KVEMPTY = 2, PB_QDFULL = 3, PB_QDEMPTY = 7, PB_MFULL = 11, PB_SFULL = 15,
       PB_PDSFULL = 17, PB_ACCDONE = 19, PB_ACCEMPTY = 20 };  // 21

template <int D, bool KEY_SOFT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_bwd_dkdv_sel_pair(const __grid_constant__ BwdArgs a) {
    using SM = PSmem<D>;
    constexpr int QS = kPairQS;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    float* qmeta = reinterpret_cast<float*>(smem + SM::kMeta);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SKB_TRACE_SEL  // items 6.. of CTA 100 (tools/trace_selp.py)
#define TRP(role, gg, ev) \
    if ((gg) >= tr0) SKB_TRB(role, (gg) - tr0, ev)
#else
#define TRP(role, gg, ev) \
    do {                  \
    } while (0)
#endif
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int ntk = (a.L + 127) / 128, ntk2 = (a.L + 255) / 256;
    const int nitems = ntk2 * a.H * a.B;
    // item wi -> (256-entry tile kt2 fastest, h, b); this CTA's keys are entries
    // [kt2 * 256 + rank * 128, +128); the query range covers both halves
    auto item = [&](int wi, int& b, int& h, int& kt2, int& nkeys, int& q_lo, int& nq) -> bool {
        kt2 = wi % ntk2;
        const int bh = wi / ntk2;
        h = bh % a.H;
        b = bh / a.H;
        const int ec = __ldg(a.ever_count + b);
        if (kt2 * 256 >= ec) return false;
        if (a.uni && 2 * ec > a.T) return false;
        const int n0 = min(128, ec - kt2 * 256), n1 = max(0, min(128, ec - kt2 * 256 - 128));
        nkeys = rank ? n1 : n0;
        int lo = INT_MAX, hi = 0;
        const int2 i0 = a.sel_items[b * ntk + 2 * kt2];
        if (i0.y > 0) lo = i0.x, hi = i0.x + 64 * i0.y;
        if (n1 > 0) {
            const int2 i1 = a.sel_items[b * ntk + 2 * kt2 + 1];
            if (i1.y > 0) lo = min(lo, i1.x), hi = max(hi, i1.x + 64 * i1.y);
        }
        q_lo = hi > 0 ? lo : 0;
        nq = hi > lo ? (hi - lo) / 64 : 0;
        return true;
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars[PB_KVFULL], 2);
        mbar_init(&bars[PB_KVLOC], kProducers + 1);
        mbar_init(&bars[PB_KVEMPTY], 1);
        for (int s = 0; s < QS; ++s) {
            mbar_init(&bars[PB_QDFULL + s], 1);
            mbar_init(&bars[PB_QDEMPTY + s], 1);
            mbar_init(&bars[PB_MFULL + s], kProducers + 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[PB_SFULL + s], 1);
            mbar_init(&bars[PB_PDSFULL + s], 2 * (kMath / 32));
        }
        mbar_init(&bars[PB_ACCDONE], 1);
        mbar_init(&bars[PB_ACCEMPTY], 2 * (kMath / 32));
        mbar_fence_init();
    }
    if (warp == kMmaWarp) tmem_alloc_pair<512>(tmem_slot);
    tc_before_sync();
    cluster_sync_all();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;
    auto lead = [&](int idx) { return peer_addr(smem_u32(&bars[idx]), 0); };

    if (warp >= kProdWarp0 && warp < kMmaWarp) {
        const int pw = warp - kProdWarp0, ptid = threadIdx.x - kProdWarp0 * 32;
        int g = 0, kit = 0, tr0 = 1 << 28;
        for (int wi = pair; wi < nitems; wi += npairs) {
            int b, h, kt2, nkeys, q_lo, nq;
            if (!item(wi, b, h, kt2, nkeys, q_lo, nq) || nq == 0) continue;
            if (kit == 6) tr0 = g;
            const int64_t bl = (int64_t)b * a.L;
            const int* elist = a.sel_order + bl + kt2 * 256 + (int)rank * 128;
            RowKeys<D, 128> kk;
            kk.fetch(pw, lane, [&](int r) { return r < nkeys ? __ldg(elist + r) : -1; });
            if (ptid == 0) TRP(6, g, 3);
            if (kit > 0) mbar_wait(&bars[PB_KVEMPTY], (kit - 1) & 1);
            if (ptid == 0) TRP(6, g, 2);
            kk.issue(sbase + SM::kK, a.k, b, h, a.L, a.H, pw, lane);
            kk.issue(sbase + SM::kV, a.v, b, h, a.L, a.H, pw, lane);
            cp_async_arrive_noinc(&bars[PB_KVLOC]);
            if (ptid == 0) mbar_arrive(&bars[PB_KVLOC]);
            if (ptid == 64) {  // relay: this CTA's rows have landed -> the even CTA's MMA thread
                mbar_wait(&bars[PB_KVLOC], kit & 1);
                fence_proxy_async();
                mbar_arrive_cluster(lead(PB_KVFULL));
            }
            ++kit;
            const float* lse2 = a.lse2 + ((int64_t)b * a.H + h) * a.L;
            const float* dlt = a.delta + ((int64_t)b * a.H + h) * a.L;
            for (int qt = 0; qt < nq; ++qt, ++g) {
                const int s = g % QS;
                if (g >= QS) mbar_wait(&bars[PB_QDEMPTY + s], ((g - QS) / QS) & 1);
                if (ptid == 0) TRP(6, g, 1);
                const int qs = q_lo + qt * 64;
                for (int c = ptid; c < 64; c += kProducers) {
                    const int i = qs + c;
                    const bool ok = i < a.L;
                    const int t = i - a.w;
                    const uint32_t mb = smem_u32(qmeta + (s * 3) * 64 + c);
                    cp_async4(mb, lse2 + (ok ? i : 0), ok);
                    cp_async4(mb + 64 * 4, dlt + (ok ? i : 0), ok);
                    cp_async4(mb + 128 * 4, a.tauf + bl + (ok && t >= 0 ? t : 0), ok && t >= 0);
                }
                cp_async_arrive_noinc(&bars[PB_MFULL + s]);
                if (ptid == 0) {
                    mbar_arrive(&bars[PB_MFULL + s]);
                    if (leader) mbar_expect_tx(&bars[PB_QDFULL + s], 2 * 2 * SM::kQT);
                    const uint32_t full = lead(PB_QDFULL + s);
                    const uint32_t q0 = sbase + SM::kQ + s * SM::kQT, d0 = sbase + SM::kDO + s * SM::kQT;
#pragma unroll
                    for (int at = 0; at < D / 64; ++at) {  // X: this CTA's 32 query rows, every column
                        tma_load_3d_pair(q0 + at * 32 * 128, &a.tm_q32, h * D + at * 64, qs + (int)rank * 32, b, full);
                        tma_load_3d_pair(d0 + at * 32 * 128, &a.tm_do32, h * D + at * 64, qs + (int)rank * 32, b, full);
                    }
                    // Y: every query row, this CTA's 64 columns
                    tma_load_3d_pair(q0 + SM::kHalf, &a.tm_q64, h * D + (int)rank * 64, qs, b, full);
                    tma_load_3d_pair(d0 + SM::kHalf, &a.tm_do64, h * D + (int)rank * 64, qs, b, full);
                }
            }
        }
    } else if (warp == kMmaWarp) {
        if (leader && lane == 0) {
            constexpr uint32_t id_s = umma_idesc(256, 64, false, false);
            constexpr uint32_t id_acc = umma_idesc(256, D, false, true);
            int g = 0, kit = 0, tr0 = 1 << 28;
            auto acc = [&](int gj, int qt, int kitn) {
                const int s = gj & 1, qs = gj % QS;
                mbar_wait(&bars[PB_PDSFULL + s], (gj >> 1) & 1);
                TRP(7, gj, 2);
                if (qt == 0 && kitn > 0) mbar_wait(&bars[PB_ACCEMPTY], (kitn - 1) & 1);
                tc_after_sync();
                const uint32_t qy = sbase + SM::kQ + qs * SM::kQT + SM::kHalf;
                const uint32_t dy = sbase + SM::kDO + qs * SM::kQT + SM::kHalf;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint32_t co = s * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
                    umma_f16_ts_pair(tDV, tS + co, desc_mnmajor(dy, 64, kk), id_acc, (qt > 0 || kk > 0) ? 1u : 0u);
                    umma_f16_ts_pair(tDK, tP + co, desc_mnmajor(qy, 64, kk), id_acc, (qt > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit_pair(&bars[PB_QDEMPTY + qs]);
            };
            for (int wi = pair; wi < nitems; wi += npairs) {
                int b, h, kt2, nkeys, q_lo, nq;
                if (!item(wi, b, h, kt2, nkeys, q_lo, nq) || nq == 0) continue;
                if (kit == 6) tr0 = g;
                mbar_wait(&bars[PB_KVFULL], kit & 1);
                TRP(7, g, 4);
                fence_proxy_async();
                tc_after_sync();
                for (int qt = 0; qt < nq; ++qt, ++g) {
                    const int s = g & 1, qs = g % QS;
                    mbar_wait(&bars[PB_QDFULL + qs], (g / QS) & 1);
                    TRP(7, g, 0);
                    tc_after_sync();
                    const uint32_t qx = sbase + SM::kQ + qs * SM::kQT, dx = sbase + SM::kDO + qs * SM::kQT;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        umma_f16_pair(tS + s * 64, desc_kmajor(sbase + SM::kK, 128, kk), desc_kmajor(qx, 32, kk), id_s,
                                      kk > 0 ? 1u : 0u);
                        umma_f16_pair(tP + s * 64, desc_kmajor(sbase + SM::kV, 128, kk), desc_kmajor(dx, 32, kk), id_s,
                                      kk > 0 ? 1u : 0u);
                    }
                    umma_commit_pair(&bars[PB_SFULL + s]);
                    TRP(7, g, 1);
                    if (qt == nq - 1) umma_commit_pair(&bars[PB_KVEMPTY]);
                    // S/dP(g) are issued after dV/dK(g - 2) (in-order MMAs), which waited
                    // for the math warps to finish with buffer s: no separate release
                    if (qt >= 1) acc(g - 1, qt - 1, kit);
                }
                acc(g - 1, nq - 1, kit);
                umma_commit_pair(&bars[PB_ACCDONE]);
                ++kit;
            }
        }
        __syncwarp();
    } else if (warp < kProdWarp0) {
        const int hf = warp >> 2;
        const int r = ((warp & 3) << 5) | lane;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sl2 = a.scale_log2;
        const float2 sl22 = make_float2(sl2, sl2);
        int g = 0, kit = 0, tr0 = 1 << 28;
        const bool trl = lane == 0 && (warp & 3) == 0;
        for (int wi = pair; wi < nitems; wi += npairs) {
            int b, h, kt2, nkeys, q_lo, nq;
            if (!item(wi, b, h, kt2, nkeys, q_lo, nq)) continue;
            if (kit == 6 && nq > 0) tr0 = g;
            const int64_t bl = (int64_t)b * a.L;
            const int e = kt2 * 256 + (int)rank * 128 + r;
            const int key = r < nkeys ? __ldg(a.sel_order + bl + e) : -1;
            const int leave = key >= 0 ? __ldg(a.leave + bl + key) : 0;
            const float uj = key >= 0 ? __ldg(a.uf + bl + key) : 0.f;
            // queries [key + w, leave + w) read this key from the selection
            // (proj/src/cache.cpp:259-311), clipped to the key's chunk
            const int lo_i = key + a.w;
            int hi_i = min(a.L, leave + a.w);
            if (a.chunk_len > 0 && key >= 0) hi_i = min(hi_i, (key / a.chunk_len + 1) * a.chunk_len);
            float colsum = 0.f;
            for (int qt = 0; qt < nq; ++qt, ++g) {
                const int s = g & 1, qs3 = g % QS;
                const int qs = q_lo + qt * 64 + hf * 32;
                if (trl) TRP(4 + hf, g, 9);
                mbar_wait(&bars[PB_SFULL + s], (g >> 1) & 1);
                mbar_wait(&bars[PB_MFULL + qs3], (g / QS) & 1);
                if (trl) TRP(4 + hf, g, 0);
                tc_after_sync();
                float sv[32], dp[32];
                tmem_ld32(tS + lane_off + s * 64 + hf * 32, sv);
                tmem_ld32(tP + lane_off + s * 64 + hf * 32, dp);
                tmem_wait_ld();
                if (SKB_BWD_EXP == 1) {  // experiment: no elementwise work
                    tc_before_sync();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(lead(PB_PDSFULL + s));
                    continue;
                }
                const float* ml = qmeta + (qs3 * 3) * 64 + hf * 32;
                const float* md = ml + 64;
                const float* mt = ml + 128;
                const int cmin = key >= 0 ? lo_i - qs : 32;
                const int cmax = key >= 0 ? hi_i - 1 - qs : -1;
                const bool full = __all_sync(0xffffffffu, cmin <= 0 && cmax >= 31);
                const int clast = max(0, min(31, a.L - 1 - qs));
                const bool sat = __all_sync(0xffffffffu, key < 0 || uj >= mt[clast] + 1.f);
                if (!full) {
#pragma unroll
                    for (int c = 0; c < 32; ++c) sv[c] = (c >= cmin && c <= cmax) ? sv[c] : -INFINITY;
                }
                colsum += sel_tile_math<KEY_SOFT>(a, sat, uj, ml, md, mt, sl2, sl22, sv, dp);
                uint32_t pk[16];
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2) pk[e2] = pack_bf16(sv[2 * e2], sv[2 * e2 + 1]);
                tmem_st16u(tS + lane_off + s * 64 + hf * 32, pk);
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2) pk[e2] = pack_bf16(dp[2 * e2], dp[2 * e2 + 1]);
                tmem_st16u(tP + lane_off + s * 64 + hf * 32, pk);
                tmem_wait_st();
                tc_before_sync();
                __syncwarp();
                if (trl) TRP(4 + hf, g, 4);
                if (lane == 0) mbar_arrive_cluster(lead(PB_PDSFULL + s));
            }
            if (key >= 0 && colsum != 0.f) atomicAdd(a.colsum + bl + key, (double)colsum);
            float dv[D / 2], dk[D / 2];
            if (nq > 0) {
                mbar_wait(&bars[PB_ACCDONE], kit & 1);
                if (trl) TRP(4 + hf, g, 5);
                tc_after_sync();
#pragma unroll
                for (int c = 0; c < D / 64; ++c) {
                    tmem_ld32(tDV + lane_off + hf * (D / 2) + c * 32, dv + c * 32);
                    tmem_ld32(tDK + lane_off + hf * (D / 2) + c * 32, dk + c * 32);
                }
                tmem_wait_ld();
                tc_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(lead(PB_ACCEMPTY));
                ++kit;
            } else {
#pragma unroll
                for (int e2 = 0; e2 < D / 2; ++e2) dv[e2] = dk[e2] = 0.f;
            }
            if (key < 0) continue;
#pragma unroll
            for (int e2 = 0; e2 < D / 2; e2 += 8) {
                const int64_t po = part_off<D>(a, b, h, key, (hf * (D / 2) + e2) >> 3);
                uint4 x, y;
                x.x = pack_bf16(dk[e2] * a.scale, dk[e2 + 1] * a.scale);
                x.y = pack_bf16(dk[e2 + 2] * a.scale, dk[e2 + 3] * a.scale);
                x.z = pack_bf16(dk[e2 + 4] * a.scale, dk[e2 + 5] * a.scale);
                x.w = pack_bf16(dk[e2 + 6] * a.scale, dk[e2 + 7] * a.scale);
                y.x = pack_bf16(dv[e2], dv[e2 + 1]);
                y.y = pack_bf16(dv[e2 + 2], dv[e2 + 3]);
                y.z = pack_bf16(dv[e2 + 4], dv[e2 + 5]);
                y.w = pack_bf16(dv[e2 + 6], dv[e2 + 7]);
                *reinterpret_cast<uint4*>(a.dk_acc + po) = x;
                *reinterpret_cast<uint4*>(a.dv_acc + po) = y;
            }
        }
    }
    tc_before_sync();
    cluster_sync_all();
    tc_after_sync();
    if (warp == kMmaWarp) tmem_dealloc_pair<512>(tmem);
#undef TRP
}

// ------------------------------------------------------------------ dQ
// Query-major over 128-key tiles [selected union | window band] (N=128 MMAs:
// narrow tiles pay a high per-instruction cost). TMEM: Q (bf16 A operand,
// loaded once by the math warps), dS (bf16), S and dP (fp32, 128 columns
// each), dQ. Per tile: S = Q K^T (TS) and dP = dO V^T (SS, dO resident in
// shared memory); the S/dP of tile j+1 run while the math warpgroups (64 keys
// each) form dS_j = P (wv dP - delta) * kappa; dQ += dS_j K (TS). Producers:
// dO and the window band by 3-D TMA, selected rows by cp.async gathers with
// keys fetched one tile ahead, per-key metadata from skb_select's block arrays.
#ifndef SKB_DQ_POLY
#define SKB_DQ_POLY 1
#endif
constexpr bool kDqPoly = SKB_DQ_POLY != 0;
constexpr int kNS = 3;  // K (+ metadata) ring depth of the dQ kernel
constexpr int kNV = 2;  // V ring depth (V is released as soon as dP is computed)

template <int D>
struct QSmem {
    static constexpr int kKT = 128 * D * 2;  // 128-key tile
    static constexpr int kDO = 0;            // dO tile (128 queries)
    static constexpr int kK = kDO + kKT;     // [kNS]
    static constexpr int kV = kK + kNS * kKT;  // [kNV]
    static constexpr int kMeta = kV + kNV * kKT;  // [kNS][key|ext|uf][128] x 4 B
    static constexpr int kFlags = kMeta + kNS * 3 * 128 * 4;  // [kNS] x 16 B
    static constexpr int kBar = kFlags + kNS * 16;
    static constexpr int kNumBars = 26;  // QB_* (25)
    static constexpr int kTmemSlot = kBar + kNumBars * 8;
    static constexpr int kAlloc = kTmemSlot + 16 + 1024;
};
enum { QB_QFULL = 0, QB_DOFULL = 1, QB_KVFULL = 2, QB_KVEMPTY = 5, QB_MFULL = 8, QB_MEMPTY = 11, QB_VFULL = 14,
       QB_VEMPTY = 16, QB_SFULL = 18, QB_SEMPTY = 19, QB_DSFULL = 20, QB_DSEMPTY = 21, QB_DQDONE = 22,
       QB_QDOEMPTY = 23, QB_DQEMPTY = 24 };  // 25

template <int D, bool KEY_SOFT>
__global__ void __launch_bounds__(kThreads, 1) k_bwd_dq_tc(const __grid_constant__ BwdArgs a) {
    using SM = QSmem<D>;
    static_assert(QB_DQDONE < SM::kNumBars, "barrier slots");
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    int* meta = reinterpret_cast<int*>(smem + SM::kMeta);
    int* tflags = reinterpret_cast<int*>(smem + SM::kFlags);

    const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bl = (int64_t)b * a.L;
    const int64_t qrow = (int64_t)b * a.nqb + qb;
    const int i0 = qb * 128;
    const int cnt = (a.R1 > 0) ? a.qb_count[qrow] : 0;
    const int n_sel = (cnt + 127) / 128;
    const int n_win = (a.w + 127 + 127) / 128;
    const int n = n_sel + n_win;
    const int jw0 = i0 - a.w + 1;
    const int* list = a.qb_list + qrow * a.qb_cap;

    if (threadIdx.x == 0) SKB_TRB(2, 31, 7);
    if (threadIdx.x == 0) {
        mbar_init(&bars[QB_QFULL], kMath / 2);
        mbar_init(&bars[QB_DOFULL], 1);
        for (int s = 0; s < kNS; ++s) {
            mbar_init(&bars[QB_KVFULL + s], kProducers + 1);
            mbar_init(&bars[QB_KVEMPTY + s], 1);
            mbar_init(&bars[QB_MFULL + s], kProducers);
            mbar_init(&bars[QB_MEMPTY + s], kMath);
        }
        for (int s = 0; s < kNV; ++s) {
            mbar_init(&bars[QB_VFULL + s], kProducers + 1);
            mbar_init(&bars[QB_VEMPTY + s], 1);
        }
        mbar_init(&bars[QB_SFULL], 1);
        mbar_init(&bars[QB_SEMPTY], kMath);
        mbar_init(&bars[QB_DSFULL], kMath);
        mbar_init(&bars[QB_DSEMPTY], 1);
        mbar_init(&bars[QB_DQDONE], 1);
        mbar_fence_init();
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tQ = tmem, tDS = tmem + 64, tS = tmem + 128, tP = tmem + 256, tDQ = tmem + 384;

    if (warp >= kProdWarp0 && warp < kMmaWarp) {
        constexpr int kAtoms = D / 64;
        const int pw = warp - kProdWarp0, ptid = threadIdx.x - kProdWarp0 * 32;
        if (ptid == 0) {
            mbar_expect_tx(&bars[QB_DOFULL], 128 * D * 2);
#pragma unroll
            for (int at = 0; at < kAtoms; ++at)
                tma_load_3d(sbase + SM::kDO + at * 128 * 128, &a.tm_do128, h * D + at * 64, i0, b, &bars[QB_DOFULL]);
        }
        RowKeys<D, 128> kcur;
        if (n_sel > 0) kcur.fetch(pw, lane, [&](int r) { return __ldg(list + r); });
        const int ma = ptid >> 5, mc = ptid & 31;  // metadata: array x 16-byte chunk (96 threads)
        const int* msrc = ma == 0 ? a.qb_list : ma == 1 ? a.qb_leave : reinterpret_cast<const int*>(a.qb_uf);
        for (int jt = 0; jt < n; ++jt) {
            const int s = jt % kNS;
            if (ptid == 0) SKB_TRB(2, jt, 0);
            if (jt >= kNS) mbar_wait(&bars[QB_MEMPTY + s], ((jt - kNS) / kNS) & 1);
            if (jt < n_sel) {
                cp_async16(smem_u32(meta + (s * 3 + ma) * 128 + mc * 4), msrc + qrow * a.qb_cap + jt * 128 + mc * 4,
                           true);
                if (ptid == 0)
                    cp_async16(smem_u32(tflags + s * 4), a.qb_flags + (qrow * (a.qb_cap / 128) + jt) * 4, true);
            }
            cp_async_arrive_noinc(&bars[QB_MFULL + s]);
            if (ptid == 0) SKB_TRB(2, jt, 1);
            // rows of tile jt of one tensor into dst, completing on bar (97 arrivals)
            auto rows = [&](uint32_t dst, const __nv_bfloat16* src, const CUtensorMap* tm, uint64_t* bar) {
                if (jt < n_sel) {
                    kcur.template issue<false>(dst, src, b, h, a.L, a.H, pw, lane);
                    cp_async_arrive_noinc(bar);
                    if (ptid == 0) mbar_arrive(bar);
                } else {
                    if (ptid == 0) {
                        mbar_expect_tx(bar, 128 * D * 2);
#pragma unroll
                        for (int at = 0; at < kAtoms; ++at)
                            tma_load_3d(dst + at * 128 * 128, tm, h * D + at * 64, jw0 + (jt - n_sel) * 128, b, bar);
                    }
                    mbar_arrive(bar);
                }
            };
            if (jt >= kNS) mbar_wait(&bars[QB_KVEMPTY + s], ((jt - kNS) / kNS) & 1);
            if (ptid == 0) SKB_TRB(2, jt, 2);
            rows(sbase + SM::kK + s * SM::kKT, a.k, &a.tm_k128, &bars[QB_KVFULL + s]);
            const int vs = jt % kNV;
            if (jt >= kNV) mbar_wait(&bars[QB_VEMPTY + vs], ((jt - kNV) / kNV) & 1);
            rows(sbase + SM::kV + vs * SM::kKT, a.v, &a.tm_v128, &bars[QB_VFULL + vs]);
            if (jt + 1 < n_sel) kcur.fetch(pw, lane, [&](int r) { return __ldg(list + (jt + 1) * 128 + r); });
        }
    } else if (warp == kMmaWarp) {
        if (lane == 0) {
            constexpr uint32_t id_s = umma_idesc(128, 128, false, false);
            constexpr uint32_t id_dq = umma_idesc(128, D, false, true);
            mbar_wait(&bars[QB_QFULL], 0);
            mbar_wait(&bars[QB_DOFULL], 0);
            tc_after_sync();
            auto sdp = [&](int j) {  // S_j = Q K_j^T (TS), dP_j = dO V_j^T (SS)
                const int ks = j % kNS;
                SKB_TRB(3, j, 8);
                mbar_wait(&bars[QB_KVFULL + ks], (j / kNS) & 1);
                mbar_wait(&bars[QB_VFULL + (j % kNV)], (j / kNV) & 1);
                SKB_TRB(3, j, 0);
                fence_proxy_async();  // cp.async (generic proxy) rows -> tensor core reads
                if (j >= 1) mbar_wait(&bars[QB_SEMPTY], (j - 1) & 1);
                tc_after_sync();
                const uint32_t kb = sbase + SM::kK + ks * SM::kKT, vb = sbase + SM::kV + (j % kNV) * SM::kKT;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    umma_f16_ts(tS, tQ + kk * 8, desc_kmajor(kb, 128, kk), id_s, kk > 0 ? 1u : 0u);
                    umma_f16(tP, desc_kmajor(sbase + SM::kDO, 128, kk), desc_kmajor(vb, 128, kk), id_s,
                             kk > 0 ? 1u : 0u);
                }
                umma_commit(&bars[QB_SFULL]);
                umma_commit(&bars[QB_VEMPTY + (j % kNV)]);
                SKB_TRB(3, j, 1);
            };
            auto dq = [&](int j) {  // dQ += dS_j K_j (TS)
                const int ks = j % kNS;
                mbar_wait(&bars[QB_DSFULL], j & 1);
                SKB_TRB(3, j, 2);
                tc_after_sync();
                const uint32_t kb = sbase + SM::kK + ks * SM::kKT;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_f16_ts(tDQ, tDS + kk * 8, desc_mnmajor(kb, 128, kk), id_dq, (j > 0 || kk > 0) ? 1u : 0u);
                umma_commit(&bars[QB_DSEMPTY]);
                umma_commit(&bars[QB_KVEMPTY + ks]);
            };
            sdp(0);
            for (int jt = 0; jt < n; ++jt) {
                if (jt + 1 < n) sdp(jt + 1);  // overlaps the math on tile jt
                dq(jt);
            }
            umma_commit(&bars[QB_DQDONE]);
        }
        __syncwarp();
    } else if (warp < kProdWarp0) {
        // query rows: two math warpgroups, each owning 64 of the 128 key columns
        const int hf = warp >> 2;
        const int r = ((warp & 3) << 5) | lane;
        const int i = i0 + r;
        const int t = i - a.w;
        const float tau_i = (t >= 0 && a.R1 > 0) ? a.tauf[bl + t] : -INFINITY;
        const int lo_win = max(i - a.w + 1, 0);
        const int64_t hl = ((int64_t)b * a.H + h) * a.L;
        const float nlse2 = i < a.L ? -a.lse2[hl + i] : -INFINITY;  // i >= L: every p = 0
        const float dlt = i < a.L ? a.delta[hl + i] : 0.f;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sl2 = a.scale_log2;
        const float2 sl22 = make_float2(sl2, sl2), nl2 = make_float2(nlse2, nlse2), ndl = make_float2(-dlt, -dlt);
        const int c0 = hf * 64;
        if (hf == 0) {  // this row of Q -> TMEM: the A operand of S
            const __nv_bfloat16* src = a.q + ((bl + (i < a.L ? i : 0)) * a.H + h) * D;
            uint32_t wq[D / 2];
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
                uint4 x = make_uint4(0u, 0u, 0u, 0u);
                if (i < a.L) x = *reinterpret_cast<const uint4*>(src + c * 8);
                wq[4 * c] = x.x, wq[4 * c + 1] = x.y, wq[4 * c + 2] = x.z, wq[4 * c + 3] = x.w;
            }
#pragma unroll
            for (int c = 0; c < D / 64; ++c) tmem_st32u(tQ + lane_off + c * 32, wq + c * 32);
            tmem_wait_st();
            tc_before_sync();
            mbar_arrive(&bars[QB_QFULL]);
        }
        float rsum = 0.f;
        for (int jt = 0; jt < n; ++jt) {
            const bool is_sel = jt < n_sel;
            const int ks = jt % kNS;
            if (lane == 0 && (warp & 3) == 0) SKB_TRB(hf, jt, 9);
            mbar_wait(&bars[QB_SFULL], jt & 1);
            if (is_sel) mbar_wait(&bars[QB_MFULL + ks], (jt / kNS) & 1);
            if (lane == 0 && (warp & 3) == 0) SKB_TRB(hf, jt, 0);
            tc_after_sync();
            float sv[64], dp[64];
            tmem_ld32(tS + lane_off + c0, sv);
            tmem_ld32(tS + lane_off + c0 + 32, sv + 32);
            tmem_ld32(tP + lane_off + c0, dp);
            tmem_ld32(tP + lane_off + c0 + 32, dp + 32);
            tmem_wait_ld();
            tc_before_sync();
            mbar_arrive(&bars[QB_SEMPTY]);  // S/dP of the next tile may overwrite now
            bool plain = true;
            if (is_sel) {
                const int* mk = meta + (ks * 3) * 128 + c0;
                const int* ml = mk + 128;
                const float* mu = reinterpret_cast<const float*>(mk + 256);
                const int fl = tflags[ks * 4];
                if (!(fl & 1)) {  // per-key interval mask j <= t < leave_j: (unsigned)(t - j) < leave_j - j
#pragma unroll
                    for (int c = 0; c < 64; c += 4) {
                        const int4 kj = *reinterpret_cast<const int4*>(mk + c);
                        const int4 ex = *reinterpret_cast<const int4*>(ml + c);
                        sv[c + 0] = ((unsigned)(t - kj.x) < (unsigned)ex.x) ? sv[c + 0] : -INFINITY;
                        sv[c + 1] = ((unsigned)(t - kj.y) < (unsigned)ex.y) ? sv[c + 1] : -INFINITY;
                        sv[c + 2] = ((unsigned)(t - kj.z) < (unsigned)ex.z) ? sv[c + 2] : -INFINITY;
                        sv[c + 3] = ((unsigned)(t - kj.w) < (unsigned)ex.w) ? sv[c + 3] : -INFINITY;
                    }
                }
                if (!(fl & 2)) {  // fractional gates present
                    plain = false;
#pragma unroll
                    for (int c = 0; c < 64; c += 4) {
                        const float4 uu = *reinterpret_cast<const float4*>(mu + c);
                        const float ua[4] = {uu.x, uu.y, uu.z, uu.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float g = __saturatef(ua[e] - tau_i);
                            const float raw = sv[c + e];
                            const float kap = KEY_SOFT ? g : 1.f;
                            // masked logits are -inf: keep them -inf under a zero gate
                            const float x = (KEY_SOFT && raw == -INFINITY) ? raw : raw * kap;
                            const float p = ex2(fmaf(x, sl2, nlse2));
                            const float wv = a.mask_st ? 1.f : g;
                            const float cc = p * fmaf(wv, dp[c + e], -dlt);
                            float gm = p * dp[c + e];
                            if (KEY_SOFT) gm += a.scale * cc * (raw == -INFINITY ? 0.f : raw);
                            rsum += (g > 0.f && g < 1.f) ? gm : 0.f;
                            dp[c + e] = cc * kap;
                        }
                    }
                }
            } else {
                const int kb = jw0 + (jt - n_sel) * 128 + c0;
                const int cmin = lo_win - kb;
                const int cmax = i - kb;
                if (__any_sync(0xffffffffu, cmin > 0 || cmax < 63)) {
#pragma unroll
                    for (int c = 0; c < 64; ++c) sv[c] = (c >= cmin && c <= cmax) ? sv[c] : -INFINITY;
                }
            }
            if (plain) {  // all gates 1: plain softmax backward, packed fp32x2
#pragma unroll
                for (int c = 0; c < 64; c += 2) {
                    float2 x = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, nl2);
                    if ((c & 7) == 6 && kDqPoly) {  // one pair in four on the FMA pipe (MUFU relief)
                        x = ex2_poly2(x);
                    } else {
                        x.x = ex2(x.x);
                        x.y = ex2(x.y);
                    }
                    const float2 d = __fmul2_rn(x, __fadd2_rn(make_float2(dp[c], dp[c + 1]), ndl));
                    dp[c] = d.x;
                    dp[c + 1] = d.y;
                }
            }
            // dS -> TMEM (packed bf16x2), once dQ of the previous tile has read the buffer
            if (jt >= 1) mbar_wait(&bars[QB_DSEMPTY], (jt - 1) & 1);
            tc_after_sync();
            {
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(dp[2 * e], dp[2 * e + 1]);
                tmem_st16u(tDS + lane_off + hf * 32, pk);
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(dp[32 + 2 * e], dp[33 + 2 * e]);
                tmem_st16u(tDS + lane_off + hf * 32 + 16, pk);
                tmem_wait_st();
            }
            tc_before_sync();
            if (lane == 0 && (warp & 3) == 0) SKB_TRB(hf, jt, 4);
            mbar_arrive(&bars[QB_MEMPTY + ks]);
            mbar_arrive(&bars[QB_DSFULL]);
        }
        mbar_wait(&bars[QB_DQDONE], 0);
        if (lane == 0 && (warp & 3) == 0) SKB_TRB(hf, 31, 5);
        tc_after_sync();
        if (i < a.L && t >= 0 && a.R1 > 0 && rsum != 0.f) atomicAdd(a.rowsum + bl + t, (double)rsum);
        __nv_bfloat16* orow = a.dq + ((bl + (i < a.L ? i : 0)) * a.H + h) * D + hf * (D / 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
            float x[32];
            tmem_ld32(tDQ + lane_off + hf * (D / 2) + c * 32, x);
            tmem_wait_ld();
            if (i < a.L) {
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    uint4 pk;
                    pk.x = pack_bf16(x[e] * a.scale, x[e + 1] * a.scale);
                    pk.y = pack_bf16(x[e + 2] * a.scale, x[e + 3] * a.scale);
                    pk.z = pack_bf16(x[e + 4] * a.scale, x[e + 5] * a.scale);
                    pk.w = pack_bf16(x[e + 6] * a.scale, x[e + 7] * a.scale);
                    *reinterpret_cast<uint4*>(orow + c * 32 + e) = pk;
                }
            }
        }
        if (lane == 0 && (warp & 3) == 0) SKB_TRB(hf, 31, 6);
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

// NQ math warpgroups (2 or 4) each own 128/NQ of a tile's 128 key columns; with
// four, every SMSP holds four math warps (the per-tile math is latency-bound
// with two: TMEM loads, MUFU and the dependent packing hide better).
template <int D, bool KEY_SOFT, int NQ>
__global__ void __launch_bounds__((4 * NQ + 4) * 32, 1) k_bwd_dq_p(const __grid_constant__ BwdArgs a) {
    constexpr int kMW = 4 * NQ;          // math warps
    constexpr int kMT = kMW * 32;        // math threads
    constexpr int kPW0 = kMW;            // first producer warp
    constexpr int kMMA = kMW + 3;        // the MMA warp
    constexpr int kColsT = 128 / NQ;     // key columns per math thread
    constexpr int kQW = D / (2 * NQ);    // 32-bit words of Q per math thread (its share of the row)
    static_assert(kQW == 16 || kQW == 32, "Q share");
    using SM = QSmem<D>;
    static_assert(QB_DQEMPTY < SM::kNumBars, "barrier slots");
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    int* meta = reinterpret_cast<int*>(smem + SM::kMeta);
    int* tflags = reinterpret_cast<int*>(smem + SM::kFlags);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SKB_TRACE_DQP  // tiles of items 6.. of the CTA (tools/trace_dqp.py)
#define TRQ(role, jj, ev) \
    if ((jj) >= tr0) SKB_TRB(role, (jj) - tr0, ev)
#else
#define TRQ(role, jj, ev) \
    do {                  \
    } while (0)
#endif
    const int n_win = (a.w + 127 + 127) / 128;
    const int nitems = a.nqb * a.H * a.B;
    // work item wi -> (query tile fastest, head, sequence)
    struct Item {
        int b, h, i0, n_sel, n, jw0;
        int64_t bl, qrow;
    };
    auto item = [&](int wi) {
        Item t;
        const int qb = wi % a.nqb, bh = wi / a.nqb;
        t.h = bh % a.H;
        t.b = bh / a.H;
        t.bl = (int64_t)t.b * a.L;
        t.qrow = (int64_t)t.b * a.nqb + qb;
        t.i0 = qb * 128;
        const int cnt = (a.R1 > 0) ? __ldg(a.qb_count + t.qrow) : 0;
        t.n_sel = (cnt + 127) / 128;
        t.n = t.n_sel + n_win;
        t.jw0 = t.i0 - a.w + 1;
        return t;
    };

    if (threadIdx.x == 0) {
        mbar_init(&bars[QB_QFULL], kMT);
        mbar_init(&bars[QB_DOFULL], 1);
        for (int s = 0; s < kNS; ++s) {
            mbar_init(&bars[QB_KVFULL + s], kProducers + 1);
            mbar_init(&bars[QB_KVEMPTY + s], 1);
            mbar_init(&bars[QB_MFULL + s], kProducers);
            mbar_init(&bars[QB_MEMPTY + s], kMT);
        }
        for (int s = 0; s < kNV; ++s) {
            mbar_init(&bars[QB_VFULL + s], kProducers + 1);
            mbar_init(&bars[QB_VEMPTY + s], 1);
        }
        mbar_init(&bars[QB_SFULL], 1);
        mbar_init(&bars[QB_SEMPTY], kMT);
        mbar_init(&bars[QB_DSFULL], kMT);
        mbar_init(&bars[QB_DSEMPTY], 1);
        mbar_init(&bars[QB_DQDONE], 1);
        mbar_init(&bars[QB_QDOEMPTY], 1);
        mbar_init(&bars[QB_DQEMPTY], kMT);
        mbar_fence_init();
    }
    if (warp == kMMA) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tQ = tmem, tDS = tmem + 64, tS = tmem + 128, tP = tmem + 256, tDQ = tmem + 384;

    if (warp >= kPW0 && warp < kMMA) {
        constexpr int kAtoms = D / 64;
        const int pw = warp - kPW0, ptid = threadIdx.x - kPW0 * 32;
        const int ma = ptid >> 5, mc = ptid & 31;  // metadata: array x 16-byte chunk (96 threads)
        const int* msrc = ma == 0 ? a.qb_list : ma == 1 ? a.qb_leave : reinterpret_cast<const int*>(a.qb_uf);
        int J = 0, it = 0, tr0 = 1 << 28;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
            const Item I = item(wi);
            if (it == 6) tr0 = J;
            const int b = I.b, h = I.h, n_sel = I.n_sel, n = I.n;
            const int* list = a.qb_list + I.qrow * a.qb_cap;
            RowKeys<D, 128> kcur;
            if (n_sel > 0) kcur.fetch(pw, lane, [&](int r) { return __ldg(list + r); });
            for (int jt = 0; jt < n; ++jt, ++J) {
                const int s = J % kNS;
                if (jt == min(1, n - 1) && ptid == 0) {
                    // dO of this item once the previous item's last dP is done
                    if (it > 0) mbar_wait(&bars[QB_QDOEMPTY], (it - 1) & 1);
                    mbar_expect_tx(&bars[QB_DOFULL], 128 * D * 2);
#pragma unroll
                    for (int at = 0; at < kAtoms; ++at)
                        tma_load_3d(sbase + SM::kDO + at * 128 * 128, &a.tm_do128, h * D + at * 64, I.i0, b,
                                    &bars[QB_DOFULL]);
                }
                if (J >= kNS) mbar_wait(&bars[QB_MEMPTY + s], ((J - kNS) / kNS) & 1);
                if (jt < n_sel) {
                    cp_async16(smem_u32(meta + (s * 3 + ma) * 128 + mc * 4),
                               msrc + I.qrow * a.qb_cap + jt * 128 + mc * 4, true);
                    if (ptid == 0)
                        cp_async16(smem_u32(tflags + s * 4), a.qb_flags + (I.qrow * (a.qb_cap / 128) + jt) * 4, true);
                }
                cp_async_arrive_noinc(&bars[QB_MFULL + s]);
                auto rows = [&](uint32_t dst, const __nv_bfloat16* src, const CUtensorMap* tm, uint64_t* bar) {
                    if (jt < n_sel) {
                        kcur.template issue<false>(dst, src, b, h, a.L, a.H, pw, lane);
                        cp_async_arrive_noinc(bar);
                        if (ptid == 0) mbar_arrive(bar);
                    } else {
                        if (ptid == 0) {
                            mbar_expect_tx(bar, 128 * D * 2);
#pragma unroll
                            for (int at = 0; at < kAtoms; ++at)
                                tma_load_3d(dst + at * 128 * 128, tm, h * D + at * 64, I.jw0 + (jt - n_sel) * 128, b,
                                            bar);
                        }
                        mbar_arrive(bar);
                    }
                };
                if (J >= kNS) mbar_wait(&bars[QB_KVEMPTY + s], ((J - kNS) / kNS) & 1);
                if (ptid == 0) TRQ(2, J, 2);
                rows(sbase + SM::kK + s * SM::kKT, a.k, &a.tm_k128, &bars[QB_KVFULL + s]);
                const int vs = J % kNV;
                if (J >= kNV) mbar_wait(&bars[QB_VEMPTY + vs], ((J - kNV) / kNV) & 1);
                rows(sbase + SM::kV + vs * SM::kKT, a.v, &a.tm_v128, &bars[QB_VFULL + vs]);
                if (jt + 1 < n_sel) kcur.fetch(pw, lane, [&](int r) { return __ldg(list + (jt + 1) * 128 + r); });
            }
        }
    } else if (warp == kMMA) {
        if (lane == 0) {
            constexpr uint32_t id_s = umma_idesc(128, 128, false, false);
            constexpr uint32_t id_dq = umma_idesc(128, D, false, true);
            int tr0 = 1 << 28;
            (void)tr0;
            auto sdp = [&](int J) {  // S_J = Q K_J^T (TS), dP_J = dO V_J^T (SS)
                const int ks = J % kNS;
                mbar_wait_fast(&bars[QB_KVFULL + ks], (J / kNS) & 1);
                mbar_wait_fast(&bars[QB_VFULL + (J % kNV)], (J / kNV) & 1);
                TRQ(3, J, 0);
                fence_proxy_async();  // cp.async (generic proxy) rows -> tensor core reads
                if (J >= 1) mbar_wait_fast(&bars[QB_SEMPTY], (J - 1) & 1);
                tc_after_sync();
                const uint32_t kb = sbase + SM::kK + ks * SM::kKT, vb = sbase + SM::kV + (J % kNV) * SM::kKT;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    umma_f16_ts(tS, tQ + kk * 8, desc_kmajor(kb, 128, kk), id_s, kk > 0 ? 1u : 0u);
                    umma_f16(tP, desc_kmajor(sbase + SM::kDO, 128, kk), desc_kmajor(vb, 128, kk), id_s,
                             kk > 0 ? 1u : 0u);
                }
                umma_commit(&bars[QB_SFULL]);
                umma_commit(&bars[QB_VEMPTY + (J % kNV)]);
                TRQ(3, J, 1);
            };
            auto dq = [&](int J, int jt, int itn) {  // dQ += dS_J K_J (TS)
                const int ks = J % kNS;
                mbar_wait_fast(&bars[QB_DSFULL], J & 1);
                TRQ(3, J, 2);
                if (jt == 0 && itn > 0) mbar_wait_fast(&bars[QB_DQEMPTY], (itn - 1) & 1);
                tc_after_sync();
                const uint32_t kb = sbase + SM::kK + ks * SM::kKT;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_f16_ts(tDQ, tDS + kk * 8, desc_mnmajor(kb, 128, kk), id_dq, (jt > 0 || kk > 0) ? 1u : 0u);
                umma_commit(&bars[QB_DSEMPTY]);
                umma_commit(&bars[QB_KVEMPTY + ks]);
            };
            int J = 0, it = 0;
            for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
                const Item I = item(wi);
                if (it == 6) tr0 = J;
                const int n = I.n;
                mbar_wait_fast(&bars[QB_QFULL], it & 1);
                TRQ(3, J, 3);
                mbar_wait_fast(&bars[QB_DOFULL], it & 1);
                TRQ(3, J, 4);
                tc_after_sync();
                sdp(J);
                if (n == 1) umma_commit(&bars[QB_QDOEMPTY]);
                for (int jt = 0; jt < n; ++jt) {
                    if (jt + 1 < n) {
                        sdp(J + jt + 1);  // overlaps the math on tile jt
                        if (jt + 2 == n) umma_commit(&bars[QB_QDOEMPTY]);  // Q / dO read for the last time
                    }
                    dq(J + jt, jt, it);
                }
                umma_commit(&bars[QB_DQDONE]);
                J += n;
            }
        }
        __syncwarp();
    } else if (warp < kPW0) {
        // query rows: two math warpgroups, each owning 64 of the 128 key columns
        const int hf = warp >> 2;
        const int r = ((warp & 3) << 5) | lane;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        // this row of Q -> TMEM (the A operand of S): warpgroup hf writes the
        // packed columns of its half of the row
        auto load_q = [&](const Item& I) {
            const int i = I.i0 + r;
            const __nv_bfloat16* src = a.q + ((I.bl + (i < a.L ? i : 0)) * a.H + I.h) * D + hf * (D / NQ);
            uint32_t wq[kQW];
#pragma unroll
            for (int c = 0; c < kQW / 4; ++c) {
                uint4 x = make_uint4(0u, 0u, 0u, 0u);
                if (i < a.L) x = *reinterpret_cast<const uint4*>(src + c * 8);
                wq[4 * c] = x.x, wq[4 * c + 1] = x.y, wq[4 * c + 2] = x.z, wq[4 * c + 3] = x.w;
            }
            if constexpr (kQW == 32) tmem_st32u(tQ + lane_off + hf * 32, wq);
            else tmem_st16u(tQ + lane_off + hf * 16, wq);
            tmem_wait_st();
            tc_before_sync();
            mbar_arrive(&bars[QB_QFULL]);
        };
        if ((int)blockIdx.x < nitems) load_q(item(blockIdx.x));
        int J = 0, it = 0, tr0 = 1 << 28;
        const bool trl = lane == 0 && (warp & 3) == 0;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
        const Item I = item(wi);
        if (it == 6) tr0 = J;
        const int b = I.b, h = I.h, n_sel = I.n_sel, n = I.n, jw0 = I.jw0;
        const int64_t bl = I.bl;
        const int i = I.i0 + r;
        if (wi + (int)gridDim.x < nitems) {  // this half of the next item's Q row, for load_q
            const Item N = item(wi + gridDim.x);
            const int ni = N.i0 + r;
            if (ni < a.L) {
                const char* src =
                    reinterpret_cast<const char*>(a.q + ((N.bl + ni) * a.H + N.h) * D + hf * (D / NQ));
#pragma unroll
                for (int c = 0; c < 2 * D / NQ; c += 128) prefetch_l2(src + c);
            }
        }
        const int t = i - a.w;
        const float tau_i = (t >= 0 && a.R1 > 0) ? a.tauf[bl + t] : -INFINITY;
        const int lo_win = max(i - a.w + 1, 0);
        const int64_t hl = ((int64_t)b * a.H + h) * a.L;
        const float nlse2 = i < a.L ? -a.lse2[hl + i] : -INFINITY;  // i >= L: every p = 0
        const float dlt = i < a.L ? a.delta[hl + i] : 0.f;
        const float sl2 = a.scale_log2;
        const float2 sl22 = make_float2(sl2, sl2), nl2 = make_float2(nlse2, nlse2), ndl = make_float2(-dlt, -dlt);
        const int c0 = hf * kColsT;
        float rsum = 0.f;
        for (int jt = 0; jt < n; ++jt, ++J) {
            const bool is_sel = jt < n_sel;
            const int ks = J % kNS;
            if (trl) TRQ(hf, J, 9);
            mbar_wait(&bars[QB_SFULL], J & 1);
            mbar_wait(&bars[QB_MFULL + ks], (J / kNS) & 1);  // every phase observed (window tiles too)
            if (trl) TRQ(hf, J, 0);
            tc_after_sync();
            float sv[kColsT], dp[kColsT];
#pragma unroll
            for (int c = 0; c < kColsT; c += 32) {
                tmem_ld32(tS + lane_off + c0 + c, sv + c);
                tmem_ld32(tP + lane_off + c0 + c, dp + c);
            }
            tmem_wait_ld();
            tc_before_sync();
            mbar_arrive(&bars[QB_SEMPTY]);  // S/dP of the next tile may overwrite now
            bool plain = true;
            if (is_sel) {
                const int* mk = meta + (ks * 3) * 128 + c0;
                const int* ml = mk + 128;
                const float* mu = reinterpret_cast<const float*>(mk + 256);
                const int fl = tflags[ks * 4];
                if (!(fl & 1)) {  // per-key interval mask j <= t < leave_j: (unsigned)(t - j) < leave_j - j
#pragma unroll
                    for (int c = 0; c < kColsT; c += 4) {
                        const int4 kj = *reinterpret_cast<const int4*>(mk + c);
                        const int4 ex = *reinterpret_cast<const int4*>(ml + c);
                        sv[c + 0] = ((unsigned)(t - kj.x) < (unsigned)ex.x) ? sv[c + 0] : -INFINITY;
                        sv[c + 1] = ((unsigned)(t - kj.y) < (unsigned)ex.y) ? sv[c + 1] : -INFINITY;
                        sv[c + 2] = ((unsigned)(t - kj.z) < (unsigned)ex.z) ? sv[c + 2] : -INFINITY;
                        sv[c + 3] = ((unsigned)(t - kj.w) < (unsigned)ex.w) ? sv[c + 3] : -INFINITY;
                    }
                }
                if (!(fl & 2)) {  // fractional gates present
                    plain = false;
                    if constexpr (!KEY_SOFT) {  // packed fp32x2 except gate saturation / support test
                        // the mask mode is uniform: one loop per mode (no per-element selects)
                        auto frac_loop = [&](auto mst_c) {
                            constexpr bool kMst = decltype(mst_c)::value;
                            float2 rs2 = make_float2(0.f, 0.f);
#pragma unroll
                            for (int c = 0; c < kColsT; c += 2) {
                                const float2 uu = *reinterpret_cast<const float2*>(mu + c);
                                const float g0 = __saturatef(uu.x - tau_i), g1 = __saturatef(uu.y - tau_i);
                                float2 p2 = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, nl2);
                                p2.x = ex2(p2.x);
                                p2.y = ex2(p2.y);
                                const float2 dp2 = make_float2(dp[c], dp[c + 1]);
                                const float2 cc2 = kMst ? __fmul2_rn(p2, __fadd2_rn(dp2, ndl))
                                                        : __fmul2_rn(p2, __ffma2_rn(make_float2(g0, g1), dp2, ndl));
                                // 0 < g < 1 <=> (bits(g) - 1) < bits(1.0) - 1 (g in [0, 1])
                                const float2 fr2 =
                                    make_float2((__float_as_uint(g0) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f,
                                                (__float_as_uint(g1) - 1u) < 0x3F7FFFFFu ? 1.f : 0.f);
                                rs2 = __ffma2_rn(__fmul2_rn(p2, dp2), fr2, rs2);
                                dp[c] = cc2.x;
                                dp[c + 1] = cc2.y;
                            }
                            rsum += rs2.x + rs2.y;
                        };
                        if (a.mask_st) frac_loop(std::true_type{});
                        else frac_loop(std::false_type{});
                    } else {
#pragma unroll
                    for (int c = 0; c < kColsT; c += 4) {
                        const float4 uu = *reinterpret_cast<const float4*>(mu + c);
                        const float ua[4] = {uu.x, uu.y, uu.z, uu.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float g = __saturatef(ua[e] - tau_i);
                            const float raw = sv[c + e];
                            const float kap = KEY_SOFT ? g : 1.f;
                            // masked logits are -inf: keep them -inf under a zero gate
                            const float x = (KEY_SOFT && raw == -INFINITY) ? raw : raw * kap;
                            const float p = ex2(fmaf(x, sl2, nlse2));
                            const float wv = a.mask_st ? 1.f : g;
                            const float cc = p * fmaf(wv, dp[c + e], -dlt);
                            float gm = p * dp[c + e];
                            if (KEY_SOFT) gm += a.scale * cc * (raw == -INFINITY ? 0.f : raw);
                            rsum += (g > 0.f && g < 1.f) ? gm : 0.f;
                            dp[c + e] = cc * kap;
                        }
                    }
                    }
                }
            } else {
                const int kb = jw0 + (jt - n_sel) * 128 + c0;
                const int cmin = lo_win - kb;
                const int cmax = i - kb;
                if (__any_sync(0xffffffffu, cmin > 0 || cmax < kColsT - 1)) {
#pragma unroll
                    for (int c = 0; c < kColsT; ++c) sv[c] = (c >= cmin && c <= cmax) ? sv[c] : -INFINITY;
                }
            }
            if (plain) {  // all gates 1: plain softmax backward, packed fp32x2
#pragma unroll
                for (int c = 0; c < kColsT; c += 2) {
                    float2 x = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl22, nl2);
                    if ((c & 7) == 6 && kDqPoly) {  // one pair in four on the FMA pipe (MUFU relief)
                        x = ex2_poly2(x);
                    } else {
                        x.x = ex2(x.x);
                        x.y = ex2(x.y);
                    }
                    const float2 d = __fmul2_rn(x, __fadd2_rn(make_float2(dp[c], dp[c + 1]), ndl));
                    dp[c] = d.x;
                    dp[c + 1] = d.y;
                }
            }
            // dS -> TMEM (packed bf16x2), once dQ of the previous tile has read the buffer
            if (J >= 1) mbar_wait(&bars[QB_DSEMPTY], (J - 1) & 1);
            tc_after_sync();
            {
                uint32_t pk[16];
#pragma unroll
                for (int part = 0; part < kColsT / 32; ++part) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(dp[32 * part + 2 * e], dp[32 * part + 2 * e + 1]);
                    tmem_st16u(tDS + lane_off + hf * (kColsT / 2) + part * 16, pk);
                }
                tmem_wait_st();
            }
            tc_before_sync();
            if (trl) TRQ(hf, J, 4);
            mbar_arrive(&bars[QB_MEMPTY + ks]);
            mbar_arrive(&bars[QB_DSFULL]);
        }
        // the next item's Q: the S MMAs of this item are complete (consumed above)
        if (wi + (int)gridDim.x < nitems) load_q(item(wi + gridDim.x));
        if (trl) TRQ(hf, J - 1, 5);
        mbar_wait(&bars[QB_DQDONE], it & 1);
        if (trl) TRQ(hf, J - 1, 6);
        tc_after_sync();
        if (i < a.L && t >= 0 && a.R1 > 0 && rsum != 0.f) atomicAdd(a.rowsum + bl + t, (double)rsum);
        __nv_bfloat16* orow = a.dq + ((bl + (i < a.L ? i : 0)) * a.H + h) * D + hf * (D / NQ);
        float xq[D / NQ];
#pragma unroll
        for (int c = 0; c < D / (32 * NQ); ++c) tmem_ld32(tDQ + lane_off + hf * (D / NQ) + c * 32, xq + c * 32);
        tmem_wait_ld();
        tc_before_sync();
        mbar_arrive(&bars[QB_DQEMPTY]);
        if (trl) TRQ(hf, J - 1, 7);
#pragma unroll
        for (int c = 0; c < D / (32 * NQ); ++c) {
            const float* x = xq + c * 32;
            if (i < a.L) {
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    uint4 pk;
                    pk.x = pack_bf16(x[e] * a.scale, x[e + 1] * a.scale);
                    pk.y = pack_bf16(x[e + 2] * a.scale, x[e + 3] * a.scale);
                    pk.z = pack_bf16(x[e + 4] * a.scale, x[e + 5] * a.scale);
                    pk.w = pack_bf16(x[e + 6] * a.scale, x[e + 7] * a.scale);
                    *reinterpret_cast<uint4*>(orow + c * 32 + e) = pk;
                }
            }
        }
        }
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == kMMA) tmem_dealloc<512>(tmem);
#undef TRQ
}

template <class K>
void set_smem(K kern, int bytes) {
    SKB_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

// dq = bf16(scale * dq32) (the fused passes accumulate dS K unscaled)
__global__ void __launch_bounds__(256) k_dq_convert(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                                    int64_t n8, float scale) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n8) return;
    const float4 x = reinterpret_cast<const float4*>(acc)[2 * i];
    const float4 y = reinterpret_cast<const float4*>(acc)[2 * i + 1];
    uint4 o;
    o.x = pack_bf16(x.x * scale, x.y * scale);
    o.y = pack_bf16(x.z * scale, x.w * scale);
    o.z = pack_bf16(y.x * scale, y.y * scale);
    o.w = pack_bf16(y.z * scale, y.w * scale);
    reinterpret_cast<uint4*>(dq)[i] = o;
}

// The fused-dQ backward (D = 128, SKB_BWD_FUSEDQ=1): dQ formed by the
// key-major passes instead of the query-major dQ pass. Measured slower at cfg3
// (bwd 4.16 vs 4.03 ms): the dQ^T read-back gates the
// next dP^T MMA into the same TMEM columns, the window pass loses a Q/dO ring
// stage to the dS^T tile, and the fp32 reductions (8 red.v4 per thread per
// tile) cost ~0.4 ms; it also makes dQ depend on the reduction order (not
// bit-reproducible across grid sizes). Kept for A/B; the default is the dQ
// pass. Chunk-wise training always takes the dQ pass: there the key-major
// passes clip a key's queries to its own chunk (dK/dV never cross a chunk
// start), while dQ and the gate-gradient row sums still collect from every
// attended key (proj/src/attention.cpp:228-234, 284-300).
// the selected pass on CTA pairs (D = 128), opt-in (SKB_BWD_PAIR=1): measured
// slower than the one-CTA pass (2.28 vs 1.69 ms at cfg3), see k_bwd_dkdv_sel_pair
inline bool sel_pair() {
    static const int on = getenv("SKB_BWD_PAIR") ? atoi(getenv("SKB_BWD_PAIR")) : 0;
    return on != 0;
}
// unified key-major pass for sequences whose ever-selected set is dense
// (SKB_BWD_UNI=0: the selected + window passes for every sequence)
inline bool uni_pass() {
    static const int on = getenv("SKB_BWD_UNI") ? atoi(getenv("SKB_BWD_UNI")) : 1;
    return on != 0;
}
inline bool fused_dq(int D, int chunk_len) {
    static const int fused = getenv("SKB_BWD_FUSEDQ") ? atoi(getenv("SKB_BWD_FUSEDQ")) : 0;
    return D == 128 && fused && chunk_len == 0;
}

template <int D, bool KS>
void launch_bwd(const BwdArgs& a0, const skb_attn_desc& d, cudaStream_t st) {
    constexpr bool kFQ = D == 128;
    BwdArgs a = a0;
    const bool fq = fused_dq(D, a.chunk_len);
    static const int persist_sel = getenv("SKB_SEL_PERSIST") ? atoi(getenv("SKB_SEL_PERSIST")) : 1;
    a.uni = (uni_pass() && !KS && !fq && persist_sel && !sel_pair() && a.chunk_len == 0 && a.R1 > 0 && a.T > 0) ? 1 : 0;
    static uint64_t attr = 0;
    if (first_on_device(&attr)) {
        set_smem(k_bwd_dkdv_tc<D, true, KS>, KSmem<D>::kAlloc);
        set_smem(k_bwd_dkdv_sel_tc<D, KS, false>, KSmem<D, kSelQS>::kAlloc);
        set_smem(k_bwd_dkdv_win_tc<D, false>, KWSmem<D>::kAlloc);
        set_smem(k_bwd_dkdv_win_tc<D, false, true>, KWSmem<D, 4, false, true>::kAlloc);
        if constexpr (kFQ) {
            set_smem(k_bwd_dkdv_sel_tc<D, KS, true>, KSmem<D, kQS, true>::kAlloc);
            set_smem(k_bwd_dkdv_win_tc<D, true>, KWSmem<D, 2, true>::kAlloc);
        }
        set_smem(k_bwd_dq_tc<D, KS>, QSmem<D>::kAlloc);
        set_smem(k_bwd_dq_p<D, KS, 2>, QSmem<D>::kAlloc);
        if constexpr (D == 128) set_smem(k_bwd_dq_p<D, KS, 4>, QSmem<D>::kAlloc);
    }
    const int64_t ndq = (int64_t)a.B * a.L * a.H * D;
    if (fq) SKB_CHECK_CUDA(cudaMemsetAsync(a.dq32, 0, (size_t)ndq * sizeof(float), st));
    if (a.R1 > 0 && a.T > 0) {
        static const int persist = getenv("SKB_SEL_PERSIST") ? atoi(getenv("SKB_SEL_PERSIST")) : 1;
        if (persist || fq) {
            const int ntk = (int)cdiv(a.L, 128);
            const int osm = kOrdCntBytes + std::min(a.T, kOrdMaxBk);
            static uint64_t oattr = 0;
            if (first_on_device(&oattr)) set_smem(k_sel_order, kOrdCntBytes + kOrdMaxBk);
            k_sel_order<<<(unsigned)a.B, kOrdThreads, osm, st>>>(a);
            SKB_CHECK_LAUNCH();
            k_sel_items<<<(unsigned)cdiv((int64_t)a.B * ntk * 32, 256), 256, 0, st>>>(a, ntk);
            SKB_CHECK_LAUNCH();
            if (a.uni) {  // dense sequences: window + selection in one key-major pass
                k_uni_items<<<dim3((unsigned)ntk, (unsigned)a.B), 128, 0, st>>>(a, ntk);
                SKB_CHECK_LAUNCH();
                const int ug = persist_grid((int64_t)ntk * d.heads * d.batch);
                static const int q128 = getenv("SKB_BWD_QTILE") ? atoi(getenv("SKB_BWD_QTILE")) : 0;  // 96 / 128: k_bwd_kmaj_q (measured slower)
                if (D == 128 && q128 == 96) {
                    static uint64_t kattr = 0;
                    if (first_on_device(&kattr)) set_smem(k_bwd_kmaj_q<96>, KQSmem<96>::kAlloc);
                    k_bwd_kmaj_q<96><<<ug, kThreads, KQSmem<96>::kAlloc, st>>>(a);
                } else if (D == 128 && q128 == 128) {
                    static uint64_t kattr = 0;
                    if (first_on_device(&kattr)) set_smem(k_bwd_kmaj_q<128>, KQSmem<128>::kAlloc);
                    k_bwd_kmaj_q<128><<<ug, kThreads, KQSmem<128>::kAlloc, st>>>(a);
                } else {
                    k_bwd_dkdv_win_tc<D, false, true><<<ug, kThreads, KWSmem<D, 4, false, true>::kAlloc, st>>>(a);
                }
                SKB_CHECK_LAUNCH();
            }
            const int64_t items = (int64_t)ntk * d.heads * d.batch;
            const int grid = persist_grid(items);
            if constexpr (kFQ) {
                if (fq) {
                    k_bwd_dkdv_sel_tc<D, KS, true><<<grid, kThreads, KSmem<D, kQS, true>::kAlloc, st>>>(a);
                } else if (sel_pair()) {
                    const int64_t items2 = cdiv(a.L, 256) * d.heads * d.batch;
                    const int npairs = (int)std::max<int64_t>(1, std::min<int64_t>(items2, persist_grid(items2 * 2) / 2));
                    static uint64_t pattr = 0;
                    if (first_on_device(&pattr)) set_smem(k_bwd_dkdv_sel_pair<D, KS>, PSmem<D>::kAlloc);
                    k_bwd_dkdv_sel_pair<D, KS><<<2 * npairs, kThreads, PSmem<D>::kAlloc, st>>>(a);
                } else {
                    k_bwd_dkdv_sel_tc<D, KS, false><<<grid, kThreads, KSmem<D, kSelQS>::kAlloc, st>>>(a);
                }
            } else {
                k_bwd_dkdv_sel_tc<D, KS, false><<<grid, kThreads, KSmem<D, kSelQS>::kAlloc, st>>>(a);
            }
        } else {
            dim3 gs((unsigned)cdiv(a.T, 128), (unsigned)d.heads, (unsigned)d.batch);
            k_bwd_dkdv_tc<D, true, KS><<<gs, kThreads, KSmem<D>::kAlloc, st>>>(a);
        }
        SKB_CHECK_LAUNCH();
    }
    {
        const int64_t items = cdiv(a.L, 128) * d.heads * d.batch;
        const int grid = persist_grid(items);
        if constexpr (kFQ) {
            if (fq) k_bwd_dkdv_win_tc<D, true><<<grid, kThreads, KWSmem<D, 2, true>::kAlloc, st>>>(a);
            else k_bwd_dkdv_win_tc<D, false><<<grid, kThreads, KWSmem<D>::kAlloc, st>>>(a);
        } else {
            k_bwd_dkdv_win_tc<D, false><<<grid, kThreads, KWSmem<D>::kAlloc, st>>>(a);
        }
        SKB_CHECK_LAUNCH();
    }
    if (fq) {
        k_dq_convert<<<(unsigned)cdiv(ndq / 8, 256), 256, 0, st>>>(a.dq32, a.dq, ndq / 8, a.scale);
        SKB_CHECK_LAUNCH();
        return;
    }
    static const int dq_persist = getenv("SKB_DQ_PERSIST") ? atoi(getenv("SKB_DQ_PERSIST")) : 1;
    if (dq_persist) {
        const int64_t items = (int64_t)a.nqb * d.heads * d.batch;
        const int grid = persist_grid(items);
        static const int quarters = getenv("SKB_DQ_QUARTERS") ? atoi(getenv("SKB_DQ_QUARTERS")) : 0;  // measured +1 %
        if (D == 128 && quarters) k_bwd_dq_p<D, KS, (D == 128 ? 4 : 2)><<<grid, 20 * 32, QSmem<D>::kAlloc, st>>>(a);
        else k_bwd_dq_p<D, KS, 2><<<grid, kThreads, QSmem<D>::kAlloc, st>>>(a);
    } else {
        dim3 gq((unsigned)a.nqb, (unsigned)d.heads, (unsigned)d.batch);
        k_bwd_dq_tc<D, KS><<<gq, kThreads, QSmem<D>::kAlloc, st>>>(a);
    }
    SKB_CHECK_LAUNCH();
}

}  // namespace

void run_attn_bwd_tc(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                     const void* o, const void* dout, const double* lse, const double* u,
                     const SelView& s, void* dq, void* dk, void* dv, double* rowsum,
                     double* colsum, void* ws, const BwdLayout& bl, cudaStream_t st) {
    (void)u;
    char* base = static_cast<char*>(ws);
    BwdArgs a{};
    {
        const int64_t HD = d.heads * d.head_dim;
        a.tm_q128 = tmap_rows3d(q, d.batch, d.seq_len, HD, 128);
        a.tm_do128 = tmap_rows3d(dout, d.batch, d.seq_len, HD, 128);
        a.tm_k64 = tmap_rows3d(k, d.batch, d.seq_len, HD, 64);
        a.tm_v64 = tmap_rows3d(v, d.batch, d.seq_len, HD, 64);
        a.tm_q64 = tmap_rows3d(q, d.batch, d.seq_len, HD, 64);
        a.tm_do64 = tmap_rows3d(dout, d.batch, d.seq_len, HD, 64);
        a.tm_q32 = tmap_rows3d(q, d.batch, d.seq_len, HD, 32);
        a.tm_q96 = tmap_rows3d(q, d.batch, d.seq_len, HD, 96);
        a.tm_do96 = tmap_rows3d(dout, d.batch, d.seq_len, HD, 96);
        a.tm_do32 = tmap_rows3d(dout, d.batch, d.seq_len, HD, 32);
        a.tm_k128 = tmap_rows3d(k, d.batch, d.seq_len, HD, 128);
        a.tm_v128 = tmap_rows3d(v, d.batch, d.seq_len, HD, 128);
        a.tm_dk_st = tmap_groups4d(dk, d.batch, d.seq_len, HD, (int)d.head_dim / 16);
        a.tm_dv_st = tmap_groups4d(dv, d.batch, d.seq_len, HD, (int)d.head_dim / 16);
    }
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.k = static_cast<const __nv_bfloat16*>(k);
    a.v = static_cast<const __nv_bfloat16*>(v);
    a.dout = static_cast<const __nv_bfloat16*>(dout);
    a.dq = static_cast<__nv_bfloat16*>(dq);
    a.dk = static_cast<__nv_bfloat16*>(dk);
    a.dv = static_cast<__nv_bfloat16*>(dv);
    a.dk_acc = reinterpret_cast<__nv_bfloat16*>(base + bl.dk_acc);
    a.dv_acc = reinterpret_cast<__nv_bfloat16*>(base + bl.dv_acc);
    float* lse2 = reinterpret_cast<float*>(base + bl.dq_acc);
    float* delta = lse2 + d.batch * d.heads * d.seq_len;
    a.lse2 = lse2;
    a.delta = delta;
    a.uf = s.uf;
    a.tauf = s.tauf;
    a.leave = s.leave;
    a.qb_count = s.qb_count;
    a.qb_list = s.qb_list;
    a.qb_leave = s.qb_leave;
    a.qb_uf = s.qb_uf;
    a.qb_flags = s.qb_flags;
    a.ever_count = s.ever_count;
    a.ever_list = s.ever_list;
    a.rowsum = rowsum;
    a.colsum = colsum;
    a.sel_items = reinterpret_cast<int2*>(base + bl.sel_items);
    a.dq32 = reinterpret_cast<float*>(base + bl.dq32);
    a.sel_order = reinterpret_cast<int*>(base + bl.sel_order);
    a.uni_hi = reinterpret_cast<int*>(base + bl.uni_hi);
    a.uni = 0;
    a.nqb = s.nqb;
    a.qb_cap = s.qb_cap;
    a.B = (int)d.batch;
    a.L = (int)d.seq_len;
    a.H = (int)d.heads;
    a.w = (int)d.window;
    a.T = std::max(0, a.L - a.w);
    a.R1 = (int)floor_k(d.k);
    const double scale = d.scale > 0.0 ? d.scale : 1.0 / std::sqrt((double)d.head_dim);
    a.scale = (float)scale;
    a.scale_log2 = (float)(scale * 1.4426950408889634);
    a.mask_st = d.mask_mode;
    a.chunk_len = (int)d.chunk_len;
    const int64_t rows = d.batch * d.seq_len * d.heads;
    const unsigned pg = (unsigned)cdiv(rows * (d.head_dim / 16), 256);  // k_bwd_prep: 2 x 16 B per thread
    if (d.head_dim == 128)
        k_bwd_prep<128><<<pg, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o), a.dout, lse, lse2, delta,
                                            a.B, a.L, a.H);
    else
        k_bwd_prep<64><<<pg, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o), a.dout, lse, lse2, delta,
                                           a.B, a.L, a.H);
    SKB_CHECK_LAUNCH();
    if (d.head_dim == 128) {
        if (d.key_mode) launch_bwd<128, true>(a, d, st);
        else launch_bwd<128, false>(a, d, st);
    } else {
        if (d.key_mode) launch_bwd<64, true>(a, d, st);
        else launch_bwd<64, false>(a, d, st);
    }
}

}  // namespace skb
