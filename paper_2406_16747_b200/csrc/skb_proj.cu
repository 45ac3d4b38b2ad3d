// Fused input projections + scoring GEMV (§8f row 2): the three projection
// GEMMs of forward_chunk (q|k|v = x Wq|Wk|Wv, proj/src/cache.cpp:204-206) as
// one hand-written tcgen05 GEMM over x, with the score raw = x . w_score
// (proj/include/sparsek/selection.hpp:72-74, called at proj/src/cache.cpp:
// 209-228) computed from the same shared-memory x tiles — x is read from HBM
// once for all four products.
//
// Persistent, one CTA per SM, work item = (128-row block of x, 256-column
// tile of [Wq | Wk | Wv]), column tile fastest so the CTAs in flight share
// their x rows in L2 and the weights (3 D^2 bf16) stay L2-resident.
// 320 threads:
//   warp 0      TMA producer: per 64-deep K step, the x tile (128 x 64) and
//               the weight tile (64 x 256, four 64-column boxes) into a
//               4-stage ring (48 KB per stage)
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer: D[128 x 256]
//               fp32 in TMEM, double-buffered across items (512 columns)
//   warps 2-5   epilogue: TMEM -> bf16 -> global rows, overlapping the next
//               item's MMAs
//   warps 6-9   score: for the row blocks whose first column tile the CTA
//               computes, thread r walks row r left to right in float64
//               (separate multiply and add: the reference's order, so raw is
//               bit-identical to skb_score_raw / the reference), streaming the
//               row from L2 (the GEMM's tile loads just brought it in) at its
//               own pace — the serial chain (4096 dependent adds at D = 4096)
//               is longer than the block's MMAs and must not hold the ring
#include <type_traits>

#include "skb_common.cuh"
#include "skb_internal.h"
#include "skb_tc.cuh"
#include "skb_tmap.h"

namespace skb {

void set_last_error(const char* msg);  // skb_capi.cu

namespace {

using namespace tc;

constexpr int kPM = 128, kPN = 256, kPK = 64;
constexpr int kPStages = 4;
constexpr int kPThreads = 320;
constexpr int kPEpiWarp0 = 2, kPScoreWarp0 = 6;

// Item -> (row block, column tile) in grouped raster order: column tiles in
// groups of kPGroup, row blocks inside a group, column tiles fastest. The items
// in flight (one per SM or pair) then touch ~kPGroup weight tiles and a few x
// row blocks — an L2-resident working set (the plain row-major order re-read
// the 96 MB of weights from HBM on every sweep). The first group holds the
// Wq tiles that carry the score, so the raw scores of every row block are
// published early for the streaming Welford.
constexpr int kPGroup = 16;
__device__ __forceinline__ void raster(int wi, int nmb, int ntn, int& mb, int& tn) {
    const int per = nmb * kPGroup;
    const int grp = wi / per, rem = wi % per;
    const int gw = min(kPGroup, ntn - grp * kPGroup);  // tiles in this group (the last may be short)
    mb = rem / gw;
    tn = grp * kPGroup + rem % gw;
}

struct ProjArgs {
    CUtensorMap tm_x;     // {K cols, M rows}, box {64, 128}
    CUtensorMap tm_w[3];  // {N cols, K rows}, box {64, 64}
    __nv_bfloat16* out[3];
    const __nv_bfloat16* x;
    const double* w_score;  // null: no score
    double* raw;
    int* ready;  // optional: ready[mb] = 1 once raw of row block mb is stored (a streaming consumer polls it)
    int M, K, N;  // N = d_model (per output); K = d_model
};

struct PSmem {
    static constexpr int kA = kPM * kPK * 2;  // 16 KB
    static constexpr int kB = kPK * kPN * 2;  // 32 KB
    static constexpr int kStage = kA + kB;
    static constexpr int kBar = kPStages * kStage;
    static constexpr int kNumBars = 2 * kPStages + 4;
    static constexpr int kTmemSlot = kBar + kNumBars * 8;
    static constexpr int kAlloc = kTmemSlot + 16 + 1024;
};
enum { PB_FULL = 0, PB_EMPTY = kPStages, PB_ACCFULL = 2 * kPStages, PB_ACCEMPTY = 2 * kPStages + 2 };

// raw = x[row, :] . w_score, left to right in float64 with separate multiply
// and add (the reference's order: bit-identical to skb_score_raw).
__device__ __forceinline__ double row_score(const ProjArgs& a, int row) {
    // 64 elements (8 x 16 B) in flight ahead of the chain: the row streams from
    // L2 at ~800-cycle latency while 64 dependent adds take longer than that
    const uint4* xr = reinterpret_cast<const uint4*>(a.x + (int64_t)row * a.K);
    const int n8 = a.K / 8;
    double acc = 0.0;
    uint4 nxt[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) nxt[j] = j < n8 ? __ldg(xr + j) : make_uint4(0, 0, 0, 0);
    for (int c0 = 0; c0 < n8; c0 += 8) {
        uint4 cur[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            cur[j] = nxt[j];
            if (c0 + 8 + j < n8) nxt[j] = __ldg(xr + c0 + 8 + j);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (c0 + j >= n8) break;
            const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&cur[j]);
            const double* w = a.w_score + (c0 + j) * 8;
            double prod[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) prod[q] = __dmul_rn((double)__bfloat162float(e[q]), __ldg(w + q));
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, prod[q]);
        }
    }
    return acc;
}
// 128-row block `blk` of raw is stored: publish it to the streaming Welford
__device__ __forceinline__ void publish(const ProjArgs& a, int blk, int r) {
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (r == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(a.ready + blk), "r"(1) : "memory");
    }
}

__global__ void __launch_bounds__(kPThreads, 1) k_proj_score(const __grid_constant__ ProjArgs a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PSmem::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + PSmem::kTmemSlot);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nmb = (a.M + kPM - 1) / kPM;
    const int ntn = 3 * (a.N / kPN);  // column tiles over [Wq | Wk | Wv]
    const int nitems = nmb * ntn;
    const int nk = a.K / kPK;
    const bool score = a.w_score != nullptr;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPStages; ++s) {
            mbar_init(&bars[PB_FULL + s], 1);
            mbar_init(&bars[PB_EMPTY + s], 1);  // the MMA commit
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[PB_ACCFULL + s], 1);
            mbar_init(&bars[PB_ACCEMPTY + s], 128);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int g = 0;
            for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x) {
                int mb, tn;
            raster(wi, nmb, ntn, mb, tn);
                const int t = tn / (a.N / kPN), n0 = (tn % (a.N / kPN)) * kPN;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int s = g % kPStages;
                    if (g >= kPStages) mbar_wait(&bars[PB_EMPTY + s], ((g - kPStages) / kPStages) & 1);
                    const uint32_t st = sbase + s * PSmem::kStage;
                    mbar_expect_tx(&bars[PB_FULL + s], PSmem::kStage);
                    tma_load_3d(st, &a.tm_x, kb * kPK, mb * kPM, 0, &bars[PB_FULL + s]);
#pragma unroll
                    for (int j = 0; j < kPN / 64; ++j)
                        tma_load_3d(st + PSmem::kA + j * (kPK * 128), &a.tm_w[t], n0 + j * 64, kb * kPK, 0,
                                    &bars[PB_FULL + s]);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc(kPM, kPN, false, true);
            int g = 0, it = 0;
            for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
                const int ab = it & 1;
                if (it >= 2) mbar_wait(&bars[PB_ACCEMPTY + ab], ((it - 2) >> 1) & 1);
                tc_after_sync();
                const uint32_t acc = tmem + ab * kPN;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int s = g % kPStages;
                    mbar_wait(&bars[PB_FULL + s], (g / kPStages) & 1);
                    tc_after_sync();
                    const uint32_t st = sbase + s * PSmem::kStage;
#pragma unroll
                    for (int kk = 0; kk < kPK / 16; ++kk)
                        umma_f16(acc, desc_kmajor(st, kPM, kk), desc_mnmajor(st + PSmem::kA, kPK, kk), idesc,
                                 (kb > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&bars[PB_EMPTY + s]);
                }
                umma_commit(&bars[PB_ACCFULL + ab]);
            }
        }
        __syncwarp();
    } else if (warp < kPScoreWarp0) {
        // epilogue: warp w reads TMEM lanes (w % 4) * 32 .. + 32 = tile rows
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        int it = 0;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
            int mb, tn;
            raster(wi, nmb, ntn, mb, tn);
            const int t = tn / (a.N / kPN), n0 = (tn % (a.N / kPN)) * kPN;
            const int ab = it & 1;
            mbar_wait(&bars[PB_ACCFULL + ab], (it >> 1) & 1);
            tc_after_sync();
            const int row = mb * kPM + r;
            __nv_bfloat16* dst = a.out[t] + (int64_t)row * a.N + n0;
#pragma unroll 1
            for (int c = 0; c < kPN / 32; ++c) {
                float v[32];
                tmem_ld32(tmem + lane_off + ab * kPN + c * 32, v);
                tmem_wait_ld();
                if (c == kPN / 32 - 1) {  // the whole accumulator is in registers: hand it back
                    tc_before_sync();
                    mbar_arrive(&bars[PB_ACCEMPTY + ab]);
                }
                if (row < a.M) {
                    uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        uint4 o;
                        o.x = pack_bf16(v[8 * e + 0], v[8 * e + 1]);
                        o.y = pack_bf16(v[8 * e + 2], v[8 * e + 3]);
                        o.z = pack_bf16(v[8 * e + 4], v[8 * e + 5]);
                        o.w = pack_bf16(v[8 * e + 6], v[8 * e + 7]);
                        d4[e] = o;
                    }
                }
            }
        }
    } else {
        // score: thread r owns row r of the row blocks whose first column tile
        // this CTA computes; it streams the row from global memory (L2-hot:
        // the GEMM's own loads just brought it in) at its own pace, so the
        // serial float64 chain never holds a stage of the GEMM's ring
        const int r = threadIdx.x - kPScoreWarp0 * 32;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x) {
            int mb, tn;
            raster(wi, nmb, ntn, mb, tn);
            if (!score || tn != 0) continue;
            const int row = mb * kPM + r;
            if (row < a.M) a.raw[row] = row_score(a, row);
            if (a.ready) publish(a, mb, r);
        }
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ CTA pair
// The same GEMM on CTA pairs (cta_group::2): a cluster of two CTAs on one TPC
// computes a 256 x 256 tile with M = 256 tcgen05.mma issued by the even CTA;
// each CTA stages its own 128 rows of x and its own 128 columns of the weight
// tile (A split by rows, B by columns), so each SM moves half the weight
// bytes of the one-CTA kernel per flop — the shape the library GEMM uses
// (and the one that keeps the SM clocks up under the power cap).
//   FULL(s)    even CTA only: both CTAs' TMA loads complete_tx on it
//   EMPTY(s)   per CTA: the multicast MMA commit
//   ACCFULL(2) per CTA: multicast commit of an item's last MMAs
//   ACCEMPTY(2) even CTA: 128 epilogue arrivals from each CTA
constexpr int kP2Stages = 6;
constexpr int kP2Threads = 320;

struct P2Smem {
    static constexpr int kA = 128 * kPK * 2;  // this CTA's 128 rows, 16 KB
    static constexpr int kB = kPK * 128 * 2;  // this CTA's 128 weight columns, 16 KB
    static constexpr int kStage = kA + kB;
    static constexpr int kBar = kP2Stages * kStage;
    static constexpr int kNumBars = 2 * kP2Stages + 4;
    static constexpr int kTmemSlot = kBar + kNumBars * 8;
    static constexpr int kAlloc = kTmemSlot + 16 + 1024;
};
enum { P2_FULL = 0, P2_EMPTY = kP2Stages, P2_ACCFULL = 2 * kP2Stages, P2_ACCEMPTY = 2 * kP2Stages + 2 };

__global__ void __launch_bounds__(kP2Threads, 1) k_proj_score2(const __grid_constant__ ProjArgs a) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P2Smem::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P2Smem::kTmemSlot);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int nmb = (a.M + 255) / 256;
    const int ntn = 3 * (a.N / kPN);
    const int nitems = nmb * ntn;
    const int nk = a.K / kPK;
    const bool score = a.w_score != nullptr;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kP2Stages; ++s) {
            mbar_init(&bars[P2_FULL + s], 1);
            mbar_init(&bars[P2_EMPTY + s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[P2_ACCFULL + s], 1);
            mbar_init(&bars[P2_ACCEMPTY + s], 256);
        }
        mbar_fence_init();
    }
    if (warp == 1) {  // both CTAs allocate the pair's accumulator columns
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_before_sync();
    cluster_sync_all();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int g = 0;
            for (int wi = pair; wi < nitems; wi += npairs) {
                int mb, tn;
            raster(wi, nmb, ntn, mb, tn);
                const int t = tn / (a.N / kPN), n0 = (tn % (a.N / kPN)) * kPN;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int s = g % kP2Stages;
                    if (g >= kP2Stages) mbar_wait(&bars[P2_EMPTY + s], ((g - kP2Stages) / kP2Stages) & 1);
                    const uint32_t st = sbase + s * P2Smem::kStage;
                    const uint32_t full = peer_addr(smem_u32(&bars[P2_FULL + s]), 0);
                    if (leader) mbar_expect_tx(&bars[P2_FULL + s], 2 * P2Smem::kStage);
                    tma_load_3d_pair(st, &a.tm_x, kb * kPK, mb * 256 + (int)rank * 128, 0, full);
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        tma_load_3d_pair(st + P2Smem::kA + j * (kPK * 128), &a.tm_w[t], n0 + (int)rank * 128 + j * 64,
                                         kb * kPK, 0, full);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (leader && lane == 0) {
            constexpr uint32_t idesc = umma_idesc(256, kPN, false, true);
            int g = 0, it = 0;
            for (int wi = pair; wi < nitems; wi += npairs, ++it) {
                const int ab = it & 1;
                if (it >= 2) mbar_wait(&bars[P2_ACCEMPTY + ab], ((it - 2) >> 1) & 1);
                tc_after_sync();
                const uint32_t acc = tmem + ab * kPN;
                for (int kb = 0; kb < nk; ++kb, ++g) {
                    const int s = g % kP2Stages;
                    mbar_wait(&bars[P2_FULL + s], (g / kP2Stages) & 1);
                    tc_after_sync();
                    const uint32_t st = sbase + s * P2Smem::kStage;
#pragma unroll
                    for (int kk = 0; kk < kPK / 16; ++kk)
                        umma_f16_pair(acc, desc_kmajor(st, 128, kk), desc_mnmajor(st + P2Smem::kA, kPK, kk), idesc,
                                      (kb > 0 || kk > 0) ? 1u : 0u);
                    umma_commit_pair(&bars[P2_EMPTY + s]);
                }
                umma_commit_pair(&bars[P2_ACCFULL + ab]);
            }
        }
        __syncwarp();
    } else if (warp < kPScoreWarp0) {
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        int it = 0;
        for (int wi = pair; wi < nitems; wi += npairs, ++it) {
            int mb, tn;
            raster(wi, nmb, ntn, mb, tn);
            const int t = tn / (a.N / kPN), n0 = (tn % (a.N / kPN)) * kPN;
            const int ab = it & 1;
            mbar_wait(&bars[P2_ACCFULL + ab], (it >> 1) & 1);
            tc_after_sync();
            const int row = mb * 256 + (int)rank * 128 + r;
            __nv_bfloat16* dst = a.out[t] + (int64_t)row * a.N + n0;
#pragma unroll 1
            for (int c = 0; c < kPN / 32; ++c) {
                float v[32];
                tmem_ld32(tmem + lane_off + ab * kPN + c * 32, v);
                tmem_wait_ld();
                if (c == kPN / 32 - 1) {  // accumulator drained: release it to the even CTA's MMA thread
                    tc_before_sync();
                    mbar_arrive_cluster(peer_addr(smem_u32(&bars[P2_ACCEMPTY + ab]), 0));
                }
                if (row < a.M) {
                    uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        uint4 o;
                        o.x = pack_bf16(v[8 * e + 0], v[8 * e + 1]);
                        o.y = pack_bf16(v[8 * e + 2], v[8 * e + 3]);
                        o.z = pack_bf16(v[8 * e + 4], v[8 * e + 5]);
                        o.w = pack_bf16(v[8 * e + 6], v[8 * e + 7]);
                        d4[e] = o;
                    }
                }
            }
        }
    } else {
        const int r = threadIdx.x - kPScoreWarp0 * 32;
        for (int wi = pair; wi < nitems; wi += npairs) {
            int mb, tn;
            raster(wi, nmb, ntn, mb, tn);
            if (!score || tn != 0) continue;
            const int row = mb * 256 + (int)rank * 128 + r;
#if defined(SKB_PROJ_EXP) && SKB_PROJ_EXP == 1
            if (row < a.M) a.raw[row] = 0.0;  // experiment: no chain (timing only)
#else
            if (row < a.M) a.raw[row] = row_score(a, row);
#endif
            if (a.ready) publish(a, mb * 2 + (int)rank, r);
        }
    }
    tc_before_sync();
    cluster_sync_all();
    tc_after_sync();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace

bool proj_supported(int64_t M, int64_t D) { return M >= 1 && D >= kPN && D % kPN == 0; }

void run_proj_score(int64_t M, int64_t D, const void* x, const void* wq, const void* wk, const void* wv,
                    const double* w_score, void* q, void* k, void* v, double* raw, int* ready, cudaStream_t st) {
    SKB_REQUIRE(proj_supported(M, D), SKB_ESHAPE, "proj: d_model must be a positive multiple of 256");
    SKB_REQUIRE(((uintptr_t)x & 15) == 0 && ((uintptr_t)wq & 15) == 0 && ((uintptr_t)wk & 15) == 0 &&
                    ((uintptr_t)wv & 15) == 0 && ((uintptr_t)q & 15) == 0 && ((uintptr_t)k & 15) == 0 &&
                    ((uintptr_t)v & 15) == 0,
                SKB_EARG, "proj: buffers must be 16-byte aligned");
    ProjArgs a{};
    a.tm_x = tmap_rows3d(x, 1, M, D, kPM);
    const void* ws[3] = {wq, wk, wv};
    for (int t = 0; t < 3; ++t) a.tm_w[t] = tmap_rows3d(ws[t], 1, D, D, kPK);
    a.out[0] = static_cast<__nv_bfloat16*>(q);
    a.out[1] = static_cast<__nv_bfloat16*>(k);
    a.out[2] = static_cast<__nv_bfloat16*>(v);
    a.x = static_cast<const __nv_bfloat16*>(x);
    a.w_score = w_score;
    a.raw = raw;
    a.ready = ready;
    a.M = (int)M;
    a.K = (int)D;
    a.N = (int)D;
    static uint64_t attr = 0;
    if (first_on_device(&attr)) {
        SKB_CHECK_CUDA(cudaFuncSetAttribute(k_proj_score, cudaFuncAttributeMaxDynamicSharedMemorySize, PSmem::kAlloc));
        SKB_CHECK_CUDA(cudaFuncSetAttribute(k_proj_score2, cudaFuncAttributeMaxDynamicSharedMemorySize, P2Smem::kAlloc));
    }
    static const int one_cta = getenv("SKB_PROJ_1CTA") ? atoi(getenv("SKB_PROJ_1CTA")) : 0;
    if (!one_cta) {  // CTA pairs (cta_group::2); `ready` is per 128-row block in both kernels
        const int64_t items = cdiv(M, 256) * 3 * (D / kPN);
        int pairs = (int)std::min<int64_t>(items, num_sms() / 2);
        static const int cap = getenv("SKB_MAX_CTAS") ? atoi(getenv("SKB_MAX_CTAS")) : 0;
        if (cap > 1) pairs = std::min(pairs, cap / 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(2 * std::max(pairs, 1)));
        cfg.blockDim = dim3(kP2Threads);
        cfg.dynamicSmemBytes = P2Smem::kAlloc;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SKB_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_proj_score2, a));
        SKB_CHECK_LAUNCH();
        return;
    }
    const int64_t items = cdiv(M, kPM) * 3 * (D / kPN);
    k_proj_score<<<persist_grid(items), kPThreads, PSmem::kAlloc, st>>>(a);
    SKB_CHECK_LAUNCH();
}

void run_score_finish_async(int64_t B, int64_t L, const skb_scoring& sc, const double* raw_in, const int* ready,
                            double* raw, double* u, double* mean, double* sdev, int* bad, cudaStream_t st);
int* score_bad_flag();
bool score_read_flag(const int* bad, cudaStream_t st);

// q|k|v = x W* and the complete score (raw, u, mean, sdev) of
// score_tokens: the fused GEMM on `st`; the Welford chain on a side stream,
// consuming each 128-row block of raw as soon as the GEMM publishes it, so
// the serial chain runs under the GEMM. Synchronises `st` (non-finite check).
void run_proj_score_fwd(int64_t B, int64_t L, int64_t D, const void* x, const void* wq, const void* wk,
                        const void* wv, const double* w_score, const skb_scoring& sc, void* q, void* k, void* v,
                        double* raw, double* u, double* mean, double* sdev, cudaStream_t st) {
    const int64_t M = B * L;
    if (!w_score) {  // scores idle (k = 0)
        run_proj_score(M, D, x, wq, wk, wv, nullptr, q, k, v, nullptr, nullptr, st);
        return;
    }
    SKB_REQUIRE(sc.slope_eps > 0.0, SKB_EARG, "ScoringParams: slope_eps must be positive");
    struct Slot {
        cudaStream_t side = nullptr;
        cudaEvent_t fork = nullptr, join = nullptr;
        int* ready = nullptr;
        int64_t cap = 0;
    };
    thread_local Slot slots[64];
    int dev = 0;
    SKB_CHECK_CUDA(cudaGetDevice(&dev));
    Slot& sl = slots[dev & 63];
    if (!sl.side) {
        SKB_CHECK_CUDA(cudaStreamCreateWithFlags(&sl.side, cudaStreamNonBlocking));
        SKB_CHECK_CUDA(cudaEventCreateWithFlags(&sl.fork, cudaEventDisableTiming));
        SKB_CHECK_CUDA(cudaEventCreateWithFlags(&sl.join, cudaEventDisableTiming));
    }
    const int64_t nmb = 2 * cdiv(M, 256);  // flags per 128-row block (both kernels)
    if (sl.cap < nmb) {
        if (sl.ready) SKB_CHECK_CUDA(cudaFree(sl.ready));
        SKB_CHECK_CUDA(cudaMalloc(&sl.ready, nmb * sizeof(int)));
        sl.cap = nmb;
    }
    int* bad = score_bad_flag();
    SKB_CHECK_CUDA(cudaMemsetAsync(sl.ready, 0, nmb * sizeof(int), st));
    SKB_CHECK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    const bool stream = sc.norm_mode != 0;
    if (stream) {  // the consumer's stream may not start before the flags are reset
        SKB_CHECK_CUDA(cudaEventRecord(sl.fork, st));
        SKB_CHECK_CUDA(cudaStreamWaitEvent(sl.side, sl.fork, 0));
    }
    // the producer GEMM is submitted before its polling consumer: streams may
    // share a hardware queue, and the GEMM never waits on the consumer, so
    // this order cannot deadlock (the other order can)
    run_proj_score(M, D, x, wq, wk, wv, w_score, q, k, v, raw, sl.ready, st);
    if (stream) {
        run_score_finish_async(B, L, sc, raw, sl.ready, raw, u, mean, sdev, bad, sl.side);
        SKB_CHECK_CUDA(cudaEventRecord(sl.join, sl.side));
        SKB_CHECK_CUDA(cudaStreamWaitEvent(st, sl.join, 0));
    } else {
        run_score_finish_async(B, L, sc, raw, nullptr, raw, u, mean, sdev, bad, st);
    }
    SKB_REQUIRE(!score_read_flag(bad, st), SKB_ENUMERIC, "score: non-finite value");
}

}  // namespace skb

extern "C" int skb_proj_score(int64_t B, int64_t L, int64_t D, const void* x, const void* wq, const void* wk,
                              const void* wv, const double* w_score, const skb_scoring* sc, void* q, void* k, void* v,
                              double* raw, double* u, double* mean, double* sdev, void* stream) {
    try {
        SKB_REQUIRE(x && wq && wk && wv && q && k && v, SKB_EARG, "proj_score: null argument");
        SKB_REQUIRE(!w_score || (sc && raw && u && mean && sdev), SKB_EARG, "proj_score: null score output");
        SKB_REQUIRE(B >= 1 && L >= 1, SKB_ESHAPE, "proj_score: empty input");
        skb::run_proj_score_fwd(B, L, D, x, wq, wk, wv, w_score, w_score ? *sc : skb_scoring{}, q, k, v, raw, u,
                                mean, sdev, static_cast<cudaStream_t>(stream));
    } catch (const skb::Error& e) {
        skb::set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        skb::set_last_error(e.what());
        return SKB_ECUDA;
    }
    return SKB_OK;
}
