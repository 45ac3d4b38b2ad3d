// K3 tensor-core forward (tcgen05 + TMEM), BF16, head_dim 64 or 128.
//
// One CTA per (128-query block, head, sequence). Key tiles of 128 rows:
//   [selected-union tiles: gathered rows, per-key interval mask
//    j <= t_i < leave_j, value gates g = sat(u_j - tau_i)]
//   ++ [window tiles: the contiguous band [i0-w+1, i0+127], band mask].
// Per tile: S = Q K^T (tcgen05, M=N=128, K=d, fp32 in TMEM, double-buffered).
// Two math warpgroups each own one half of every tile's keys (64 columns) and
// run an independent online softmax over them with their own accumulator
// O_h += P~_h V_h (TS-MMA: P~ = P*g packed to bf16 in TMEM over the consumed
// S columns) — no per-tile exchange between the halves; the two partial
// softmaxes are merged once in the epilogue. Softmax statistics use the
// ungated P: proj/src/cache.cpp:358-393 (softmax over Sel U W, value gates
// applied after, no renormalisation).
//
// Producers (3 warps) fill K/V stages with cp.async row gathers whose keys
// were fetched one tile ahead, and copy the block's precomputed per-tile
// metadata (keys, leave, u, fast-path flags from skb_select) — no dependent
// global loads on the pipeline. The O rescale of the lazy softmax (exponent
// base moves only when the max grows by > 2^8) is the only place the math
// waits for a PV MMA.
#include "skb_common.cuh"
#include "skb_internal.h"
#include "skb_tc.cuh"
#include "skb_tmap.h"

#ifndef SKB_EXP
#define SKB_EXP 0
#endif

#ifdef SKB_TRACE
// Timeline probe (experiment builds only): clock64 stamps of one CTA's
// pipeline events, read back with skb_debug_trace().
__device__ unsigned long long g_skb_trace[4096];
#define SKB_TR(role, jt, ev)                                                                         \
    do {                                                                                              \
        if (blockIdx.x == 100 && blockIdx.y == 0 && blockIdx.z == 0 && (jt) < 16)                  \
            g_skb_trace[(role) * 256 + (jt) * 16 + (ev)] = clock64();                                \
    } while (0)
extern "C" int skb_debug_trace(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_skb_trace, sizeof(unsigned long long) * (n < 4096 ? n : 4096));
}
#else
#define SKB_TR(role, jt, ev) \
    do {                     \
    } while (0)
#endif

namespace skb {

namespace {

using namespace tc;

constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleSlack = 8.0f;  // lazy rescale threshold (log2 units)
#ifndef SKB_POLY_MASK
#define SKB_POLY_MASK 0
#endif
#ifndef SKB_POLY_PAIR
#define SKB_POLY_PAIR -1
#endif
constexpr int kPolyPair = SKB_POLY_PAIR;  // which key pair of every 8 uses the polynomial exp2 (-1: none)
constexpr int kPolyMask = SKB_POLY_MASK;  // bit e/2: key pair e of every 8 uses the polynomial exp2

struct FwdArgs {
    CUtensorMap tm_q;   // 3-D row tiles (box 64 x 128)
    CUtensorMap tm_k;
    CUtensorMap tm_v;
    CUtensorMap tg_k;   // 2-D row gathers (box 64 x 1)
    CUtensorMap tg_v;
    const __nv_bfloat16* q;
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    __nv_bfloat16* o;
    double* lse;
    const float* tauf;
    const int* qb_count;
    const int* qb_list;
    const int* qb_leave;
    const float* qb_uf;
    const int* qb_flags;
    int nqb, qb_cap;
    int B, L, H, w, T, R1;
    float scale_log2;
    int mask_st;
};

#ifndef SKB_FWD_KS
#define SKB_FWD_KS 3
#endif
constexpr int kKS = SKB_FWD_KS;  // K + metadata ring depth (V ring: 2)

template <int D>
struct FwdSmem {
    static constexpr int kTile = 128 * D * 2;  // bytes of a 128-row bf16 tile
    static constexpr int kQ = 0;
    static constexpr int kK = kQ + kTile;          // [kKS]
    static constexpr int kV = kK + kKS * kTile;    // [2]
    static constexpr int kMeta = kV + 2 * kTile;   // [kKS][key|leave|uf][128] x 4 B
    static constexpr int kFlags = kMeta + kKS * 3 * 128 * 4;  // [kKS] (16 B apart)
    static constexpr int kRed = kFlags + kKS * 16;            // [2 halves][m|l][128] f32
    static constexpr int kBar = kRed + 2 * 2 * 128 * 4;
    static constexpr int kNumBars = 30;
    static constexpr int kTmemSlot = kBar + kNumBars * 8;
    static constexpr int kBytes = kTmemSlot + 16;
    static constexpr int kAlloc = kBytes + 1024;  // room to align the base to 1024
};

// PFULL is per (S stage, half): a warpgroup may finish tile j+1 before the MMA
// warp consumes tile j's P~, so one barrier per half could run two phases ahead.
enum { B_QFULL = 0, B_KFULL = 1, B_KEMPTY = 4, B_MFULL = 7, B_MEMPTY = 10, B_VFULL = 13, B_VEMPTY = 15,
       B_SFULL = 17, B_SEMPTY = 19, B_PFULL = 21, B_PVDONE = 25, B_ODONE = 27,
       B_QEMPTY = 28, B_OEMPTY = 29 };  // 30 barriers (28 in the non-persistent kernel)

template <int D, bool KEY_SOFT>
__global__ void __launch_bounds__(kThreads, 1) k_fwd_tc(const __grid_constant__ FwdArgs a) {
    using SM = FwdSmem<D>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    // keep the shared address space visible to the compiler (LDS/STS, not generic)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    int* meta = reinterpret_cast<int*>(smem + SM::kMeta);
    int* tflags = reinterpret_cast<int*>(smem + SM::kFlags);
    float* red = reinterpret_cast<float*>(smem + SM::kRed);

    const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bl = (int64_t)b * a.L;
    const int64_t qrow = (int64_t)b * a.nqb + qb;
    const int i0 = qb * 128;
    const int cnt = (a.R1 > 0) ? a.qb_count[qrow] : 0;
    const int n_sel = (cnt + 127) / 128;
    const int n_win = (a.w + 127 + 127) / 128;
    const int n = n_sel + n_win;
    const int jw0 = i0 - a.w + 1;  // first key of the window band

    if (threadIdx.x == 0) {
        mbar_init(&bars[B_QFULL], 1);
        for (int s = 0; s < kKS; ++s) {
            mbar_init(&bars[B_KFULL + s], kProducers + 1);
            mbar_init(&bars[B_KEMPTY + s], 1);
            mbar_init(&bars[B_MFULL + s], kProducers);
            mbar_init(&bars[B_MEMPTY + s], kMath);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[B_VFULL + s], kProducers + 1);
            mbar_init(&bars[B_VEMPTY + s], 1);
            mbar_init(&bars[B_SFULL + s], 1);
            mbar_init(&bars[B_SEMPTY + s], kMath);
            mbar_init(&bars[B_PFULL + 2 * s], kMath / 2);
            mbar_init(&bars[B_PFULL + 2 * s + 1], kMath / 2);
            mbar_init(&bars[B_PVDONE + s], 1);
        }
        mbar_init(&bars[B_ODONE], 1);
        mbar_fence_init();
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tO = tmem + 256;  // O half h at tO + h * 128

    if (warp >= kProdWarp0 && warp < kMmaWarp) {
        // ------------------------------------------------------------ producers
        // Selected-union tiles: cp.async row gathers (keys fetched one tile
        // ahead; TMA tile::gather4 moves only 512 B per op and measured slower).
        // Q and the window band: 3-D TMA row tiles (OOB rows -> 0), issued by
        // one thread. Every FULL barrier counts 96 thread arrivals + 1 (the TMA
        // expect_tx on band tiles, a plain arrival on gathered ones).
        constexpr int kAtoms = D / 64;
        constexpr uint32_t kTileBytes = 128 * D * 2;
        const int pw = warp - kProdWarp0, ptid = threadIdx.x - kProdWarp0 * 32;
        if (ptid == 0) {
            mbar_expect_tx(&bars[B_QFULL], kTileBytes);
#pragma unroll
            for (int at = 0; at < kAtoms; ++at)
                tma_load_3d(sbase + SM::kQ + at * 128 * 128, &a.tm_q, h * D + at * 64, i0, b, &bars[B_QFULL]);
        }
        const int* list = a.qb_list + qrow * a.qb_cap;
        RowKeys<D, 128> kcur, kprev;
        if (n_sel > 0) kcur.fetch(pw, lane, [&](int r) { return __ldg(list + r); });
        const int ma = ptid >> 5, mc = ptid & 31;  // metadata: array, 16-byte chunk
        const int* msrc = ma == 0 ? a.qb_list : ma == 1 ? a.qb_leave : reinterpret_cast<const int*>(a.qb_uf);
        auto load_rows = [&](int jt, uint32_t dst, const RowKeys<D, 128>& keys, const __nv_bfloat16* src,
                             const CUtensorMap* tm3, uint64_t* bar) {
            if (SKB_EXP == 5 || SKB_EXP == 7 || SKB_EXP == 8) {  // experiment: no loads at all
                mbar_arrive(bar);
                if (ptid == 0) mbar_arrive(bar);
            } else if (jt < n_sel) {
                keys.template issue<false>(dst, src, b, h, a.L, a.H, pw, lane);  // union keys are valid
                cp_async_arrive_noinc(bar);
                if (ptid == 0) mbar_arrive(bar);
            } else {
                if (ptid == 0) {
                    mbar_expect_tx(bar, kTileBytes);
#pragma unroll
                    for (int at = 0; at < kAtoms; ++at)
                        tma_load_3d(dst + at * 128 * 128, tm3, h * D + at * 64, jw0 + (jt - n_sel) * 128, b, bar);
                }
                mbar_arrive(bar);
            }
        };
        // K + metadata run one tile ahead of V so a softmax never waits for a V gather
        for (int jt = 0; jt <= n; ++jt) {
            RowKeys<D, 128> knext;
            if (ptid == 0) SKB_TR(2, jt, 0);
            if (jt < n) {
                const int ks = jt % kKS;
                if (jt >= kKS) mbar_wait(&bars[B_MEMPTY + ks], ((jt - kKS) / kKS) & 1);
                if (jt < n_sel) {
                    cp_async16(smem_u32(meta + (ks * 3 + ma) * 128 + mc * 4),
                               msrc + qrow * a.qb_cap + jt * 128 + mc * 4, true);
                    if (ptid == 0)
                        cp_async16(smem_u32(tflags + ks * 4), a.qb_flags + (qrow * (a.qb_cap / 128) + jt) * 4, true);
                }
                cp_async_arrive_noinc(&bars[B_MFULL + ks]);
                if (jt >= kKS) mbar_wait(&bars[B_KEMPTY + ks], ((jt - kKS) / kKS) & 1);
                if (ptid == 0) SKB_TR(2, jt, 1);
                load_rows(jt, sbase + SM::kK + ks * SM::kTile, kcur, a.k, &a.tm_k, &bars[B_KFULL + ks]);
                if (ptid == 0) SKB_TR(2, jt, 2);
                if (jt + 1 < n_sel) knext.fetch(pw, lane, [&](int r) { return __ldg(list + (jt + 1) * 128 + r); });
            }
            if (jt >= 1) {
                const int j = jt - 1, vs = j & 1;
                if (j >= 2) mbar_wait(&bars[B_VEMPTY + vs], ((j - 2) >> 1) & 1);
                if (ptid == 0) SKB_TR(2, j, 3);
                load_rows(j, sbase + SM::kV + vs * SM::kTile, kprev, a.v, &a.tm_v, &bars[B_VFULL + vs]);
                if (ptid == 0) SKB_TR(2, j, 4);
            }
            kprev = kcur;
            kcur = knext;
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc_qk = umma_idesc(128, 128, false, false);
            constexpr uint32_t idesc_pv = umma_idesc(128, D, false, true);
            mbar_wait_fast(&bars[B_QFULL], 0);
            fence_proxy_async();
            auto pv = [&](int j) {
                mbar_wait_fast(&bars[B_VFULL + (j & 1)], (j >> 1) & 1);
                fence_proxy_async();
                const uint32_t vb = sbase + SM::kV + (j & 1) * SM::kTile;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    mbar_wait_fast(&bars[B_PFULL + 2 * (j & 1) + hf], (j >> 1) & 1);
                    SKB_TR(3, j, 2 + hf);
                    tc_after_sync();
                    // P~ of this half: 64 keys packed over the first 32 of its own S columns
                    const uint32_t pa = tS + (j & 1) * 128 + hf * 64;
#pragma unroll
                    for (int kk = 0; kk < ((SKB_EXP == 4 || SKB_EXP == 7) ? 0 : 4); ++kk)
                        umma_f16_ts(tO + hf * 128, pa + kk * 8, desc_mnmajor(vb, 128, hf * 4 + kk), idesc_pv,
                                    (j > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&bars[B_PVDONE + hf]);
                }
                umma_commit(&bars[B_VEMPTY + (j & 1)]);
            };
            for (int jt = 0; jt < n; ++jt) {
                const int s = jt & 1;
                const int ks = jt % kKS;
                SKB_TR(3, jt, 8);
                mbar_wait_fast(&bars[B_KFULL + ks], (jt / kKS) & 1);
                SKB_TR(3, jt, 0);
                fence_proxy_async();
                if (jt >= 2) mbar_wait_fast(&bars[B_SEMPTY + s], ((jt - 2) >> 1) & 1);
                tc_after_sync();
                const uint32_t kb = sbase + SM::kK + ks * SM::kTile;
#pragma unroll
                for (int kk = 0; kk < ((SKB_EXP == 4 || SKB_EXP == 7) ? 0 : D / 16); ++kk)
                    umma_f16(tS + s * 128, desc_kmajor(sbase + SM::kQ, 128, kk), desc_kmajor(kb, 128, kk),
                             idesc_qk, kk > 0 ? 1u : 0u);
                umma_commit(&bars[B_SFULL + s]);
                SKB_TR(3, jt, 1);
                umma_commit(&bars[B_KEMPTY + ks]);
                if (jt >= 1) pv(jt - 1);
            }
            pv(n - 1);
            umma_commit(&bars[B_ODONE]);  // every MMA of the CTA complete
        }
        __syncwarp();
    } else if (warp < kProdWarp0) {
        // ------------------------------------------------------------ math (warps 0-7)
        const int hf = warp >> 2;                // key half: 0 -> tile cols 0..63, 1 -> 64..127
        const int r = ((warp & 3) << 5) | lane;  // tile row = TMEM lane
        const int c0 = hf * 64;
        const int i = i0 + r;
        const int t = i - a.w;
        const float tau_i = (t >= 0 && a.R1 > 0) ? a.tauf[bl + t] : -INFINITY;
        const int lo_win = max(i - a.w + 1, 0);
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tOh = tO + hf * 128;
        const float sl2 = a.scale_log2;
        float m = -INFINITY, l = 0.f;  // this half's running max (log2 units) and sum
        float sv[64];
        for (int jt = 0; jt < n; ++jt) {
            const int s = jt & 1;
            const bool is_sel = jt < n_sel;
            const int ks = jt % kKS;
            if (lane == 0) SKB_TR(hf, jt, 9);
            mbar_wait(&bars[B_SFULL + s], (jt >> 1) & 1);
            if (lane == 0) SKB_TR(hf, jt, 0);
            if (is_sel) mbar_wait(&bars[B_MFULL + ks], (jt / kKS) & 1);
            tc_after_sync();
            tmem_ld32(tS + lane_off + s * 128 + c0, sv);
            tmem_ld32(tS + lane_off + s * 128 + c0 + 32, sv + 32);
            tmem_wait_ld();
            if (lane == 0 && (warp & 3) == 0) SKB_TR(hf, jt, 1);
            tc_before_sync();
            mbar_arrive(&bars[B_SEMPTY + s]);

#if SKB_EXP == 1 || SKB_EXP == 4 || SKB_EXP == 8
            if (true) {  // experiment: no softmax work (pipeline without the math)
                tc_before_sync();
                mbar_arrive(&bars[B_MEMPTY + ks]);
                mbar_arrive(&bars[B_PFULL + 2 * s + hf]);
                continue;
            }
#endif
            const int* mk = meta + (ks * 3) * 128 + c0;
            const int* ml = mk + 128;
            const float* mu = reinterpret_cast<const float*>(mk + 256);
            int fl = 3;
            if (is_sel && SKB_EXP != 3) {
                fl = tflags[ks * 4];
                if (KEY_SOFT) {  // gated logits (proj/src/cache.cpp:368-369)
#pragma unroll
                    for (int c = 0; c < 64; c += 4) {
                        const float4 uu = *reinterpret_cast<const float4*>(mu + c);
                        sv[c + 0] *= __saturatef(uu.x - tau_i);
                        sv[c + 1] *= __saturatef(uu.y - tau_i);
                        sv[c + 2] *= __saturatef(uu.z - tau_i);
                        sv[c + 3] *= __saturatef(uu.w - tau_i);
                    }
                }
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
            } else {
                // this row's window band inside the tile: columns [cmin, cmax]
                const int kb = jw0 + (jt - n_sel) * 128 + c0;
                const int cmin = lo_win - kb;
                const int cmax = i - kb;
                if (SKB_EXP != 3 && __any_sync(0xffffffffu, cmin > 0 || cmax < 63)) {
#pragma unroll
                    for (int c = 0; c < 64; ++c) sv[c] = (c >= cmin && c <= cmax) ? sv[c] : -INFINITY;
                }
            }
            float mx[8];  // 8 independent chains: the row max is not a 64-deep dependency
#pragma unroll
            for (int e = 0; e < 8; ++e) mx[e] = fmaxf(sv[e], sv[8 + e]);
#pragma unroll
            for (int c = 16; c < 64; c += 8)
#pragma unroll
                for (int e = 0; e < 8; ++e) mx[e] = fmaxf(mx[e], sv[c + e]);
            const float mr = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                   fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            if (lane == 0 && (warp & 3) == 0) SKB_TR(hf, jt, 2);
            const float mt = mr * sl2;  // scale > 0: max commutes with scaling
            float fac = 1.f;
            bool need = false;
            if (mt > m + kRescaleSlack) {
                if (m != -INFINITY) {
                    fac = ex2(m - mt);
                    l *= fac;
                    need = true;
                }
                m = mt;
            }
            const float nmb = m == -INFINITY ? 0.f : -m;  // fully masked so far: avoid -inf - -inf
            // packed fp32x2 arithmetic: one FFMA2 / FADD2 per two keys
            const float2 sl22 = make_float2(sl2, sl2), nmb2 = make_float2(nmb, nmb);
            float2 ps[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                            make_float2(0.f, 0.f)};
#pragma unroll
            for (int c = 0; c < 64; c += 8)
#pragma unroll
                for (int e = 0; e < 8; e += 2) {
                    float2 x = __ffma2_rn(make_float2(sv[c + e], sv[c + e + 1]), sl22, nmb2);
                    if (SKB_EXP == 6) {  // experiment: no exponentials at all
                    } else if (e == kPolyPair || ((kPolyMask >> (e >> 1)) & 1)) {  // pairs on the FMA pipe, the rest on MUFU
                        x = ex2_poly2(x);
                    } else {
                        x.x = ex2(x.x);  // masked: exp2(-inf) = 0
                        x.y = ex2(x.y);
                    }
                    ps[e >> 1] = __fadd2_rn(ps[e >> 1], x);
                    sv[c + e] = x.x;
                    sv[c + e + 1] = x.y;
                }
            const float2 pq = __fadd2_rn(__fadd2_rn(ps[0], ps[1]), __fadd2_rn(ps[2], ps[3]));
            l += pq.x + pq.y;
            if (lane == 0 && (warp & 3) == 0) SKB_TR(hf, jt, 3);
            if (is_sel && !a.mask_st && !(fl & 2)) {  // value gates (cache.cpp:381-382)
#pragma unroll
                for (int c = 0; c < 64; c += 4) {
                    const float4 uu = *reinterpret_cast<const float4*>(mu + c);
                    sv[c + 0] *= __saturatef(uu.x - tau_i);
                    sv[c + 1] *= __saturatef(uu.y - tau_i);
                    sv[c + 2] *= __saturatef(uu.z - tau_i);
                    sv[c + 3] *= __saturatef(uu.w - tau_i);
                }
            }
            if (__any_sync(0xffffffffu, need)) {
                // O_h must hold PV(jt-1) before it is rescaled; PV(jt-2) is
                // already complete (S(jt) was committed after it)
                mbar_wait(&bars[B_PVDONE + hf], (jt - 1) & 1);
                tc_after_sync();
                float ov[32];
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    const uint32_t ta = tOh + lane_off + c * 32;
                    tmem_ld32(ta, ov);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) ov[e] *= fac;
                    tmem_st32(ta, ov);
                }
            }
            // P~ (this half's 64 keys) -> TMEM over the tile's consumed S
            // columns, packed bf16x2: the A operand of this half's PV MMA
            {
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[2 * e], sv[2 * e + 1]);
                tmem_st16u(tS + lane_off + s * 128 + c0, pk);
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[32 + 2 * e], sv[33 + 2 * e]);
                tmem_st16u(tS + lane_off + s * 128 + c0 + 16, pk);
                tmem_wait_st();
            }
            tc_before_sync();
            if (lane == 0 && (warp & 3) == 0) SKB_TR(hf, jt, 4);
            mbar_arrive(&bars[B_MEMPTY + ks]);  // every tile (the producer waits on each stage)
            mbar_arrive(&bars[B_PFULL + 2 * s + hf]);
        }
        // epilogue: merge the two halves' softmaxes; half h writes O columns
        // [h*D/2, (h+1)*D/2) = (O_0 f_0 + O_1 f_1) / (l_0 f_0 + l_1 f_1)
        red[(hf * 2 + 0) * 128 + r] = m;
        red[(hf * 2 + 1) * 128 + r] = l;
        math_bar();
        const float mo = red[((hf ^ 1) * 2 + 0) * 128 + r];
        const float lo = red[((hf ^ 1) * 2 + 1) * 128 + r];
        const float M = fmaxf(m, mo);
        const float fs = (m == -INFINITY) ? 0.f : ex2(m - M);
        const float fo = (mo == -INFINITY) ? 0.f : ex2(mo - M);
        const float lrow = l * fs + lo * fo;
        const float f0 = hf == 0 ? fs : fo, f1 = hf == 0 ? fo : fs;
        mbar_wait(&bars[B_ODONE], 0);
        tc_after_sync();
        const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
        __nv_bfloat16* orow = a.o + ((bl + (i < a.L ? i : 0)) * a.H + h) * D + hf * (D / 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
            float o0[32], o1[32];
            tmem_ld32(tO + lane_off + hf * (D / 2) + c * 32, o0);
            tmem_ld32(tO + 128 + lane_off + hf * (D / 2) + c * 32, o1);
            tmem_wait_ld();
            if (i < a.L) {
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    uint4 pk;
                    pk.x = pack_bf16((o0[e] * f0 + o1[e] * f1) * inv, (o0[e + 1] * f0 + o1[e + 1] * f1) * inv);
                    pk.y = pack_bf16((o0[e + 2] * f0 + o1[e + 2] * f1) * inv, (o0[e + 3] * f0 + o1[e + 3] * f1) * inv);
                    pk.z = pack_bf16((o0[e + 4] * f0 + o1[e + 4] * f1) * inv, (o0[e + 5] * f0 + o1[e + 5] * f1) * inv);
                    pk.w = pack_bf16((o0[e + 6] * f0 + o1[e + 6] * f1) * inv, (o0[e + 7] * f0 + o1[e + 7] * f1) * inv);
                    *reinterpret_cast<uint4*>(orow + c * 32 + e) = pk;
                }
            }
        }
        if (hf == 0 && i < a.L) a.lse[((int64_t)b * a.H + h) * a.L + i] = (double)((M + __log2f(lrow)) * kLn2);
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

template <int D, bool KEY_SOFT>
__global__ void __launch_bounds__(kThreads, 1) k_fwd_p(const __grid_constant__ FwdArgs a) {
    using SM = FwdSmem<D>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    // keep the shared address space visible to the compiler (LDS/STS, not generic)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBar);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::kTmemSlot);
    int* meta = reinterpret_cast<int*>(smem + SM::kMeta);
    int* tflags = reinterpret_cast<int*>(smem + SM::kFlags);
    float* red = reinterpret_cast<float*>(smem + SM::kRed);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SKB_TRACE_FWDP  // tiles of items 3.. of CTA 100 (tools/trace_fwdp.py)
#define TRF(role, jj, ev) \
    if ((jj) >= tr0) SKB_TR(role, (jj) - tr0, ev)
#else
#define TRF(role, jj, ev) \
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
        t.jw0 = t.i0 - a.w + 1;  // first key of the window band
        return t;
    };

    if (threadIdx.x == 0) {
        mbar_init(&bars[B_QFULL], 1);
        for (int s = 0; s < kKS; ++s) {
            mbar_init(&bars[B_KFULL + s], kProducers + 1);
            mbar_init(&bars[B_KEMPTY + s], 1);
            mbar_init(&bars[B_MFULL + s], kProducers);
            mbar_init(&bars[B_MEMPTY + s], kMathArrivals);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars[B_VFULL + s], kProducers + 1);
            mbar_init(&bars[B_VEMPTY + s], 1);
            mbar_init(&bars[B_SFULL + s], 1);
            mbar_init(&bars[B_SEMPTY + s], kMathArrivals);
            mbar_init(&bars[B_PFULL + 2 * s], kMathArrivals / 2);
            mbar_init(&bars[B_PFULL + 2 * s + 1], kMathArrivals / 2);
            mbar_init(&bars[B_PVDONE + s], 1);
        }
        mbar_init(&bars[B_ODONE], 1);
        mbar_init(&bars[B_QEMPTY], 1);
        mbar_init(&bars[B_OEMPTY], kMathArrivals);
        mbar_fence_init();
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tO = tmem + 256;  // O half h at tO + h * 128

    if (warp >= kProdWarp0 && warp < kMmaWarp) {
        // ------------------------------------------------------------ producers
        // Selected-union tiles: cp.async row gathers (keys fetched one tile
        // ahead; TMA tile::gather4 moves only 512 B per op and measured slower).
        // Q and the window band: 3-D TMA row tiles (OOB rows -> 0), issued by
        // one thread. Every FULL barrier counts 96 thread arrivals + 1 (the TMA
        // expect_tx on band tiles, a plain arrival on gathered ones).
        constexpr int kAtoms = D / 64;
        constexpr uint32_t kTileBytes = 128 * D * 2;
        const int pw = warp - kProdWarp0, ptid = threadIdx.x - kProdWarp0 * 32;
        const int ma = ptid >> 5, mc = ptid & 31;  // metadata: array, 16-byte chunk
        const int* msrc = ma == 0 ? a.qb_list : ma == 1 ? a.qb_leave : reinterpret_cast<const int*>(a.qb_uf);
        int J = 0, it = 0, tr0 = 1 << 28;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
            const Item I = item(wi);
            const int b = I.b, h = I.h, n_sel = I.n_sel, n = I.n, jw0 = I.jw0;
            const int64_t qrow = I.qrow;
            if (it == 3) tr0 = J;
            if (ptid == 0) {  // Q once the previous item's last S MMA has read it
                if (it > 0) mbar_wait(&bars[B_QEMPTY], (it - 1) & 1);
                mbar_expect_tx(&bars[B_QFULL], kTileBytes);
#pragma unroll
                for (int at = 0; at < kAtoms; ++at)
                    tma_load_3d(sbase + SM::kQ + at * 128 * 128, &a.tm_q, h * D + at * 64, I.i0, b, &bars[B_QFULL]);
            }
            const int* list = a.qb_list + qrow * a.qb_cap;
            RowKeys<D, 128> kcur, kprev;
            if (n_sel > 0) kcur.fetch(pw, lane, [&](int r) { return __ldg(list + r); });
            auto load_rows = [&](int jt, uint32_t dst, const RowKeys<D, 128>& keys, const __nv_bfloat16* src,
                                 const CUtensorMap* tm3, uint64_t* bar) {
                if (jt < n_sel) {
                    keys.template issue<false>(dst, src, b, h, a.L, a.H, pw, lane);  // union keys are valid
                    cp_async_arrive_noinc(bar);
                    if (ptid == 0) mbar_arrive(bar);
                } else {
                    if (ptid == 0) {
                        mbar_expect_tx(bar, kTileBytes);
#pragma unroll
                        for (int at = 0; at < kAtoms; ++at)
                            tma_load_3d(dst + at * 128 * 128, tm3, h * D + at * 64, jw0 + (jt - n_sel) * 128, b, bar);
                    }
                    mbar_arrive(bar);
                }
            };
            // K + metadata run one tile ahead of V so a softmax never waits for a V gather
            for (int jt = 0; jt <= n; ++jt) {
                RowKeys<D, 128> knext;
                if (jt < n) {
                    const int JJ = J + jt;
                    const int ks = JJ % kKS;
                    if (JJ >= kKS) mbar_wait(&bars[B_MEMPTY + ks], ((JJ - kKS) / kKS) & 1);
                    if (jt < n_sel) {
                        cp_async16(smem_u32(meta + (ks * 3 + ma) * 128 + mc * 4),
                                   msrc + qrow * a.qb_cap + jt * 128 + mc * 4, true);
                        if (ptid == 0)
                            cp_async16(smem_u32(tflags + ks * 4), a.qb_flags + (qrow * (a.qb_cap / 128) + jt) * 4,
                                       true);
                    }
                    cp_async_arrive_noinc(&bars[B_MFULL + ks]);
                    if (JJ >= kKS) mbar_wait(&bars[B_KEMPTY + ks], ((JJ - kKS) / kKS) & 1);
                    if (ptid == 0) TRF(2, JJ, 1);
                    load_rows(jt, sbase + SM::kK + ks * SM::kTile, kcur, a.k, &a.tm_k, &bars[B_KFULL + ks]);
                    if (jt + 1 < n_sel)
                        knext.fetch(pw, lane, [&](int r) { return __ldg(list + (jt + 1) * 128 + r); });
                }
                if (jt >= 1) {
                    const int j = jt - 1, JJ = J + j, vs = JJ & 1;
                    if (JJ >= 2) mbar_wait(&bars[B_VEMPTY + vs], ((JJ - 2) >> 1) & 1);
                    if (ptid == 0) TRF(2, JJ, 3);
                    load_rows(j, sbase + SM::kV + vs * SM::kTile, kprev, a.v, &a.tm_v, &bars[B_VFULL + vs]);
                }
                kprev = kcur;
                kcur = knext;
            }
            J += n;
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc_qk = umma_idesc(128, 128, false, false);
            constexpr uint32_t idesc_pv = umma_idesc(128, D, false, true);
            int tr0 = 1 << 28;
            auto pv = [&](int J, int j, int itn) {
                mbar_wait_fast(&bars[B_VFULL + (J & 1)], (J >> 1) & 1);
                TRF(3, J, 2);
                fence_proxy_async();
                if (j == 0 && itn > 0) mbar_wait_fast(&bars[B_OEMPTY], (itn - 1) & 1);  // O read out
                const uint32_t vb = sbase + SM::kV + (J & 1) * SM::kTile;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    mbar_wait_fast(&bars[B_PFULL + 2 * (J & 1) + hf], (J >> 1) & 1);
                    TRF(3, J, 3 + hf);
                    tc_after_sync();
                    // P~ of this half: 64 keys packed over the first 32 of its own S columns
                    const uint32_t pa = tS + (J & 1) * 128 + hf * 64;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_f16_ts(tO + hf * 128, pa + kk * 8, desc_mnmajor(vb, 128, hf * 4 + kk), idesc_pv,
                                    (j > 0 || kk > 0) ? 1u : 0u);
                }
                // one completion for both halves (a commit costs the issuing thread ~90
                // cycles; the math waits on it only to rescale O, rarely)
                umma_commit(&bars[B_PVDONE]);
                umma_commit(&bars[B_VEMPTY + (J & 1)]);
                TRF(3, J, 5);
            };
            int J = 0, it = 0;
            for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
                const Item I = item(wi);
                const int n = I.n;
                if (it == 3) tr0 = J;
                mbar_wait_fast(&bars[B_QFULL], it & 1);
                for (int jt = 0; jt < n; ++jt) {
                    const int JJ = J + jt, s = JJ & 1, ks = JJ % kKS;
                    mbar_wait_fast(&bars[B_KFULL + ks], (JJ / kKS) & 1);
                    TRF(3, JJ, 0);
                    fence_proxy_async();
                    if (JJ >= 2) mbar_wait_fast(&bars[B_SEMPTY + s], ((JJ - 2) >> 1) & 1);
                    tc_after_sync();
                    const uint32_t kb = sbase + SM::kK + ks * SM::kTile;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        umma_f16(tS + s * 128, desc_kmajor(sbase + SM::kQ, 128, kk), desc_kmajor(kb, 128, kk),
                                 idesc_qk, kk > 0 ? 1u : 0u);
                    umma_commit(&bars[B_SFULL + s]);
                    umma_commit(&bars[B_KEMPTY + ks]);
                    TRF(3, JJ, 1);
                    if (jt == n - 1) umma_commit(&bars[B_QEMPTY]);
                    if (jt >= 1) pv(JJ - 1, jt - 1, it);
                }
                pv(J + n - 1, n - 1, it);
                umma_commit(&bars[B_ODONE]);  // every MMA of the item complete
                J += n;
            }
        }
        __syncwarp();
    } else if (warp < kProdWarp0) {
        // ------------------------------------------------------------ math (warps 0-7)
        const int hf = warp >> 2;                // key half: 0 -> tile cols 0..63, 1 -> 64..127
        const int r = ((warp & 3) << 5) | lane;  // tile row = TMEM lane
        const int c0 = hf * 64;
        int J = 0, it = 0, tr0 = 1 << 28;
        const bool trl = lane == 0 && (warp & 3) == 0;
        for (int wi = blockIdx.x; wi < nitems; wi += gridDim.x, ++it) {
        const Item I = item(wi);
        const int b = I.b, h = I.h, n_sel = I.n_sel, n = I.n, jw0 = I.jw0;
        const int64_t bl = I.bl;
        if (it == 3) tr0 = J;
        const int i = I.i0 + r;
        const int t = i - a.w;
        const float tau_i = (t >= 0 && a.R1 > 0) ? a.tauf[bl + t] : -INFINITY;
        const int lo_win = max(i - a.w + 1, 0);
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tOh = tO + hf * 128;
        const float sl2 = a.scale_log2;
        float m = -INFINITY, l = 0.f;  // this half's running max (log2 units) and sum
        float sv[64];
        for (int jt = 0; jt < n; ++jt, ++J) {
            const int s = J & 1;
            const bool is_sel = jt < n_sel;
            const int ks = J % kKS;
            if (trl) TRF(hf, J, 9);
            mbar_wait(&bars[B_SFULL + s], (J >> 1) & 1);
            mbar_wait(&bars[B_MFULL + ks], (J / kKS) & 1);  // every phase observed (window tiles too)
            tc_after_sync();
            tmem_ld32(tS + lane_off + s * 128 + c0, sv);
            tmem_ld32(tS + lane_off + s * 128 + c0 + 32, sv + 32);
            tmem_wait_ld();
            tc_before_sync();
            warp_arrive(&bars[B_SEMPTY + s]);
            if (trl) TRF(hf, J, 0);

#if SKB_EXP == 1 || SKB_EXP == 4 || SKB_EXP == 8
            if (true) {  // experiment: no softmax work (pipeline without the math)
                tc_before_sync();
                mbar_arrive(&bars[B_MEMPTY + ks]);
                warp_arrive(&bars[B_PFULL + 2 * s + hf]);
                continue;
            }
#endif
            const int* mk = meta + (ks * 3) * 128 + c0;
            const int* ml = mk + 128;
            const float* mu = reinterpret_cast<const float*>(mk + 256);
            int fl = 3;
            if (is_sel && SKB_EXP != 3) {
                fl = tflags[ks * 4];
                if (KEY_SOFT) {  // gated logits (proj/src/cache.cpp:368-369)
#pragma unroll
                    for (int c = 0; c < 64; c += 4) {
                        const float4 uu = *reinterpret_cast<const float4*>(mu + c);
                        sv[c + 0] *= __saturatef(uu.x - tau_i);
                        sv[c + 1] *= __saturatef(uu.y - tau_i);
                        sv[c + 2] *= __saturatef(uu.z - tau_i);
                        sv[c + 3] *= __saturatef(uu.w - tau_i);
                    }
                }
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
            } else {
                // this row's window band inside the tile: columns [cmin, cmax]
                const int kb = jw0 + (jt - n_sel) * 128 + c0;
                const int cmin = lo_win - kb;
                const int cmax = i - kb;
                if (SKB_EXP != 3 && __any_sync(0xffffffffu, cmin > 0 || cmax < 63)) {
#pragma unroll
                    for (int c = 0; c < 64; ++c) sv[c] = (c >= cmin && c <= cmax) ? sv[c] : -INFINITY;
                }
            }
            float mx[8];  // 8 independent chains: the row max is not a 64-deep dependency
#pragma unroll
            for (int e = 0; e < 8; ++e) mx[e] = fmaxf(sv[e], sv[8 + e]);
#pragma unroll
            for (int c = 16; c < 64; c += 8)
#pragma unroll
                for (int e = 0; e < 8; ++e) mx[e] = fmaxf(mx[e], sv[c + e]);
            const float mr = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                   fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            const float mt = mr * sl2;  // scale > 0: max commutes with scaling
            float fac = 1.f;
            bool need = false;
            if (mt > m + kRescaleSlack) {
                if (m != -INFINITY) {
                    fac = ex2(m - mt);
                    l *= fac;
                    need = true;
                }
                m = mt;
            }
            const float nmb = m == -INFINITY ? 0.f : -m;  // fully masked so far: avoid -inf - -inf
            // packed fp32x2 arithmetic: one FFMA2 / FADD2 per two keys
            const float2 sl22 = make_float2(sl2, sl2), nmb2 = make_float2(nmb, nmb);
            float2 ps[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                            make_float2(0.f, 0.f)};
#pragma unroll
            for (int c = 0; c < 64; c += 8)
#pragma unroll
                for (int e = 0; e < 8; e += 2) {
                    float2 x = __ffma2_rn(make_float2(sv[c + e], sv[c + e + 1]), sl22, nmb2);
                    if (SKB_EXP == 6) {  // experiment: no exponentials at all
                    } else if (e == kPolyPair || ((kPolyMask >> (e >> 1)) & 1)) {  // pairs on the FMA pipe, the rest on MUFU
                        x = ex2_poly2(x);
                    } else {
                        x.x = ex2(x.x);  // masked: exp2(-inf) = 0
                        x.y = ex2(x.y);
                    }
                    ps[e >> 1] = __fadd2_rn(ps[e >> 1], x);
                    sv[c + e] = x.x;
                    sv[c + e + 1] = x.y;
                }
            const float2 pq = __fadd2_rn(__fadd2_rn(ps[0], ps[1]), __fadd2_rn(ps[2], ps[3]));
            l += pq.x + pq.y;
            if (is_sel && !a.mask_st && !(fl & 2)) {  // value gates (cache.cpp:381-382)
#pragma unroll
                for (int c = 0; c < 64; c += 4) {
                    const float4 uu = *reinterpret_cast<const float4*>(mu + c);
                    sv[c + 0] *= __saturatef(uu.x - tau_i);
                    sv[c + 1] *= __saturatef(uu.y - tau_i);
                    sv[c + 2] *= __saturatef(uu.z - tau_i);
                    sv[c + 3] *= __saturatef(uu.w - tau_i);
                }
            }
            if (__any_sync(0xffffffffu, need)) {
                // O_h must hold PV(jt-1) before it is rescaled; PV(jt-2) is
                // already complete (S(jt) was committed after it)
                mbar_wait(&bars[B_PVDONE], (J - 1) & 1);
                tc_after_sync();
                float ov[32];
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    const uint32_t ta = tOh + lane_off + c * 32;
                    tmem_ld32(ta, ov);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) ov[e] *= fac;
                    tmem_st32(ta, ov);
                }
            }
            // P~ (this half's 64 keys) -> TMEM over the tile's consumed S
            // columns, packed bf16x2: the A operand of this half's PV MMA
            {
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[2 * e], sv[2 * e + 1]);
                tmem_st16u(tS + lane_off + s * 128 + c0, pk);
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(sv[32 + 2 * e], sv[33 + 2 * e]);
                tmem_st16u(tS + lane_off + s * 128 + c0 + 16, pk);
                tmem_wait_st();
            }
            tc_before_sync();
            if (trl) TRF(hf, J, 4);
            warp_arrive(&bars[B_MEMPTY + ks]);  // every tile (the producer waits on each stage)
            warp_arrive(&bars[B_PFULL + 2 * s + hf]);
        }
        // epilogue: merge the two halves' softmaxes; half h writes O columns
        // [h*D/2, (h+1)*D/2) = (O_0 f_0 + O_1 f_1) / (l_0 f_0 + l_1 f_1)
        red[(hf * 2 + 0) * 128 + r] = m;
        red[(hf * 2 + 1) * 128 + r] = l;
        math_bar();
        const float mo = red[((hf ^ 1) * 2 + 0) * 128 + r];
        const float lo = red[((hf ^ 1) * 2 + 1) * 128 + r];
        math_bar();  // red is rewritten by the next item
        const float M = fmaxf(m, mo);
        const float fs = (m == -INFINITY) ? 0.f : ex2(m - M);
        const float fo = (mo == -INFINITY) ? 0.f : ex2(mo - M);
        const float lrow = l * fs + lo * fo;
        const float f0 = hf == 0 ? fs : fo, f1 = hf == 0 ? fo : fs;
        mbar_wait(&bars[B_ODONE], it & 1);
        tc_after_sync();
        const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
        __nv_bfloat16* orow = a.o + ((bl + (i < a.L ? i : 0)) * a.H + h) * D + hf * (D / 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
            float o0[32], o1[32];
            tmem_ld32(tO + lane_off + hf * (D / 2) + c * 32, o0);
            tmem_ld32(tO + 128 + lane_off + hf * (D / 2) + c * 32, o1);
            tmem_wait_ld();
            if (i < a.L) {
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    uint4 pk;
                    pk.x = pack_bf16((o0[e] * f0 + o1[e] * f1) * inv, (o0[e + 1] * f0 + o1[e + 1] * f1) * inv);
                    pk.y = pack_bf16((o0[e + 2] * f0 + o1[e + 2] * f1) * inv, (o0[e + 3] * f0 + o1[e + 3] * f1) * inv);
                    pk.z = pack_bf16((o0[e + 4] * f0 + o1[e + 4] * f1) * inv, (o0[e + 5] * f0 + o1[e + 5] * f1) * inv);
                    pk.w = pack_bf16((o0[e + 6] * f0 + o1[e + 6] * f1) * inv, (o0[e + 7] * f0 + o1[e + 7] * f1) * inv);
                    *reinterpret_cast<uint4*>(orow + c * 32 + e) = pk;
                }
            }
        }
        tc_before_sync();
        warp_arrive(&bars[B_OEMPTY]);
        if (hf == 0 && i < a.L) a.lse[((int64_t)b * a.H + h) * a.L + i] = (double)((M + __log2f(lrow)) * kLn2);
        }
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
#undef TRF
}

template <int D, bool KS>
void launch_fwd(const FwdArgs& a, dim3 grid, cudaStream_t st) {
    using SM = FwdSmem<D>;
    static uint64_t attr = 0;
    if (first_on_device(&attr)) {
        SKB_CHECK_CUDA(cudaFuncSetAttribute(k_fwd_tc<D, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            SM::kAlloc));
        SKB_CHECK_CUDA(cudaFuncSetAttribute(k_fwd_p<D, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            SM::kAlloc));
    }
    static const int persist = getenv("SKB_FWD_PERSIST") ? atoi(getenv("SKB_FWD_PERSIST")) : 1;
    if (persist) {
        const int64_t items = (int64_t)grid.x * grid.y * grid.z;
        const int g = persist_grid(items);
        k_fwd_p<D, KS><<<g, kThreads, SM::kAlloc, st>>>(a);
    } else {
        k_fwd_tc<D, KS><<<grid, kThreads, SM::kAlloc, st>>>(a);
    }
    SKB_CHECK_LAUNCH();
}

}  // namespace

bool tc_supported(const skb_attn_desc& d) {
    return d.dtype == SKB_BF16 && (d.head_dim == 64 || d.head_dim == 128) && d.window >= 1 &&
           d.seq_len >= 1;
}

void run_attn_fwd_tc(const skb_attn_desc& d, const void* q, const void* k, const void* v,
                     const double* u, const SelView& s, void* o, double* lse, void* ws,
                     cudaStream_t st) {
    (void)u;
    (void)ws;
    FwdArgs a{};
    {
        const int64_t HD = d.heads * d.head_dim;
        a.tm_q = tmap_rows3d(q, d.batch, d.seq_len, HD, 128);
        a.tm_k = tmap_rows3d(k, d.batch, d.seq_len, HD, 128);
        a.tm_v = tmap_rows3d(v, d.batch, d.seq_len, HD, 128);
        a.tg_k = tmap_gather2d(k, d.batch * d.seq_len, HD);
        a.tg_v = tmap_gather2d(v, d.batch * d.seq_len, HD);
    }
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.k = static_cast<const __nv_bfloat16*>(k);
    a.v = static_cast<const __nv_bfloat16*>(v);
    a.o = static_cast<__nv_bfloat16*>(o);
    a.lse = lse;
    a.tauf = s.tauf;
    a.qb_count = s.qb_count;
    a.qb_list = s.qb_list;
    a.qb_leave = s.qb_leave;
    a.qb_uf = s.qb_uf;
    a.qb_flags = s.qb_flags;
    a.nqb = s.nqb;
    a.qb_cap = s.qb_cap;
    a.B = (int)d.batch;
    a.L = (int)d.seq_len;
    a.H = (int)d.heads;
    a.w = (int)d.window;
    a.T = std::max(0, a.L - a.w);
    a.R1 = (int)floor_k(d.k);
    const double scale = d.scale > 0.0 ? d.scale : 1.0 / std::sqrt((double)d.head_dim);
    a.scale_log2 = (float)(scale * 1.4426950408889634);
    a.mask_st = d.mask_mode;
    dim3 grid((unsigned)s.nqb, (unsigned)d.heads, (unsigned)d.batch);
    if (d.head_dim == 128) {
        if (d.key_mode) launch_fwd<128, true>(a, grid, st);
        else launch_fwd<128, false>(a, grid, st);
    } else {
        if (d.key_mode) launch_fwd<64, true>(a, grid, st);
        else launch_fwd<64, false>(a, grid, st);
    }
}

}  // namespace skb
