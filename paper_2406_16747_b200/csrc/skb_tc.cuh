// sm_100a building blocks for the tensor-core SparseK kernels: mbarriers,
// TMEM allocation and loads, tcgen05.mma issue/commit, UMMA shared-memory
// descriptors for 128B-swizzled tiles, and the cp.async row gather that
// writes that swizzle.
//
// Tile layout (all bf16 operands): a tile of R rows x C columns (C = 64 or
// 128) is stored as C/64 "atom columns" of R x 128 B; inside each, row r
// occupies 128 B at r*128 and its 16-byte chunk c sits at chunk (c ^ (r & 7))
// — the canonical SWIZZLE_128B layout. The same bytes serve as a K-major
// operand (rows = M/N, columns = K) or an MN-major operand (rows = K,
// columns = M/N).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace skb {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Barrier waits. SKB_WAIT_MODE selects the polling primitive (experiment
// hook): 0 try_wait with a suspend-time hint, 1 plain try_wait (the hardware
// picks the suspend window), 2 test_wait with an explicit nanosleep backoff.
#ifndef SKB_WAIT_MODE
#define SKB_WAIT_MODE 1
#endif
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
#if SKB_WAIT_MODE == 0
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(1000000u)
        : "memory");
#elif SKB_WAIT_MODE == 1
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (!ok) __nanosleep(64);
#endif
    return ok != 0;
}
// Wait for the phase with the given parity to complete. A wait that never
// completes (a pipeline bug) traps after ~seconds instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_slow(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t spins = 0;
    while (!mbar_try_wait(addr, parity)) {
        if (++spins > (1u << 26)) __trap();
    }
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// A try_wait costs ~150 cycles even on a completed phase, ~3x a test_wait
// (tools/probes/mma_rate.cu): every wait tests first. On the single
// MMA-issuing thread that time is tensor-pipe idle time once its queue drains.
#ifndef SKB_WAIT_TEST_FIRST
#define SKB_WAIT_TEST_FIRST 1
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if (SKB_WAIT_TEST_FIRST && mbar_test(bar, parity)) return;
    mbar_wait_slow(bar, parity);
}
// (kept for the call sites on MMA-issuing threads)
#ifndef SKB_MMA_SPIN  // 1: the MMA-issuing thread polls with test_wait (no suspend window)
#define SKB_MMA_SPIN 0
#endif
__device__ __forceinline__ void mbar_wait_fast(uint64_t* bar, uint32_t parity) {
    if (SKB_WAIT_TEST_FIRST && mbar_test(bar, parity)) return;
    if (SKB_MMA_SPIN) {
        uint32_t spins = 0;
        while (!mbar_test(bar, parity))
            if (++spins > (1u << 28)) __trap();
        return;
    }
    mbar_wait_slow(bar, parity);
}
// cp.async completion of this thread's prior copies arrives on the barrier.
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* addr) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(addr));
}
// 4-D tiled store shared -> global (bulk-group completion)
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// bulk L2 prefetch of [addr, addr + bytes) (16-byte aligned, multiple of 16)
__device__ __forceinline__ void prefetch_l2_bulk(const void* addr, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(addr), "r"(bytes) : "memory");
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 3-D tiled box load {c0 = column, c1 = row, c2 = sequence} (OOB -> zeros)
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// L2 prefetch of one 3-D tile box (no shared-memory destination, no barrier)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(c0), "r"(c1),
                 "r"(c2)
                 : "memory");
}
// four gathered rows of one 64-column box (2-D map, box {64, 1}); lands as
// four consecutive 128-byte rows, swizzled by their shared-memory address
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                            int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
// plain bulk copy global -> shared (bytes % 16 == 0, both 16-byte aligned)
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ------------------------------------------------------------------ cp.async
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
}

// Byte offset of (row r, 16-byte chunk c) inside a swizzled tile with R rows.
__device__ __forceinline__ uint32_t sw_off(int r, int c, int R) {
    return (uint32_t)((c >> 3) * (R * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// ------------------------------------------------------------------ fences
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ------------------------------------------------------------------ TMEM
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // one full warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}

// 32 lanes x 32 columns of fp32: thread t of the warp receives lane (base lane + t).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
        "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
        "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
        "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
        "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ UMMA
// Shared-memory matrix descriptor, SWIZZLE_128B, version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}
// Instruction descriptor: BF16 x BF16 -> F32, dense.
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N, bool a_mn_major, bool b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn_major ? 1u : 0u) << 15) |
           ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[tmem] * B[smem]: A (M x K, bf16, K-major) lives in TMEM — lane
// m holds row m, each 32-bit column two consecutive K elements (low half first).
__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}
// 32 lanes x 16 columns of fp32.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 lanes x 8 columns of raw 32-bit words.
__device__ __forceinline__ void tmem_st8u(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
// 32 lanes x 32 columns of raw 32-bit words (e.g. a bf16 row as an A operand).
__device__ __forceinline__ void tmem_st32u(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
// 32 lanes x 16 columns of packed bf16x2 (the A-operand layout above).
__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// Arrive on `bar` once every tcgen05 op this thread issued so far has completed.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// The start-address field of a descriptor is (addr >> 4) & 0x3FFF and shared
// memory stays below 2^18 bytes, so desc(base + off) = desc(base) + off / 16:
// the descriptor of a tile is built once and each K slice adds an immediate
// (keeps the single-thread MMA issue loop short).
// K-major operand with R rows (M or N) and K = 64*katoms columns: descriptor for
// the 16-wide K slice kk (0 .. 4*katoms-1).
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int R, int kk) {
    return umma_desc(base, 16, 1024) + (uint64_t)(((kk >> 2) * R * 128 + (kk & 3) * 32) >> 4);
}
// MN-major operand stored as K rows x (64*natoms) columns (R = number of K
// rows in the tile): descriptor for the 16-deep K slice kk.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int R, int kk) {
    return umma_desc(base, (uint32_t)(R * 128), 1024) + (uint64_t)((kk * 16 * 128) >> 4);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
// exp2 of two values on the FMA/ALU pipes (the MUFU unit is the softmax
// bottleneck: 16 ex2/clk/SM): Cody-Waite split x = n + f with the 1.5*2^23
// rounding trick, 2^f by a degree-3 minimax polynomial on [-1/2, 1/2]
// (max relative error 7.5e-5, far below the bf16 P~ it feeds), 2^n added
// into the exponent bits. Inputs below -126 (masked: -inf) give ~1e-38.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -126.f);  // n >= -126 keeps the exponent field non-negative
    x.y = fmaxf(x.y, -126.f);
    const float2 magic = make_float2(12582912.f, 12582912.f);
    const float2 t = __fadd2_rn(x, magic);
    const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));
    float2 p = __ffma2_rn(make_float2(0.05517098f, 0.05517098f), f, make_float2(0.2426097f, 0.2426097f));
    p = __ffma2_rn(p, f, make_float2(0.69326097f, 0.69326097f));
    p = __ffma2_rn(p, f, make_float2(0.99992816f, 0.99992816f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ------------------------------------------------------------------ CTA shape
// 384 threads: warps 0-3 and 4-7 are two math warpgroups that split every
// tile's columns (each thread owns one TMEM lane = tile row and half the
// columns, so each SM sub-partition runs two math warps), warps 8-10 are
// cp.async producers, warp 11 owns TMEM and issues tcgen05.mma (one thread).
constexpr int kThreads = 384;
constexpr int kMath = 256;
constexpr int kProducers = 96;
constexpr int kProdWarp0 = 8;
constexpr int kMmaWarp = 11;
// One arrival per warp (barrier count = warps): the warp's lanes order their
// prior work (tcgen05 fences included) before lane 0's release-arrive.
#ifndef SKB_WARP_ARRIVE
#define SKB_WARP_ARRIVE 1
#endif
constexpr int kMathArrivals = SKB_WARP_ARRIVE ? kMath / 32 : kMath;  // math-warp arrivals per phase
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
    if (!SKB_WARP_ARRIVE) {
        mbar_arrive(bar);
        return;
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

// Named barrier over the 256 math threads (id 1; 0 is __syncthreads).
__device__ __forceinline__ void math_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// one math warpgroup (128 threads); ids 2 and 3
__device__ __forceinline__ void wg_bar(int hf) { asm volatile("bar.sync %0, 128;" ::"r"(2 + hf) : "memory"); }

// Load an R-row tile of a [B, L, H, D] bf16 tensor into the swizzled layout.
// keyfn(row) gives the source row (< 0 or >= L: zero-filled). The producer
// warps stride over row groups (one group = the rows a warp covers per copy).
// All row keys are fetched first (independent loads, one latency), then the
// copies are issued — a gathered key must not sit on each copy's critical path.
template <int D, int R, class KeyFn>
__device__ __forceinline__ void load_tile(uint32_t dst, const __nv_bfloat16* base, int b, int h, int L, int H,
                                          int pw, int lane, KeyFn keyfn) {
    constexpr int kChunks = D / 8;              // 16-byte chunks per row
    constexpr int kRowsPerIter = 32 / kChunks;  // rows per warp per copy
    constexpr int kGroups = R / kRowsPerIter;
    constexpr int kPW = kProducers / 32;
    constexpr int kIters = (kGroups + kPW - 1) / kPW;
    const int sub = lane / kChunks, ch = lane % kChunks;
    int keys[kIters];
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const int g = pw + kPW * it;
        keys[it] = g < kGroups ? keyfn(g * kRowsPerIter + sub) : -1;
    }
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const int g = pw + kPW * it;
        if (g < kGroups) {
            const int r = g * kRowsPerIter + sub;
#if defined(SKB_EXP) && SKB_EXP == 2
            const bool ok = false;  // experiment: no gathers (zero fill)
#else
            const bool ok = keys[it] >= 0 && keys[it] < L;
#endif
            const __nv_bfloat16* src = base + (((int64_t)b * L + (ok ? keys[it] : 0)) * H + h) * D + ch * 8;
            cp_async16(dst + sw_off(r, ch, R), src, ok);
        }
    }
}

// Row keys of one R-row tile for this producer thread, fetched ahead of the
// copies so a gathered key is never on a copy's critical path.
template <int D, int R>
struct RowKeys {
    static constexpr int kChunks = D / 8;
    static constexpr int kRowsPerIter = 32 / kChunks;
    static constexpr int kGroups = R / kRowsPerIter;
    static constexpr int kPW = kProducers / 32;
    static constexpr int kIters = (kGroups + kPW - 1) / kPW;
    int k[kIters];

    // k[it] holds the raw key (no arithmetic on it here, so a prefetch never
    // waits for its loads); issue() turns it into the row index
    template <class KeyFn>
    __device__ __forceinline__ void fetch(int pw, int lane, KeyFn keyfn) {
        const int sub = lane / kChunks;
#pragma unroll
        for (int it = 0; it < kIters; ++it) {
            const int g = pw + kPW * it;
            k[it] = g < kGroups ? keyfn(g * kRowsPerIter + sub) : -1;
        }
    }
    // cp.async the rows into the 128B-swizzled tile. CHECKED: keys < 0 or
    // >= L are zero-filled; unchecked callers guarantee valid keys.
    template <bool CHECKED = true>
    __device__ __forceinline__ void issue(uint32_t dst, const __nv_bfloat16* base, int b, int h, int L, int H, int pw,
                                          int lane) const {
        const int sub = lane / kChunks, ch = lane % kChunks;
        // one IMAD.WIDE per row: src = basec + key * row_bytes
        const uint64_t basec = reinterpret_cast<uint64_t>(base + ((int64_t)b * L * H + h) * D) + (uint64_t)(ch * 16);
        const uint32_t row_bytes = (uint32_t)(H * D * 2);
        const uint32_t dcol = (uint32_t)((ch >> 3) * (R * 128));
#pragma unroll
        for (int it = 0; it < kIters; ++it) {
            const int g = pw + kPW * it;
            if (g < kGroups) {
                const int r = g * kRowsPerIter + sub;
#if defined(SKB_EXP) && SKB_EXP == 2
                const bool ok = false;  // experiment: no gathers (zero fill)
#else
                const bool ok = !CHECKED || (unsigned)k[it] < (unsigned)L;
#endif
                const uint32_t key = (CHECKED && !ok) ? 0u : (uint32_t)k[it];
                cp_async16(dst + dcol + r * 128 + (((ch & 7) ^ (r & 7)) << 4),
                           reinterpret_cast<const void*>(basec + (uint64_t)key * row_bytes), ok);
            }
        }
    }
};

// ------------------------------------------------------------------ CTA pairs
// cta_group::2: a cluster of two CTAs (one TPC); the even CTA issues M = 256
// MMAs whose A rows are split between the CTAs (128 each) and whose B columns
// are split in halves, each CTA staging its own half at the same offset.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA tile load whose completion is signalled on the even CTA's barrier
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
        : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// A from TMEM (each CTA's own 128 lanes), B from shared memory
__device__ __forceinline__ void umma_f16_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on `bar` in both CTAs of the pair once the pair's prior MMAs completed
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem) {  // one full warp in each CTA
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}

__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace tc
}  // namespace skb
