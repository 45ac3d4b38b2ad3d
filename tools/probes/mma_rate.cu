// Issue-rate probe for the tcgen05 MMA shapes the backward uses (one CTA per
// SM, one thread issuing back-to-back MMAs on resident smem/TMEM operands):
// cycles per instruction against the floor max(M,128) N / 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_16747_b200/csrc \
//        tools/probes/mma_rate.cu -o tools/probes/mma_rate -lcuda
#include <cstdio>
#include <cstdlib>

#include "skb_tc.cuh"

using namespace skb::tc;

constexpr int kIters = 256;

// pattern: 0 SS 128x64 (K-major A 128 rows, K-major B 64 rows)
//          1 SS 128x128 (K-major A, K-major B 128 rows)
//          2 TS 128x128 (A in TMEM, B MN-major 64 rows of K)
//          3 the selected dK/dV tile: 8 x (S^T, dP^T) SS 128x64 + 4 x (dV, dK) TS 128x128
//          4 SS 128x256 (K-major A, K-major B 256 rows)
//          5 SS 128x128 B MN-major (A K-major)
//          6 TS 128x64 (A in TMEM, B MN-major)
__global__ void __launch_bounds__(128, 1) k_probe(int pattern, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bars2[3];
    const uint32_t sb = smem_u32(smem);
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0, 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bars2[0], 1);
        mbar_init(&bars2[1], 1);
        mbar_init(&bars2[2], 1);
        mbar_fence_init();
        mbar_arrive(&bars2[2]);  // phase 0 complete: waits on parity 0 succeed at once
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
    fence_async_smem();
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tm = tslot;
    long long t0 = 0, t1 = 0;
    if ((pattern == 19 || pattern == 20) && threadIdx.x >= 32) {  // warps 1-3: tcgen05.ld traffic on lanes of their quarter
        const int w = threadIdx.x >> 5;
        const uint32_t lane_off = (uint32_t)(w * 32) << 16;
        float v[32], acc = 0.f;
        for (int it = 0; it < (pattern == 19 ? 600 : 300); ++it) {
            tmem_ld32(tm + lane_off + (it & 3) * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) acc += v[c];
        }
        if (acc == 12345.f) out[2] = 1;
    }
    if (threadIdx.x == 0) {
        const uint32_t id64 = umma_idesc(128, 64, false, false);
        const uint32_t id128 = umma_idesc(128, 128, false, false);
        const uint32_t id256 = umma_idesc(128, 256, false, false);
        const uint32_t id128mn = umma_idesc(128, 128, false, true);
        const uint32_t id64mn = umma_idesc(128, 64, false, true);
        const uint32_t A = sb, B = sb + 32768, B2 = sb + 65536;
        int n = 0;
        for (int it = -8; it < kIters; ++it) {
            if (it == 0) {
                umma_commit(&bar);
                mbar_wait(&bar, 0);
                t0 = clock64();
            }
            switch (pattern) {
                case 0:
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id64, 1), ++n;
                    break;
                case 1:
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm, desc_kmajor(A, 128, kk), desc_kmajor(B, 128, kk), id128, 1), ++n;
                    break;
                case 2:
                    for (int kk = 0; kk < 8; ++kk) umma_f16_ts(tm + 256, tm + (kk & 3) * 8, desc_mnmajor(B, 64, kk & 3), id128mn, 1), ++n;
                    break;
                case 3:
                    for (int kk = 0; kk < 8; ++kk) {
                        umma_f16(tm, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id64, 1);
                        umma_f16(tm + 64, desc_kmajor(B2, 128, kk), desc_kmajor(B, 64, kk), id64, 1);
                        n += 2;
                    }
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_ts(tm + 256, tm + 128 + kk * 8, desc_mnmajor(B, 64, kk), id128mn, 1);
                        umma_f16_ts(tm + 384, tm + 192 + kk * 8, desc_mnmajor(B2, 64, kk), id128mn, 1);
                        n += 2;
                    }
                    break;
                case 4:
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm, desc_kmajor(A, 128, kk), desc_kmajor(B, 256, kk), id256, 1), ++n;
                    break;
                case 5:
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm, desc_kmajor(A, 128, kk), desc_mnmajor(B, 64, kk & 3), id128mn, 1), ++n;
                    break;
                case 7:  // SS 128x64, 2 accumulators alternating
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm + (kk & 1) * 64, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id64, 1), ++n;
                    break;
                case 8:  // SS 128x64, 4 accumulators
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm + (kk & 3) * 64, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id64, 1), ++n;
                    break;
                case 9:  // TS 128x128, 2 accumulators
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16_ts(tm + 256 + (kk & 1) * 128, tm + (kk & 3) * 8, desc_mnmajor(B, 64, kk & 3), id128mn, 1), ++n;
                    break;
                case 10:  // SS 128x128, 2 accumulators
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm + (kk & 1) * 128, desc_kmajor(A, 128, kk), desc_kmajor(B, 128, kk), id128, 1), ++n;
                    break;
                case 11:  // SS 128x256, 2 accumulators
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm + (kk & 1) * 256, desc_kmajor(A, 128, kk), desc_kmajor(B, 256, kk), id256, 1), ++n;
                    break;
                case 12:  // SS 128x32, 4 accumulators
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm + (kk & 3) * 32, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), umma_idesc(128, 32, false, false), 1), ++n;
                    break;
                case 13: case 14: case 15: case 16: {  // TMEM hazard: SS N=64 writes at wc, TS reads A at 0 (D at 384)
                    const uint32_t wc = pattern == 13 ? 64 : pattern == 14 ? 128 : pattern == 15 ? 256 : 320;
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(tm + wc, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id64, kk > 0), ++n;
                    for (int kk = 0; kk < 4; ++kk)
                        umma_f16_ts(tm + 384, tm + kk * 8, desc_mnmajor(B, 64, kk), id128mn, 1), ++n;
                    break;
                }
                case 19: case 20:
                    for (int kk = 0; kk < 8; ++kk) {
                        umma_f16(tm + 256, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id64, 1);
                        umma_f16(tm + 320, desc_kmajor(B2, 128, kk), desc_kmajor(B, 64, kk), id64, 1);
                        n += 2;
                    }
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_ts(tm + 384, tm + 128 + kk * 8, desc_mnmajor(B, 64, kk), id128mn, 1);
                        umma_f16_ts(tm + 384, tm + 192 + kk * 8, desc_mnmajor(B2, 64, kk), id128mn, 1);
                        n += 2;
                    }
                    break;
                case 21: case 22: {  // the selected tile, commits, two waits on a completed barrier
                    for (int kk = 0; kk < 8; ++kk) {
                        umma_f16(tm, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id64, 1);
                        umma_f16(tm + 64, desc_kmajor(B2, 128, kk), desc_kmajor(B, 64, kk), id64, 1);
                        n += 2;
                    }
                    umma_commit(&bars2[0]);
                    if (pattern == 21) mbar_wait(&bars2[2], 0);
                    else {
                        uint32_t ok;
                        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                     : "=r"(ok) : "r"(smem_u32(&bars2[2])), "r"(0u) : "memory");
                        if (!ok) mbar_wait(&bars2[2], 0);
                    }
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_ts(tm + 256, tm + 128 + kk * 8, desc_mnmajor(B, 64, kk), id128mn, 1);
                        umma_f16_ts(tm + 384, tm + 192 + kk * 8, desc_mnmajor(B2, 64, kk), id128mn, 1);
                        n += 2;
                    }
                    umma_commit(&bars2[1]);
                    if (pattern == 21) mbar_wait(&bars2[2], 0);
                    else {
                        uint32_t ok;
                        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                     : "=r"(ok) : "r"(smem_u32(&bars2[2])), "r"(0u) : "memory");
                        if (!ok) mbar_wait(&bars2[2], 0);
                    }
                    break;
                }
                case 17: case 18: {  // the selected tile with its commits (17) and commits + waits on a
                    // barrier the previous iteration's commit completes (18: one iteration of slack)
                    for (int kk = 0; kk < 8; ++kk) {
                        umma_f16(tm, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id64, 1);
                        umma_f16(tm + 64, desc_kmajor(B2, 128, kk), desc_kmajor(B, 64, kk), id64, 1);
                        n += 2;
                    }
                    umma_commit(&bars2[0]);
                    if (pattern == 18 && it > -7) mbar_wait(&bars2[1], (it + 7) & 1);
                    for (int kk = 0; kk < 4; ++kk) {
                        umma_f16_ts(tm + 256, tm + 128 + kk * 8, desc_mnmajor(B, 64, kk), id128mn, 1);
                        umma_f16_ts(tm + 384, tm + 192 + kk * 8, desc_mnmajor(B2, 64, kk), id128mn, 1);
                        n += 2;
                    }
                    umma_commit(&bars2[1]);
                    break;
                }
                case 6:
                    for (int kk = 0; kk < 8; ++kk) umma_f16_ts(tm + 256, tm + (kk & 3) * 8, desc_mnmajor(B, 64, kk & 3), id64mn, 1), ++n;
                    break;
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 1);
        t1 = clock64();
        if (blockIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = n;
        }
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (threadIdx.x < 32) tmem_dealloc<512>(tm);
    (void)bars2;
}

// ---- CTA pairs (cta_group::2, cluster of 2): M = 256, the even CTA issues
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
    asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void mma_pair_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
    asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(d), "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
// pattern: 0 SS 256x64, 1 SS 256x128, 2 TS 256x128 (B MN-major), 3 the pair's selected tile:
// 8 x (S^T, dP^T) SS 256x64 + 4 x (dV, dK) TS 256x128, 4 TS 256x64
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_probe2(int pattern, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sb = smem_u32(smem);
    const bool leader = cl_rank() == 0;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0, 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_async_smem();
    tc_before_sync();
    cl_sync();
    tc_after_sync();
    const uint32_t tm = tslot;
    if (threadIdx.x == 0 && leader) {
        const uint32_t id64 = umma_idesc(256, 64, false, false);
        const uint32_t id128 = umma_idesc(256, 128, false, false);
        const uint32_t id128mn = umma_idesc(256, 128, false, true);
        const uint32_t id64mn = umma_idesc(256, 64, false, true);
        const uint32_t A = sb, B = sb + 32768, B2 = sb + 65536;
        int n = 0;
        long long t0 = 0;
        for (int it = -8; it < kIters; ++it) {
            if (it == 0) {
                commit_pair(&bar);
                mbar_wait(&bar, 0);
                t0 = clock64();
            }
            switch (pattern) {
                case 0:
                    for (int kk = 0; kk < 8; ++kk) mma_pair(tm + (kk & 1) * 64, desc_kmajor(A, 128, kk), desc_kmajor(B, 32, kk), id64), ++n;
                    break;
                case 1:
                    for (int kk = 0; kk < 8; ++kk) mma_pair(tm + (kk & 1) * 128, desc_kmajor(A, 128, kk), desc_kmajor(B, 64, kk), id128), ++n;
                    break;
                case 2:
                    for (int kk = 0; kk < 8; ++kk) mma_pair_ts(tm + 256 + (kk & 1) * 128, tm + (kk & 3) * 8, desc_mnmajor(B, 64, kk & 3), id128mn), ++n;
                    break;
                case 3:
                    for (int kk = 0; kk < 8; ++kk) {
                        mma_pair(tm, desc_kmajor(A, 128, kk), desc_kmajor(B, 32, kk), id64);
                        mma_pair(tm + 64, desc_kmajor(B2, 128, kk), desc_kmajor(B, 32, kk), id64);
                        n += 2;
                    }
                    for (int kk = 0; kk < 4; ++kk) {
                        mma_pair_ts(tm + 256, tm + 128 + kk * 8, desc_mnmajor(B, 64, kk), id128mn);
                        mma_pair_ts(tm + 384, tm + 192 + kk * 8, desc_mnmajor(B2, 64, kk), id128mn);
                        n += 2;
                    }
                    break;
                case 4:
                    for (int kk = 0; kk < 8; ++kk) mma_pair_ts(tm + 256 + (kk & 1) * 64, tm + (kk & 3) * 8, desc_mnmajor(B, 64, kk & 3), id64mn), ++n;
                    break;
            }
        }
        commit_pair(&bar);
        mbar_wait(&bar, 1);
        const long long t1 = clock64();
        if (blockIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = n;
        }
    } else if (threadIdx.x == 0) {
        mbar_wait(&bar, 0);
        mbar_wait(&bar, 1);
    }
    tc_before_sync();
    cl_sync();
    tc_after_sync();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    long long* d;
    cudaMalloc(&d, 32);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024 + 1024);
    const char* names[] = {"SS 128x64  (S^T/dP^T)", "SS 128x128", "TS 128x128 (dV/dK)", "sel tile (16 SS64 + 8 TS128)",
                           "SS 128x256", "SS 128x128 B MN-major", "TS 128x64", "SS 128x64 2 acc", "SS 128x64 4 acc",
                           "TS 128x128 2 acc", "SS 128x128 2 acc", "SS 128x256 2 acc", "SS 128x32 4 acc",
                           "8 SS64 @64 + 4 TS(A@0)", "8 SS64 @128 + 4 TS(A@0)", "8 SS64 @256 + 4 TS(A@0)",
                           "8 SS64 @320 + 4 TS(A@0)", "sel tile + 2 commits", "sel tile + commits + wait(prev)",
                           "sel tile, 3 warps tcgen05.ld (long)", "sel tile, 3 warps tcgen05.ld (short)",
                           "sel tile + commits + 2 try_wait(done)", "sel tile + commits + 2 test_wait(done)"};
    const double floor_[] = {32, 64, 64, (16 * 32 + 8 * 64) / 24.0, 128, 64, 32, 32, 32, 64, 64, 128, 16, 42.7, 42.7, 42.7, 42.7, 42.7, 42.7, 42.7, 42.7, 42.7, 42.7};
    for (int p = 0; p < 23; ++p) {
        k_probe<<<148, 128, 160 * 1024 + 1024>>>(p, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            printf("%s: %s\n", names[p], cudaGetErrorString(e));
            return 1;
        }
        const int n0 = (int)(h[1] * kIters / (kIters + 8));
        printf("%-32s cycles/instr %.1f (floor %.1f)\n", names[p], (double)h[0] / n0, floor_[p]);
    }
    cudaFuncSetAttribute(k_probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024 + 1024);
    const char* names2[] = {"pair SS 256x64", "pair SS 256x128", "pair TS 256x128", "pair sel tile (16 SS64 + 8 TS128)",
                            "pair TS 256x64"};
    for (int p = 0; p < 5; ++p) {
        k_probe2<<<148, 128, 160 * 1024 + 1024>>>(p, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            printf("%s: %s\n", names2[p], cudaGetErrorString(e));
            return 1;
        }
        const int n0 = (int)(h[1] * kIters / (kIters + 8));
        printf("%-32s cycles/instr %.1f (per SM-pair)\n", names2[p], (double)h[0] / n0);
    }
    return 0;
}
