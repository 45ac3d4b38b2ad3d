// TMEM read throughput per SM: W warps each tcgen05.ld 32 lanes x 32 columns (4 KB per warp-load)
// repeatedly; bytes per SM cycle (one CTA per SM, 148 CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2406_16747_b200/csrc \
//        tools/probes/tmem_ld_rate.cu -o tools/probes/tmem_ld_rate
#include <cstdio>

#include "skb_tc.cuh"

using namespace skb::tc;

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_ld(long long* out, float* sink, int iters) {
    __shared__ uint32_t tslot;
    if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tm = tslot;
    const int w = threadIdx.x >> 5;
    const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        float v[32];
        tmem_ld32(tm + lane_off + ((it + w) & 15) * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c) acc += v[c];
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (acc == 1234.5f) sink[threadIdx.x] = acc;
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

template <int NW>
void run(long long* d, float* s) {
    const int iters = 2048;
    k_ld<NW><<<148, NW * 32>>>(d, s, iters);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)NW * iters * 4096;
    printf("%2d warps: %.1f B/cycle/SM (%.0f cycles per 4 KB warp-load per warp)\n", NW, bytes / h,
           (double)h / iters);
}

int main() {
    long long* d;
    float* s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 4096);
    run<4>(d, s);
    run<8>(d, s);
    run<16>(d, s);
    return 0;
}
