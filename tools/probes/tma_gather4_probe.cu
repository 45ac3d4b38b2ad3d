// Probe: TMA tile::gather4 semantics on sm_100a (box shape, swizzle placement).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tma_gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3, int col, int bytes,
                        uint16_t* out, int* status) {
    __shared__ __align__(1024) uint8_t buf[4096];
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 0xEE;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(buf + 512)),
            "l"(&tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su(&bar))
            : "memory");
        uint32_t ok = 0;
        for (long it = 0; it < 20000000 && !ok; ++it) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(su(&bar)) : "memory");
        }
        *status = ok ? 1 : -1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

int main() {
    const int ROWS = 64, COLS = 256;  // bf16 matrix; value = row*1000 + col (as raw u16)
    std::vector<uint16_t> h(ROWS * COLS);
    for (int r = 0; r < ROWS; ++r)
        for (int c = 0; c < COLS; ++c) h[r * COLS + c] = (uint16_t)(r * 256 + c);
    uint16_t* d;
    cudaMalloc(&d, h.size() * 2);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    uint16_t* out;
    int* st;
    cudaMalloc(&out, 4096);
    cudaMalloc(&st, 4);
    for (int boxrows : {1, 4}) {
        CUtensorMap tm;
        cuuint64_t gdim[2] = {(cuuint64_t)COLS, (cuuint64_t)ROWS};
        cuuint64_t gstr[1] = {(cuuint64_t)COLS * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)boxrows};
        cuuint32_t es[2] = {1, 1};
        CUresult rc = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, gdim, gstr, box, es,
                                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("boxrows=%d encode rc=%d\n", boxrows, (int)rc);
        if (rc) continue;
        int r[4] = {5, 17, 2, 40};
        k_probe<<<1, 128>>>(tm, r[0], r[1], r[2], r[3], 64, 512, out, st);
        cudaError_t e = cudaDeviceSynchronize();
        int hs = 0;
        std::vector<uint16_t> ho(2048);
        cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(ho.data(), out, 4096, cudaMemcpyDeviceToHost);
        printf("  launch=%s status=%d\n", cudaGetErrorString(e), hs);
        if (e) { cudaDeviceReset(); return 1; }
        // dump row-chunk placement in the 512B destination (buf+512 => smem rows 4..7 of a 1024-aligned tile)
        for (int row = 0; row < 4; ++row) {
            printf("  dst row %d:", row);
            for (int ch = 0; ch < 8; ++ch) {
                uint16_t v = ho[(512 + row * 128 + ch * 16) / 2];
                if (v == 0xEEEE) printf(" ----");
                else printf(" r%02d/c%03d", v / 256, v % 256);
            }
            printf("\n");
        }
    }
    return 0;
}
