// Shared helpers for the sm_100a SparseK kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "sparsek_b200.h"

namespace skb {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SKB_CHECK_CUDA(expr)                                                               \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw ::skb::Error(SKB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define SKB_CHECK_LAUNCH() SKB_CHECK_CUDA(cudaGetLastError())

#define SKB_REQUIRE(cond, code, msg)                       \
    do {                                                   \
        if (!(cond)) throw ::skb::Error((code), (msg));    \
    } while (0)

constexpr int kQBlock = 128;   // queries per attention block (and union list granule)
constexpr int kChunk = 32;     // push times per tau chunk (one per lane)

inline int64_t floor_k(double k) { return k > 0.0 ? (int64_t)floor(k) : 0; }
inline int64_t ceil_k(double k) { return k > 0.0 ? (int64_t)ceil(k) : 0; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- device
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <class T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ float tof(float x) { return x; }
__device__ __forceinline__ float tof(double x) { return (float)x; }
__device__ __forceinline__ float tof(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ void store_from_f(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_from_f(double* p, float v) { *p = (double)v; }
__device__ __forceinline__ void store_from_f(__nv_bfloat16* p, float v) { *p = __float2bfloat16(v); }

__device__ __forceinline__ double ld_as_double(const void* p, int dtype, int64_t i) {
    if (dtype == SKB_F64) return static_cast<const double*>(p)[i];
    if (dtype == SKB_F32) return (double)static_cast<const float*>(p)[i];
    return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}

}  // namespace skb
