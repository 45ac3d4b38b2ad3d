// Host-side TMA descriptors for [B, L, H, D] bf16 tensors (sm_100a).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "skb_common.cuh"

namespace skb {

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        SKB_CHECK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        SKB_REQUIRE(p != nullptr && q == cudaDriverEntryPointSuccess, SKB_ECUDA,
                    "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D view {H*D columns, L rows, B sequences}, box {64 columns, box_rows rows,
// 1}, SWIZZLE_128B: one 64-column atom of a row tile per load; rows outside
// [0, L) of a sequence are zero-filled.
inline CUtensorMap tmap_rows3d(const void* base, int64_t B, int64_t L, int64_t HD, int box_rows) {
    CUtensorMap m;
    cuuint64_t gdim[3] = {(cuuint64_t)HD, (cuuint64_t)L, (cuuint64_t)B};
    cuuint64_t gstr[2] = {(cuuint64_t)HD * 2, (cuuint64_t)(L * HD * 2)};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult rc = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gdim, gstr, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SKB_REQUIRE(rc == CUDA_SUCCESS, SKB_ECUDA, "cuTensorMapEncodeTiled (3d) failed");
    return m;
}

// 4-D view {8 elements, L rows, H*D/8 16-byte chunks, B} of a [B, L, H, D]
// tensor, box {8, 32, chunks, 1}: a box lands in shared memory as
// [chunk][32 rows][8 elements], the "32-key group" layout of the dK/dV
// epilogue staging (skb_attn_tc_bwd.cu part_off), stored with one TMA store.
inline CUtensorMap tmap_groups4d(const void* base, int64_t B, int64_t L, int64_t HD, int box_chunks) {
    CUtensorMap m;
    cuuint64_t gdim[4] = {8, (cuuint64_t)L, (cuuint64_t)(HD / 8), (cuuint64_t)B};
    cuuint64_t gstr[3] = {(cuuint64_t)HD * 2, 16, (cuuint64_t)(L * HD * 2)};
    cuuint32_t box[4] = {8, 32, (cuuint32_t)box_chunks, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult rc = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), gdim, gstr, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SKB_REQUIRE(rc == CUDA_SUCCESS, SKB_ECUDA, "cuTensorMapEncodeTiled (groups4d) failed");
    return m;
}

// 2-D view {H*D columns, B*L rows}, box {64, 1}: the row-gather (tile::gather4) map.
inline CUtensorMap tmap_gather2d(const void* base, int64_t rows, int64_t HD) {
    CUtensorMap m;
    cuuint64_t gdim[2] = {(cuuint64_t)HD, (cuuint64_t)rows};
    cuuint64_t gstr[1] = {(cuuint64_t)HD * 2};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult rc = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstr, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SKB_REQUIRE(rc == CUDA_SUCCESS, SKB_ECUDA, "cuTensorMapEncodeTiled (gather) failed");
    return m;
}

}  // namespace skb
