// Host-side TMA descriptor construction.  The driver entry point is resolved
// through the runtime (cudaGetDriverEntryPoint) so the library does not link
// libcuda directly.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstring>

namespace flame {

inline PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D bf16 tensor map [groups][rows][inner] with a (box_inner x box_rows x 1)
// box and 128-byte swizzle (box_inner * 2 must be <= 128), or the 64-byte one
// (box_inner * 2 <= 64) when asked.  Out-of-bounds
// elements read as zero, which is what pads ragged M / N tiles.
inline bool make_tmap_bf16_3d_swz(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows,
                                  uint64_t groups, uint64_t row_stride_bytes,
                                  uint64_t group_stride_bytes, uint32_t box_inner, uint32_t box_rows,
                                  CUtensorMapSwizzle swizzle) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  std::memset(map, 0, sizeof(*map));
  if (groups < 1) groups = 1;
  if (group_stride_bytes == 0) group_stride_bytes = rows * row_stride_bytes;
  if (group_stride_bytes == 0) group_stride_bytes = 16;
  cuuint64_t dims[3] = {inner, rows, groups};
  cuuint64_t strides[2] = {row_stride_bytes, group_stride_bytes};
  cuuint32_t box[3] = {box_inner, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline bool make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows,
                              uint64_t groups, uint64_t row_stride_bytes,
                              uint64_t group_stride_bytes, uint32_t box_inner, uint32_t box_rows) {
  return make_tmap_bf16_3d_swz(map, base, inner, rows, groups, row_stride_bytes, group_stride_bytes, box_inner,
                               box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Same for fp32 operands (the tf32 GEMM): box_inner * 4 <= 128.
inline bool make_tmap_f32_3d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows, uint64_t groups,
                             uint64_t row_stride_bytes, uint64_t group_stride_bytes, uint32_t box_inner,
                             uint32_t box_rows) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  std::memset(map, 0, sizeof(*map));
  if (groups < 1) groups = 1;
  if (group_stride_bytes == 0) group_stride_bytes = rows * row_stride_bytes;
  if (group_stride_bytes == 0) group_stride_bytes = 16;
  cuuint64_t dims[3] = {inner, rows, groups};
  cuuint64_t strides[2] = {row_stride_bytes, group_stride_bytes};
  cuuint32_t box[3] = {box_inner, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Output map for the GEMM epilogue's TMA stores: [groups][rows][cols] of
// bf16 (2-byte) or fp32 (4-byte) elements, box 32 cols x 32 rows; swizzle
// matches a 32-column row (64 B -> SW64, 128 B -> SW128).
inline bool make_tmap_out_3d(CUtensorMap* map, void* base, int elem_bytes, uint64_t cols,
                             uint64_t rows, uint64_t groups, uint64_t row_stride_bytes,
                             uint64_t group_stride_bytes) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  std::memset(map, 0, sizeof(*map));
  if (groups < 1) groups = 1;
  if (group_stride_bytes == 0) group_stride_bytes = rows * row_stride_bytes;
  if (group_stride_bytes == 0) group_stride_bytes = 16;
  cuuint64_t dims[3] = {cols, rows, groups};
  cuuint64_t strides[2] = {row_stride_bytes, group_stride_bytes};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const bool f32 = elem_bytes == 4;
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base,
                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace flame
