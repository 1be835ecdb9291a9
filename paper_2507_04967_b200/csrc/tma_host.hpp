// Host-side TMA descriptor construction (cuTensorMapEncodeTiled through the runtime's driver
// entry point, so the library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "dtype.hpp"
#include <cstdint>
#include <stdexcept>
#include <string>

namespace iolmh {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D K-major operand [rows x inner] with a row stride in bytes; box = 128 bytes of inner x box_rows,
// SWIZZLE_128B (matches smem_desc_k_sw128 on the device). Out-of-bounds elements read as zero.
inline CUtensorMap make_kmajor_map(const void* ptr, CUtensorMapDataType dt, int elem_bytes,
                                   uint64_t inner, uint64_t rows, uint64_t row_stride_bytes,
                                   uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / elem_bytes), box_rows};
  cuuint32_t es[2] = {1, 1};
  if ((row_stride_bytes % 16) != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
    throw std::runtime_error("TMA operand must be 16-byte aligned with a 16-byte row stride");
  CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed with code " + std::to_string(r));
  return m;
}

// fp16 row tensor [rows x inner] read in boxes of box_inner elements x box_rows, swizzled over the
// box's row span (128/64/32 B -> SWIZZLE_128B/64B/32B). Used by the prefill attention for the q
// buffer and the paged KV pool.
inline CUtensorMap make_rows_map_h16(const void* ptr, uint64_t inner, uint64_t rows, uint64_t row_stride_bytes,
                                      uint32_t box_inner, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t es[2] = {1, 1};
  const uint32_t span = box_inner * 2;
  const CUtensorMapSwizzle sw = span == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : span == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : span == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                             : CU_TENSOR_MAP_SWIZZLE_NONE;
  if (sw == CU_TENSOR_MAP_SWIZZLE_NONE || (row_stride_bytes % 16) != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
    throw std::runtime_error("row TMA map: unsupported box width or misaligned tensor");
  CUresult r = encode_fn()(&m, H16_TMA, 2, const_cast<void*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed with code " + std::to_string(r));
  return m;
}

// Packed int4 weights [rows x ceil(K/2) bytes] (two codes per byte, low nibble = even column: the
// bundle's q4 layout, model.cpp:164-176) read in unswizzled boxes of 32 bytes (64 codes) x 128 rows.
// Out-of-bounds bytes read as 0 (codes -8): they only ever meet zero-filled activations (k >= K) or
// output columns the epilogue masks (n >= N).
inline CUtensorMap make_w4_map(const void* ptr, uint64_t K, uint64_t rows, uint64_t row_stride_bytes) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(K + 1) / 2, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  if ((row_stride_bytes % 16) != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
    throw std::runtime_error("int4 weight map must be 16-byte aligned with a 16-byte row stride");
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled (int4 weights) failed with code " + std::to_string(r));
  return m;
}

// GEMM output boxes of 32 x 32 for the TMA epilogue: fp32 [rows x cols] with SWIZZLE_128B (the
// epilogue's swz() staging layout), fp16 [rows x cols] with SWIZZLE_64B.
inline CUtensorMap make_out_map(const void* ptr, bool f32, uint64_t cols, uint64_t rows, uint64_t row_stride_bytes) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  if ((row_stride_bytes % 16) != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
    throw std::runtime_error("output map must be 16-byte aligned with a 16-byte row stride");
  CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : H16_TMA, 2,
                           const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (GEMM output) failed: " + std::to_string(r));
  return m;
}

// Residual stream x (fp32 [rows x cols]) as the target of the 2:4 GEMM's TMA reduce-add epilogue:
// boxes of 32 channels x 8 tokens, no swizzle (the staging tile is plain row-major [8][32] floats).
inline CUtensorMap make_resid_map(const float* ptr, uint64_t cols, uint64_t rows, uint64_t row_stride_bytes) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {32, 8};
  cuuint32_t es[2] = {1, 1};
  if ((row_stride_bytes % 16) != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
    throw std::runtime_error("residual map must be 16-byte aligned with a 16-byte row stride");
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (residual) failed: " + std::to_string(r));
  return m;
}

}  // namespace iolmh
