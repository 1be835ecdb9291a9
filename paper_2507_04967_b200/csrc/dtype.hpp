// The 16-bit element type of every GEMM operand, KV page, attention operand (q, K, V, P) and
// intermediate activation the engine stores (h, q, z, g): IEEE binary16. fp16 carries 3 more
// mantissa bits than fp16 (relative rounding 2^-11 vs 2^-8) at the same tensor-core rate and the
// same bytes, so the GPU path stays ~8x closer to the reference's f32 arithmetic (BASELINE.json:
// "rel <= 1e-2 in fp16/fp16"); activations of these models stay far inside its range (|x| < 65504).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

using h16 = __half;
using h16x2 = __half2;
// tcgen05 instruction descriptor a/b format of kind::f16 for h16 operands (0 = f16, 1 = fp16)
constexpr unsigned H16_FMT = 0;
#define H16_TMA CU_TENSOR_MAP_DATA_TYPE_FLOAT16

// Host: IEEE binary16 bit pattern of a small integer (|v| <= 2048 is exact).
inline unsigned short f16_bits_of_int(int v) {
  if (v == 0) return 0;
  const unsigned short sign = v < 0 ? 0x8000 : 0;
  unsigned a = static_cast<unsigned>(v < 0 ? -v : v);
  int e = 0;
  while ((a >> e) > 1) ++e;  // a in [2^e, 2^(e+1))
  const unsigned mant = (a << (10 - e)) & 0x3FF;
  return static_cast<unsigned short>(sign | ((e + 15) << 10) | mant);
}
