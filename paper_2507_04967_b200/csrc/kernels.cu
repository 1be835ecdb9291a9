// Non-GEMM kernels of the prompt() hot path on sm_100a:
//   embed_ln_kernel   x = tok_embed[id] + pos_embed[pos]; h = LN1(x)       (runtime.cpp:122-141)
//   ln_kernel         h = LN(x) -> fp16 GEMM operand                        (numerics.cpp:158-177)
//   attn_prefill      causal flash attention over paged KV, mma.sync tiles  (runtime.cpp:152-174)
//   attn_decode       one query per sequence, split by absolute 32-key chunks
//   head_argmax       final LN + tied head (fp32) + greedy argmax           (runtime.cpp:202-215,
//                                                                            numerics.cpp:190-197)
//   lcp / decode helpers
#include <algorithm>
#include <cstdlib>
#include <cfloat>
#include <cmath>

#include "kernels.cuh"
#include "launch.hpp"
#include "ptx.cuh"

namespace iolmk {

constexpr int PAGE = 16;

// ------------------------------------------------------------------ per-token int8 (W8A8)
// Activation quantization rule (the reference has none; modelled on its RTN weight
// rule, quant.cpp:23-38, applied per token): s = amax/127 (amax == 0 -> 1), inv = 1/s (IEEE fp32),
// q = clamp(rint(x * inv)) with the fp32 product rounded to nearest-even. |x * inv| <= 127 * (1 +
// 2^-22), so the clamp never clips a code. Restated bit-for-bit in oracle/iolm_oracle.c
// orc_quant_rows_s8. Evaluated on the FMA/ALU pipes instead of the XU
// (cvt.rni.sat.s8.f32 is an XU conversion at a quarter of the FMA rate): after the clamp to
// [-128, 127], adding 1.5 * 2^23 rounds to the nearest integer with ties to even (the sum's ulp is 1)
// and leaves the two's-complement code in the low byte of the sum's bit pattern - the same result
// as cvt.rni.sat.s8.f32 for every finite input.
__device__ __forceinline__ int8_t quant_one(float x, float /*s*/, float inv_s) {
  const float y = fminf(fmaxf(x * inv_s, -128.f), 127.f);
  return static_cast<int8_t>(__float_as_int(__fadd_rn(y, 12582912.f)) & 0xff);
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------------------------ LayerNorm
// One warp per row. Two-pass mean / variance in fp32 over the row held in registers. Writes the
// fp16 GEMM operand, or (Q8) per-token int8 codes + the row scale for the W8A8 GEMMs.
template <int MAXV>
__device__ __forceinline__ void ln_load_row(const float* __restrict__ xr, int d, int lane, float4 (&v)[MAXV]) {
  const int nv = d >> 2;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) v[i] = reinterpret_cast<const float4*>(xr)[idx];
  }
}

template <int MAXV, bool Q8 = false>
__device__ __forceinline__ void ln_finish_row(float4 (&v)[MAXV], int d, const float* __restrict__ g,
                                              const float* __restrict__ b, h16* __restrict__ hr,
                                              int lane, int8_t* __restrict__ q8 = nullptr,
                                              float* __restrict__ qscale = nullptr);

template <int MAXV, bool Q8 = false>
__device__ __forceinline__ void ln_row_warp(const float* __restrict__ xr, int d, const float* __restrict__ g,
                                            const float* __restrict__ b, h16* __restrict__ hr,
                                            int lane, int8_t* __restrict__ q8 = nullptr,
                                            float* __restrict__ qscale = nullptr) {
  float4 v[MAXV];
  ln_load_row<MAXV>(xr, d, lane, v);
  ln_finish_row<MAXV, Q8>(v, d, g, b, hr, lane, q8, qscale);
}

template <int MAXV, bool Q8>
__device__ __forceinline__ void ln_finish_row(float4 (&v)[MAXV], int d, const float* __restrict__ g,
                                              const float* __restrict__ b, h16* __restrict__ hr,
                                              int lane, int8_t* __restrict__ q8, float* __restrict__ qscale) {
  const int nv = d >> 2;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / static_cast<float>(d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int idx = lane + 32 * i;
    if (idx < nv) {
      const float a = v[i].x - mean, bb = v[i].y - mean, c = v[i].z - mean, e = v[i].w - mean;
      q += (a * a + bb * bb) + (c * c + e * e);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float inv = 1.0f / sqrtf(q / static_cast<float>(d) + 1e-5f);
  if constexpr (Q8) {
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int idx = lane + 32 * i;
      if (idx < nv) {
        const float4 gg = reinterpret_cast<const float4*>(g)[idx];
        const float4 bb = reinterpret_cast<const float4*>(b)[idx];
        v[i].x = (v[i].x - mean) * inv * gg.x + bb.x;
        v[i].y = (v[i].y - mean) * inv * gg.y + bb.y;
        v[i].z = (v[i].z - mean) * inv * gg.z + bb.z;
        v[i].w = (v[i].w - mean) * inv * gg.w + bb.w;
        amax = fmaxf(fmaxf(amax, fmaxf(fabsf(v[i].x), fabsf(v[i].y))), fmaxf(fabsf(v[i].z), fabsf(v[i].w)));
      }
    }
    amax = warp_max(amax);
    const float s = amax == 0.f ? 1.f : amax / 127.0f;
    const float sd = s;
    const float inv_sd = 1.0f / s;
    if (lane == 0) *qscale = s;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int idx = lane + 32 * i;
      if (idx < nv) {
        char4 c;
        c.x = quant_one(v[i].x, sd, inv_sd);
        c.y = quant_one(v[i].y, sd, inv_sd);
        c.z = quant_one(v[i].z, sd, inv_sd);
        c.w = quant_one(v[i].w, sd, inv_sd);
        reinterpret_cast<char4*>(q8)[idx] = c;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int idx = lane + 32 * i;
      if (idx < nv) {
        const float4 gg = reinterpret_cast<const float4*>(g)[idx];
        const float4 bb = reinterpret_cast<const float4*>(b)[idx];
        uint2 w;
        w.x = pack_h16x2((v[i].x - mean) * inv * gg.x + bb.x, (v[i].y - mean) * inv * gg.y + bb.y);
        w.y = pack_h16x2((v[i].z - mean) * inv * gg.z + bb.z, (v[i].w - mean) * inv * gg.w + bb.w);
        reinterpret_cast<uint2*>(hr)[idx] = w;
      }
    }
  }
}

// 4 resident CTAs (32 rows in flight per SM): the kernel is bound by the latency of its row loads
// (ncu: 65% long-scoreboard stalls at 3 CTAs / 24 warps), so the register cap buys occupancy.
template <int MAXV, bool Q8>
__global__ void __launch_bounds__(256, MAXV <= 10 ? 4 : 2) ln_kernel(const float* __restrict__ x, int M, int d,
                                                 const float* __restrict__ g, const float* __restrict__ b,
                                                 h16* __restrict__ h, int ldh, int8_t* __restrict__ q8,
                                                 float* __restrict__ qscale) {
  pdl_sync();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= M) return;
  if constexpr (Q8)
    ln_row_warp<MAXV, true>(x + static_cast<size_t>(row) * d, d, g, b, nullptr, threadIdx.x & 31,
                            q8 + static_cast<size_t>(row) * ldh, qscale + row);
  else
    ln_row_warp<MAXV>(x + static_cast<size_t>(row) * d, d, g, b, h + static_cast<size_t>(row) * ldh,
                      threadIdx.x & 31);
}

// Streaming LayerNorm: persistent warps walk rows gw, gw + nw, ... and load row i+1 into registers
// before normalising row i, so every warp always has a row's loads in flight (the one-row-per-warp
// kernel above idles its memory traffic during each row's reductions). Same arithmetic.
// gb_smem: the gain / bias rows are first copied to shared memory (every row re-reads them: 2 x d
// floats per row from L1 otherwise), dynamic smem = 2 d floats.
__device__ __forceinline__ void ln_stage_gb(const float*& g, const float*& b, int d, int gb_smem) {
  if (!gb_smem) return;
  extern __shared__ __align__(16) float ln_gb[];
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    ln_gb[i] = g[i];
    ln_gb[d + i] = b[i];
  }
  __syncthreads();
  g = ln_gb;
  b = ln_gb + d;
}

template <int MAXV, bool Q8>
__global__ void __launch_bounds__(256, 2) ln_stream_kernel(const float* __restrict__ x, int M, int d,
                                                           const float* g, const float* b,
                                                           h16* __restrict__ h, int ldh,
                                                           int8_t* __restrict__ q8, float* __restrict__ qscale,
                                                           int gb_smem) {
  pdl_sync();
  ln_stage_gb(g, b, d, gb_smem);
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * 8;
  int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  float4 cur[MAXV], nxt[MAXV];
  if (row < M) ln_load_row<MAXV>(x + static_cast<size_t>(row) * d, d, lane, cur);
  for (; row < M; row += nw) {
    const int nrow = row + nw;
    if (nrow < M) ln_load_row<MAXV>(x + static_cast<size_t>(nrow) * d, d, lane, nxt);
    if constexpr (Q8)
      ln_finish_row<MAXV, true>(cur, d, g, b, nullptr, lane, q8 + static_cast<size_t>(row) * ldh, qscale + row);
    else
      ln_finish_row<MAXV>(cur, d, g, b, h + static_cast<size_t>(row) * ldh, lane);
#pragma unroll
    for (int i = 0; i < MAXV; ++i) cur[i] = nxt[i];
  }
}

// Wide-row streaming LayerNorm (d = 2048-4096): a PAIR of warps owns each row (64 threads,
// float4 index t + 64 i), so the per-thread row slice and its prefetched successor fit in registers
// at 2 CTAs x 8 warps per SM. Partial sums are combined through shared memory under a 64-thread
// named barrier per pair (ids 1-4); the arithmetic per element is the one-warp kernel's.
template <int MAXV, bool Q8>
__global__ void __launch_bounds__(256, 2) ln_stream2_kernel(const float* __restrict__ x, int M, int d,
                                                            const float* g, const float* b,
                                                            h16* __restrict__ h, int ldh,
                                                            int8_t* __restrict__ q8, float* __restrict__ qscale,
                                                            int gb_smem) {
  pdl_sync();
  ln_stage_gb(g, b, d, gb_smem);
  __shared__ float red[4][2][3][2];  // [pair][row parity][reduction][half]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1, t = half * 32 + lane;
  const int nv = d >> 2;
  const int np = gridDim.x * 4;
  auto pair_sum = [&](float v, int par, int k, bool is_max) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float w = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmaxf(v, w) : v + w;
    }
    if (lane == 0) red[pair][par][k][half] = v;
    asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
    const float a = red[pair][par][k][0], c = red[pair][par][k][1];
    return is_max ? fmaxf(a, c) : a + c;  // same order in both warps: identical result
  };
  auto load = [&](int row, float4 (&v)[MAXV]) {
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(row) * d);
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
      const int idx = t + 64 * i;
      if (idx < nv) v[i] = xr[idx];
    }
  };
  float4 cur[MAXV], nxt[MAXV];
  int row = blockIdx.x * 4 + pair, par = 0;
  if (row < M) load(row, cur);
  for (; row < M; row += np, par ^= 1) {
    if (row + np < M) load(row + np, nxt);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i)
      if (t + 64 * i < nv) s += (cur[i].x + cur[i].y) + (cur[i].z + cur[i].w);
    const float mean = pair_sum(s, par, 0, false) / static_cast<float>(d);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < MAXV; ++i)
      if (t + 64 * i < nv) {
        const float a = cur[i].x - mean, bb = cur[i].y - mean, c = cur[i].z - mean, e = cur[i].w - mean;
        q += (a * a + bb * bb) + (c * c + e * e);
      }
    const float inv = 1.0f / sqrtf(pair_sum(q, par, 1, false) / static_cast<float>(d) + 1e-5f);
    if constexpr (Q8) {
      float amax = 0.f;
#pragma unroll
      for (int i = 0; i < MAXV; ++i) {
        const int idx = t + 64 * i;
        if (idx < nv) {
          const float4 gg = reinterpret_cast<const float4*>(g)[idx];
          const float4 bb = reinterpret_cast<const float4*>(b)[idx];
          cur[i].x = (cur[i].x - mean) * inv * gg.x + bb.x;
          cur[i].y = (cur[i].y - mean) * inv * gg.y + bb.y;
          cur[i].z = (cur[i].z - mean) * inv * gg.z + bb.z;
          cur[i].w = (cur[i].w - mean) * inv * gg.w + bb.w;
          amax = fmaxf(fmaxf(amax, fmaxf(fabsf(cur[i].x), fabsf(cur[i].y))), fmaxf(fabsf(cur[i].z), fabsf(cur[i].w)));
        }
      }
      amax = pair_sum(amax, par, 2, true);
      const float sd = amax == 0.f ? 1.f : amax / 127.0f;
      const float inv_sd = 1.0f / sd;
      if (t == 0) qscale[row] = sd;
      char4* qr = reinterpret_cast<char4*>(q8 + static_cast<size_t>(row) * ldh);
#pragma unroll
      for (int i = 0; i < MAXV; ++i) {
        const int idx = t + 64 * i;
        if (idx < nv) {
          char4 c;
          c.x = quant_one(cur[i].x, sd, inv_sd);
          c.y = quant_one(cur[i].y, sd, inv_sd);
          c.z = quant_one(cur[i].z, sd, inv_sd);
          c.w = quant_one(cur[i].w, sd, inv_sd);
          qr[idx] = c;
        }
      }
    } else {
      uint2* hr = reinterpret_cast<uint2*>(h + static_cast<size_t>(row) * ldh);
#pragma unroll
      for (int i = 0; i < MAXV; ++i) {
        const int idx = t + 64 * i;
        if (idx < nv) {
          const float4 gg = reinterpret_cast<const float4*>(g)[idx];
          const float4 bb = reinterpret_cast<const float4*>(b)[idx];
          uint2 w;
          w.x = pack_h16x2((cur[i].x - mean) * inv * gg.x + bb.x, (cur[i].y - mean) * inv * gg.y + bb.y);
          w.y = pack_h16x2((cur[i].z - mean) * inv * gg.z + bb.z, (cur[i].w - mean) * inv * gg.w + bb.w);
          hr[idx] = w;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < MAXV; ++i) cur[i] = nxt[i];
  }
}

// Bandwidth-oriented LayerNorm: persistent CTAs, a producer warp streams groups of 8 consecutive x
// rows (one contiguous block) with cp.async.bulk into an LN_STAGES-deep smem ring; each of the 8
// compute warps normalises one row of the group from smem (same arithmetic as ln_row_warp).
constexpr int LN_STAGES = 2;
template <int MAXV, bool Q8>
__global__ void __launch_bounds__(288) ln_bulk_kernel(const float* __restrict__ x, int M, int d,
                                                      const float* __restrict__ g, const float* __restrict__ b,
                                                      h16* __restrict__ h, int ldh, int8_t* __restrict__ q8,
                                                      float* __restrict__ qscale) {
  pdl_sync();
  extern __shared__ __align__(128) uint8_t lsm[];
  const uint32_t sbase = (smem_u32(lsm) + 127u) & ~127u;
  float* ring = reinterpret_cast<float*>(lsm + (sbase - smem_u32(lsm)));
  const int group_floats = 8 * d;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + LN_STAGES * group_floats);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + LN_STAGES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ngroups = (M + 7) / 8;
  if (threadIdx.x == 0) {
    for (int s = 0; s < LN_STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      int it = 0;
      for (int gi = blockIdx.x; gi < ngroups; gi += gridDim.x, ++it) {
        const int s = it % LN_STAGES;
        mbar_wait(empty0 + 8 * s, ((it / LN_STAGES) & 1) ^ 1u);
        const int rows = min(8, M - gi * 8);
        const uint32_t bytes = static_cast<uint32_t>(rows) * d * 4;
        mbar_expect_tx(full0 + 8 * s, bytes);
        bulk_load(smem_u32(ring + s * group_floats), x + static_cast<size_t>(gi) * 8 * d, bytes, full0 + 8 * s);
      }
    }
    return;
  }
  int it = 0;
  for (int gi = blockIdx.x; gi < ngroups; gi += gridDim.x, ++it) {
    const int s = it % LN_STAGES;
    mbar_wait(full0 + 8 * s, (it / LN_STAGES) & 1);
    const int row = gi * 8 + warp;
    if (row < M) {
      const float* xr = ring + s * group_floats + warp * d;
      if constexpr (Q8)
        ln_row_warp<MAXV, true>(xr, d, g, b, nullptr, lane, q8 + static_cast<size_t>(row) * ldh, qscale + row);
      else
        ln_row_warp<MAXV>(xr, d, g, b, h + static_cast<size_t>(row) * ldh, lane);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
  }
}

// Per-token int8 quantization of a fp16 activation matrix (attention output z, GELU output g).
// One warp per row. CH > 0: the row (cols = 256*CH, multiple of 8) stays in registers between the
// amax and the code pass; CH == 0: generic two-pass version (any width).
template <int CH>
__global__ void __launch_bounds__(256, CH == 0 ? 8 : 4) quant_rows_kernel(const h16* __restrict__ src, int lds, int M,
                                                         int cols, int8_t* __restrict__ dst, int ldd,
                                                         float* __restrict__ scale) {
  pdl_sync();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= M) return;
  const int lane = threadIdx.x & 31;
  const h16* r = src + static_cast<size_t>(row) * lds;
  int8_t* o = dst + static_cast<size_t>(row) * ldd;
  if constexpr (CH > 0) {
    uint4 u[CH];
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int c = (lane + 32 * i) * 8;
      u[i] = c < cols ? *reinterpret_cast<const uint4*>(r + c) : make_uint4(0, 0, 0, 0);
      const h16x2* h2 = reinterpret_cast<const h16x2*>(&u[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h2[j]);
        amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
      }
    }
    amax = warp_max(amax);
    const float sd = amax == 0.f ? 1.f : amax / 127.0f;
    const float inv_sd = 1.0f / sd;
    if (lane == 0) scale[row] = sd;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c >= cols) break;
      const h16x2* h2 = reinterpret_cast<const h16x2*>(&u[i]);
      uint2 w;
      int8_t* wb = reinterpret_cast<int8_t*>(&w);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h2[j]);
        wb[2 * j] = quant_one(f.x, sd, inv_sd);
        wb[2 * j + 1] = quant_one(f.y, sd, inv_sd);
      }
      *reinterpret_cast<uint2*>(o + c) = w;
    }
  } else {
    const int cols8 = cols & ~7;
    float amax = 0.f;
    for (int c = cols8 + lane; c < cols; c += 32) amax = fmaxf(amax, fabsf(__half2float(r[c])));
    for (int c = lane * 8; c < cols8; c += 256) {
      const uint4 u = *reinterpret_cast<const uint4*>(r + c);
      const h16x2* h2 = reinterpret_cast<const h16x2*>(&u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h2[j]);
        amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
      }
    }
    amax = warp_max(amax);
    const float sd = amax == 0.f ? 1.f : amax / 127.0f;
    const float inv_sd = 1.0f / sd;
    if (lane == 0) scale[row] = sd;
    for (int c = cols8 + lane; c < cols; c += 32) o[c] = quant_one(__half2float(r[c]), sd, inv_sd);
    for (int c = lane * 8; c < cols8; c += 256) {
      const uint4 u = *reinterpret_cast<const uint4*>(r + c);
      const h16x2* h2 = reinterpret_cast<const h16x2*>(&u);
      uint2 w;
      int8_t* wb = reinterpret_cast<int8_t*>(&w);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h2[j]);
        wb[2 * j] = quant_one(f.x, sd, inv_sd);
        wb[2 * j + 1] = quant_one(f.y, sd, inv_sd);
      }
      *reinterpret_cast<uint2*>(o + c) = w;
    }
  }
}

// Wide rows (1024 < cols <= 4096, cols % 8 == 0): a pair of warps per row, the row slice and the
// next row's slice in registers (16-B chunks t + 64 i), amax combined under a 64-thread named barrier.
// Same per-element rule as quant_rows_kernel.
template <int CH>
__global__ void __launch_bounds__(256, 2) quant_rows2_kernel(const h16* __restrict__ src, int lds, int M,
                                                             int cols, int8_t* __restrict__ dst, int ldd,
                                                             float* __restrict__ scale) {
  pdl_sync();
  __shared__ float red[4][2][2];  // [pair][row parity][half]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1, t = half * 32 + lane;
  const int nch = cols >> 3;  // 16-byte chunks per row
  const int np = gridDim.x * 4;
  auto load = [&](int row, uint4 (&u)[CH]) {
    const uint4* r = reinterpret_cast<const uint4*>(src + static_cast<size_t>(row) * lds);
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int c = t + 64 * i;
      u[i] = c < nch ? r[c] : make_uint4(0, 0, 0, 0);
    }
  };
  uint4 cur[CH], nxt[CH];
  int row = blockIdx.x * 4 + pair, par = 0;
  if (row < M) load(row, cur);
  for (; row < M; row += np, par ^= 1) {
    if (row + np < M) load(row + np, nxt);
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const h16x2* h2 = reinterpret_cast<const h16x2*>(&cur[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(h2[j]);
        amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
      }
    }
    amax = warp_max(amax);
    if (lane == 0) red[pair][par][half] = amax;
    asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
    amax = fmaxf(red[pair][par][0], red[pair][par][1]);
    const float sd = amax == 0.f ? 1.f : amax / 127.0f;
    const float inv_sd = 1.0f / sd;
    if (t == 0) scale[row] = sd;
    uint2* o = reinterpret_cast<uint2*>(dst + static_cast<size_t>(row) * ldd);
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int c = t + 64 * i;
      if (c < nch) {
        const h16x2* h2 = reinterpret_cast<const h16x2*>(&cur[i]);
        uint2 w;
        int8_t* wb = reinterpret_cast<int8_t*>(&w);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __half22float2(h2[j]);
          wb[2 * j] = quant_one(f.x, sd, inv_sd);
          wb[2 * j + 1] = quant_one(f.y, sd, inv_sd);
        }
        o[c] = w;
      }
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) cur[i] = nxt[i];
  }
}

// token id of step row m: prompt tokens come from the id table, generated tokens from the
// per-slot "last token" register written by head_argmax_kernel.
template <int MAXV, bool Q8>
__global__ void __launch_bounds__(256)
    embed_ln_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ tok_src,
                    const int* __restrict__ tok_slot, const int* __restrict__ tok_pos,
                    const int32_t* __restrict__ last_tok, int M, int d, const float* __restrict__ tok_embed,
                    const float* __restrict__ pos_embed, float* __restrict__ x, const float* __restrict__ g,
                    const float* __restrict__ b, h16* __restrict__ h, int ldh, int8_t* __restrict__ q8,
                    float* __restrict__ qscale) {
  pdl_sync();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= M) return;
  const int lane = threadIdx.x & 31;
  const int64_t src = tok_src[row];
  const int id = src >= 0 ? ids[src] : last_tok[tok_slot[row]];
  const float4* te = reinterpret_cast<const float4*>(tok_embed + static_cast<size_t>(id) * d);
  const float4* pe = reinterpret_cast<const float4*>(pos_embed + static_cast<size_t>(tok_pos[row]) * d);
  float4* xr = reinterpret_cast<float4*>(x + static_cast<size_t>(row) * d);
  for (int i = lane; i < (d >> 2); i += 32) {
    const float4 a = te[i], c = pe[i];
    xr[i] = make_float4(a.x + c.x, a.y + c.y, a.z + c.z, a.w + c.w);
  }
  __syncwarp();
  if constexpr (Q8)
    ln_row_warp<MAXV, true>(x + static_cast<size_t>(row) * d, d, g, b, nullptr, lane,
                            q8 + static_cast<size_t>(row) * ldh, qscale + row);
  else
    ln_row_warp<MAXV>(x + static_cast<size_t>(row) * d, d, g, b, h + static_cast<size_t>(row) * ldh, lane);
}

// ------------------------------------------------------------------ attention (prefill, mma.sync)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma_h16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 64 queries of one group x one head per CTA (4 warps x 16 query rows). Keys stream in blocks of
// PF_KB = 32 absolute positions (two KV pages): thread 0 issues one TMA per page slab (the pool is a
// 2D tensor of HD-wide rows, swizzled like the GEMM operands) into a PF_ST-deep ring with mbarrier
// completion, so no thread computes a load address and no warp waits on another at a CTA barrier.
// Work is skipped per 16-key chunk (one page) beyond a warp's last query, and the causal mask is
// applied only in chunks that straddle the diagonal. A query's arithmetic depends only on its own
// position and the K/V values (chunks are aligned to absolute positions): batch-invariant.
constexpr int PF_KB = 32;
template <int HD>
struct PfCfg {
  static constexpr int CB = HD < 64 ? HD : 64;   // elements per TMA box row (<= 128 B)
  static constexpr int CBB = CB * 2;             // bytes per box row = swizzle span
  static constexpr int NCB = HD / CB;            // boxes per HD-wide row
  static constexpr uint32_t SWM = CBB == 128 ? 7 : (CBB == 64 ? 3 : 1);
  static constexpr int ST = HD >= 128 ? 3 : 4;   // ring depth (blocks in flight)
  static constexpr int MINB = HD >= 128 ? 3 : 5; // resident CTAs per SM (smem-limited)
  static constexpr uint32_t Q_BYTES = 64 * HD * 2;
  static constexpr uint32_t KT_BYTES = PF_KB * HD * 2;  // one K (or V) tile
  static constexpr uint32_t STAGE_BYTES = 2 * KT_BYTES;
  static constexpr size_t SMEM = 1024 + Q_BYTES + ST * STAGE_BYTES + 64;
};

// Byte offset of element (r, c) in a [R x HD] fp16 tile stored as NCB swizzled [R x CB] boxes.
template <int HD>
__device__ __forceinline__ uint32_t pf_off(int R, int r, int c) {
  using C = PfCfg<HD>;
  const uint32_t b = static_cast<uint32_t>(c / C::CB) * R * C::CBB + r * C::CBB + (c % C::CB) * 2;
  return b ^ (((b >> 7) & C::SWM) << 4);
}

template <int HD, bool MASK>
__global__ void __launch_bounds__(128, PfCfg<HD>::MINB) attn_prefill_kernel(const __grid_constant__ AttnParams p) {
  pdl_sync();
  using C = PfCfg<HD>;
  constexpr int ST = C::ST;
  extern __shared__ __align__(1024) uint8_t pf_smem[];
  const uint32_t sraw = smem_u32(pf_smem);
  const uint32_t sQ = (sraw + 1023u) & ~1023u;
  uint8_t* gQ = pf_smem + (sQ - sraw);
  const uint32_t sKV = sQ + C::Q_BYTES;
  const uint32_t bars = sKV + ST * C::STAGE_BYTES;  // full[ST], empty[ST], q
  const AttnGroup grp = p.groups[blockIdx.x];
  const int head = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int last_key = grp.pos0 + grp.nq - 1;
  const int nblocks = last_key / PF_KB + 1;
  const int* pt = p.page_table + static_cast<size_t>(grp.slot) * p.max_pages;

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(bars + 8 * s, 1);
      mbar_init(bars + 8 * (ST + s), 4);
    }
    mbar_init(bars + 16 * ST, 1);
    mbar_fence_init();
  }
  __syncthreads();

  // warp 0 is also the producer: lanes hold 32 page ids at a time, lane 0 issues the TMAs
  int pid_base = -(1 << 20), pid = 0;
  auto issue_block = [&](int kb) {
    const uint32_t full = bars + 8 * (kb % ST);
    const uint32_t dst = sKV + (kb % ST) * C::STAGE_BYTES;
    const int pg0 = kb * (PF_KB / PAGE);
    const int npg = min(PF_KB / PAGE, last_key / PAGE - pg0 + 1);
    if (pg0 + npg > pid_base + 32 || pg0 < pid_base) {
      pid_base = pg0;
      pid = pid_base + lane < p.max_pages ? __ldg(pt + pid_base + lane) : 0;
    }
    if (lane == 0) mbar_expect_tx(full, npg * 2 * PAGE * HD * 2);
    for (int j = 0; j < npg; ++j) {
      const int page = __shfl_sync(0xffffffffu, pid, pg0 + j - pid_base);
      if (lane == 0) {
        const int rk = ((page * 2 + 0) * p.heads + head) * PAGE;
        const int rv = rk + p.heads * PAGE;
#pragma unroll
        for (int cb = 0; cb < C::NCB; ++cb) {
          const uint32_t o = cb * PF_KB * C::CBB + j * PAGE * C::CBB;
          tma_load_2d(dst + o, &p.kv_map, full, cb * C::CB, rk);
          tma_load_2d(dst + C::KT_BYTES + o, &p.kv_map, full, cb * C::CB, rv);
        }
      }
    }
  };
  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&p.kv_map);
      mbar_expect_tx(bars + 16 * ST, C::Q_BYTES);
#pragma unroll
      for (int cb = 0; cb < C::NCB; ++cb)
        tma_load_2d(sQ + cb * 64 * C::CBB, &p.q_map, bars + 16 * ST, head * HD + cb * C::CB, grp.m0);
    }
    for (int kb = 0; kb < min(ST, nblocks); ++kb) issue_block(kb);
  }

  const int qrow0 = warp * 16 + gq;  // this thread's rows qrow0 and qrow0 + 8
  const int qpos0 = grp.pos0 + qrow0, qpos1 = qpos0 + 8;
  const bool warp_active = warp * 16 < grp.nq;
  const int warp_min_pos = grp.pos0 + warp * 16;
  const int warp_max_pos = grp.pos0 + min(grp.nq - 1, warp * 16 + 15);
  float m_i[2] = {-INFINITY, -INFINITY};
  float l_i[2] = {0.f, 0.f};
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  uint32_t qf[HD / 16][4];
  if (warp_active) {
    mbar_wait(bars + 16 * ST, 0);
#pragma unroll
    for (int kc = 0; kc < HD / 16; ++kc)
      ldsm_x4(qf[kc], gQ + pf_off<HD>(64, warp * 16 + (lane & 15), kc * 16 + (lane >> 4) * 8));
  }

  for (int kb = 0; kb < nblocks; ++kb) {
    if (warp == 0 && kb >= 1 && kb - 1 + ST < nblocks) {
      // refill the stage block kb-1 used once every warp has released it
      mbar_wait(bars + 8 * (ST + (kb - 1) % ST), ((kb - 1) / ST) & 1);
      issue_block(kb - 1 + ST);
    }
    mbar_wait(bars + 8 * (kb % ST), (kb / ST) & 1);
    const int key0 = kb * PF_KB;
    if (warp_active && key0 <= warp_max_pos) {  // warp-uniform
      const uint8_t* sK = pf_smem + (sKV + (kb % ST) * C::STAGE_BYTES - sraw);
      const uint8_t* sV = sK + C::KT_BYTES;
      const bool need1 = key0 + 16 <= warp_max_pos;  // second 16-key chunk visible to this warp
      float s[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < HD / 16; ++kc) {
#pragma unroll
        for (int np = 0; np < 2; ++np) {
          if (np == 1 && !need1) break;
          uint32_t b[4];
          ldsm_x4(b, sK + pf_off<HD>(PF_KB, np * 16 + (lane & 7) + (lane >> 4) * 8, kc * 16 + ((lane >> 3) & 1) * 8));
          mma_h16(s[2 * np], qf[kc], b[0], b[1]);
          mma_h16(s[2 * np + 1], qf[kc], b[2], b[3]);
        }
      }
      // chunks entirely at or below the warp's first query need no causal mask (warp-uniform)
      const bool full0 = !MASK && key0 + 15 <= warp_min_pos;
      const bool full1 = !MASK && key0 + 31 <= warp_min_pos;
      float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const bool full = nt < 2 ? full0 : full1;
        if (nt >= 2 && !need1) {
#pragma unroll
          for (int e = 0; e < 4; ++e) s[nt][e] = -INFINITY;
          continue;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = s[nt][e];
          if (!full) {
            const int key = key0 + nt * 8 + 2 * tq + (e & 1);
            bool ok = key <= (e < 2 ? qpos0 : qpos1);
            if (MASK) ok = ok && key <= last_key && p.key_mask[key];
            v = ok ? v : -INFINITY;
            s[nt][e] = v;
          }
          mx[e >> 1] = fmaxf(mx[e >> 1], v);
        }
      }
      float alpha[2], msub[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
        const float mnew = fmaxf(m_i[r], mx[r] * p.scale_log2);
        alpha[r] = mnew == -INFINITY ? 1.f : ex2_approx(m_i[r] - mnew);
        m_i[r] = mnew;
        l_i[r] *= alpha[r];
        // rows with no visible key yet contribute exact zeros: ex2(-inf) = +0
        msub[r] = mnew == -INFINITY ? 0.f : mnew;
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        if (nt >= 2 && !need1) break;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float pv = ex2_approx(fmaf(s[nt][e], p.scale_log2, -msub[e >> 1]));
          s[nt][e] = pv;
          l_i[e >> 1] += pv;
        }
      }
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        o[i][0] *= alpha[0];
        o[i][1] *= alpha[0];
        o[i][2] *= alpha[1];
        o[i][3] *= alpha[1];
      }
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        if (kc == 1 && !need1) break;
        uint32_t a[4];
        a[0] = pack_h16x2(s[2 * kc][0], s[2 * kc][1]);
        a[1] = pack_h16x2(s[2 * kc][2], s[2 * kc][3]);
        a[2] = pack_h16x2(s[2 * kc + 1][0], s[2 * kc + 1][1]);
        a[3] = pack_h16x2(s[2 * kc + 1][2], s[2 * kc + 1][3]);
#pragma unroll
        for (int dn = 0; dn < HD / 16; ++dn) {
          uint32_t b[4];
          ldsm_x4_t(b, sV + pf_off<HD>(PF_KB, kc * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, dn * 16 + (lane >> 4) * 8));
          mma_h16(o[2 * dn], a, b[0], b[1]);
          mma_h16(o[2 * dn + 1], a, b[2], b[3]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bars + 8 * (ST + kb % ST));
  }
  if (!warp_active) return;
  float inv[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    float l = l_i[r];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    inv[r] = l > 0.f ? 1.f / l : 0.f;
  }
  // stage the warp's 16 x HD output tile in its own (consumed) Q rows, then coalesced 16-B stores
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int col = i * 8 + 2 * tq;
    *reinterpret_cast<uint32_t*>(gQ + pf_off<HD>(64, qrow0, col)) = pack_h16x2(o[i][0] * inv[0], o[i][1] * inv[0]);
    *reinterpret_cast<uint32_t*>(gQ + pf_off<HD>(64, qrow0 + 8, col)) = pack_h16x2(o[i][2] * inv[1], o[i][3] * inv[1]);
  }
  __syncwarp();
  constexpr int CPR = HD / 8;  // 16-B chunks per row
#pragma unroll
  for (int it = 0; it < 16 * CPR / 32; ++it) {
    const int idx = it * 32 + lane;
    const int r = idx / CPR, c = (idx % CPR) * 8;
    const int row = warp * 16 + r;
    if (row < grp.nq)
      *reinterpret_cast<uint4*>(p.z + static_cast<size_t>(grp.m0 + row) * p.ldz + head * HD + c) =
          *reinterpret_cast<const uint4*>(gQ + pf_off<HD>(64, row, c));
  }
}

// ------------------------------------------------------------------ attention (decode)
// One CTA per (decode sequence, group of hg heads). A page's K rows for heads h0 .. h0+hg-1 are one
// contiguous run of hg*PAGE pool rows (and so are its V rows), so a producer warp moves each page
// of the group with two swizzled TMA boxes into an nst-deep ring (mbarrier completion) while one
// compute warp per head runs the online softmax on the tensor cores: S^T = K q (m16n8k16 with q as
// the single live B column) and O^T += V^T p^T (V through ldmatrix.trans, p as the live B column),
// so a 16-key page costs 2*HD/16 MMAs and HD/8 ldmatrix per warp instead of per-lane dot products.
// Work is chunked by page (absolute 16-position blocks), so a query's arithmetic never depends on
// the batch composition.
constexpr int DSTAGES_MAX = 4;
template <int HD>
struct DecCfg {
  static constexpr int HG_MAX = HD >= 128 ? 8 : 16;  // heads per CTA = compute warps
  static constexpr size_t smem(int hg, int nst) {
    return 1024 + static_cast<size_t>(nst) * 2 * hg * PAGE * HD * 2 + 16 * DSTAGES_MAX + hg * HD * 2;
  }
};

// Block = hg compute warps (warp h owns head h0+h) + 1 producer warp.
template <int HD>
__global__ void __launch_bounds__(32 * 17) attn_decode_kernel(const __grid_constant__ AttnParams p, int hg,
                                                              int n_hgroups, int nst) {
  pdl_sync();
  using C = PfCfg<HD>;
  extern __shared__ __align__(1024) uint8_t dsm[];
  const uint32_t sraw = smem_u32(dsm);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  uint8_t* gbase = dsm + (sbase - sraw);
  const int R = hg * PAGE;                            // rows of one K (or V) tile
  const uint32_t HALF = static_cast<uint32_t>(R) * HD * 2;
  const uint32_t STAGE = 2 * HALF;
  const uint32_t full0 = sbase + nst * STAGE, empty0 = full0 + 8 * DSTAGES_MAX;
  h16* sOut = reinterpret_cast<h16*>(gbase + nst * STAGE + 16 * DSTAGES_MAX);

  const int gi = blockIdx.x / n_hgroups;
  const int hgi = blockIdx.x - gi * n_hgroups;
  const AttnGroup grp = p.groups[gi];
  const int h0 = hgi * hg;
  const int nh = min(hg, p.heads - h0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int last = grp.pos0;
  const int npages = last / PAGE + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, hg);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == hg) {  // producer: lanes hold 32 page ids at a time, lane 0 issues the boxes
    const int* pt = p.page_table + static_cast<size_t>(grp.slot) * p.max_pages;
    if (lane == 0) tma_prefetch_desc(&p.kvg_map);
    int pid = 0, s = 0;
    uint32_t ph = 0;
    for (int pg = 0; pg < npages; ++pg) {
      if ((pg & 31) == 0) pid = pg + lane < p.max_pages ? __ldg(pt + pg + lane) : 0;
      const int page = __shfl_sync(0xffffffffu, pid, pg & 31);
      if (lane == 0) {
        mbar_wait(empty0 + 8 * s, ph ^ 1u);
        mbar_expect_tx(full0 + 8 * s, STAGE);
        const int rk = (page * 2 * p.heads + h0) * PAGE;
        const int rv = rk + p.heads * PAGE;
        const uint32_t dst = sbase + s * STAGE;
#pragma unroll
        for (int cb = 0; cb < C::NCB; ++cb) {
          tma_load_2d(dst + cb * R * C::CBB, &p.kvg_map, full0 + 8 * s, cb * C::CB, rk);
          tma_load_2d(dst + HALF + cb * R * C::CBB, &p.kvg_map, full0 + 8 * s, cb * C::CB, rv);
        }
      }
      if (++s == nst) s = 0, ph ^= 1u;
    }
    return;
  }

  const int h = warp;  // this warp's head within the group
  const bool active = h < nh;
  const int gq = lane >> 2, tq = lane & 3;
  // q as column 0 of the B operand: lanes with gq == 0 hold dims 16ks + 2tq (+1) and 16ks + 8 + 2tq (+1)
  uint32_t qb[HD / 16][2];
#pragma unroll
  for (int ks = 0; ks < HD / 16; ++ks) qb[ks][0] = qb[ks][1] = 0u;
  if (active && gq == 0) {
    const h16* qr = p.q + static_cast<size_t>(grp.m0) * p.ldq + (h0 + h) * HD;
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      qb[ks][0] = *reinterpret_cast<const uint32_t*>(qr + ks * 16 + 2 * tq);
      qb[ks][1] = *reinterpret_cast<const uint32_t*>(qr + ks * 16 + 8 + 2 * tq);
    }
  }
  float o[HD / 16][4];
#pragma unroll
  for (int i = 0; i < HD / 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m = -INFINITY, l = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int pg = 0; pg < npages; ++pg) {
    mbar_wait(full0 + 8 * s, ph);
    if (active) {
      const uint8_t* sK = gbase + s * STAGE;
      const uint8_t* sV = sK + HALF;
      float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < HD / 16; ++ks) {
        uint32_t a[4];
        ldsm_x4(a, sK + pf_off<HD>(R, h * PAGE + (lane & 15), ks * 16 + (lane >> 4) * 8));
        mma_h16(sc, a, qb[ks][0], qb[ks][1]);
      }
      // lanes tq == 0: sc[0] = score of key gq, sc[2] = score of key gq + 8 (of this page)
      const int key0 = pg * PAGE + gq, key1 = key0 + 8;
      const bool ok0 = key0 <= last && (!p.key_mask || p.key_mask[key0]);
      const bool ok1 = key1 <= last && (!p.key_mask || p.key_mask[key1]);
      const float s0 = ok0 ? sc[0] * p.scale_log2 : -INFINITY;
      const float s1 = ok1 ? sc[2] * p.scale_log2 : -INFINITY;
      float cmax = fmaxf(s0, s1);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, off));
      const float mnew = fmaxf(m, cmax);
      const float alpha = mnew == -INFINITY ? 1.f : ex2_approx(m - mnew);
      const float msub = mnew == -INFINITY ? 0.f : mnew;
      const float p0 = ex2_approx(s0 - msub), p1 = ex2_approx(s1 - msub);
      float psum = p0 + p1;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) psum += __shfl_xor_sync(0xffffffffu, psum, off);
      l = l * alpha + psum;
      m = mnew;
      // p^T as column 0 of the B operand: lane t < 4 needs keys 2t, 2t+1 (b0) and 8+2t, 9+2t (b1)
      const uint32_t pk = pack_h16x2(p0, p1);
      const uint32_t u = __shfl_sync(0xffffffffu, pk, (lane & 3) * 8);
      const uint32_t w = __shfl_sync(0xffffffffu, pk, (lane & 3) * 8 + 4);
      const uint32_t b0 = lane < 4 ? __byte_perm(u, w, 0x5410) : 0u;
      const uint32_t b1 = lane < 4 ? __byte_perm(u, w, 0x7632) : 0u;
#pragma unroll
      for (int mt = 0; mt < HD / 16; ++mt) {
        o[mt][0] *= alpha;
        o[mt][2] *= alpha;
        uint32_t a[4];
        ldsm_x4_t(a, sV + pf_off<HD>(R, h * PAGE + (lane & 7) + (lane >> 4) * 8, mt * 16 + ((lane >> 3) & 1) * 8));
        mma_h16(o[mt], a, b0, b1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
    if (++s == nst) s = 0, ph ^= 1u;
  }
  if (!active) return;
  // lanes tq == 0 hold O[16mt + gq] (o[mt][0]) and O[16mt + gq + 8] (o[mt][2])
  const float inv = l > 0.f ? 1.f / l : 0.f;
  h16* so = sOut + h * HD;
  if (tq == 0) {
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      so[mt * 16 + gq] = __float2half_rn(o[mt][0] * inv);
      so[mt * 16 + gq + 8] = __float2half_rn(o[mt][2] * inv);
    }
  }
  __syncwarp();
  if (lane < HD / 8)
    *reinterpret_cast<uint4*>(p.z + static_cast<size_t>(grp.m0) * p.ldz + (h0 + h) * HD + lane * 8) =
        *reinterpret_cast<const uint4*>(so + lane * 8);
}

// ------------------------------------------------------------------ head + argmax
// 8 rows per CTA: final LN in fp32, logits = y * tok_embed^T with the fp32 embedding (transposed
// copy, coalesced over the vocabulary), greedy argmax (strict >, ties to the lowest id). 8 rows and
// 32-row E^T chunks keep two CTAs per SM (~2000 rows per step = 256 CTAs; 16 rows / 64-row chunks
// left one under-filled CTA per SM). Every logit's k order is unchanged (ascending k).
constexpr int HEAD_ROWS = 8;
constexpr int HEAD_KC = 32;
__global__ void __launch_bounds__(256)
    head_argmax_kernel(const float* __restrict__ x, int d, const int* __restrict__ rows, int n_rows,
                       const float* __restrict__ g, const float* __restrict__ b,
                       const float* __restrict__ embed_t, int V, const int* __restrict__ row_slot,
                       int32_t* __restrict__ next_tok, int32_t* __restrict__ last_tok,
                       float* __restrict__ logits_out) {
  pdl_sync();
  extern __shared__ float sy[];  // [HEAD_ROWS][d] then [HEAD_ROWS][V]
  float* slog = sy + HEAD_ROWS * d;
  const int r0 = blockIdx.x * HEAD_ROWS;
  const int nr = min(HEAD_ROWS, n_rows - r0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < nr; r += 8) {
    const float* xr = x + static_cast<size_t>(rows[r0 + r]) * d;
    float s = 0.f;
    for (int i = lane; i < d; i += 32) s += xr[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s / static_cast<float>(d);
    float q = 0.f;
    for (int i = lane; i < d; i += 32) {
      const float t = xr[i] - mean;
      q += t * t;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = 1.0f / sqrtf(q / static_cast<float>(d) + 1e-5f);
    for (int i = lane; i < d; i += 32) sy[r * d + i] = (xr[i] - mean) * inv * g[i] + b[i];
  }
  for (int r = nr; r < HEAD_ROWS; ++r)
    for (int i = threadIdx.x; i < d; i += blockDim.x) sy[r * d + i] = 0.f;
  __syncthreads();
  // logits = y * E^T: E^T streamed through a 2-stage cp.async ring of KC-row chunks (16-byte
  // copies, the next chunk in flight during the FMAs); each thread owns one vocabulary column and
  // accumulates all HEAD_ROWS rows in fp32, 4 k at a time.
  constexpr int KC = HEAD_KC;
  float* set0 = slog + HEAD_ROWS * V;  // [2][KC][V]
  const int chunk_floats = KC * V;     // multiple of 4 (KC = 32)
  float acc[HEAD_ROWS];
#pragma unroll
  for (int r = 0; r < HEAD_ROWS; ++r) acc[r] = 0.f;
  const int v = threadIdx.x;
  const int nchunks = (d + KC - 1) / KC;
  auto issue = [&](int c) {
    const int k0 = c * KC;
    const int nf = min(KC, d - k0) * V;  // d % 4 == 0, V*kc*4 bytes 16-aligned when kc % 4 == 0
    float* dst = set0 + (c & 1) * chunk_floats;
    const float* src = embed_t + static_cast<size_t>(k0) * V;
    for (int i = threadIdx.x * 4; i < nf; i += blockDim.x * 4) cp_async16(dst + i, src + i, true);
    cp_async_commit();
  };
  issue(0);
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      issue(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int k0 = c * KC;
    const int kc = min(KC, d - k0);
    const float* set = set0 + (c & 1) * chunk_floats;
    if (v < V) {
      for (int k = 0; k < kc; k += 4) {
        const float e0 = set[k * V + v], e1 = set[(k + 1) * V + v], e2 = set[(k + 2) * V + v],
                    e3 = set[(k + 3) * V + v];
#pragma unroll
        for (int r = 0; r < HEAD_ROWS; ++r) {
          const float4 y4 = *reinterpret_cast<const float4*>(sy + r * d + k0 + k);
          acc[r] = fmaf(y4.x, e0, acc[r]);
          acc[r] = fmaf(y4.y, e1, acc[r]);
          acc[r] = fmaf(y4.z, e2, acc[r]);
          acc[r] = fmaf(y4.w, e3, acc[r]);
        }
      }
    }
    __syncthreads();  // stage (c & 1) is refilled by the next iteration's prefetch
  }
  if (v < V) {
#pragma unroll
    for (int r = 0; r < HEAD_ROWS; ++r) slog[r * V + v] = acc[r];
  }
  __syncthreads();
  for (int r = warp; r < nr; r += 8) {
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int v = lane; v < V; v += 32) {
      const float val = slog[r * V + v];
      if (val > best || (val == best && v < bi)) {
        best = val;
        bi = v;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (bi == 0x7fffffff) bi = 0;  // all-NaN row: argmax_row returns index 0
    if (lane == 0) {
      next_tok[r0 + r] = bi;
      if (last_tok) last_tok[row_slot[r0 + r]] = bi;
    }
    if (logits_out)
      for (int v = lane; v < V; v += 32) logits_out[static_cast<size_t>(r0 + r) * V + v] = slog[r * V + v];
  }
}

// ------------------------------------------------------------------ misc
// Longest common prefix (in tokens) of every row with row 0, bounded by `limit`.
__global__ void lcp_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ offsets, int64_t n_rows,
                           int limit, int* __restrict__ out) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= n_rows || r == 0) return;
  const int32_t* a = ids + offsets[0];
  const int32_t* b = ids + offsets[r];
  const int n = static_cast<int>(min(static_cast<int64_t>(limit), offsets[r + 1] - offsets[r]));
  int i = 0;
  while (i < n && a[i] == b[i]) ++i;
  atomicMin(out, i);
}

__global__ void check_ids_kernel(const int32_t* __restrict__ ids, int64_t n, int V, int* __restrict__ bad) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n && (ids[i] < 0 || ids[i] >= V)) atomicMin(bad, 0);
}

// Weight decode: bundle payload -> device GEMM operand (row-major [rows x ld], zero padded).
__global__ void decode_dense_h16_kernel(const float* __restrict__ src, int rows, int cols, h16* dst,
                                         int ld) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(rows) * ld) return;
  const int r = static_cast<int>(i / ld), c = static_cast<int>(i % ld);
  dst[i] = c < cols ? __float2half_rn(src[static_cast<size_t>(r) * cols + c]) : __float2half_rn(0.f);
}

// q8 / q4 / sparse24 payload -> dequantized fp16 value code*scale (model.cpp:153-199).
__global__ void decode_quant_h16_kernel(const uint8_t* __restrict__ p, int enc, int rows, int cols,
                                         h16* dst, int ld) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(rows) * ld) return;
  const int r = static_cast<int>(i / ld), c = static_cast<int>(i % ld);
  float v = 0.f;
  if (c < cols) {
    if (enc == 1) {
      const float s = reinterpret_cast<const float*>(p + static_cast<size_t>(rows) * cols)[r];
      v = static_cast<float>(reinterpret_cast<const int8_t*>(p)[static_cast<size_t>(r) * cols + c]) * s;
    } else if (enc == 2) {
      const size_t rb = (static_cast<size_t>(cols) + 1) / 2;
      float s;
      memcpy(&s, p + rows * rb + 4ull * r, 4);
      const uint8_t byte = p[r * rb + c / 2];
      const int nib = (c & 1) ? (byte >> 4) : (byte & 0xF);
      v = static_cast<float>(nib - 8) * s;
    } else if (enc == 3 && c < (cols & ~3)) {  // tail columns past the last whole group stay 0 (model.cpp:178-199)
      const size_t groups = cols / 4, irb = (groups + 1) / 2;
      const int8_t* codes = reinterpret_cast<const int8_t*>(p);
      const uint8_t* idx = p + static_cast<size_t>(rows) * groups * 2;
      float s;
      memcpy(&s, idx + rows * irb + 4ull * r, 4);
      const size_t gidx = c / 4;
      const uint8_t byte = idx[r * irb + gidx / 2];
      const int nib = (gidx & 1) ? (byte >> 4) : (byte & 0xF);
      const int p0 = nib & 3, p1 = (nib >> 2) & 3, j = c & 3;
      if (j == p0) v = static_cast<float>(codes[(r * groups + gidx) * 2]) * s;
      if (j == p1) v = static_cast<float>(codes[(r * groups + gidx) * 2 + 1]) * s;
    }
  }
  dst[i] = __float2half_rn(v);
}

// Quantized payload -> the integer codes only (exact as fp16 for |code| <= 127), zero padded;
// scales[r] receives the per-row f32 scale. The scale is applied in the GEMM epilogue.
template <typename T>
__global__ void decode_codes_kernel(const uint8_t* __restrict__ p, int enc, int rows, int cols, T* dst, int ld,
                                    float* __restrict__ scales) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(rows) * ld) return;
  const int r = static_cast<int>(i / ld), c = static_cast<int>(i % ld);
  int code = 0;
  size_t scale_off = 0;
  if (enc == 1) {
    scale_off = static_cast<size_t>(rows) * cols;
    if (c < cols) code = reinterpret_cast<const int8_t*>(p)[static_cast<size_t>(r) * cols + c];
  } else if (enc == 2) {
    const size_t rb = (static_cast<size_t>(cols) + 1) / 2;
    scale_off = rows * rb;
    if (c < cols) {
      const uint8_t byte = p[r * rb + c / 2];
      code = ((c & 1) ? (byte >> 4) : (byte & 0xF)) - 8;
    }
  } else if (enc == 3) {
    const size_t groups = cols / 4, irb = (groups + 1) / 2;
    const int8_t* codes = reinterpret_cast<const int8_t*>(p);
    const uint8_t* idx = p + static_cast<size_t>(rows) * groups * 2;
    scale_off = static_cast<size_t>(rows) * groups * 2 + rows * irb;
    if (c < (cols & ~3)) {  // the tail past the last whole group stays 0, as in model.cpp:178-199
      const size_t gidx = c / 4;
      const uint8_t byte = idx[r * irb + gidx / 2];
      const int nib = (gidx & 1) ? (byte >> 4) : (byte & 0xF);
      const int j = c & 3;
      if (j == (nib & 3)) code = codes[(r * groups + gidx) * 2];
      if (j == ((nib >> 2) & 3)) code = codes[(r * groups + gidx) * 2 + 1];
    }
  }
  if constexpr (sizeof(T) == 1) dst[i] = static_cast<int8_t>(code);
  else dst[i] = __int2half_rn(code);
  if (c == 0) {
    float s;
    memcpy(&s, p + scale_off + 4ull * r, 4);
    scales[r] = s;
  }
}

__global__ void transpose_f32_kernel(const float* __restrict__ src, int rows, int cols, float* __restrict__ dst) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(rows) * cols) return;
  const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
  dst[static_cast<size_t>(c) * rows + r] = src[i];
}

}  // namespace iolmk

// ====================================================================== host launchers
namespace iolmh {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("IOLM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
using namespace iolmk;

static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
// decode attention CTA shape (IOLM_DEC_HG / IOLM_DEC_STAGES override, for A/B measurements)
static int decode_stages() {
  static const int v = std::max(2, std::min(DSTAGES_MAX, env_int("IOLM_DEC_STAGES", 3)));
  return v;
}
int decode_heads_per_cta(int heads, int hd) {
  static const int cap = env_int("IOLM_DEC_HG", 0);
  // measured on C1 (20 heads, hd 64): 5 heads per CTA 6.49 TB/s, 4 heads 6.74, 2 heads 6.83 -
  // smaller groups give more resident CTAs per SM for the short decode sequences
  const int hmax = std::min(hd >= 128 ? 8 : 16, cap > 0 ? cap : 4);
  const int ngrp = (heads + hmax - 1) / hmax;
  const int per = (heads + ngrp - 1) / ngrp;
  // uneven split (e.g. 10 heads -> 4 + 4 + 2, a half-idle last CTA): prefer a divisor of the head
  // count in [hmax/2, hmax] (10 -> 5 x 2; measured C3 +0.8%, profiles/r01_dec_hg_ab.jsonl)
  if (cap == 0 && heads % per != 0)
    for (int h = hmax; h >= (hmax + 1) / 2 && h >= 2; --h)
      if (heads % h == 0) return h;
  return per;
}

static inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

void launch_ln(const float* x, int M, int d, const float* g, const float* b, h16* h, int ldh,
               cudaStream_t st, int8_t* q8, float* qscale) {
  if (M <= 0) return;
  const int nv = (d / 4 + 31) / 32;
  const int sms = device_sms();
  // gain / bias staged in shared memory for the fp16 output (measured: C1 LN 237 -> 224 ms; the int8
  // output variant is 3-6% slower with it, C3 / C4). IOLM_LN_GB_SMEM=0 / 1 forces it off / on (A/B).
  static const int gb_env = [] {
    const char* e = std::getenv("IOLM_LN_GB_SMEM");
    return e == nullptr ? -1 : (std::string(e) != "0" ? 1 : 0);
  }();
  const int gbf = gb_env >= 0 ? gb_env : (q8 ? 0 : 1);
  const size_t gbs = gbf ? 2ull * d * sizeof(float) : 0;
  if (std::getenv("IOLM_LN_LEGACY") == nullptr && nv > 10 && nv <= 32 && d % 4 == 0) {
    const int grid_s = std::min<int>((M + 3) / 4, sms * 2);
    const int v2 = (d / 4 + 63) / 64;  // float4 per thread with two warps per row
    if (v2 <= 8) {
      if (q8) launch_k<false>(ln_stream2_kernel<8, true>, grid_s, 256, gbs, st, x, M, d, g, b, h, ldh, q8, qscale, gbf);
      else launch_k<false>(ln_stream2_kernel<8, false>, grid_s, 256, gbs, st, x, M, d, g, b, h, ldh, q8, qscale, gbf);
    } else {
      if (q8) launch_k<false>(ln_stream2_kernel<16, true>, grid_s, 256, gbs, st, x, M, d, g, b, h, ldh, q8, qscale, gbf);
      else launch_k<false>(ln_stream2_kernel<16, false>, grid_s, 256, gbs, st, x, M, d, g, b, h, ldh, q8, qscale, gbf);
    }
    CUDA_OK(cudaGetLastError());
    return;
  }
  if (std::getenv("IOLM_LN_LEGACY") == nullptr && nv <= 10) {
    const int grid_s = std::min<int>((M + 7) / 8, sms * 2);
#define LNS(V)                                                                                             \
  do {                                                                                                     \
    if (q8) launch_k<false>(ln_stream_kernel<V, true>, grid_s, 256, gbs, st, x, M, d, g, b, h, ldh, q8, qscale, gbf);     \
    else launch_k<false>(ln_stream_kernel<V, false>, grid_s, 256, gbs, st, x, M, d, g, b, h, ldh, q8, qscale, gbf);       \
  } while (0)
    switch (nv) {
      case 1: LNS(1); break;
      case 2: LNS(2); break;
      case 3: LNS(3); break;
      case 4: LNS(4); break;
      case 5: LNS(5); break;
      case 6: LNS(6); break;
      case 8: LNS(8); break;
      default: LNS(10); break;
    }
#undef LNS
    CUDA_OK(cudaGetLastError());
    return;
  }
  const size_t bsmem = 256 + static_cast<size_t>(LN_STAGES) * 8 * d * 4;
  // the bulk-streamed variant pays off for the int8 (W8A8) output; the fp16 output keeps the
  // register-resident one-warp-per-row kernel (measured faster at d = 1280)
  if (q8 && d % 128 == 0 && (nv == 10 || nv == 16 || nv == 8 || nv == 4) && bsmem <= 200 * 1024) {
    const int per_sm = bsmem <= 100 * 1024 ? 2 : 1;
    const int grid_b = std::min<int>((M + 7) / 8, sms * per_sm);
#define LNB(V)                                                                                          \
  do {                                                                                                  \
    ensure_smem(ln_bulk_kernel<V, true>, 200 * 1024);                                                   \
    ensure_smem(ln_bulk_kernel<V, false>, 200 * 1024);                                                  \
    if (q8) launch_k<false>(ln_bulk_kernel<V, true>, grid_b, 288, bsmem, st, x, M, d, g, b, h, ldh, q8, qscale);      \
    else launch_k<false>(ln_bulk_kernel<V, false>, grid_b, 288, bsmem, st, x, M, d, g, b, h, ldh, q8, qscale);        \
  } while (0)
    switch (nv) {
      case 4: LNB(4); break;
      case 8: LNB(8); break;
      case 10: LNB(10); break;
      default: LNB(16); break;
    }
#undef LNB
    CUDA_OK(cudaGetLastError());
    return;
  }
  const unsigned grid = blocks_for(M, 8);
#define LNK(V)                                                                     \
  do {                                                                             \
    if (q8) launch_k(ln_kernel<V, true>, grid, 256, 0, st, x, M, d, g, b, h, ldh, q8, qscale); \
    else launch_k(ln_kernel<V, false>, grid, 256, 0, st, x, M, d, g, b, h, ldh, q8, qscale);   \
  } while (0)
  switch (nv) {
    case 1: LNK(1); break;
    case 2: LNK(2); break;
    case 3: LNK(3); break;
    case 4: LNK(4); break;
    case 5: LNK(5); break;
    case 6: LNK(6); break;
    case 8: LNK(8); break;
    case 10: LNK(10); break;
    case 12: LNK(12); break;
    case 16: LNK(16); break;
    default:
      if (nv <= 16) LNK(16);
      else if (nv <= 32) LNK(32);
      else throw Unsupported("layernorm: d_model > 4096");
  }
#undef LNK
  CUDA_OK(cudaGetLastError());
}

void launch_quant_rows(const h16* src, int lds, int M, int cols, int8_t* dst, int ldd, float* scale,
                       cudaStream_t st) {
  if (M <= 0) return;
  if (lds % 8 != 0 || ldd % 8 != 0) throw Unsupported("quant_rows: leading dimensions must be multiples of 8");
  const unsigned grid = blocks_for(M, 8);
  const int ch = (cols + 255) / 256;
  if (cols % 8 != 0) launch_k(quant_rows_kernel<0>, grid, 256, 0, st, src, lds, M, cols, dst, ldd, scale);
  // register-resident rows up to 1280 columns (measured, profiles/r02_experiments.md: C2-W8A8's 1280-wide
  // attention output 223.6 -> 217.4 ms with the row in registers, while 2560 columns - C3's GELU output
  // - lose 9% against the two-pass kernel); wider rows take the two-pass kernel (its second read hits
  // L2) at 8 CTAs per SM: these launches are bound by load latency, not bytes
  else if (ch <= 4) launch_k(quant_rows_kernel<4>, grid, 256, 0, st, src, lds, M, cols, dst, ldd, scale);
  else if (ch <= 5) launch_k(quant_rows_kernel<5>, grid, 256, 0, st, src, lds, M, cols, dst, ldd, scale);
  else if (cols > 3072 && cols <= 5120) {  // measured: two-warp rows win at 4096 (C4 FFN), lose at 2560
    const int sms = device_sms();
    const int grid2 = std::min<int>((M + 3) / 4, sms * 2);
    if (cols <= 4096) launch_k<false>(quant_rows2_kernel<8>, grid2, 256, 0, st, src, lds, M, cols, dst, ldd, scale);
    else launch_k<false>(quant_rows2_kernel<10>, grid2, 256, 0, st, src, lds, M, cols, dst, ldd, scale);
  } else launch_k(quant_rows_kernel<0>, grid, 256, 0, st, src, lds, M, cols, dst, ldd, scale);
  CUDA_OK(cudaGetLastError());
}

void launch_embed_ln(const int32_t* ids, const int64_t* tok_src, const int* tok_slot, const int* tok_pos,
                     const int32_t* last_tok, int M, int d, const float* tok_embed, const float* pos_embed, float* x,
                     const float* g, const float* b, h16* h, int ldh, cudaStream_t st, int8_t* q8,
                     float* qscale) {
  if (M <= 0) return;
  const unsigned grid = blocks_for(M, 8);
  const int nv = (d / 4 + 31) / 32;
#define EMB(V)                                                                                        \
  do {                                                                                                \
    if (q8)                                                                                           \
      launch_k(embed_ln_kernel<V, true>, grid, 256, 0, st, ids, tok_src, tok_slot, tok_pos, last_tok, M, d, \
                                                     tok_embed, pos_embed, x, g, b, h, ldh, q8, qscale); \
    else                                                                                              \
      launch_k(embed_ln_kernel<V, false>, grid, 256, 0, st, ids, tok_src, tok_slot, tok_pos, last_tok, M, d, \
                                                      tok_embed, pos_embed, x, g, b, h, ldh, q8, qscale); \
  } while (0)
  switch (nv) {
    case 1: EMB(1); break;
    case 2: EMB(2); break;
    case 4: EMB(4); break;
    case 8: EMB(8); break;
    case 10: EMB(10); break;
    case 16: EMB(16); break;
    default:
      if (nv <= 16) EMB(16);
      else if (nv <= 32) EMB(32);
      else throw Unsupported("embed: d_model > 4096");
  }
#undef EMB
  CUDA_OK(cudaGetLastError());
}

void launch_attention(const AttnParams& prefill, const AttnParams& decode, int hd, cudaStream_t st) {
#define ATT(HD)                                                                                     \
  do {                                                                                              \
    constexpr int smem = static_cast<int>(PfCfg<HD>::SMEM);                                         \
    ensure_smem(attn_prefill_kernel<HD, false>, smem, 100);                                         \
    ensure_smem(attn_prefill_kernel<HD, true>, smem);                                               \
    if (prefill.n_groups > 0) {                                                                     \
      const dim3 grid(prefill.n_groups, prefill.heads);                                             \
      if (prefill.key_mask)                                                                         \
        launch_k(attn_prefill_kernel<HD, true>, grid, 128, smem, st, prefill);                            \
      else                                                                                          \
        launch_k(attn_prefill_kernel<HD, false>, grid, 128, smem, st, prefill);                           \
    }                                                                                               \
    if (decode.n_groups > 0) {                                                                      \
      const int hg = decode_heads_per_cta(decode.heads, HD);                                        \
      const int ngrp = (decode.heads + hg - 1) / hg;                                                \
      const int nst = decode_stages();                                                              \
      const size_t sm = DecCfg<HD>::smem(hg, nst);                                                  \
      ensure_smem(attn_decode_kernel<HD>, sm, 100);                                                 \
      launch_k(attn_decode_kernel<HD>, decode.n_groups * ngrp, 32 * (hg + 1), sm, st, decode, hg, ngrp, nst); \
    }                                                                                               \
  } while (0)
  switch (hd) {
    case 16: ATT(16); break;
    case 32: ATT(32); break;
    case 64: ATT(64); break;
    case 128: ATT(128); break;
    default: throw Unsupported("attention: head_dim must be 16, 32, 64 or 128");
  }
#undef ATT
  CUDA_OK(cudaGetLastError());
}

// Head-row compaction of the last layer (engine.cu, Engine::launch_step): row c of xc / zc <- row
// rows[c] of x (fp32 residual stream, d) and z (fp16 attention output, kh). One CTA per row.
__global__ void __launch_bounds__(128) gather_head_rows_kernel(const float* __restrict__ x, int d,
                                                               const h16* __restrict__ z, int ldz, int kh,
                                                               const int* __restrict__ rows, float* __restrict__ xc,
                                                               h16* __restrict__ zc, int ldzc) {
  pdl_sync();
  const int c = blockIdx.x, r = rows[c];
  const float4* xs = reinterpret_cast<const float4*>(x + static_cast<size_t>(r) * d);
  float4* xd = reinterpret_cast<float4*>(xc + static_cast<size_t>(c) * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) xd[i] = xs[i];
  const uint4* zs = reinterpret_cast<const uint4*>(z + static_cast<size_t>(r) * ldz);
  uint4* zd = reinterpret_cast<uint4*>(zc + static_cast<size_t>(c) * ldzc);
  for (int i = threadIdx.x; i < kh / 8; i += blockDim.x) zd[i] = zs[i];
}

void launch_gather_head_rows(const float* x, int d, const h16* z, int ldz, int kh, const int* rows, int n_rows,
                             float* xc, h16* zc, int ldzc, cudaStream_t st) {
  if (n_rows <= 0) return;
  if (d % 4 != 0 || kh % 8 != 0 || ldz % 8 != 0 || ldzc % 8 != 0)
    throw Unsupported("gather_head_rows: d must be a multiple of 4, kh / ld a multiple of 8");
  launch_k(gather_head_rows_kernel, n_rows, 128, 0, st, x, d, z, ldz, kh, rows, xc, zc, ldzc);
  CUDA_OK(cudaGetLastError());
}

void launch_head(const float* x, int d, const int* rows, int n_rows, const float* g, const float* b,
                 const float* embed_t, int V, const int* row_slot, int32_t* next_tok, int32_t* last_tok,
                 float* logits_out, cudaStream_t st) {
  if (n_rows <= 0) return;
  if (V > 256) throw Unsupported("head: vocabulary larger than the CTA");
  if (d % 4 != 0) throw Unsupported("head: d_model must be a multiple of 4");
  const size_t smem = sizeof(float) * (HEAD_ROWS * (d + V) + 2 * HEAD_KC * V) + 16;
  if (smem > 48 * 1024) ensure_smem(head_argmax_kernel, smem);
  launch_k(head_argmax_kernel, blocks_for(n_rows, HEAD_ROWS), 256, smem, st, x, d, rows, n_rows, g, b, embed_t, V,
                                                                       row_slot, next_tok, last_tok, logits_out);
  CUDA_OK(cudaGetLastError());
}

void launch_lcp(const int32_t* ids, const int64_t* offsets, int64_t n_rows, int limit, int* out, cudaStream_t st) {
  if (n_rows > 1) lcp_kernel<<<blocks_for(n_rows, 256), 256, 0, st>>>(ids, offsets, n_rows, limit, out);
  CUDA_OK(cudaGetLastError());
}

void launch_check_ids(const int32_t* ids, int64_t n, int V, int* bad, cudaStream_t st) {
  if (n > 0) check_ids_kernel<<<blocks_for(n, 256), 256, 0, st>>>(ids, n, V, bad);
  CUDA_OK(cudaGetLastError());
}

void launch_decode_weight(const void* payload, int enc, int rows, int cols, h16* dst, int ld,
                          cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(rows) * ld;
  if (enc == 0)
    decode_dense_h16_kernel<<<blocks_for(n, 256), 256, 0, st>>>(static_cast<const float*>(payload), rows, cols,
                                                                 dst, ld);
  else
    decode_quant_h16_kernel<<<blocks_for(n, 256), 256, 0, st>>>(static_cast<const uint8_t*>(payload), enc, rows,
                                                                 cols, dst, ld);
  CUDA_OK(cudaGetLastError());
}

void launch_decode_codes(const void* payload, int enc, int rows, int cols, void* dst, bool int8, int ld,
                         float* scales, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(rows) * ld;
  if (enc < 1 || enc > 3) throw Unsupported("decode_codes: not a quantized encoding");
  if (int8)
    decode_codes_kernel<int8_t><<<blocks_for(n, 256), 256, 0, st>>>(static_cast<const uint8_t*>(payload), enc, rows,
                                                                    cols, static_cast<int8_t*>(dst), ld, scales);
  else
    decode_codes_kernel<h16><<<blocks_for(n, 256), 256, 0, st>>>(
        static_cast<const uint8_t*>(payload), enc, rows, cols, static_cast<h16*>(dst), ld, scales);
  CUDA_OK(cudaGetLastError());
}

void launch_transpose(const float* src, int rows, int cols, float* dst, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(rows) * cols;
  transpose_f32_kernel<<<blocks_for(n, 256), 256, 0, st>>>(src, rows, cols, dst);
  CUDA_OK(cudaGetLastError());
}

}  // namespace iolmh
