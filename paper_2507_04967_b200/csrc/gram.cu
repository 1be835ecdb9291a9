// Calibration Gram matrix on the GPU: H = scale * X^T X in f64 (the Hessian of
// GPTQ / compensated 2:4 sparsification).
//
// Reference: build_hessian (proj/src/calib.cpp:64-74) -> fastmath::gram_accumulate
// (proj/src/fastmath.cpp:79-100): for every sample row s in order, acc[i][j] += double(x_si) *
// double(x_sj) for j >= i, then h = scale * acc mirrored to the lower triangle. Each product of two
// f32 values is EXACT in f64 (24 + 24 <= 53 mantissa bits), so an FMA and a multiply-then-add round
// identically, and the only rounding per step is the addition. Each output element here is one
// thread's sequential f64 sum over s = 0, 1, ... in the same order, so H is bit-identical to the
// reference's (the skipped x_si == 0 terms add +-0 to an accumulator that is never -0).
//
// Tiling: 64 x 64 output tiles of the upper triangle, 256 threads x 4 x 4 f64 accumulators, samples
// staged 32 at a time in shared memory as f32. f64 FMA throughput, not bandwidth, bounds it.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "capi_util.hpp"
#include "launch.hpp"

namespace iolmk {

constexpr int GT = 64;  // output tile
constexpr int GS = 32;  // samples per smem stage

__global__ void __launch_bounds__(256) gram_f64_kernel(const float* __restrict__ x, int rows, int cols,
                                                       const int2* __restrict__ tiles, double scale,
                                                       double* __restrict__ h) {
  __shared__ float As[GS][GT];
  __shared__ float Bs[GS][GT];
  const int2 t = tiles[blockIdx.x];
  const int i0 = t.x * GT, j0 = t.y * GT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int s0 = 0; s0 < rows; s0 += GS) {
    for (int e = threadIdx.x; e < GS * GT; e += 256) {
      const int ss = e / GT, c = e % GT, s = s0 + ss;
      As[ss][c] = (s < rows && i0 + c < cols) ? x[static_cast<size_t>(s) * cols + i0 + c] : 0.f;
      Bs[ss][c] = (s < rows && j0 + c < cols) ? x[static_cast<size_t>(s) * cols + j0 + c] : 0.f;
    }
    __syncthreads();
    const int ns = min(GS, rows - s0);
    for (int ss = 0; ss < ns; ++ss) {  // ascending sample order (the reference's)
      double a[4], b[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        a[k] = static_cast<double>(As[ss][ty * 4 + k]);
        b[k] = static_cast<double>(Bs[ss][tx * 4 + k]);
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + ty * 4 + p, j = j0 + tx * 4 + q;
      if (i < cols && j < cols && j >= i) {
        const double v = scale * acc[p][q];
        h[static_cast<size_t>(i) * cols + j] = v;
        h[static_cast<size_t>(j) * cols + i] = v;
      }
    }
}

}  // namespace iolmk

extern "C" int iolm_cuda_gram(int device, const float* x, int64_t rows, int32_t cols, double scale, double* h) {
  using namespace iolmh;
  return guarded([&] {
    if (!x || !h || rows < 1 || cols < 1) throw ContractViolation("gram: bad arguments");
    CUDA_OK(cudaSetDevice(device));
    const int nt = (cols + iolmk::GT - 1) / iolmk::GT;
    std::vector<int2> tiles;
    for (int a = 0; a < nt; ++a)
      for (int b = a; b < nt; ++b) tiles.push_back(make_int2(a, b));
    float* dx = nullptr;
    double* dh = nullptr;
    int2* dt = nullptr;
    const size_t xb = static_cast<size_t>(rows) * cols * sizeof(float);
    const size_t hb = static_cast<size_t>(cols) * cols * sizeof(double);
    cudaStream_t st = nullptr;
    auto release = [&] {
      if (dx) cudaFree(dx);
      if (dh) cudaFree(dh);
      if (dt) cudaFree(dt);
      if (st) cudaStreamDestroy(st);
    };
    try {
      CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      CUDA_OK(cudaMalloc(&dx, xb));
      CUDA_OK(cudaMalloc(&dh, hb));
      CUDA_OK(cudaMalloc(&dt, tiles.size() * sizeof(int2)));
      CUDA_OK(cudaMemcpyAsync(dx, x, xb, cudaMemcpyHostToDevice, st));
      CUDA_OK(cudaMemcpyAsync(dt, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
      iolmk::gram_f64_kernel<<<static_cast<unsigned>(tiles.size()), 256, 0, st>>>(dx, static_cast<int>(rows), cols, dt,
                                                                                 scale, dh);
      CUDA_OK(cudaGetLastError());
      CUDA_OK(cudaMemcpyAsync(h, dh, hb, cudaMemcpyDeviceToHost, st));
      CUDA_OK(cudaStreamSynchronize(st));
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}
