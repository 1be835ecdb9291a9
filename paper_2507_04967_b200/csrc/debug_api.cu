// Kernel-level C entry points used by the parity tests: they run the production kernels on
// host-provided operands (device allocation, H2D, launch, D2H inside).
#include <vector>

#include "capi_util.hpp"
#include "launch.hpp"
#include "tma_host.hpp"

using namespace iolmh;

namespace {

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { CUDA_OK(cudaMalloc(&p, n * sizeof(T) + 16)); }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

int sm_count() {
  int dev = 0, n = 0;
  CUDA_OK(cudaGetDevice(&dev));
  CUDA_OK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

}  // namespace

extern "C" int iolm_cuda_debug_gemm_bf16(const uint16_t* A, const uint16_t* W, float* C,
                                         int32_t M, int32_t N, int32_t K, int32_t bn,
                                         int32_t epi) {
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0 || (K % 8) != 0)
      throw ContractViolation("debug_gemm: need positive M,N and K % 8 == 0");
    DevBuf<uint16_t> dA(static_cast<size_t>(M) * K), dW(static_cast<size_t>(N) * K);
    DevBuf<float> dC(static_cast<size_t>(M) * N);
    DevBuf<__nv_bfloat16> dG(static_cast<size_t>(M) * N);
    CUDA_OK(cudaMemcpy(dA.p, A, sizeof(uint16_t) * M * K, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dW.p, W, sizeof(uint16_t) * N * K, cudaMemcpyHostToDevice));
    CUtensorMap ta = make_kmajor_map(dA.p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, M, 2ull * K, 128);
    CUtensorMap tb = make_kmajor_map(dW.p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, N, 2ull * K, 128);
    iolmk::GemmEpi ep;
    ep.M = M;
    ep.N = N;
    if (epi == iolmk::EPI_F32) {
      ep.out = dC.p;
      ep.ldo = N;
    } else if (epi == iolmk::EPI_GELU_BF16 || epi == iolmk::EPI_BF16) {
      if (N % 8 != 0) throw ContractViolation("debug_gemm: bf16 epilogue needs N % 8 == 0");
      ep.out = dG.p;
      ep.ldo = N;
    } else if (epi == iolmk::EPI_RESID_F32) {
      CUDA_OK(cudaMemcpy(dC.p, C, sizeof(float) * M * N, cudaMemcpyHostToDevice));
      ep.out = dC.p;
      ep.ldo = N;
    } else {
      throw ContractViolation("debug_gemm: unsupported epilogue");
    }
    launch_gemm(bn == 256, false, epi, ta, tb, M, N, K, ep, nullptr, sm_count());
    CUDA_OK(cudaDeviceSynchronize());
    if (epi == iolmk::EPI_GELU_BF16 || epi == iolmk::EPI_BF16) {
      std::vector<__nv_bfloat16> h(static_cast<size_t>(M) * N);
      CUDA_OK(cudaMemcpy(h.data(), dG.p, h.size() * 2, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < h.size(); ++i) C[i] = __bfloat162float(h[i]);
    } else {
      CUDA_OK(cudaMemcpy(C, dC.p, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
    }
  });
}

extern "C" int iolm_cuda_debug_gemm_s8(const int8_t* A, const int8_t* W, int32_t* C, int32_t M, int32_t N,
                                       int32_t K, int32_t pair) {
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0 || (K % 16) != 0)
      throw ContractViolation("debug_gemm_s8: need positive M,N and K % 16 == 0");
    DevBuf<int8_t> dA(static_cast<size_t>(M) * K), dW(static_cast<size_t>(N) * K);
    DevBuf<int32_t> dC(static_cast<size_t>(M) * N);
    CUDA_OK(cudaMemcpy(dA.p, A, static_cast<size_t>(M) * K, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dW.p, W, static_cast<size_t>(N) * K, cudaMemcpyHostToDevice));
    CUtensorMap ta = make_kmajor_map(dA.p, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, K, M, K, 128);
    CUtensorMap tb = make_kmajor_map(dW.p, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, K, N, K, 128);
    iolmk::GemmEpi ep;
    ep.M = M;
    ep.N = N;
    ep.out = dC.p;
    ep.ldo = N;
    launch_gemm(pair != 0, true, iolmk::EPI_S32, ta, tb, M, N, K, ep, nullptr, sm_count());
    CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaMemcpy(C, dC.p, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost));
  });
}
