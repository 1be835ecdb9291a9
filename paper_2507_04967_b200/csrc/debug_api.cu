// Kernel-level C entry points used by the parity tests: they run the production kernels on
// host-provided operands (device allocation, H2D, launch, D2H inside).
#include <vector>

#include "capi_util.hpp"
#include "launch.hpp"
#include "tma_host.hpp"

namespace iolmh {
void launch_quant_rows(const __nv_bfloat16* src, int lds, int M, int cols, int8_t* dst, int ldd, float* scale,
                       cudaStream_t st);
}

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

extern "C" int iolm_cuda_debug_quant_rows_bf16(const uint16_t* x, int32_t n, int32_t d, int8_t* codes,
                                               float* scales) {
  return guarded([&] {
    if (n <= 0 || d <= 0 || d % 8 != 0) throw ContractViolation("debug_quant_rows: need d % 8 == 0");
    DevBuf<uint16_t> dx(static_cast<size_t>(n) * d);
    DevBuf<int8_t> dc(static_cast<size_t>(n) * d);
    DevBuf<float> ds(n);
    CUDA_OK(cudaMemcpy(dx.p, x, sizeof(uint16_t) * n * d, cudaMemcpyHostToDevice));
    launch_quant_rows(reinterpret_cast<const __nv_bfloat16*>(dx.p), d, n, d, dc.p, d, ds.p, nullptr);
    CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaMemcpy(codes, dc.p, static_cast<size_t>(n) * d, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(scales, ds.p, sizeof(float) * n, cudaMemcpyDeviceToHost));
  });
}

// Device-only GEMM timing for kernel tuning: random operands, `iters` back-to-back launches timed
// with CUDA events; returns the mean ms per launch. epi: 0 f32, 1 bf16, 2 gelu, 3 resid, 5 s32.
extern "C" int iolm_cuda_debug_gemm_time(int32_t M, int32_t N, int32_t K, int32_t epi, int32_t pair, int32_t i8,
                                         int32_t iters, float* ms_out) {
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0 || iters <= 0) throw ContractViolation("debug_gemm_time: bad sizes");
    const size_t eb = i8 ? 1 : 2;
    DevBuf<uint8_t> dA(static_cast<size_t>(M) * K * eb), dW(static_cast<size_t>(N) * K * eb);
    DevBuf<float> dC(static_cast<size_t>(M) * N), ws(N), as(M);
    CUDA_OK(cudaMemset(dA.p, 0x11, static_cast<size_t>(M) * K * eb));
    CUDA_OK(cudaMemset(dW.p, 0x13, static_cast<size_t>(N) * K * eb));
    CUDA_OK(cudaMemset(dC.p, 0, sizeof(float) * M * N));
    CUDA_OK(cudaMemset(ws.p, 0, sizeof(float) * N));
    CUDA_OK(cudaMemset(as.p, 0, sizeof(float) * M));
    const auto dt = i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap ta = make_kmajor_map(dA.p, dt, static_cast<int>(eb), K, M, eb * K, 128);
    CUtensorMap tb = make_kmajor_map(dW.p, dt, static_cast<int>(eb), K, N, eb * K, 128);
    iolmk::GemmEpi ep;
    ep.M = M;
    ep.N = N;
    ep.out = dC.p;
    ep.ldo = N;
    if (i8) {
      ep.a_scale = as.p;
      ep.w_scale = ws.p;
    }
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    launch_gemm(pair != 0, i8 != 0, epi, ta, tb, M, N, K, ep, nullptr, sm_count());
    CUDA_OK(cudaEventRecord(e0));
    for (int i = 0; i < iters; ++i) launch_gemm(pair != 0, i8 != 0, epi, ta, tb, M, N, K, ep, nullptr, sm_count());
    CUDA_OK(cudaEventRecord(e1));
    CUDA_OK(cudaEventSynchronize(e1));
    float ms = 0;
    CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}
