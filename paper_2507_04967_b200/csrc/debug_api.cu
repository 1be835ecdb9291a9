// Kernel-level C entry points used by the parity tests: they run the production kernels on
// host-provided operands (device allocation, H2D, launch, D2H inside).
#include <cstdlib>
#include <string>
#include <vector>

#include "capi_util.hpp"
#include "launch.hpp"
#include "sparse24.hpp"
#include "tma_host.hpp"

namespace iolmh {
void launch_quant_rows(const h16* src, int lds, int M, int cols, int8_t* dst, int ldd, float* scale,
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

extern "C" int iolm_cuda_debug_gemm_f16(const uint16_t* A, const uint16_t* W, float* C,
                                         int32_t M, int32_t N, int32_t K, int32_t bn,
                                         int32_t epi) {
  static const bool use_tma_epi =
      std::getenv("IOLM_GEMM_TMA_EPI") == nullptr || std::string(std::getenv("IOLM_GEMM_TMA_EPI")) != "0";
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0 || (K % 8) != 0)
      throw ContractViolation("debug_gemm: need positive M,N and K % 8 == 0");
    DevBuf<uint16_t> dA(static_cast<size_t>(M) * K), dW(static_cast<size_t>(N) * K);
    DevBuf<float> dC(static_cast<size_t>(M) * N);
    DevBuf<h16> dG(static_cast<size_t>(M) * N);
    CUDA_OK(cudaMemcpy(dA.p, A, sizeof(uint16_t) * M * K, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dW.p, W, sizeof(uint16_t) * N * K, cudaMemcpyHostToDevice));
    CUtensorMap ta = make_kmajor_map(dA.p, H16_TMA, 2, K, M, 2ull * K, 128);
    CUtensorMap tb = make_kmajor_map(dW.p, H16_TMA, 2, K, N, 2ull * K, 128);
    iolmk::GemmEpi ep;
    ep.M = M;
    ep.N = N;
    if (epi == iolmk::EPI_F32) {
      ep.out = dC.p;
      ep.ldo = N;
    } else if (epi == iolmk::EPI_GELU_H16 || epi == iolmk::EPI_H16) {
      if (N % 8 != 0) throw ContractViolation("debug_gemm: fp16 epilogue needs N % 8 == 0");
      ep.out = dG.p;
      ep.ldo = N;
    } else if (epi == iolmk::EPI_RESID_F32) {
      CUDA_OK(cudaMemcpy(dC.p, C, sizeof(float) * M * N, cudaMemcpyHostToDevice));
      ep.out = dC.p;
      ep.ldo = N;
    } else {
      throw ContractViolation("debug_gemm: unsupported epilogue");
    }
    // the TMA store / reduce-add epilogue, as the engine runs it (N multiple of 8 keeps rows 16-B aligned)
    CUtensorMap tc;
    const CUtensorMap* out_map = nullptr;
    if (use_tma_epi && N % 8 == 0 && (epi == iolmk::EPI_RESID_F32 || epi == iolmk::EPI_GELU_H16 || epi == iolmk::EPI_H16)) {
      tc = epi == iolmk::EPI_RESID_F32 ? make_out_map(dC.p, true, N, M, 4ull * N) : make_out_map(dG.p, false, N, M, 2ull * N);
      out_map = &tc;
    }
    launch_gemm(bn == 256, false, epi, ta, tb, M, N, K, ep, nullptr, sm_count(), out_map);
    CUDA_OK(cudaDeviceSynchronize());
    if (epi == iolmk::EPI_GELU_H16 || epi == iolmk::EPI_H16) {
      std::vector<h16> h(static_cast<size_t>(M) * N);
      CUDA_OK(cudaMemcpy(h.data(), dG.p, h.size() * 2, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < h.size(); ++i) C[i] = __half2float(h[i]);
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

extern "C" int iolm_cuda_debug_quant_rows_f16(const uint16_t* x, int32_t n, int32_t d, int8_t* codes,
                                               float* scales) {
  return guarded([&] {
    if (n <= 0 || d <= 0 || d % 8 != 0) throw ContractViolation("debug_quant_rows: need d % 8 == 0");
    DevBuf<uint16_t> dx(static_cast<size_t>(n) * d);
    DevBuf<int8_t> dc(static_cast<size_t>(n) * d);
    DevBuf<float> ds(n);
    CUDA_OK(cudaMemcpy(dx.p, x, sizeof(uint16_t) * n * d, cudaMemcpyHostToDevice));
    launch_quant_rows(reinterpret_cast<const h16*>(dx.p), d, n, d, dc.p, d, ds.p, nullptr);
    CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaMemcpy(codes, dc.p, static_cast<size_t>(n) * d, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(scales, ds.p, sizeof(float) * n, cudaMemcpyDeviceToHost));
  });
}

// Device-only GEMM timing for kernel tuning: random operands, `iters` back-to-back launches timed
// with CUDA events; returns the mean ms per launch. epi: 0 f32, 1 fp16, 2 gelu, 3 resid, 5 s32.
extern "C" int iolm_cuda_debug_gemm_time(int32_t M, int32_t N, int32_t K, int32_t epi, int32_t pair, int32_t i8,
                                         int32_t iters, float* ms_out) {
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0 || iters <= 0) throw ContractViolation("debug_gemm_time: bad sizes");
    const size_t eb = i8 ? 1 : 2;
    if (i8 == 2 && K % 32 != 0) throw ContractViolation("debug_gemm_time: W4 needs K % 32 == 0");
    DevBuf<uint8_t> dA(static_cast<size_t>(M) * K * 2), dW(static_cast<size_t>(N) * K * eb);
    DevBuf<float> dC(static_cast<size_t>(M) * N), ws(N), as(M);
    CUDA_OK(cudaMemset(dA.p, 0x11, static_cast<size_t>(M) * K * 2));
    CUDA_OK(cudaMemset(dW.p, 0x13, static_cast<size_t>(N) * K * eb));
    CUDA_OK(cudaMemset(dC.p, 0, sizeof(float) * M * N));
    CUDA_OK(cudaMemset(ws.p, 0, sizeof(float) * N));
    CUDA_OK(cudaMemset(as.p, 0, sizeof(float) * M));
    const auto dt = i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : H16_TMA;
    const bool w4 = i8 == 2;  // W4A16: fp16 activations, packed int4 weights (K/2 bytes per row)
    const auto dt_a = w4 ? H16_TMA : dt;
    const size_t eb_a = w4 ? 2 : eb;
    if (w4) i8 = 0;
    CUtensorMap ta = make_kmajor_map(dA.p, dt_a, static_cast<int>(eb_a), K, M, eb_a * K, 128);
    CUtensorMap tb = w4 ? make_w4_map(dW.p, K, N, static_cast<uint64_t>(K) / 2)
                        : make_kmajor_map(dW.p, dt, static_cast<int>(eb), K, N, eb * K, 128);
    iolmk::GemmEpi ep;
    ep.M = M;
    ep.N = N;
    ep.out = dC.p;
    ep.ldo = N;
    if (i8 || w4) ep.w_scale = ws.p;
    if (i8) ep.a_scale = as.p;
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    static const bool use_tma_epi =
        std::getenv("IOLM_GEMM_TMA_EPI") == nullptr || std::string(std::getenv("IOLM_GEMM_TMA_EPI")) != "0";
    CUtensorMap tc;
    const CUtensorMap* out_map = nullptr;
    if (use_tma_epi && N % 8 == 0 && (epi == iolmk::EPI_RESID_F32 || epi == iolmk::EPI_GELU_H16 || epi == iolmk::EPI_H16)) {
      tc = make_out_map(dC.p, epi == iolmk::EPI_RESID_F32, N, M, (epi == iolmk::EPI_RESID_F32 ? 4ull : 2ull) * N);
      out_map = &tc;
    }
    auto go = [&] {
      if (w4) launch_gemm_w4(pair != 0, epi, ta, tb, M, N, K, ep, nullptr, sm_count(), out_map);
      else launch_gemm(pair != 0, i8 != 0, epi, ta, tb, M, N, K, ep, nullptr, sm_count(), out_map);
    };
    go();
    CUDA_OK(cudaEventRecord(e0));
    for (int i = 0; i < iters; ++i) go();
    CUDA_OK(cudaEventRecord(e1));
    CUDA_OK(cudaEventSynchronize(e1));
    float ms = 0;
    CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

// 2:4 sparse W8A8 GEMM through the sparse tensor cores: X_s8 [T x K] times the sparse24_q8 payload
// W [N x K] (the bundle's own bytes, proj/src/model.cpp:255-290). epi 5: raw int32 accumulators
// into out_s32 [T x N]; epi 0: acc * a_scale[t] * w_scale[n] into out_f32 (w_scale from the payload).
extern "C" int iolm_cuda_debug_gemm_sp24(const int8_t* X, const uint8_t* payload, int32_t T, int32_t N, int32_t K,
                                         int32_t epi, const float* a_scale, int32_t* out_s32, float* out_f32) {
  return guarded([&] {
    if (T <= 0 || N <= 0 || K <= 0 || K % 16 != 0)
      throw ContractViolation("debug_gemm_sp24: need positive T, N and K % 16 == 0");
    if (epi != iolmk::EPI_S32 && epi != iolmk::EPI_F32) throw ContractViolation("debug_gemm_sp24: epi 0 or 5");
    if (!sp24_check(payload, N, K)) throw Unsupported("debug_gemm_sp24: positions not ascending");
    const Sp24Layout l = sp24_layout(N, K);
    std::vector<int8_t> codes(l.code_bytes(), 0);
    std::vector<uint8_t> meta(l.meta_bytes(), 0x44);
    std::vector<float> scales(N);
    sp24_append(l, payload, N, K, 0, codes.data(), meta.data(), scales.data());
    DevBuf<int8_t> dX(static_cast<size_t>(T) * K), dW(codes.size());
    DevBuf<uint8_t> dE(meta.size());
    DevBuf<float> dS(N), dA(T), dC(static_cast<size_t>(T) * N);
    CUDA_OK(cudaMemcpy(dX.p, X, static_cast<size_t>(T) * K, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dW.p, codes.data(), codes.size(), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dE.p, meta.data(), meta.size(), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dS.p, scales.data(), sizeof(float) * N, cudaMemcpyHostToDevice));
    iolmk::GemmEpi ep;
    ep.M = T;
    ep.N = N;
    ep.out = dC.p;
    ep.ldo = N;
    if (epi == iolmk::EPI_F32) {
      CUDA_OK(cudaMemcpy(dA.p, a_scale, sizeof(float) * T, cudaMemcpyHostToDevice));
      ep.a_scale = dA.p;
      ep.w_scale = dS.p;
    }
    launch_gemm_sp(epi, sp24_codes_map(l, dW.p), sp24_act_map(dX.p, K, T, K), sp24_meta_map(l, dE.p), K,
                   l.katoms_pad, ep, nullptr, sm_count());
    CUDA_OK(cudaDeviceSynchronize());
    if (epi == iolmk::EPI_S32)
      CUDA_OK(cudaMemcpy(out_s32, dC.p, sizeof(int32_t) * T * N, cudaMemcpyDeviceToHost));
    else
      CUDA_OK(cudaMemcpy(out_f32, dC.p, sizeof(float) * T * N, cudaMemcpyDeviceToHost));
  });
}

// 2:4 sparse fp16 GEMM (tcgen05.mma.sp kind::f16): X_h16 [T x K] (uint16 bit patterns) times the
// sparse24_q8 payload's kept codes as exact fp16 integers; out_f32 [T x N] = acc * w_scale[n] (the
// W8A16 2:4 path the engine runs for sparse24_q8 bundles without act_quant).
extern "C" int iolm_cuda_debug_gemm_sp24_f16(const uint16_t* X, const uint8_t* payload, int32_t T, int32_t N,
                                              int32_t K, float* out_f32) {
  return guarded([&] {
    if (T <= 0 || N <= 0 || K <= 0 || K % 16 != 0)
      throw ContractViolation("debug_gemm_sp24_h16: need positive T, N and K % 16 == 0");
    if (!sp24_check(payload, N, K)) throw Unsupported("debug_gemm_sp24_h16: positions not ascending");
    const Sp24Layout l = sp24_layout(N, K, true);
    std::vector<uint8_t> codes(l.code_bytes(), 0);
    std::vector<uint8_t> meta(l.meta_bytes(), 0x44);
    std::vector<float> scales(N);
    sp24_append(l, payload, N, K, 0, codes.data(), meta.data(), scales.data());
    sp24_finalize(l, meta.data());
    DevBuf<uint16_t> dX(static_cast<size_t>(T) * K);
    DevBuf<uint8_t> dW(codes.size()), dE(meta.size());
    DevBuf<float> dS(N), dC(static_cast<size_t>(T) * N);
    CUDA_OK(cudaMemcpy(dX.p, X, sizeof(uint16_t) * T * K, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dW.p, codes.data(), codes.size(), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dE.p, meta.data(), meta.size(), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dS.p, scales.data(), sizeof(float) * N, cudaMemcpyHostToDevice));
    iolmk::GemmEpi ep;
    ep.M = T;
    ep.N = N;
    ep.out = dC.p;
    ep.ldo = N;
    ep.w_scale = dS.p;
    launch_gemm_sp(iolmk::EPI_F32, sp24_codes_map(l, dW.p), sp24_act_map_h16(dX.p, K, T, K), sp24_meta_map(l, dE.p),
                   K, l.katoms_pad, ep, nullptr, sm_count(), true);
    CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaMemcpy(out_f32, dC.p, sizeof(float) * T * N, cudaMemcpyDeviceToHost));
  });
}

// Device-only timing of the sparse GEMM (kernel tuning): every group keeps positions (0, 1).
static void sp24_time(int32_t T, int32_t N, int32_t K, int32_t epi, int32_t iters, bool f16, float* ms_out) {
  if (T <= 0 || N <= 0 || K <= 0 || K % 16 != 0 || iters <= 0) throw ContractViolation("debug_gemm_sp24_time");
  const Sp24Layout l = sp24_layout(N, K, f16);
  const size_t xb = static_cast<size_t>(T) * K * (f16 ? 2 : 1);
  DevBuf<uint8_t> dX(xb), dW(l.code_bytes());
  DevBuf<uint8_t> dE(l.meta_bytes());
  DevBuf<float> dS(N), dA(T), dC(static_cast<size_t>(T) * N);
  CUDA_OK(cudaMemset(dX.p, 0x11, xb));
  CUDA_OK(cudaMemset(dW.p, 0x13, l.code_bytes()));
  CUDA_OK(cudaMemset(dE.p, 0x44, l.meta_bytes()));
  CUDA_OK(cudaMemset(dS.p, 0, sizeof(float) * N));
  CUDA_OK(cudaMemset(dA.p, 0, sizeof(float) * T));
  CUDA_OK(cudaMemset(dC.p, 0, sizeof(float) * T * N));
  iolmk::GemmEpi ep;
  ep.M = T;
  ep.N = N;
  ep.out = dC.p;
  ep.ldo = N;
  ep.a_scale = f16 ? nullptr : dA.p;
  ep.w_scale = dS.p;
  const CUtensorMap ta = sp24_codes_map(l, dW.p), te = sp24_meta_map(l, dE.p);
  const CUtensorMap tb = f16 ? sp24_act_map_h16(dX.p, K, T, K) : sp24_act_map(reinterpret_cast<int8_t*>(dX.p), K, T, K);
  cudaEvent_t e0, e1;
  CUDA_OK(cudaEventCreate(&e0));
  CUDA_OK(cudaEventCreate(&e1));
  launch_gemm_sp(epi, ta, tb, te, K, l.katoms_pad, ep, nullptr, sm_count(), f16);
  CUDA_OK(cudaEventRecord(e0));
  for (int i = 0; i < iters; ++i) launch_gemm_sp(epi, ta, tb, te, K, l.katoms_pad, ep, nullptr, sm_count(), f16);
  CUDA_OK(cudaEventRecord(e1));
  CUDA_OK(cudaEventSynchronize(e1));
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
  *ms_out = ms / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

extern "C" int iolm_cuda_debug_gemm_sp24_time(int32_t T, int32_t N, int32_t K, int32_t epi, int32_t iters,
                                              float* ms_out) {
  return guarded([&] { sp24_time(T, N, K, epi, iters, false, ms_out); });
}

extern "C" int iolm_cuda_debug_gemm_sp24_f16_time(int32_t T, int32_t N, int32_t K, int32_t epi, int32_t iters,
                                                   float* ms_out) {
  return guarded([&] { sp24_time(T, N, K, epi, iters, true, ms_out); });
}

extern "C" int iolm_cuda_debug_gemm_w4(const uint16_t* A, const uint8_t* payload, float* C, int32_t M, int32_t N,
                                       int32_t K, int32_t pair) {
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0 || K % 8 != 0) throw ContractViolation("debug_gemm_w4: need K % 8 == 0");
    const size_t rb = static_cast<size_t>(K + 1) / 2, ld4 = (rb + 15) / 16 * 16;
    DevBuf<uint16_t> dA(static_cast<size_t>(M) * K);
    DevBuf<uint8_t> dW(static_cast<size_t>(N) * ld4);
    DevBuf<float> dS(N), dC(static_cast<size_t>(M) * N);
    CUDA_OK(cudaMemcpy(dA.p, A, sizeof(uint16_t) * M * K, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy2D(dW.p, ld4, payload, rb, rb, N, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dS.p, payload + rb * N, sizeof(float) * N, cudaMemcpyHostToDevice));
    CUtensorMap ta = make_kmajor_map(dA.p, H16_TMA, 2, K, M, 2ull * K, 128);
    CUtensorMap tb = make_w4_map(dW.p, K, N, ld4);
    iolmk::GemmEpi ep;
    ep.M = M;
    ep.N = N;
    ep.out = dC.p;
    ep.ldo = N;
    ep.w_scale = dS.p;
    launch_gemm_w4(pair != 0, iolmk::EPI_F32, ta, tb, M, N, K, ep, nullptr, sm_count());
    CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaMemcpy(C, dC.p, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
  });
}
