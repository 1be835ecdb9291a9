// Host launchers for the tcgen05 GEMM instantiations.
#include "gemm_sm100.cuh"
#include "launch.hpp"

namespace iolmh {

using namespace iolmk;

template <int BN, int EPI>
static void launch_one(const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                       const GemmEpi& ep, cudaStream_t st, int grid_cap) {
  using Cfg = GemmCfg<BN>;
  static bool configured = false;
  if (!configured) {
    CUDA_OK(cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, EPI>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(Cfg::SMEM)));
    configured = true;
  }
  const int tiles = ((M + Cfg::BM - 1) / Cfg::BM) * ((N + BN - 1) / BN);
  const int grid = tiles < grid_cap ? tiles : grid_cap;
  if (grid <= 0) return;
  gemm_bf16_tn_kernel<BN, EPI><<<grid, 192, Cfg::SMEM, st>>>(A, B, M, N, K, ep);
  CUDA_OK(cudaGetLastError());
}

template <int BN>
static void dispatch_epi(int epi, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                         const GemmEpi& ep, cudaStream_t st, int grid_cap) {
  switch (epi) {
    case EPI_F32: return launch_one<BN, EPI_F32>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_BF16: return launch_one<BN, EPI_BF16>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_GELU_BF16: return launch_one<BN, EPI_GELU_BF16>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_RESID_F32: return launch_one<BN, EPI_RESID_F32>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_QKV: return launch_one<BN, EPI_QKV>(A, B, M, N, K, ep, st, grid_cap);
    default: throw Unsupported("gemm: unknown epilogue");
  }
}

void launch_gemm_bf16(int bn, int epi, const CUtensorMap& A, const CUtensorMap& B, int M, int N,
                      int K, const GemmEpi& ep, cudaStream_t st, int grid_cap) {
  if (M <= 0 || N <= 0) return;
  if (bn == 256)
    dispatch_epi<256>(epi, A, B, M, N, K, ep, st, grid_cap);
  else if (bn == 128)
    dispatch_epi<128>(epi, A, B, M, N, K, ep, st, grid_cap);
  else
    throw Unsupported("gemm: BN must be 128 or 256");
}

}  // namespace iolmh
