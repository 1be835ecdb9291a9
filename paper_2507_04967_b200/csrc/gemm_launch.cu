// Host launchers for the tcgen05 GEMM instantiations.
//   fp16 x fp16 -> fp32 (kind::f16) and s8 x s8 -> s32 (kind::i8, W8A8), each as
//   2-SM pairs (CG = 2, 256 x 256 tiles, clusters of 2) or single-CTA (CG = 1, 128 x 128 tiles).
// Every TMA box is 128 rows x 128 bytes, so one tensor map per operand serves both shapes.
#include "gemm_sm100.cuh"
#include "launch.hpp"

namespace iolmh {

using namespace iolmk;

// Output tensor map of the launch in flight (ep.tma_out): set by launch_gemm / launch_gemm_w4.
static thread_local const CUtensorMap* g_out_map = nullptr;

template <int BN, int EPI, int CG, bool I8, bool W4 = false>
static void launch_one(const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K, const GemmEpi& ep,
                       cudaStream_t st, int grid_cap) {
  using Cfg = GemmCfg<BN, CG, W4>;
  auto kern = gemm_tn_kernel<BN, EPI, CG, I8, W4>;
  ensure_smem(kern, Cfg::SMEM);
  const int tiles = ((M + Cfg::TILE_M - 1) / Cfg::TILE_M) * ((N + BN - 1) / BN);
  int groups = std::min(tiles, grid_cap / CG);
  if (groups <= 0) return;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(groups * CG);
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1 + pdl_attr(&attr[1]);  // the kernel calls pdl_sync() after its prologue
  CUDA_OK(cudaLaunchKernelEx(&cfg, kern, A, B, ep.tma_out ? *g_out_map : A, M, N, K, ep));
}

template <int BN, int CG, bool I8>
static void dispatch_epi(int epi, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                         const GemmEpi& ep, cudaStream_t st, int grid_cap) {
  switch (epi) {
    case EPI_F32:
      if constexpr (!I8) return launch_one<BN, EPI_F32, CG, I8>(A, B, M, N, K, ep, st, grid_cap);
      break;
    case EPI_S32:
      if constexpr (I8) return launch_one<BN, EPI_S32, CG, I8>(A, B, M, N, K, ep, st, grid_cap);
      break;
    case EPI_H16: return launch_one<BN, EPI_H16, CG, I8>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_GELU_H16: return launch_one<BN, EPI_GELU_H16, CG, I8>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_RESID_F32: return launch_one<BN, EPI_RESID_F32, CG, I8>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_QKV: return launch_one<BN, EPI_QKV, CG, I8>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_NONE: return launch_one<BN, EPI_NONE, CG, I8>(A, B, M, N, K, ep, st, grid_cap);
    default: break;
  }
  throw Unsupported("gemm: epilogue not instantiated for this operand type");
}

// W4A16: B is the packed int4 weight map (make_w4_map), expanded to fp16 in shared memory.
template <int BN, int CG>
static void dispatch_w4(int epi, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K, const GemmEpi& ep,
                        cudaStream_t st, int grid_cap) {
  switch (epi) {
    case EPI_F32: return launch_one<BN, EPI_F32, CG, false, true>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_H16: return launch_one<BN, EPI_H16, CG, false, true>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_GELU_H16: return launch_one<BN, EPI_GELU_H16, CG, false, true>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_RESID_F32: return launch_one<BN, EPI_RESID_F32, CG, false, true>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_QKV: return launch_one<BN, EPI_QKV, CG, false, true>(A, B, M, N, K, ep, st, grid_cap);
    case EPI_NONE: return launch_one<BN, EPI_NONE, CG, false, true>(A, B, M, N, K, ep, st, grid_cap);
    default: break;
  }
  throw Unsupported("gemm_w4: epilogue not instantiated");
}

void launch_gemm_w4(bool pair, int epi, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                    const GemmEpi& ep_in, cudaStream_t st, int grid_cap, const CUtensorMap* out_map) {
  if (M <= 0 || N <= 0) return;
  GemmEpi ep = ep_in;
  ep.tma_out = out_map != nullptr && (epi == EPI_RESID_F32 || epi == EPI_H16 || epi == EPI_GELU_H16);
  g_out_map = out_map;
  if (pair) dispatch_w4<256, 2>(epi, A, B, M, N, K, ep, st, grid_cap);
  else dispatch_w4<128, 1>(epi, A, B, M, N, K, ep, st, grid_cap);
  CUDA_OK(cudaGetLastError());
}

// pair = true: 2-SM 256x256 tiles; false: single-CTA 128x128 tiles.
void launch_gemm(bool pair, bool i8, int epi, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                 const GemmEpi& ep_in, cudaStream_t st, int grid_cap, const CUtensorMap* out_map) {
  if (M <= 0 || N <= 0) return;
  GemmEpi ep = ep_in;
  ep.tma_out = out_map != nullptr && (epi == EPI_RESID_F32 || epi == EPI_H16 || epi == EPI_GELU_H16);
  g_out_map = out_map;
  if (pair) {
    if (i8) dispatch_epi<256, 2, true>(epi, A, B, M, N, K, ep, st, grid_cap);
    else dispatch_epi<256, 2, false>(epi, A, B, M, N, K, ep, st, grid_cap);
  } else {
    if (i8) dispatch_epi<128, 1, true>(epi, A, B, M, N, K, ep, st, grid_cap);
    else dispatch_epi<128, 1, false>(epi, A, B, M, N, K, ep, st, grid_cap);
  }
  CUDA_OK(cudaGetLastError());
}

}  // namespace iolmh
