// 2:4 sparse weights on the sparse tensor cores: load-time repack of the bundle's sparse24_q8
// payload into the device layout of gemm_sp_kernel, and its host launcher.
//
// Bundle layout (proj/docs/format.md:62, writer proj/src/model.cpp:255-290, reader :177-199):
//   codes  int8 [rows x groups x 2]      the two kept codes of each group of 4, group-major
//   idx    u8   [rows x ceil(groups/2)]  nibble p0 | p1 << 2 per group, low nibble = even group
//   scales f32  [rows]
// Device layout:
//   codes  int8 [N x ld_c], ld_c = round_up(K/2, 16): the same kept-code stream, re-pitched for TMA
//   meta   u8   [(mtile, katom) -> 128 rows x 16 B]: 16 bytes of a row's nibble stream per 128
//          logical K, atoms of 128 rows, ordered (mtile, katom); absent groups hold 0x4 (p0 = 0,
//          p1 = 1: a valid pattern over zero operands)
#include <cstring>
#include <vector>

#include "gemm_sp_sm100.cuh"
#include "launch.hpp"
#include "sparse24.hpp"
#include "tma_host.hpp"

namespace iolmh {

using namespace iolmk;

Sp24Layout sp24_layout(int N, int K, bool f16) {
  Sp24Layout l;
  l.N = N;
  l.K = K;
  l.f16 = f16;
  l.ld_c = ((K / 2) * (f16 ? 2 : 1) + 15) / 16 * 16;
  // int8: a stage is 256 logical K = 2 atoms; fp16: 128 logical K = 1 atom
  l.katoms_pad = f16 ? (K + 127) / 128 : 2 * ((K + SpCfg::BK - 1) / SpCfg::BK);
  l.mtiles = 2 * ((N + SpCfg::TILE_M - 1) / SpCfg::TILE_M);
  return l;
}

bool sp24_check(const uint8_t* payload, int rows, int cols) {
  if (cols % 4 != 0) return false;
  const size_t groups = static_cast<size_t>(cols) / 4;
  const size_t idx_row_bytes = (groups + 1) / 2;
  const uint8_t* idx = payload + static_cast<size_t>(rows) * groups * 2;
  for (int r = 0; r < rows; ++r)
    for (size_t g = 0; g < groups; ++g) {
      const uint8_t b = idx[r * idx_row_bytes + g / 2];
      const int nib = (g % 2 == 0) ? (b & 0xf) : (b >> 4);
      if ((nib & 3) >= ((nib >> 2) & 3)) return false;  // the MMA needs ascending positions
    }
  return true;
}

void sp24_append(const Sp24Layout& l, const uint8_t* payload, int rows, int cols, int row0, void* codes_out,
                 uint8_t* meta, float* scales) {
  const size_t groups = static_cast<size_t>(cols) / 4;
  const size_t idx_row_bytes = (groups + 1) / 2;
  const uint8_t* idx = payload + static_cast<size_t>(rows) * groups * 2;
  const uint8_t* sc = idx + static_cast<size_t>(rows) * idx_row_bytes;
  for (int r = 0; r < rows; ++r) {
    const int gr = row0 + r;
    const uint8_t* src = payload + static_cast<size_t>(r) * groups * 2;
    uint8_t* dst = static_cast<uint8_t*>(codes_out) + static_cast<size_t>(gr) * l.ld_c;
    if (!l.f16) {
      std::memcpy(dst, src, groups * 2);
    } else {  // |code| <= 127 is exact in fp16
      for (size_t i = 0; i < groups * 2; ++i) {
        const uint16_t h = f16_bits_of_int(static_cast<int8_t>(src[i]));
        std::memcpy(dst + 2 * i, &h, 2);
      }
    }
    const int mt = gr / 128, rr = gr % 128;
    for (size_t b = 0; b < idx_row_bytes; ++b) {
      uint8_t v = idx[r * idx_row_bytes + b];
      if ((groups % 2) == 1 && b + 1 == idx_row_bytes) v = static_cast<uint8_t>((v & 0x0f) | 0x40);
      const size_t ka = b / 16;
      meta[((static_cast<size_t>(mt) * l.katoms_pad + ka) * 128 + rr) * 16 + (b % 16)] = v;
    }
    std::memcpy(scales + gr, sc + static_cast<size_t>(r) * 4, 4);
  }
}

// kind::f16 reads one 32-bit metadata word per lane per MMA (32 logical K = 8 groups) with the halves
// of rows r and r + 8 (r % 16 < 8) interleaved: lane r holds [row r groups 0-3 | row r+8 groups 0-3]
// and lane r + 8 holds [row r groups 4-7 | row r+8 groups 4-7] (measured with profiles/sp16_probe.py:
// identity activations expose the positions the tensor core applied). kind::i8 takes each row's own
// 64 bits per MMA unchanged.
void sp24_finalize(const Sp24Layout& l, uint8_t* meta) {
  if (!l.f16) return;
  const size_t atoms = static_cast<size_t>(l.mtiles) * l.katoms_pad;
  for (size_t a = 0; a < atoms; ++a)
    for (int blk = 0; blk < 128; blk += 16)
      for (int i = 0; i < 8; ++i) {
        uint8_t* ra = meta + (a * 128 + blk + i) * 16;
        uint8_t* rb = ra + 8 * 16;
        for (int w = 0; w < 4; ++w) {
          uint32_t A, B;
          std::memcpy(&A, ra + 4 * w, 4);
          std::memcpy(&B, rb + 4 * w, 4);
          const uint32_t na = (A & 0xFFFFu) | (B << 16), nb = (A >> 16) | (B & 0xFFFF0000u);
          std::memcpy(ra + 4 * w, &na, 4);
          std::memcpy(rb + 4 * w, &nb, 4);
        }
      }
}

CUtensorMap sp24_codes_map(const Sp24Layout& l, const void* d_codes) {
  if (l.f16)
    return make_kmajor_map(d_codes, H16_TMA, 2, static_cast<uint64_t>(l.K / 2), l.N,
                           static_cast<uint64_t>(l.ld_c), 128);
  return make_kmajor_map(d_codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, static_cast<uint64_t>(l.K / 2), l.N,
                         static_cast<uint64_t>(l.ld_c), 128);
}

CUtensorMap sp24_meta_map(const Sp24Layout& l, const uint8_t* d_meta) {
  CUtensorMap m;
  cuuint64_t dims[2] = {16, static_cast<cuuint64_t>(l.meta_bytes() / 16)};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {16, l.f16 ? 128u : 256u};  // one stage: 1 (fp16) or 2 (int8) 128-row atoms
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(d_meta), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (sparse metadata) failed: " + std::to_string(r));
  return m;
}

CUtensorMap sp24_act_map(const int8_t* act, int K, int rows, int ld) {
  return make_kmajor_map(act, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, static_cast<uint64_t>(K), rows,
                         static_cast<uint64_t>(ld), SpCfg::BN_CTA);
}

CUtensorMap sp24_act_map_h16(const void* act, int K, int rows, int ld) {
  return make_kmajor_map(act, H16_TMA, 2, static_cast<uint64_t>(K), rows,
                         2ull * static_cast<uint64_t>(ld), SpCfg::BN_CTA);
}

template <int EPI, bool F16>
static void launch_sp_one(const CUtensorMap& A, const CUtensorMap& B, const CUtensorMap& E, const CUtensorMap& X,
                          int K, int katoms_pad, const GemmEpi& ep, cudaStream_t st, int grid_cap) {
  auto kern = gemm_sp_kernel<EPI, F16>;
  ensure_smem(kern, SpCfg::SMEM);
  const int tiles = ((ep.N + SpCfg::TILE_M - 1) / SpCfg::TILE_M) * ((ep.M + SpCfg::BN - 1) / SpCfg::BN);
  const int groups = std::min(tiles, grid_cap / 2);
  if (groups <= 0) return;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(groups * 2);
  cfg.blockDim = dim3(SpCfg::THREADS);
  cfg.dynamicSmemBytes = SpCfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1 + pdl_attr(&attr[1]);  // the kernel calls pdl_sync() after its prologue
  CUDA_OK(cudaLaunchKernelEx(&cfg, kern, A, B, E, X, K, katoms_pad, ep));
}

template <bool F16>
static void launch_sp(int epi, const CUtensorMap& A, const CUtensorMap& B, const CUtensorMap& E, const CUtensorMap& X,
                      int K, int katoms_pad, const GemmEpi& ep, cudaStream_t st, int grid_cap) {
  switch (epi) {
    case EPI_S32:
      if constexpr (F16) throw Unsupported("gemm_sp: raw accumulators are int8-only");
      else launch_sp_one<EPI_S32, false>(A, B, E, X, K, katoms_pad, ep, st, grid_cap);
      break;
    case EPI_F32: launch_sp_one<EPI_F32, F16>(A, B, E, X, K, katoms_pad, ep, st, grid_cap); break;
    case EPI_H16: launch_sp_one<EPI_H16, F16>(A, B, E, X, K, katoms_pad, ep, st, grid_cap); break;
    case EPI_GELU_H16: launch_sp_one<EPI_GELU_H16, F16>(A, B, E, X, K, katoms_pad, ep, st, grid_cap); break;
    case EPI_RESID_F32: launch_sp_one<EPI_RESID_F32, F16>(A, B, E, X, K, katoms_pad, ep, st, grid_cap); break;
    case EPI_QKV: launch_sp_one<EPI_QKV, F16>(A, B, E, X, K, katoms_pad, ep, st, grid_cap); break;
    case EPI_NONE: launch_sp_one<EPI_NONE, F16>(A, B, E, X, K, katoms_pad, ep, st, grid_cap); break;
    default: throw Unsupported("gemm_sp: epilogue not instantiated");
  }
}

void launch_gemm_sp(int epi, const CUtensorMap& A, const CUtensorMap& B, const CUtensorMap& E, int K, int katoms_pad,
                    const GemmEpi& ep, cudaStream_t st, int grid_cap, bool f16, const CUtensorMap* resid_map) {
  if (ep.M <= 0 || ep.N <= 0) return;
  CUtensorMap X = A;  // unused unless epi == EPI_RESID_F32
  if (epi == EPI_RESID_F32) {
    if (resid_map != nullptr) X = *resid_map;
    else X = make_resid_map(static_cast<const float*>(ep.out), ep.N, ep.M, 4ull * ep.ldo);
  }
  if (f16) launch_sp<true>(epi, A, B, E, X, K, katoms_pad, ep, st, grid_cap);
  else launch_sp<false>(epi, A, B, E, X, K, katoms_pad, ep, st, grid_cap);
  CUDA_OK(cudaGetLastError());
}

}  // namespace iolmh
