// Host-side API of the 2:4 sparse tensor-core path (sparse24.cu, kernel in gemm_sp_sm100.cuh).
#pragma once
#include <cuda.h>
#include <cstddef>
#include <cstdint>

#include "gemm_sm100.cuh"

namespace iolmh {

// Device layout of one stacked sparse weight group [N x K] (see sparse24.cu).
struct Sp24Layout {
  int N = 0, K = 0;
  bool f16 = false;    // kept codes stored as fp16 (kind::f16 kernel) instead of int8 (kind::i8)
  int ld_c = 0;        // compressed row pitch in bytes (K/2 elements rounded up to 16 bytes)
  int katoms_pad = 0;  // metadata atoms (128 logical K each) per 128-row tile, padded to whole stages
  int mtiles = 0;      // 128-row metadata tiles, padded to whole 256-row pair tiles
  size_t meta_bytes() const { return static_cast<size_t>(mtiles) * katoms_pad * 128 * 16; }
  size_t code_bytes() const { return static_cast<size_t>(N) * ld_c; }
};

Sp24Layout sp24_layout(int N, int K, bool f16 = false);
// True when a sparse24_q8 payload [rows x cols] can run on the sparse MMA (cols % 4 == 0 and
// every group lists two ascending positions, as ModelBundle::append_sparse24_q8 enforces).
bool sp24_check(const uint8_t* payload, int rows, int cols);
// Repacks one tensor's payload into rows [row0, row0 + rows) of the group's host staging buffers
// (codes [N x ld_c] zero-filled, meta [meta_bytes] filled with 0x44, scales [N]).
// codes: int8 [N x ld_c], or for l.f16 the same codes as exact fp16 integers (uint16 bit patterns).
void sp24_append(const Sp24Layout& l, const uint8_t* payload, int rows, int cols, int row0, void* codes,
                 uint8_t* meta, float* scales);
// After every tensor of a group is appended: the kind::f16 metadata layout (a no-op for int8).
void sp24_finalize(const Sp24Layout& l, uint8_t* meta);
CUtensorMap sp24_codes_map(const Sp24Layout& l, const void* d_codes);
CUtensorMap sp24_meta_map(const Sp24Layout& l, const uint8_t* d_meta);
// int8 activation operand [rows x K] (row pitch ld bytes) in the sparse kernel's 112-row boxes.
CUtensorMap sp24_act_map(const int8_t* act, int K, int rows, int ld);
// fp16 activation operand [rows x K] (row pitch ld elements) for the kind::f16 sparse kernel.
CUtensorMap sp24_act_map_h16(const void* act, int K, int rows, int ld);
// C = X * W^T with W the sparse operand: ep.M = tokens, ep.N = output channels.
void launch_gemm_sp(int epi, const CUtensorMap& A, const CUtensorMap& B, const CUtensorMap& E, int K, int katoms_pad,
                    const iolmk::GemmEpi& ep, cudaStream_t st, int grid_cap, bool f16 = false, const CUtensorMap* resid_map = nullptr);

}  // namespace iolmh
