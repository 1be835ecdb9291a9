// 2:4 structured-sparse W8A8 GEMM on the sparse tensor cores (tcgen05.mma.sp.cta_group::2.kind::i8).
//
//   C[T x N] = X[T x K] * W[N x K]^T,  W 2:4-sparse along K (the reference's sparse24_q8 bundle
//   encoding, proj/src/model.cpp:255-290 / decode at :177-199), X the per-token int8 activations.
//
// The sparse operand of tcgen05.mma.sp is A, so the roles are swapped relative to the dense GEMM:
// the MMA computes C^T = W * X^T with M = output channels (W rows, 128 per CTA, 256 per CTA pair)
// and N = tokens (BN = 224 per pair tile, 112 staged per CTA). The accumulator in TMEM therefore
// holds one output channel per lane and one token per column, which makes the epilogue naturally
// coalesced: for a fixed token, the 32 lanes of a warp own 32 consecutive output channels.
//
// Operands per pipeline stage (256 logical K):
//   A  compressed weights: 128 rows x 128 B (256 logical K -> 128 kept int8 per row), SWIZZLE_128B;
//      the bundle's kept-code stream (2 codes per group of 4, group-major) IS the compressed
//      K-major layout the MMA expects, so the codes are only re-pitched, never reordered.
//   B  activations: 112 rows x 256 B as two SWIZZLE_128B boxes of 128 K each.
//   E  metadata: 128 rows x 32 B (1 bit per logical element: per group of 4 the two 2-bit
//      positions p0 | p1 << 2, low nibble = even group; exactly the bundle's nibble stream).
//      The loader pre-tiles it into 128-row x 16-B atoms (sparse24_repack in sparse24.cu); the MMA
//      warp copies each stage's two atoms smem -> TMEM with tcgen05.cp.128x128b into a per-stage
//      column slot, so a slot is rewritten only after the MMAs that read it have committed.
// TMEM (512 columns): two 224-column int32 accumulators + STAGES x 8 metadata columns.
//
// Reduction order: per output element, ascending K blocks and ascending MMA k-steps, identical for
// every M / batch composition, and integer-exact: the int32 accumulators equal the dense kind::i8
// GEMM over the expanded weights bit-for-bit (tests/test_sparse_gpu.py).
#pragma once
#include "gemm_sm100.cuh"

namespace iolmk {

struct SpCfg {
  static constexpr int BM = 128;       // output channels per CTA (TMEM lanes)
  static constexpr int TILE_M = 256;   // per CTA pair
  static constexpr int BN = 224;       // tokens per pair tile (MMA N)
  static constexpr int BN_CTA = 112;   // tokens staged per CTA
  static constexpr int BK = 256;       // logical K per stage
  static constexpr int STAGES = 4;
  static constexpr uint32_t A_BYTES = BM * 128;
  static constexpr uint32_t B_BOX = BN_CTA * 128;
  static constexpr uint32_t B_BYTES = 2 * B_BOX;
  static constexpr uint32_t E_BYTES = BM * 32;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES + E_BYTES;
  static constexpr uint32_t E_COL0 = 2 * BN;  // metadata slots after the two accumulators
  static constexpr uint32_t TMEM_COLS = 512;
  // 16 epilogue warps: 4 per TMEM lane quarter, each draining 56 of the tile's 224 token columns
  // (chunks of 16, 16, 16, 8). Twice the warps of the first version: the epilogue is latency-bound
  // (per-chunk dependency chains), so warps per scheduler, not instructions, set its rate.
  static constexpr int EPI_WARPS = 16;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int WTOK = BN / (EPI_WARPS / 4);  // 56 tokens per epilogue warp
  static constexpr int CHUNK = 16;                   // tokens per tcgen05.ld
  static constexpr int NCH = (WTOK + CHUNK - 1) / CHUNK;
  static constexpr size_t SMEM =
      1024 + STAGES * STAGE_BYTES + 256 + EPI_WARPS * WTOK * sizeof(QkvRow) + EPI_WARPS * 64 * sizeof(float);
  static_assert(E_COL0 + 8 * STAGES <= TMEM_COLS, "TMEM budget");
  static_assert(EPI_WARPS * 1024 <= EPI_WARPS * WTOK * 24, "RESID staging tiles fit in the QKV row area");
};

// kind::i8 instruction descriptor with the sparse flag (bit 2): s8 x s8 -> s32, K-major A/B.
__host__ __device__ constexpr uint32_t idesc_i8_sp(int M, int N) { return idesc_i8(M, N) | (1u << 2); }
// kind::f16 with the sparse flag: fp16 x fp16 -> f32 (the W16A16 / W8A16 path: A = the kept weight
// codes as exact fp16 integers, B = fp16 activations; the per-channel scale is applied in the epilogue).
__host__ __device__ constexpr uint32_t idesc_f16_sp(int M, int N) { return idesc_f16(M, N, H16_FMT) | (1u << 2); }

__device__ __forceinline__ void umma_f16_sp_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t tmem_e,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(tmem_e), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_i8_sp_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t tmem_e,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%3], %4, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(tmem_e), "r"(idesc), "r"(accumulate)
      : "memory");
}
// smem -> TMEM copy of a 128-row x 16-byte matrix (lane i <- row i), issued for both CTAs of the pair.
__device__ __forceinline__ void tmem_cp_128x128b_pair(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
// Descriptor of a non-swizzled K-major smem matrix of 16-byte rows: 8-row core matrices of 128 B
// stacked contiguously (SBO = 128 B).
__device__ __forceinline__ uint64_t smem_desc_rows16(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(128 >> 4) << 16;  // LBO (single 16-B column: unused)
  d |= static_cast<uint64_t>(128 >> 4) << 32;  // SBO: next 8 rows
  d |= static_cast<uint64_t>(1) << 46;         // sm_100 descriptor version
  return d;                                    // layout type 0: SWIZZLE_NONE
}

__device__ __forceinline__ void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// tmA: compressed weights [N rows x K/2 bytes]; tmB: activations [T rows x K bytes] (box 112 rows);
// tmE: metadata atoms [rows x 16 B] (box 256 rows). ep.M = tokens T, ep.N = output channels.
//
// F16 = true: the same pipeline over fp16 operands (tcgen05.mma.sp kind::f16). A 128-byte operand row
// then holds 64 kept fp16 = 128 logical K, so a stage covers 128 logical K with ONE metadata atom
// (128 rows x 16 B -> 4 TMEM columns, one per 32-K MMA) instead of two; A / B / E tiles keep their
// byte shapes (B: 112 tokens x 128 K x 2 B as two 64-K SWIZZLE_128B boxes). Epilogue: acc * s_w.
template <int EPI, bool F16 = false>
__global__ void __launch_bounds__(SpCfg::THREADS, 1)
    gemm_sp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmX, int K,
                   int katoms_pad, GemmEpi ep) {
  using C = SpCfg;
  constexpr int STAGES = C::STAGES;
  constexpr int BKL = F16 ? 128 : C::BK;                     // logical K per stage
  constexpr int A_EL = F16 ? 64 : 128;                        // kept elements per stage row (128 B)
  constexpr int B_EL = F16 ? 64 : 128;                        // activation elements per 128-B box row
  constexpr int E_ROWS = F16 ? 128 : 256;                     // metadata atom rows per stage
  constexpr uint32_t STAGE_TX = C::A_BYTES + C::B_BYTES + (F16 ? C::E_BYTES / 2 : C::E_BYTES);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sA = base;
  const uint32_t sB = sA + STAGES * C::A_BYTES;
  const uint32_t sE = sB + STAGES * C::B_BYTES;
  const uint32_t bars = sE + STAGES * C::E_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * STAGES + 4);
  const uint32_t* tmem_slot_ptr = reinterpret_cast<const uint32_t*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), C::EPI_WARPS * 2);
    }
    mbar_fence_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmE);
  }
  if (warp == 1) tmem_alloc2(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  pdl_sync();

  const int T = ep.M, N = ep.N;
  const int w_tiles = (N + C::TILE_M - 1) / C::TILE_M;
  const int t_tiles = (T + C::BN - 1) / C::BN;
  const int num_tiles = w_tiles * t_tiles;
  const int kbs = (K + BKL - 1) / BKL;
  const int group = blockIdx.x / 2, n_groups = gridDim.x / 2;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t leader_full0 = mapa_shared(full_bar(0), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = group; tile < num_tiles; tile += n_groups) {
        const int tt = tile / w_tiles;
        const int wt = tile - tt * w_tiles;
        const int wrow = wt * C::TILE_M + static_cast<int>(rank) * C::BM;
        const int trow = tt * C::BN + static_cast<int>(rank) * C::BN_CTA;
        const int erow = (wt * 2 + static_cast<int>(rank)) * katoms_pad * 128;
        for (int kb = 0; kb < kbs; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          const uint32_t lf = leader_full0 + 8u * stage;
          if (leader) mbar_expect_tx(full_bar(stage), 2 * STAGE_TX);
          tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, lf, kb * A_EL, wrow);
          tma_load_2d_pair(sB + stage * C::B_BYTES, &tmB, lf, kb * BKL, trow);
          tma_load_2d_pair(sB + stage * C::B_BYTES + C::B_BOX, &tmB, lf, kb * BKL + B_EL, trow);
          tma_load_2d_pair(sE + stage * C::E_BYTES, &tmE, lf, 0, erow + kb * E_ROWS);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = F16 ? idesc_f16_sp(C::TILE_M, C::BN) : idesc_i8_sp(C::TILE_M, C::BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = group; tile < num_tiles; tile += n_groups) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * C::BN);
        for (int kb = 0; kb < kbs; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint32_t ecol = tmem_base + C::E_COL0 + 8u * stage;
          const uint32_t se = sE + stage * C::E_BYTES;
          tmem_cp_128x128b_pair(ecol, smem_desc_rows16(se));
          if constexpr (!F16) tmem_cp_128x128b_pair(ecol + 4u, smem_desc_rows16(se + 2048u));
          const uint64_t ad = smem_desc_k_sw128(sA + stage * C::A_BYTES);
          const uint64_t bd0 = smem_desc_k_sw128(sB + stage * C::B_BYTES);
          const uint64_t bd1 = smem_desc_k_sw128(sB + stage * C::B_BYTES + C::B_BOX);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t accum = (kb | kk) != 0 ? 1u : 0u;
            // A advances 32 compressed bytes per MMA (64 logical K of int8 / 32 of fp16); B 64 bytes
            // inside its 128-byte box; E 64 (int8) or 32 (fp16) metadata bits = 2 or 1 TMEM columns
            const uint64_t bd = (kk < 2 ? bd0 : bd1) + 4u * (kk & 1);
            // kind::f16: the metadata address must be 2-column aligned; an odd column is selected
            // with the instruction descriptor's sparse id2 field (bits [0, 2))
            if constexpr (F16) umma_f16_sp_pair(d, ad + 2u * kk, bd, (ecol + kk) & ~1u, idesc | ((ecol + kk) & 1u), accum);
            else umma_i8_sp_pair(d, ad + 2u * kk, bd, ecol + 2u * kk, idesc, accum);
          }
          umma_commit_pair_mc(empty_bar(stage), 0x3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit_pair_mc(tfull_bar(acc), 0x3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1u;
      }
    }
    __syncwarp();
  } else {
    const int e = warp - 2;
    const int q = warp & 3;                      // TMEM lane quarter
    const int c_begin = (e >> 2) * C::WTOK;      // this warp's token columns [c_begin, c_begin + 56)
    constexpr int NCH = C::NCH;
    const uint32_t leader_tempty0 = mapa_shared(tempty_bar(0), 0);
    QkvRow* s_rows = reinterpret_cast<QkvRow*>(smem_raw + (bars + 256 - raw)) + e * C::WTOK;
    // the warp's 56 per-token activation scales (+ padding to 64): read back as warp-uniform
    // float4 broadcasts (4 LDS per 16 tokens instead of 16 shuffles)
    float* s_as = reinterpret_cast<float*>(smem_raw + (bars + 256 - raw) + C::EPI_WARPS * C::WTOK * sizeof(QkvRow)) +
                  e * 64;
    const bool has_ws = ep.w_scale != nullptr;
    const size_t head_stride = static_cast<size_t>(ep.page_size) << ep.hd_shift;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = group; tile < num_tiles; tile += n_groups) {
      const int tt = tile / w_tiles;
      const int wt = tile - tt * w_tiles;
      const int tw0 = tt * C::BN + c_begin;  // first token of this warp's half tile
      const int ch = wt * C::TILE_M + static_cast<int>(rank) * C::BM + q * 32 + lane;  // this thread's channel
      const bool ch_ok = ch < N;
      // Per-tile operands are fetched BEFORE waiting for the accumulator, so their global-memory
      // latency overlaps the mainloop instead of stalling every chunk: the channel's weight scale,
      // one activation scale per (chunk, lane & 15) token, and (QKV) the 112 token destinations.
      const float w_sc = has_ws && ch_ok ? ep.w_scale[ch] : 1.f;
      __syncwarp();  // the previous tile's readers of s_as are done
      for (int i = lane; i < 64; i += 32) {
        const int t = tw0 + i;
        s_as[i] = ep.a_scale != nullptr ? (i < C::WTOK && t < T ? ep.a_scale[t] : 0.f) : 1.f;
      }
      __syncwarp();
      int region = 0, off = ch;
      if constexpr (EPI == EPI_QKV) {
        if (ch >= ep.kh) {
          const int c = ch - ep.kh;
          region = c >= ep.kh ? 2 : 1;
          const int cc = region == 2 ? c - ep.kh : c;
          off = static_cast<int>((cc >> ep.hd_shift) * head_stride) + (cc & (ep.hd - 1));
        }
        for (int i = lane; i < C::WTOK; i += 32) s_rows[i] = tw0 + i < T ? qkv_row(ep, tw0 + i) : QkvRow{};
        __syncwarp();
      }
      // RESID: this warp's 8-token x 32-channel staging tile (in the QKV destination area, unused
      // by this epilogue): x += v leaves through TMA reduce-add boxes, so x is never loaded into
      // registers and there is one shared store per element instead of a global load + store
      // (1 KB per warp from the 256-aligned start of the area: TMA sources must be 128-byte aligned)
      float* stage = reinterpret_cast<float*>(smem_raw + (bars + 256 - raw) + e * 1024);
      const uint32_t stage_addr = smem_u32(stage);
      const int ch0 = wt * C::TILE_M + static_cast<int>(rank) * C::BM + q * 32;  // the warp's first channel
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * C::BN);
      if constexpr (EPI == EPI_NONE) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(leader_tempty0 + 8u * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1u;
        continue;
      }
      uint32_t r[2][16];
      tmem_ld_32x32b_x16(tbase + c_begin, r[0]);
#pragma unroll
      for (int ci = 0; ci < NCH; ++ci) {
        const int t0 = tw0 + ci * C::CHUNK;  // first token of the chunk
        constexpr int JN_FULL = C::CHUNK;
        const int jn = (ci + 1) * C::CHUNK <= C::WTOK ? JN_FULL : C::WTOK - ci * C::CHUNK;  // tokens in chunk
        tmem_ld_wait();
        if (ci + 1 < NCH) {
          if ((ci + 2) * C::CHUNK <= C::WTOK) tmem_ld_32x32b_x16(tbase + c_begin + (ci + 1) * C::CHUNK, r[(ci + 1) & 1]);
          else tmem_ld_32x32b_x8(tbase + c_begin + (ci + 1) * C::CHUNK, r[(ci + 1) & 1]);
        }
        const uint32_t(&rc)[16] = r[ci & 1];
        if (t0 < T) {
          if constexpr (EPI == EPI_S32) {
            int32_t* o = static_cast<int32_t*>(ep.out);
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < jn && ch_ok && t0 + j < T) o[static_cast<size_t>(t0 + j) * ep.ldo + ch] = static_cast<int32_t>(rc[j]);
          } else {
            float v[16];
            float as[16];
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(as + j) = *reinterpret_cast<const float4*>(s_as + ci * C::CHUNK + j);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              // same operations as the dense epilogues: int8 (acc * s_a[token]) * s_w[ch], fp16 codes
              // acc * s_w[ch], each rounded (explicit _rn: no FMA contraction into the residual add)
              if constexpr (F16) v[j] = __fmul_rn(__uint_as_float(rc[j]), w_sc);
              else v[j] = __fmul_rn(__fmul_rn(static_cast<float>(static_cast<int32_t>(rc[j])), as[j]), w_sc);
            }
            if constexpr (EPI == EPI_GELU_H16) {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = gelu_tanh(v[j]);
            }
            if constexpr (EPI == EPI_F32) {
              float* o = static_cast<float*>(ep.out);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (j < jn && ch_ok && t0 + j < T) o[static_cast<size_t>(t0 + j) * ep.ldo + ch] = v[j];
            } else if constexpr (EPI == EPI_RESID_F32) {
              // two 8-token boxes per chunk; TMA clips tokens >= T and channels >= N. The tile is
              // reused only once the previous box has been read out of shared memory.
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                if (h * 8 < jn && t0 + h * 8 < T) {
                  if (lane == 0) bulk_wait_read0();
                  __syncwarp();
#pragma unroll
                  for (int j = 0; j < 8; ++j)  // rows past T (inside the tensor map) add +0
                    stage[j * 32 + lane] = t0 + h * 8 + j < T ? v[h * 8 + j] : 0.f;
                  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                  __syncwarp();
                  if (lane == 0) {
                    tma_reduce_add_2d(&tmX, stage_addr, ch0, t0 + h * 8);
                    bulk_commit();
                  }
                }
              }
            } else {
              // fp16 outputs: lane pairs exchange one value so that every store is a 4-byte
              // channel pair; even lanes write token j, odd lanes token j + 1
              const bool odd = lane & 1;
              const int c0 = ch & ~1;
              if constexpr (EPI != EPI_QKV) {
                if (jn == C::CHUNK && t0 + C::CHUNK <= T && c0 + 1 < N) {
                  // whole chunk in range: one 4-byte store per token pair, pointer stepped by 2 rows
                  uint32_t* dst = reinterpret_cast<uint32_t*>(static_cast<h16*>(ep.out) +
                                                              static_cast<size_t>(t0 + (odd ? 1 : 0)) * ep.ldo + c0);
                  const size_t step = static_cast<size_t>(ep.ldo);  // 2 rows of fp16 = ldo uint32
#pragma unroll
                  for (int j = 0; j < 16; j += 2) {
                    const float send = odd ? v[j] : v[j + 1];
                    const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                    *dst = odd ? pack_h16x2(recv, v[j + 1]) : pack_h16x2(v[j], recv);
                    dst += step;
                  }
                  continue;
                }
              }
#pragma unroll
              for (int j = 0; j < 16; j += 2) {
                const float send = odd ? v[j] : v[j + 1];
                const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                const int jj = j + (odd ? 1 : 0);
                const int tok = t0 + jj;
                const uint32_t packed = odd ? pack_h16x2(recv, v[j + 1]) : pack_h16x2(v[j], recv);
                if (jj < jn && tok < T && c0 < N) {
                  h16* dst;
                  if constexpr (EPI == EPI_QKV) {
                    const QkvRow& rw = s_rows[ci * C::CHUNK + jj];
                    dst = (region == 0 ? rw.q : region == 1 ? rw.k : rw.v) + (off & ~1);
                  } else {
                    dst = static_cast<h16*>(ep.out) + static_cast<size_t>(tok) * ep.ldo + c0;
                  }
                  if (c0 + 1 < N) {
                    *reinterpret_cast<uint32_t*>(dst) = packed;
                  } else {
                    *dst = __ushort_as_half(static_cast<unsigned short>(packed & 0xffffu));
                  }
                }
              }
            }
          }
        }
      }
      if constexpr (EPI == EPI_QKV) __syncwarp();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(leader_tempty0 + 8u * acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1u;
    }
    if constexpr (EPI == EPI_RESID_F32) {
      if (lane == 0) bulk_wait0();  // every reduce-add into x complete before the grid ends
      __syncwarp();
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace iolmk
