// Persistent, warp-specialised tcgen05 GEMM for sm_100a:  C[M x N] = A[M x K] * W[N x K]^T
//
//   A  : activations, K-major (row-major [M x K]), bf16 (or int8 for the W8A8 variant)
//   W  : weights as stored in the bundle, [out x in] = [N x K] row-major, i.e. also K-major
//        (the reference applies x * W^T via transposed copies, runtime.cpp:80-85; on the GPU the
//        bundle layout is already the K-major B operand, so no transpose is materialised)
//
// Roles (192 threads, one CTA per SM, persistent over output tiles):
//   warp 0      : TMA producer (one elected lane) - A and W tiles into a STAGES-deep smem ring
//   warp 1      : TMEM allocator + MMA issuer (one elected lane), tcgen05.mma into a
//                 double-buffered fp32 accumulator in TMEM (2 x BN columns)
//   warps 2..5  : epilogue - tcgen05.ld 32 lanes x 32 columns per step, fused op, global store
//
// Reduction order per output element is fixed by K alone (BK-blocks ascending, UMMA_K steps
// ascending inside a block) and never depends on M, the tile a row lands in, or the batch, which is
// what keeps batch_decode(P)[i] == batch_decode({P[i]}) bitwise on the GPU (the invariant the
// reference proves for its CPU matmul, test_model.cpp:240-267).
#pragma once
#include "ptx.cuh"

namespace iolmk {

enum EpiMode : int {
  EPI_F32 = 0,        // out f32 [M x ldo]
  EPI_BF16 = 1,       // out bf16 [M x ldo]
  EPI_GELU_BF16 = 2,  // out bf16 gelu(acc)
  EPI_RESID_F32 = 3,  // resid f32 [M x ldo] += acc   (x += z*Wo^T, x += g*Wout^T)
  EPI_QKV = 4,        // cols [0,kh) -> q bf16; [kh,2kh) -> K pages; [2kh,3kh) -> V pages
  EPI_S32 = 5,        // raw int32 accumulators [M x ldo] (integer GEMM parity tests)
};

struct GemmEpi {
  int M = 0, N = 0;
  void* out = nullptr;
  int ldo = 0;
  // QKV scatter into the paged KV pool of one layer. Page layout: [page][K|V][head][PAGE][hd].
  __nv_bfloat16* kv_layer = nullptr;
  const int* tok_slot = nullptr;
  const int* tok_pos = nullptr;
  const int* page_table = nullptr;
  int max_pages = 0;
  int kh = 0, hd = 0, heads = 0, page_size = 16;
  // W8A8 dequant epilogue: acc_i32 * a_scale[row] * w_scale[col]
  const float* a_scale = nullptr;
  const float* w_scale = nullptr;
};

// Tile configuration. CG = 2 runs the 2-SM UMMA: a CTA pair computes a 256 x BN tile, each CTA
// stages its own 128 rows of A and half (BN/2 rows) of the W tile, the leader CTA issues
// tcgen05.mma.cta_group::2, and each CTA drains its 128 accumulator lanes from its own TMEM.
template <int BN, int CG>
struct GemmCfg {
  static constexpr int BM = 128;        // rows per CTA
  static constexpr int TILE_M = BM * CG;
  static constexpr int BN_CTA = BN / CG;  // W rows staged per CTA
  static constexpr int BK_BYTES = 128;  // one 128-byte swizzle row per operand row
  static constexpr int STAGES = CG == 2 ? (BN >= 256 ? 6 : 8) : (BN >= 256 ? 4 : 6);
  static constexpr uint32_t A_BYTES = BM * BK_BYTES;
  static constexpr uint32_t B_BYTES = BN_CTA * BK_BYTES;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr int EPI_WARPS = 8;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr size_t SMEM = 1024 + STAGES * STAGE_BYTES + 256;
};

template <int EPI>
__device__ __forceinline__ void epi_apply(const GemmEpi& ep, int m, int n0, float (&v)[32]) {
  const int N = ep.N;
  if constexpr (EPI == EPI_GELU_BF16) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(v[j]);
  }
  if constexpr (EPI == EPI_BF16 || EPI == EPI_GELU_BF16) {
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(ep.out) + static_cast<size_t>(m) * ep.ldo + n0;
    if (n0 + 32 <= N && (ep.ldo & 7) == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 w;
        w.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
        w.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
        w.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
        w.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
        reinterpret_cast<uint4*>(o)[j] = w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) o[j] = __float2bfloat16_rn(v[j]);
    }
  } else if constexpr (EPI == EPI_F32) {
    float* o = static_cast<float*>(ep.out) + static_cast<size_t>(m) * ep.ldo + n0;
    if (n0 + 32 <= N && (ep.ldo & 3) == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        reinterpret_cast<float4*>(o)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) o[j] = v[j];
    }
  } else if constexpr (EPI == EPI_RESID_F32) {
    float* o = static_cast<float*>(ep.out) + static_cast<size_t>(m) * ep.ldo + n0;
    if (n0 + 32 <= N && (ep.ldo & 3) == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 x = reinterpret_cast<float4*>(o)[j];
        x.x += v[4 * j];
        x.y += v[4 * j + 1];
        x.z += v[4 * j + 2];
        x.w += v[4 * j + 3];
        reinterpret_cast<float4*>(o)[j] = x;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) o[j] += v[j];
    }
  } else if constexpr (EPI == EPI_QKV) {
    const int kh = ep.kh;
    const int slot = ep.tok_slot[m];
    const int pos = ep.tok_pos[m];
    const int page = ep.page_table[static_cast<size_t>(slot) * ep.max_pages + pos / ep.page_size];
    const int in_page = pos % ep.page_size;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + 8 * j;
      if (n >= N) break;
      uint4 w;
      w.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
      w.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
      w.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
      w.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
      __nv_bfloat16* dst;
      if (n < kh) {
        dst = static_cast<__nv_bfloat16*>(ep.out) + static_cast<size_t>(m) * ep.ldo + n;
      } else {
        const int c = n - kh;
        const int which = c >= kh ? 1 : 0;
        const int cc = c - which * kh;
        const int head = cc / ep.hd;
        const int dim = cc - head * ep.hd;
        dst = ep.kv_layer +
              ((static_cast<size_t>(page) * 2 + which) * ep.heads + head) * ep.page_size * ep.hd +
              static_cast<size_t>(in_page) * ep.hd + dim;
      }
      *reinterpret_cast<uint4*>(dst) = w;
    }
  }
}

template <int BN, int EPI, int CG, bool I8>
__global__ void __launch_bounds__(GemmCfg<BN, CG>::THREADS, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, GemmEpi ep) {
  using C = GemmCfg<BN, CG>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sA = base;
  const uint32_t sB = base + STAGES * C::A_BYTES;
  const uint32_t bars = sB + STAGES * C::B_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * STAGES + 4);
  const uint32_t* tmem_slot_ptr = reinterpret_cast<const uint32_t*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);  // pair: the leader's expect_tx covers both CTAs' bytes
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), C::EPI_WARPS * CG);
    }
    mbar_fence_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc2(tmem_slot, C::TMEM_COLS);
    else tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;

  const int m_tiles = (M + C::TILE_M - 1) / C::TILE_M;
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int kbs = (K * (I8 ? 1 : 2) + C::BK_BYTES - 1) / C::BK_BYTES;  // 128-byte K blocks
  constexpr int KELEMS = I8 ? 128 : 64;                                // K elements per block
  const int group = blockIdx.x / CG, n_groups = gridDim.x / CG;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t leader_full0 = CG == 2 ? mapa_shared(full_bar(0), 0) : full_bar(0);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = group; tile < num_tiles; tile += n_groups) {
        const int mt = tile / n_tiles;
        const int nt = tile - mt * n_tiles;
        const int arow = mt * C::TILE_M + static_cast<int>(rank) * C::BM;
        const int brow = nt * BN + static_cast<int>(rank) * C::BN_CTA;
        for (int kb = 0; kb < kbs; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          if constexpr (CG == 2) {
            const uint32_t lf = leader_full0 + 8u * stage;
            // The peer's bytes may land on the leader's barrier before the leader's expect_tx of
            // the same phase: the transaction count goes transiently negative, which the
            // barrier allows; the phase cannot complete before the leader's arrive.
            if (leader) mbar_expect_tx(full_bar(stage), 2 * C::STAGE_BYTES);
            tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, lf, kb * KELEMS, arow);
            tma_load_2d_pair(sB + stage * C::B_BYTES, &tmB, lf, kb * KELEMS, brow);
          } else {
            mbar_expect_tx(full_bar(stage), C::STAGE_BYTES);
            tma_load_2d(sA + stage * C::A_BYTES, &tmA, full_bar(stage), kb * KELEMS, arow);
            tma_load_2d(sB + stage * C::B_BYTES, &tmB, full_bar(stage), kb * KELEMS, brow);
          }
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
      constexpr uint32_t idesc = I8 ? idesc_i8(128 * CG, BN) : idesc_f16(128 * CG, BN, 1);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = group; tile < num_tiles; tile += n_groups) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < kbs; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          const uint64_t ad = smem_desc_k_sw128(sA + stage * C::A_BYTES);
          const uint64_t bd = smem_desc_k_sw128(sB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t accum = (kb | kk) != 0 ? 1u : 0u;
            if constexpr (CG == 2) {
              if constexpr (I8) umma_i8_pair(d, ad + 2u * kk, bd + 2u * kk, idesc, accum);
              else umma_f16_pair(d, ad + 2u * kk, bd + 2u * kk, idesc, accum);
            } else {
              if constexpr (I8) umma_i8(d, ad + 2u * kk, bd + 2u * kk, idesc, accum);
              else umma_f16(d, ad + 2u * kk, bd + 2u * kk, idesc, accum);
            }
          }
          if constexpr (CG == 2) umma_commit_pair_mc(empty_bar(stage), 0x3);
          else umma_commit(empty_bar(stage));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if constexpr (CG == 2) umma_commit_pair_mc(tfull_bar(acc), 0x3);
        else umma_commit(tfull_bar(acc));
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1u;
      }
    }
    __syncwarp();
  } else {
    const int e = warp - 2;
    const int q = warp & 3;             // TMEM lane quarter this warp may access
    const int c_begin = (e >> 2) * (BN / 2);  // column half handled by this warp
    const uint32_t leader_tempty0 = CG == 2 ? mapa_shared(tempty_bar(0), 0) : tempty_bar(0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = group; tile < num_tiles; tile += n_groups) {
      const int mt = tile / n_tiles;
      const int nt = tile - mt * n_tiles;
      const int m = mt * C::TILE_M + static_cast<int>(rank) * C::BM + q * 32 + lane;
      if constexpr (EPI == EPI_RESID_F32) {
        // warm L2 with this thread's residual row segment while the MMAs of the tile run
        if (m < M) {
          const float* xr = static_cast<const float*>(ep.out) + static_cast<size_t>(m) * ep.ldo + nt * BN + c_begin;
#pragma unroll
          for (int c = 0; c < BN / 2; c += 32)
            if (nt * BN + c_begin + c < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + c));
        }
      }
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
#pragma unroll 1
      for (int c = c_begin; c < c_begin + BN / 2; c += 32) {
        const int n0 = nt * BN + c;
        if (n0 >= N) break;  // warp-uniform
        uint32_t r[32];
        tmem_ld_32x32b_x32(tbase + c, r);
        tmem_ld_wait();
        if (m < M) {
          if constexpr (EPI == EPI_S32) {
            int32_t* o = static_cast<int32_t*>(ep.out) + static_cast<size_t>(m) * ep.ldo + n0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + j < N) o[j] = static_cast<int32_t>(r[j]);
          } else {
            float v[32];
            if constexpr (I8) {
              const float sa = ep.a_scale[m];
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int n = min(n0 + j, N - 1);
                v[j] = static_cast<float>(static_cast<int32_t>(r[j])) * sa * ep.w_scale[n];
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            }
            epi_apply<EPI>(ep, m, n0, v);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(leader_tempty0 + 8u * acc);
        else mbar_arrive(tempty_bar(acc));
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1u;
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc2(tmem_base, C::TMEM_COLS);
    else tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace iolmk
