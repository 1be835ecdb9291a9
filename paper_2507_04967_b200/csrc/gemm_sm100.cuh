// Persistent, warp-specialised tcgen05 GEMM for sm_100a:  C[M x N] = A[M x K] * W[N x K]^T
//
//   A  : activations, K-major (row-major [M x K]), fp16 (or int8 for the W8A8 variant)
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
  EPI_H16 = 1,       // out fp16 [M x ldo]
  EPI_GELU_H16 = 2,  // out fp16 gelu(acc)
  EPI_RESID_F32 = 3,  // resid f32 [M x ldo] += acc   (x += z*Wo^T, x += g*Wout^T)
  EPI_QKV = 4,        // cols [0,kh) -> q fp16; [kh,2kh) -> K pages; [2kh,3kh) -> V pages
  EPI_S32 = 5,        // raw int32 accumulators [M x ldo] (integer GEMM parity tests)
  EPI_NONE = 6,       // kernel tuning only: accumulators are drained but not read (mainloop rate)
};

struct GemmEpi {
  int M = 0, N = 0;
  void* out = nullptr;
  int ldo = 0;
  // QKV scatter into the paged KV pool of one layer. Page layout: [page][K|V][head][PAGE][hd].
  h16* kv_layer = nullptr;
  const int* tok_slot = nullptr;
  const int* tok_pos = nullptr;
  const int* page_table = nullptr;
  int max_pages = 0;
  int kh = 0, hd = 0, heads = 0, page_size = 16;
  int hd_shift = 0;  // log2(hd); hd is 16/32/64/128
  // W8A8 dequant epilogue: acc_i32 * a_scale[row] * w_scale[col]
  const float* a_scale = nullptr;
  const float* w_scale = nullptr;
  // RESID / H16 / GELU: write full 32 x 32 chunks with TMA (store, or reduce-add into x) from the
  // warp's staging tile instead of per-thread global stores (the kernel's tmC describes `out`)
  int tma_out = 0;
};

// Tile configuration. CG = 2 runs the 2-SM UMMA: a CTA pair computes a 256 x BN tile, each CTA
// stages its own 128 rows of A and half (BN/2 rows) of the W tile, the leader CTA issues
// tcgen05.mma.cta_group::2, and each CTA drains its 128 accumulator lanes from its own TMEM.
// W4 = true: W4A16. The weights stay int4 (the bundle's q4 nibbles, re-pitched) in HBM; TMA
// stages the packed tile (BN_CTA rows x 32 B per 64 K) and CONV_WARPS converter warps expand it
// in shared memory into the fp16 SWIZZLE_128B operand tile the MMA reads (code - 8, exact in fp16;
// the per-channel scale is applied in the epilogue as for the other code forms).
template <int BN, int CG, bool W4 = false>
struct GemmCfg {
  static constexpr int BM = 128;        // rows per CTA
  static constexpr int TILE_M = BM * CG;
  static constexpr int BN_CTA = BN / CG;  // W rows staged per CTA
  static constexpr int BK_BYTES = 128;  // one 128-byte swizzle row per operand row
  // 8 epilogue warps (2 per TMEM lane quarter). 16 warps were measured too: no gain here (this
  // epilogue stages through smem and competes with the MMA for it), unlike the sparse kernel's.
  static constexpr int EPI_WARPS = 8;
  static constexpr int STAGES = CG == 2 ? (BN >= 256 ? 5 : 7) : (BN >= 256 ? 4 : 5);
  static constexpr uint32_t A_BYTES = BM * BK_BYTES;
  static constexpr uint32_t B_BYTES = BN_CTA * BK_BYTES;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr int CONV_WARPS = W4 ? 4 : 0;
  static constexpr uint32_t RAW_BYTES = W4 ? BN_CTA * 32 : 0;  // packed int4 per stage
  static constexpr int THREADS = 64 + 32 * EPI_WARPS + 32 * CONV_WARPS;
  static constexpr size_t SMEM = 1024 + STAGES * (STAGE_BYTES + RAW_BYTES) + 2048 +
                                 EPI_WARPS * 5120;  // rings, barriers + scales, 1 KB-aligned warp tiles
  static_assert(!W4 || BN_CTA == 128, "W4 converter maps one thread per staged weight row");
};

// Expands 4 packed bytes (8 int4 codes, low nibble first) into 4 f16x2 words of (nibble - 8):
// fp16(1024 + n) has bit pattern 0x6400 | n, and 1024 + n - 1032 is exact in fp16. Byte permutes build
// the 0x64nn halves (12 instructions per 8 codes).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ void int4x8_to_h16(uint32_t x, uint32_t (&w)[4]) {
  const uint32_t lo = x & 0x0F0F0F0Fu, hi = (x >> 4) & 0x0F0F0F0Fu;  // codes 0,2,4,6 / 1,3,5,7
  const uint32_t u = prmt(lo, hi, 0x5140u), v = prmt(lo, hi, 0x7362u);  // codes 0..3 / 4..7 in order
  const uint32_t c64 = 0x64646464u;
  const uint32_t t[4] = {prmt(u, c64, 0x4140u), prmt(u, c64, 0x4342u), prmt(v, c64, 0x4140u),
                         prmt(v, c64, 0x4342u)};
  const h16x2 off = __floats2half2_rn(1032.f, 1032.f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h16x2 h = __hsub2(*reinterpret_cast<const h16x2*>(&t[i]), off);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int EPI>
__device__ __forceinline__ void epi_apply(const GemmEpi& ep, int m, int n0, float (&v)[32]) {
  const int N = ep.N;
  if constexpr (EPI == EPI_GELU_H16) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(v[j]);
  }
  if constexpr (EPI == EPI_H16 || EPI == EPI_GELU_H16) {
    h16* o = static_cast<h16*>(ep.out) + static_cast<size_t>(m) * ep.ldo + n0;
    if (n0 + 32 <= N && (ep.ldo & 7) == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 w;
        w.x = pack_h16x2(v[8 * j + 0], v[8 * j + 1]);
        w.y = pack_h16x2(v[8 * j + 2], v[8 * j + 3]);
        w.z = pack_h16x2(v[8 * j + 4], v[8 * j + 5]);
        w.w = pack_h16x2(v[8 * j + 6], v[8 * j + 7]);
        reinterpret_cast<uint4*>(o)[j] = w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) o[j] = __float2half_rn(v[j]);
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
    // row context (kbase/vbase) is resolved once per tile by the caller: see QkvRow
    (void)N;
  }
}

// Per-row destinations of the QKV epilogue, resolved once per tile: the q row and the K/V rows of
// this token's page slot (page layout [page][K|V][head][PAGE][hd]).
struct QkvRow {
  h16* q;
  h16* k;  // head 0 of this token's K row
  h16* v;
};
__device__ __forceinline__ QkvRow qkv_row(const GemmEpi& ep, int m) {
  QkvRow r;
  const int slot = ep.tok_slot[m];
  const int pos = ep.tok_pos[m];
  const int page = ep.page_table[static_cast<size_t>(slot) * ep.max_pages + (pos >> 4)];
  const size_t head_stride = static_cast<size_t>(ep.page_size) << ep.hd_shift;
  h16* kp = ep.kv_layer + static_cast<size_t>(page) * 2 * ep.heads * head_stride +
                      (static_cast<size_t>(pos & 15) << ep.hd_shift);
  r.q = static_cast<h16*>(ep.out) + static_cast<size_t>(m) * ep.ldo;
  r.k = kp;
  r.v = kp + ep.heads * head_stride;
  return r;
}
__device__ __forceinline__ void qkv_store(const GemmEpi& ep, const QkvRow& row, int n0, const float (&v)[32]) {
  const int kh = ep.kh;
  const size_t head_stride = static_cast<size_t>(ep.page_size) << ep.hd_shift;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int n = n0 + 8 * j;
    if (n >= ep.N) break;
    uint4 w;
    w.x = pack_h16x2(v[8 * j + 0], v[8 * j + 1]);
    w.y = pack_h16x2(v[8 * j + 2], v[8 * j + 3]);
    w.z = pack_h16x2(v[8 * j + 4], v[8 * j + 5]);
    w.w = pack_h16x2(v[8 * j + 6], v[8 * j + 7]);
    h16* dst;
    if (n < kh) {
      dst = row.q + n;
    } else {
      const int c = n - kh;
      const bool is_v = c >= kh;
      const int cc = is_v ? c - kh : c;
      const int head = cc >> ep.hd_shift;
      dst = (is_v ? row.v : row.k) + head * head_stride + (cc & (ep.hd - 1));
    }
    *reinterpret_cast<uint4*>(dst) = w;
  }
}

// Coalesced epilogue of one warp's 32 x 32 fp32 chunk (thread t holds row m_base + t). The values
// go through a per-warp smem tile with an XOR swizzle of the eight 16-byte column groups by
// (row & 7), so both the row-wise (thread = row) and the column-wise (8 lanes = one 128-byte row
// segment) accesses are bank-conflict free; every global access is then a full 128-byte row
// segment instead of 32 half-sector writes.
__device__ __forceinline__ int swz(int r, int g) { return r * 32 + ((g ^ (r & 7)) << 2); }

template <int EPI>
__device__ __forceinline__ void warp_tile_epilogue(const GemmEpi& ep, float* tile, int m_base, int n0, float (&v)[32],
                                                   int lane, const QkvRow* rows = nullptr,
                                                   const CUtensorMap* tmC = nullptr, uint32_t* seq = nullptr) {
  const int rr = lane >> 3, gg = lane & 7;  // coalesced phase: row rr + 4i, column group gg
  if constexpr (EPI == EPI_GELU_H16) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(v[j]);
  }
  if constexpr (EPI == EPI_RESID_F32 || EPI == EPI_H16 || EPI == EPI_GELU_H16) {
    if (ep.tma_out) {
      if constexpr (EPI != EPI_RESID_F32) {
        // fp16 boxes are 2 KB: the warp's 4 KB tile holds two, used alternately, so writing this
        // chunk only waits for the store issued two chunks ago (not the previous one) to be read
        tile += ((*seq)++ & 1u) * 512;
        if (lane == 0) bulk_wait_read1();
      } else {
        // the tile may still be the source of this warp's previous bulk store
        if (lane == 0) bulk_wait_read0();
      }
      __syncwarp();
      if constexpr (EPI == EPI_RESID_F32) {
        // fp32 32 x 32 box in the SWIZZLE_128B layout (16-byte chunk g of row r at g ^ (r & 7)):
        // exactly swz(); TMA adds it into x in L2 - no read of x on the SM
#pragma unroll
        for (int g = 0; g < 8; ++g)
          *reinterpret_cast<float4*>(tile + swz(lane, g)) = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
      } else {
        // fp16 32 x 32 box, SWIZZLE_64B: 16-byte chunk k of 64-byte row r at k ^ ((r >> 1) & 3)
        uint8_t* trow = reinterpret_cast<uint8_t*>(tile) + lane * 64;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint4 w;
          w.x = pack_h16x2(v[8 * k + 0], v[8 * k + 1]);
          w.y = pack_h16x2(v[8 * k + 2], v[8 * k + 3]);
          w.z = pack_h16x2(v[8 * k + 4], v[8 * k + 5]);
          w.w = pack_h16x2(v[8 * k + 6], v[8 * k + 7]);
          *reinterpret_cast<uint4*>(trow + ((k ^ ((lane >> 1) & 3)) << 4)) = w;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if constexpr (EPI == EPI_RESID_F32) tma_reduce_add_2d(tmC, smem_u32(tile), n0, m_base);
        else tma_store_2d(tmC, smem_u32(tile), n0, m_base);
        bulk_commit();
      }
      return;
    }
  }
#pragma unroll
  for (int g = 0; g < 8; ++g)
    *reinterpret_cast<float4*>(tile + swz(lane, g)) = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
  __syncwarp();
  if constexpr (EPI == EPI_RESID_F32) {
    float* xb = static_cast<float*>(ep.out) + n0 + gg * 4;
    float4 xo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = m_base + rr + 4 * i;
      xo[i] = row < ep.M ? *reinterpret_cast<const float4*>(xb + static_cast<size_t>(row) * ep.ldo)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = m_base + rr + 4 * i;
      const float4 a = *reinterpret_cast<const float4*>(tile + swz(rr + 4 * i, gg));
      if (row < ep.M)
        *reinterpret_cast<float4*>(xb + static_cast<size_t>(row) * ep.ldo) =
            make_float4(xo[i].x + a.x, xo[i].y + a.y, xo[i].z + a.z, xo[i].w + a.w);
    }
  } else if constexpr (EPI == EPI_QKV) {
    // 4 lanes x 16 B per row segment, 8 rows per instruction; destinations per row from `rows`
    const int r8 = lane >> 2, q4 = lane & 3;
    const int n = n0 + q4 * 8;
    const int kh = ep.kh;
    const size_t head_stride = static_cast<size_t>(ep.page_size) << ep.hd_shift;
    int region = 0, off = n;  // 0: q, 1: K, 2: V
    if (n >= kh) {
      const int c = n - kh;
      region = c >= kh ? 2 : 1;
      const int cc = region == 2 ? c - kh : c;
      off = static_cast<int>((cc >> ep.hd_shift) * head_stride) + (cc & (ep.hd - 1));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int lr = r8 + 8 * i;
      const float4 a = *reinterpret_cast<const float4*>(tile + swz(lr, 2 * q4));
      const float4 b = *reinterpret_cast<const float4*>(tile + swz(lr, 2 * q4 + 1));
      if (m_base + lr < ep.M) {
        uint4 w;
        w.x = pack_h16x2(a.x, a.y);
        w.y = pack_h16x2(a.z, a.w);
        w.z = pack_h16x2(b.x, b.y);
        w.w = pack_h16x2(b.z, b.w);
        const QkvRow& rw = rows[lr];
        h16* dst = (region == 0 ? rw.q : region == 1 ? rw.k : rw.v) + off;
        *reinterpret_cast<uint4*>(dst) = w;
      }
    }
  } else {  // fp16 output: 4 lanes x 16 B = one 64-byte row segment, 8 rows per instruction
    const int r8 = lane >> 2, q4 = lane & 3;
    h16* ob = static_cast<h16*>(ep.out) + n0 + q4 * 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int lr = r8 + 8 * i;
      const float4 a = *reinterpret_cast<const float4*>(tile + swz(lr, 2 * q4));
      const float4 b = *reinterpret_cast<const float4*>(tile + swz(lr, 2 * q4 + 1));
      const int row = m_base + lr;
      if (row < ep.M) {
        uint4 w;
        w.x = pack_h16x2(a.x, a.y);
        w.y = pack_h16x2(a.z, a.w);
        w.z = pack_h16x2(b.x, b.y);
        w.w = pack_h16x2(b.z, b.w);
        *reinterpret_cast<uint4*>(ob + static_cast<size_t>(row) * ep.ldo) = w;
      }
    }
  }
  __syncwarp();
}

template <int BN, int EPI, int CG, bool I8, bool W4 = false>
__global__ void __launch_bounds__(GemmCfg<BN, CG, W4>::THREADS, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, int M, int N, int K, GemmEpi ep) {
  using C = GemmCfg<BN, CG, W4>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sA = base;
  const uint32_t sB = base + STAGES * C::A_BYTES;
  const uint32_t sRaw = sB + STAGES * C::B_BYTES;  // W4: packed int4 staging ring
  const uint32_t bars = sRaw + STAGES * C::RAW_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * STAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * STAGES + 4);
  const uint32_t* tmem_slot_ptr = reinterpret_cast<const uint32_t*>(smem_raw + (tmem_slot - raw));
  auto raw_full_bar = [&](int s) { return bars + 8u * (2 * STAGES + 5 + s); };  // W4, CTA-local

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // pair: the leader's expect_tx covers both CTAs' TMA bytes; W4 adds one arrival per CTA
      // from the converter warp that expanded that CTA's B tile of the stage
      mbar_init(full_bar(s), W4 ? 1 + CG : 1);
      mbar_init(empty_bar(s), 1);
      if constexpr (W4) mbar_init(raw_full_bar(s), 1);
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
  pdl_sync();

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
          if constexpr (W4) {
            // A as usual; the packed weight tile goes to this CTA's raw ring (local barrier)
            mbar_expect_tx(raw_full_bar(stage), C::RAW_BYTES);
            tma_load_2d(sRaw + stage * C::RAW_BYTES, &tmB, raw_full_bar(stage), kb * 32, brow);
            if constexpr (CG == 2) {
              if (leader) mbar_expect_tx(full_bar(stage), 2 * C::A_BYTES);
              tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, leader_full0 + 8u * stage, kb * KELEMS, arow);
            } else {
              mbar_expect_tx(full_bar(stage), C::A_BYTES);
              tma_load_2d(sA + stage * C::A_BYTES, &tmA, full_bar(stage), kb * KELEMS, arow);
            }
          } else if constexpr (CG == 2) {
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
      constexpr uint32_t idesc = I8 ? idesc_i8(128 * CG, BN) : idesc_f16(128 * CG, BN, H16_FMT);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = group; tile < num_tiles; tile += n_groups) {
        mbar_wait(tempty_bar(acc), acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < kbs; ++kb) {
          if constexpr (W4 && CG == 2) mbar_wait_acq_cluster(full_bar(stage), phase);  // peer converters
          else mbar_wait(full_bar(stage), phase);
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
  } else if (W4 && warp >= 2 + C::EPI_WARPS) {
    // converters: warp cw expands every CONV_WARPS-th stage on its own (4 stages in flight, so the
    // per-stage fence / barrier latency of one warp overlaps the others' conversion work). Lane l
    // expands rows l, l + 32, l + 64, l + 96: 32 packed bytes (64 codes) -> one 128-byte
    // SWIZZLE_128B row of the B tile (16-byte chunk c lands at chunk c ^ (r & 7)).
    const int cw = warp - (2 + C::EPI_WARPS);
    const uint32_t leader_full0 = CG == 2 ? mapa_shared(full_bar(0), 0) : full_bar(0);
    int stage = 0, seq = 0;
    uint32_t phase = 0;
    for (int tile = group; tile < num_tiles; tile += n_groups) {
      for (int kb = 0; kb < kbs; ++kb, ++seq) {
        if (seq % C::CONV_WARPS == cw) {
          mbar_wait(raw_full_bar(stage), phase);
          const uint4* src = reinterpret_cast<const uint4*>(smem_raw + (sRaw + stage * C::RAW_BYTES - raw));
          uint8_t* dst = smem_raw + (sB + stage * C::B_BYTES - raw);
#pragma unroll
          for (int i = 0; i < C::BN_CTA / 32; ++i) {
            const int r = lane + 32 * i;
            const uint4 p0 = src[2 * r], p1 = src[2 * r + 1];
            const uint32_t words[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
            uint8_t* dst_row = dst + r * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              uint32_t w[4];
              int4x8_to_h16(words[c], w);
              *reinterpret_cast<uint4*>(dst_row + ((c ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
          fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
          if constexpr (CG == 2) fence_release_smem_cluster();  // ... and to the leader's MMA issue
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_relaxed_cluster(leader_full0 + 8u * stage);
            else mbar_arrive(full_bar(stage));
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else {
    const int e = warp - 2;
    const int q = warp & 3;                   // TMEM lane quarter this warp may access
    constexpr int WCOLS = BN / (C::EPI_WARPS / 4);  // columns drained per warp per tile
    const int c_begin = (e >> 2) * WCOLS;        // this warp's column range
    constexpr int NCH = WCOLS / 32;              // 32-column chunks per warp per tile
    const uint32_t leader_tempty0 = CG == 2 ? mapa_shared(tempty_bar(0), 0) : tempty_bar(0);
    float* s_scale = reinterpret_cast<float*>(smem_raw + (bars + 512 - raw));  // [BN] per tile
    uint8_t* s_warp = smem_raw + (bars + 2048 - raw) + e * 5120;  // 1024-byte aligned (TMA swizzle)
    float* s_tile = reinterpret_cast<float*>(s_warp);                 // 32 x 32 fp32 (4 KB)
    QkvRow* s_rows = reinterpret_cast<QkvRow*>(s_warp + 4096);        // the warp's 32 row destinations
    const bool has_ws = ep.w_scale != nullptr;
    uint32_t store_seq = 0;  // bulk stores issued by this warp (staging half selection)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = group; tile < num_tiles; tile += n_groups) {
      const int mt = tile / n_tiles;
      const int nt = tile - mt * n_tiles;
      const int m = mt * C::TILE_M + static_cast<int>(rank) * C::BM + q * 32 + lane;
      const bool row_ok = m < M;
      // stage this tile's per-column weight scales once (all epilogue warps, named barrier 1)
      if (has_ws) {
        asm volatile("bar.sync 1, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
        for (int i = threadIdx.x - 64; i < BN; i += 32 * C::EPI_WARPS) {
          const int n = nt * BN + i;
          s_scale[i] = n < N ? ep.w_scale[n] : 0.f;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
      }
      float a_sc = 1.f;
      if constexpr (I8) a_sc = row_ok ? ep.a_scale[m] : 0.f;
      QkvRow qrow{};
      if constexpr (EPI == EPI_QKV) {
        if (row_ok) qrow = qkv_row(ep, m);
        s_rows[lane] = qrow;
        __syncwarp();
      }
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
      if constexpr (EPI == EPI_NONE) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_remote(leader_tempty0 + 8u * acc);
          else mbar_arrive(tempty_bar(acc));
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1u;
        continue;
      }
      // TMEM loads double-buffered across chunks: chunk c+1 is in flight while c is processed
      uint32_t r[2][32];
      tmem_ld_32x32b_x32(tbase + c_begin, r[0]);
#pragma unroll
      for (int ci = 0; ci < NCH; ++ci) {
        const int c = c_begin + ci * 32;
        const int n0 = nt * BN + c;
        tmem_ld_wait();
        if (ci + 1 < NCH) tmem_ld_32x32b_x32(tbase + c + 32, r[(ci + 1) & 1]);
        const uint32_t(&rc)[32] = r[ci & 1];
        const int m_base = mt * C::TILE_M + static_cast<int>(rank) * C::BM + q * 32;  // warp's first row
        if constexpr (EPI == EPI_RESID_F32 || EPI == EPI_H16 || EPI == EPI_GELU_H16 || EPI == EPI_QKV) {
          // full 32-column chunk with aligned rows: coalesced path through the warp's smem tile
          // (QKV: a chunk never straddles q/K/V or a head when hd >= 32)
          const bool full = n0 + 32 <= N && (ep.ldo & 7) == 0 && (EPI != EPI_QKV || ep.hd_shift >= 5);
          if (full && m_base < M) {
            float v[32];
            if constexpr (I8) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = static_cast<float>(static_cast<int32_t>(rc[j])) * a_sc * s_scale[c + j];
            } else if (has_ws) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rc[j]) * s_scale[c + j];
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rc[j]);
            }
            warp_tile_epilogue<EPI>(ep, s_tile, m_base, n0, v, lane, s_rows, &tmC, &store_seq);
            continue;
          }
        }
        if (row_ok && n0 < N) {
          if constexpr (EPI == EPI_S32) {
            int32_t* o = static_cast<int32_t*>(ep.out) + static_cast<size_t>(m) * ep.ldo + n0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + j < N) o[j] = static_cast<int32_t>(rc[j]);
          } else {
            float v[32];
            if constexpr (I8) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = static_cast<float>(static_cast<int32_t>(rc[j])) * a_sc * s_scale[c + j];
            } else {
              if (has_ws) {  // W8A16 / W4A16: codes as exact fp16 integers, scale here
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rc[j]) * s_scale[c + j];
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rc[j]);
              }
            }
            if constexpr (EPI == EPI_QKV) {
              qkv_store(ep, qrow, n0, v);
            } else {
              epi_apply<EPI>(ep, m, n0, v);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_remote(leader_tempty0 + 8u * acc);
        else mbar_arrive(tempty_bar(acc));
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1u;
    }
    if (ep.tma_out && lane == 0) bulk_wait0();  // this warp's bulk stores / reductions are complete
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
