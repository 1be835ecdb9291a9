// Causal prefill attention on the 5th-generation tensor cores (tcgen05 + TMEM), flash style.
//
// Reference: the attention loop of ModelRuntime::advance (runtime.cpp:152-174) with softmax_row
// (numerics.cpp:130-156): per query, s_j = (q . k_j) / sqrt(hd) for keys j <= t, softmax, z = sum p_j v_j.
//
// Persistent CTAs walk work items = (up to 128 consecutive prompt tokens of one row, one head); the
// producer prefetches the next item's Q (double-buffered) and K/V blocks (one ring across items)
// and the MMA warp starts the next item's S while the softmax warps finish the current one. Roles:
//   warp 0    : TMA producer - the Q tile once, then K and V page slabs (KB keys per block, 16-key
//               pages resolved through the page table) into an NST-deep ring
//   warp 1    : TMEM allocator + MMA issuer (one lane):
//                 S_j  = Q K_j^T           tcgen05.mma kind::f16, M 128, N KB, K hd (A, B K-major)
//                 Ob_j = P_j V_j           tcgen05.mma kind::f16, M 128, N hd, K KB (B = V MN-major)
//               S_{j+1} is issued before Ob_j so the tensor core runs while block j's softmax does
//   warps 2-5 : softmax / correction, thread i <-> query row i (TMEM lane i): reads S_j from TMEM,
//               online softmax in fp32 (exp2), writes P_j (fp16) into a swizzled smem tile (the A
//               operand of the PV MMA), then accumulates O = O * alpha_j + Ob_j in registers
// TMEM: S double-buffered (2 x KB columns) + Ob double-buffered (2 x hd columns).
// Keys are processed in blocks aligned to absolute positions, so a query's arithmetic never depends
// on which other queries share its tile (batch invariance, test_model.cpp:240-267).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "kernels.cuh"
#include "launch.hpp"
#include "ptx.cuh"

namespace iolmk {

namespace {
constexpr int TC_PAGE = 16;

template <int HD>
struct TcCfg {
  static constexpr int KB = 64;                     // keys per block (4 pages)
  static constexpr int NCH = HD / 64;               // 64-wide (128-byte) hd chunks
  static constexpr int NST = 3;                     // K/V ring depth
  static constexpr uint32_t Q_BYTES = 128 * HD * 2;
  static constexpr uint32_t KT_BYTES = KB * HD * 2;  // one K (or V) block
  static constexpr uint32_t STAGE_BYTES = 2 * KT_BYTES;
  static constexpr uint32_t P_BYTES = 128 * KB * 2;
  static constexpr uint32_t TMEM_COLS = HD == 64 ? 256 : 512;  // hd 64: two CTAs per SM
  static constexpr uint32_t S_COL = 0, O_COL = 2 * KB;
  static constexpr size_t SMEM = 1024 + 2 * Q_BYTES + NST * STAGE_BYTES + 2 * P_BYTES + 256;
  static_assert(2 * KB + 2 * HD <= TMEM_COLS, "TMEM budget");
};

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// MN-major SWIZZLE_128B operand (the V block as the B operand of P V): 8-row (key) x 128-byte
// (64 hd) atoms; SBO = next 8 keys (1024 B), LBO = next 64-wide hd chunk.
__device__ __forceinline__ uint64_t smem_desc_mn_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
}  // namespace

// Walks a CTA's work items in order: item = blockIdx.x + k * gridDim.x over groups x heads,
// each item a run of key blocks; the global block index g drives every ring / buffer parity.
struct TcCursor {
  int item, kb, nkb, g, qi;  // qi: ordinal of the item within this CTA (Q double buffer)
};

template <int HD, bool MASK>
__global__ void __launch_bounds__(192, HD == 64 ? 2 : 1) attn_prefill_tc_kernel(const __grid_constant__ AttnParams p) {
  using C = TcCfg<HD>;
  constexpr int KB = C::KB, NST = C::NST;
  extern __shared__ __align__(1024) uint8_t tsm[];
  const uint32_t raw = smem_u32(tsm);
  const uint32_t sQ = (raw + 1023u) & ~1023u;  // two Q buffers
  const uint32_t sKV = sQ + 2 * C::Q_BYTES;
  const uint32_t sP = sKV + NST * C::STAGE_BYTES;
  const uint32_t bars = sP + 2 * C::P_BYTES;
  auto kv_full = [&](int s) { return bars + 8u * s; };
  auto kv_empty = [&](int s) { return bars + 8u * (NST + s); };
  auto s_full = [&](int b) { return bars + 8u * (2 * NST + b); };
  auto s_empty = [&](int b) { return bars + 8u * (2 * NST + 2 + b); };
  auto p_full = [&](int b) { return bars + 8u * (2 * NST + 4 + b); };
  auto o_full = [&](int b) { return bars + 8u * (2 * NST + 6 + b); };
  auto o_empty = [&](int b) { return bars + 8u * (2 * NST + 8 + b); };
  auto q_full = [&](int b) { return bars + 8u * (2 * NST + 10 + b); };
  auto q_empty = [&](int b) { return bars + 8u * (2 * NST + 12 + b); };
  const uint32_t tmem_slot = bars + 8u * (2 * NST + 14);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = p.n_groups * p.heads;
  auto item_nkb = [&](int item) {
    const AttnGroup& g = p.groups[item / p.heads];
    return (g.pos0 + g.nq - 1) / KB + 1;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(kv_full(s), 1);
      mbar_init(kv_empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full(b), 1);
      mbar_init(s_empty(b), 4);
      mbar_init(p_full(b), 4);
      mbar_init(o_full(b), 1);
      mbar_init(o_empty(b), 4);
      mbar_init(q_full(b), 1);
      mbar_init(q_empty(b), 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  // zero the K/V ring once: rows of a partial last block keep finite values (p = 0 times stale V
  // must stay 0), and the async-proxy TMA writes are ordered after these generic writes
  for (uint32_t i = threadIdx.x; i < NST * C::STAGE_BYTES / 16; i += blockDim.x)
    *reinterpret_cast<uint4*>(tsm + (sKV - raw) + 16 * i) = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<const uint32_t*>(tsm + (tmem_slot - raw));
  pdl_sync();

  if (warp == 0) {  // ------------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&p.kv_map);
      tma_prefetch_desc(&p.q_map);
    }
    int g = 0, qi = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++qi) {
      const AttnGroup grp = p.groups[item / p.heads];
      const int head = item % p.heads;
      const int last_key = grp.pos0 + grp.nq - 1;
      const int nkb = last_key / KB + 1;
      const int* pt = p.page_table + static_cast<size_t>(grp.slot) * p.max_pages;
      const int qb = qi & 1;
      if (lane == 0) {
        mbar_wait(q_empty(qb), ((qi >> 1) & 1) ^ 1u);
        mbar_expect_tx(q_full(qb), C::Q_BYTES);
#pragma unroll
        for (int cb = 0; cb < C::NCH; ++cb)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            tma_load_2d(sQ + qb * C::Q_BYTES + cb * 128 * 128 + h * 64 * 128, &p.q_map, q_full(qb),
                        head * HD + cb * 64, grp.m0 + h * 64);
      }
      int pid_base = -(1 << 20), pid = 0;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % NST;
        const int pg0 = kb * (KB / TC_PAGE);
        const int npg = min(KB / TC_PAGE, last_key / TC_PAGE - pg0 + 1);  // pages of the slot actually used
        if (pg0 + npg > pid_base + 32 || pg0 < pid_base) {
          pid_base = pg0;
          pid = pid_base + lane < p.max_pages ? __ldg(pt + pid_base + lane) : 0;
        }
        if (lane == 0) {
          mbar_wait(kv_empty(s), ((g / NST) & 1) ^ 1u);
          mbar_expect_tx(kv_full(s), npg * 2 * TC_PAGE * HD * 2);
        }
        const uint32_t dst = sKV + s * C::STAGE_BYTES;
        for (int j = 0; j < npg; ++j) {
          const int page = __shfl_sync(0xffffffffu, pid, pg0 + j - pid_base);
          if (lane == 0) {
            const int rk = ((page * 2 + 0) * p.heads + head) * TC_PAGE;
            const int rv = rk + p.heads * TC_PAGE;
#pragma unroll
            for (int cb = 0; cb < C::NCH; ++cb) {
              const uint32_t o = cb * KB * 128 + j * TC_PAGE * 128;
              tma_load_2d(dst + o, &p.kv_map, kv_full(s), cb * 64, rk);
              tma_load_2d(dst + C::KT_BYTES + o, &p.kv_map, kv_full(s), cb * 64, rv);
            }
          }
        }
      }
    }
  } else if (warp == 1) {  // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_f16(128, KB, H16_FMT);
      constexpr uint32_t idesc_o = idesc_f16(128, HD, H16_FMT) | (1u << 16);  // B (V) MN-major
      // S blocks run ahead of PV blocks, across item boundaries; whichever MMA has its inputs ready
      // is issued first (non-blocking polls), so a PV never waits behind the next block's K/V load
      TcCursor sc{static_cast<int>(blockIdx.x), 0, 0, 0, 0};
      if (sc.item < n_items) sc.nkb = item_nkb(sc.item);
      TcCursor pc = sc;
      auto advance = [&](TcCursor& c) {
        ++c.g;
        if (++c.kb == c.nkb) {
          c.kb = 0;
          c.item += gridDim.x;
          ++c.qi;
          c.nkb = c.item < n_items ? item_nkb(c.item) : 0;
        }
      };
      while (pc.item < n_items) {
        if (sc.item < n_items) {
          const int s = sc.g % NST, b = sc.g & 1, qb = sc.qi & 1;
          if ((sc.kb != 0 || mbar_test_wait(q_full(qb), (sc.qi >> 1) & 1)) &&
              mbar_test_wait(kv_full(s), (sc.g / NST) & 1) && mbar_test_wait(s_empty(b), ((sc.g >> 1) & 1) ^ 1u)) {
            tc_fence_after();
            const uint32_t d = tmem + C::S_COL + b * KB;
            const uint32_t sK = sKV + s * C::STAGE_BYTES;
            const uint32_t sq = sQ + qb * C::Q_BYTES;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
              const uint32_t cb = kk / 4, ko = (kk % 4) * 32;
              umma_f16(d, smem_desc_k_sw128(sq + cb * 128 * 128 + ko), smem_desc_k_sw128(sK + cb * KB * 128 + ko),
                       idesc_s, kk ? 1u : 0u);
            }
            umma_commit(s_full(b));
            if (sc.kb + 1 == sc.nkb) umma_commit(q_empty(qb));  // the item's last read of its Q tile
            advance(sc);
          }
        }
        if (pc.g < sc.g) {  // S(pc) issued
          const int s = pc.g % NST, b = pc.g & 1;
          if (mbar_test_wait(p_full(b), (pc.g >> 1) & 1) && mbar_test_wait(o_empty(b), ((pc.g >> 1) & 1) ^ 1u)) {
            tc_fence_after();
            const uint32_t d = tmem + C::O_COL + b * HD;
            const uint32_t sV = sKV + s * C::STAGE_BYTES + C::KT_BYTES;
            const uint32_t pb = sP + b * C::P_BYTES;
#pragma unroll
            for (int kk = 0; kk < KB / 16; ++kk) {
              const uint32_t pch = kk / 4, po = (kk % 4) * 32;  // P: 64-key chunks of 128-byte rows
              umma_f16(d, smem_desc_k_sw128(pb + pch * 128 * 128 + po), smem_desc_mn_sw128(sV + kk * 2048, KB * 128),
                       idesc_o, kk ? 1u : 0u);
            }
            umma_commit(o_full(b));
            umma_commit(kv_empty(s));
            advance(pc);
          }
        }
      }
    }
  } else {  // ------------------------------------------------------------------ softmax warps
    const int q = warp & 3;           // TMEM lane quarter
    const int row = q * 32 + lane;    // query row of the tile = TMEM lane
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float o[HD];
    auto accumulate = [&](int g, float alpha) {  // O = O * alpha + Ob_g
      const int b = g & 1;
      mbar_wait(o_full(b), (g >> 1) & 1);
      tc_fence_after();
      // all TMEM loads of the block in flight before one wait (each load-wait pair is a full
      // TMEM round trip)
      uint32_t r[HD];
#pragma unroll
      for (int c = 0; c < HD; c += 32)
        tmem_ld_32x32b_x32(lane_base + C::O_COL + b * HD + c, *reinterpret_cast<uint32_t(*)[32]>(r + c));
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < HD; ++i) o[i] = fmaf(o[i], alpha, __uint_as_float(r[i]));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty(b));
    };
    int g = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const AttnGroup grp = p.groups[item / p.heads];
      const int head = item % p.heads;
      const int last_key = grp.pos0 + grp.nq - 1;
      const int nkb = last_key / KB + 1;
      const bool row_ok = row < grp.nq;
      const int qpos = grp.pos0 + row;
      float m_run = -INFINITY, l_run = 0.f, alpha_prev = 1.f;
#pragma unroll
      for (int i = 0; i < HD; ++i) o[i] = 0.f;
      const bool warp_live = q * 32 < grp.nq;  // warp-uniform: a warp of padding rows skips its work
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int b = g & 1;
        const int key0 = kb * KB;
        mbar_wait(s_full(b), (g >> 1) & 1);
        tc_fence_after();
        if (!warp_live) {  // its P rows only feed output rows that are never stored
          __syncwarp();
          if (lane == 0) {  // p_full before s_empty (see below)
            mbar_arrive(p_full(b));
            mbar_arrive(s_empty(b));
          }
          if (kb > 0) {
            mbar_wait(o_full((g - 1) & 1), ((g - 1) >> 1) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(o_empty((g - 1) & 1));
          }
          continue;
        }
        // the block's S row in registers (one TMEM round trip), masked row max
        uint32_t sr[KB];
#pragma unroll
        for (int c = 0; c < KB; c += 32)
          tmem_ld_32x32b_x32(lane_base + C::S_COL + b * KB + c, *reinterpret_cast<uint32_t(*)[32]>(sr + c));
        tmem_ld_wait();
        // S(g) is in registers: release its TMEM buffer now, so S(g + 2) overlaps this softmax (P(g)
        // is still protected: it is read by PV(g), which accumulate(g) waits for before P(g + 2))
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty(b));
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < KB; ++i) {
          const int key = key0 + i;
          bool ok = row_ok && key <= qpos;
          if (MASK) ok = ok && key <= last_key && p.key_mask[key];
          if (!ok) sr[i] = __float_as_uint(-INFINITY);
          mx = fmaxf(mx, __uint_as_float(sr[i]));
        }
        const float mnew = fmaxf(m_run, mx * p.scale_log2);
        const float alpha = mnew == -INFINITY ? 1.f : ex2f(m_run - mnew);
        const float msub = mnew == -INFINITY ? 0.f : mnew;
        m_run = mnew;
        l_run *= alpha;
        // pass 2: P = exp2(s * scale - m) as fp16 into the swizzled A tile of the PV MMA
        uint8_t* prow = tsm + (sP + b * C::P_BYTES - raw) + row * 128;
#pragma unroll
        for (int c = 0; c < KB; c += 32) {
          float pv[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            // masked keys hold -inf: ex2(-inf) = +0 (rows with no visible key have msub = 0)
            pv[i] = ex2f(fmaf(__uint_as_float(sr[c + i]), p.scale_log2, -msub));
            l_run += pv[i];
          }
          // 32 keys = 4 16-byte chunks of this row; chunk g4 of 64-key region `region` lands at
          // region base + row * 128 + ((chunk ^ (row & 7)) << 4)
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4) {
            const int kc = c + g4 * 8;
            const int region = kc / 64, cg = (kc % 64) / 8;
            uint4 w;
            w.x = pack_h16x2(pv[g4 * 8 + 0], pv[g4 * 8 + 1]);
            w.y = pack_h16x2(pv[g4 * 8 + 2], pv[g4 * 8 + 3]);
            w.z = pack_h16x2(pv[g4 * 8 + 4], pv[g4 * 8 + 5]);
            w.w = pack_h16x2(pv[g4 * 8 + 6], pv[g4 * 8 + 7]);
            *reinterpret_cast<uint4*>(prow + region * 128 * 128 + ((cg ^ (row & 7)) << 4)) = w;
          }
        }
        tc_fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (generic writes) -> tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full(b));
        if (kb > 0) accumulate(g - 1, alpha_prev);
        alpha_prev = alpha;
      }
      if (warp_live) {
        accumulate(g - 1, alpha_prev);
      } else {
        mbar_wait(o_full((g - 1) & 1), ((g - 1) >> 1) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(o_empty((g - 1) & 1));
      }
      if (row_ok) {
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        h16* zr = p.z + static_cast<size_t>(grp.m0 + row) * p.ldz + head * HD;
#pragma unroll
        for (int c = 0; c < HD; c += 8) {
          uint4 w;
          w.x = pack_h16x2(o[c + 0] * inv, o[c + 1] * inv);
          w.y = pack_h16x2(o[c + 2] * inv, o[c + 3] * inv);
          w.z = pack_h16x2(o[c + 4] * inv, o[c + 5] * inv);
          w.w = pack_h16x2(o[c + 6] * inv, o[c + 7] * inv);
          *reinterpret_cast<uint4*>(zr + c) = w;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ hd 64: head-pair tiles
// Short prompt chunks (<= 64 queries per group, hd 64) leave a 128-lane tile half empty, so one
// item stacks the SAME 64 queries for two heads h, h+1: Q rows 0-63 = head h, 64-127 = head h+1.
//   S' = Q [K_h ; K_h+1]^T   M 128, N 64 (32 keys of each head), K 64     -> lanes of head x read
//                                                                          their own 32 columns
//   O' += P [V_h | V_h+1]    M 128, N 128 (hd of both heads), K 32 keys  -> lanes of head x read
//                                                                          their own 64 columns
// Both heads see the same key positions, so P (128 x 32 keys) needs no zero blocks: the other
// head's columns of S' / O' are simply never read. Keys stream in 32-position blocks (two pages),
// aligned to absolute positions exactly like attn_prefill_kernel (the mma.sync kernel).
// O accumulates in TMEM across an item's blocks (no per-block TMEM round trip): P is formed against
// a per-row reference max m_ref that only moves when a block's max exceeds it by more than
// HP_RESCALE (log2 units; then the warp rescales its O rows in TMEM once PV of the previous block
// has landed), so p <= 2^HP_RESCALE and l, O share one reference - the quotient O / l is the
// softmax of the reference (numerics.cpp:130-156) up to fp rounding. oracle/iolm_oracle.c
// flash_head_gpu restates this rule for the W8A8 rounding-point checker.
// TMEM 256 columns (S double-buffered 2 x 64, O 128), ~97 KB smem: two CTAs per SM, each a
// producer warp, an MMA warp and one softmax warpgroup.
constexpr float HP_RESCALE = 8.0f;
template <int HD, int QB, int NST_, bool PT = false>
struct HpCfg {
  static constexpr int HPT = HD == 64 ? 2 : 1;          // heads per 128-lane tile
  static constexpr int QPT = 128 / HPT;                 // queries per tile
  static constexpr int NCH = HD / 64;                   // 64-column (128-byte) chunks per row
  static constexpr int KB = 32;                         // keys per block (2 pages)
  static constexpr int NST = NST_;                      // K/V ring depth
  static constexpr int QBUF = QB;                       // Q tiles (next item's Q prefetched when 2)
  static constexpr uint32_t Q_BYTES = 128 * HD * 2;     // 128 rows x HD, NCH chunk regions of 16 KB
  static constexpr uint32_t KCH_BYTES = HPT * KB * 128; // one 64-column chunk of the K block
  static constexpr uint32_t KT_BYTES = NCH * KCH_BYTES; // K block (also V): HPT x KB keys x HD
  static constexpr uint32_t STAGE_BYTES = 2 * KT_BYTES; // K then V
  static constexpr uint32_t P_BYTES = PT ? 0 : 128 * KB * 2;  // 128 rows x 64 B, SWIZZLE_64B K-major (PT: in TMEM)
  static constexpr uint32_t TMEM_COLS = 256;
  static constexpr uint32_t S_COL = 0, O_COL = 128;     // S: 2 x HPT*KB columns; O: HPT*HD = 128
  static constexpr size_t SMEM = 1024 + QB * Q_BYTES + NST * STAGE_BYTES + 2 * P_BYTES + 256;
  static_assert(HPT * HD == 128 && SMEM <= 115712, "128 O columns, two CTAs per SM");
};

// K-major SWIZZLE_64B operand (the P tile: 64-byte rows, 8-row atoms of 512 B, SBO = 512).
__device__ __forceinline__ uint64_t smem_desc_k_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;  // SWIZZLE_64B
  return d;
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int HD, int QB, int NSTG, bool PT>
__global__ void __launch_bounds__(192, 2) attn_prefill_hp_kernel(const __grid_constant__ AttnParams p) {
  // PT: P lives in TMEM over the consumed S columns of its block and PV takes A from TMEM
  // (tcgen05.mma ... [a_tmem]): no shared-memory P tile, no generic -> async proxy fence
  using C = HpCfg<HD, QB, NSTG, PT>;
  constexpr int KB = C::KB, NST = C::NST, HPT = C::HPT, QPT = C::QPT, NCH = C::NCH;
  extern __shared__ __align__(1024) uint8_t tsm[];
  const uint32_t raw = smem_u32(tsm);
  const uint32_t sQ = (raw + 1023u) & ~1023u;  // two Q buffers
  const uint32_t sKV = sQ + QB * C::Q_BYTES;
  const uint32_t sP = sKV + NST * C::STAGE_BYTES;
  const uint32_t bars = sP + 2 * C::P_BYTES;
  auto kv_full = [&](int s) { return bars + 8u * s; };
  auto kv_empty = [&](int s) { return bars + 8u * (NST + s); };
  auto s_full = [&](int b) { return bars + 8u * (2 * NST + b); };
  auto s_empty = [&](int b) { return bars + 8u * (2 * NST + 2 + b); };
  auto p_full = [&](int b) { return bars + 8u * (2 * NST + 4 + b); };
  auto p_empty = [&](int b) { return bars + 8u * (2 * NST + 6 + b); };  // PV of the buffer's block done
  auto q_full = [&](int b) { return bars + 8u * (2 * NST + 8 + b); };
  auto q_empty = [&](int b) { return bars + 8u * (2 * NST + 10 + b); };
  const uint32_t o_empty = bars + 8u * (2 * NST + 12);  // the item's O read by every softmax warp
  const uint32_t tmem_slot = bars + 8u * (2 * NST + 13);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npairs = (p.heads + HPT - 1) / HPT;  // head slots per group
  const int n_items = p.n_groups * npairs;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(kv_full(s), 1);
      mbar_init(kv_empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full(b), 1);
      mbar_init(s_empty(b), 4);
      mbar_init(p_full(b), 4);
      mbar_init(p_empty(b), 1);
      mbar_init(q_full(b), 1);
      mbar_init(q_empty(b), 1);
    }
    mbar_init(o_empty, 4);
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  // finite Q / K / V everywhere: columns of the other head (or of a missing odd head) are multiplied
  // but never read, and must not carry NaN bit patterns into rows that are read
  for (uint32_t i = threadIdx.x; i < (QB * C::Q_BYTES + NST * C::STAGE_BYTES) / 16; i += blockDim.x)
    *reinterpret_cast<uint4*>(tsm + (sQ - raw) + 16 * i) = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<const uint32_t*>(tsm + (tmem_slot - raw));
  pdl_sync();

  // Item metadata is loaded one item AHEAD in every role (group record, page ids, block count):
  // a dependent global load at each item boundary stalled all three roles (ncu: the item-start
  // instructions were the top stall sites).
  auto load_grp = [&](int item) {
    return item < n_items ? p.groups[item / npairs] : AttnGroup{0, 0, 1, 0};
  };
  if (warp == 0) {  // ------------------------------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&p.kv_map);
      tma_prefetch_desc(&p.q_map);
    }
    auto load_pids = [&](const AttnGroup& gr, int item) {
      return item < n_items && lane < p.max_pages ? __ldg(p.page_table + static_cast<size_t>(gr.slot) * p.max_pages + lane)
                                                  : 0;
    };
    int g = 0, qi = 0;
    AttnGroup grp = load_grp(blockIdx.x);
    int pid0 = load_pids(grp, blockIdx.x);
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++qi) {
      const AttnGroup ngrp = load_grp(item + gridDim.x);  // in flight during this item
      const int npid0 = load_pids(ngrp, item + gridDim.x);
      const int h0 = HPT * (item % npairs);
      const int nh = min(HPT, p.heads - h0);  // live heads of the tile (1 for an odd last pair)
      const int last_key = grp.pos0 + grp.nq - 1;
      const int nkb = last_key / KB + 1;
      const int* pt = p.page_table + static_cast<size_t>(grp.slot) * p.max_pages;
      const int qb = qi % QB;
      if (lane == 0) {
        mbar_wait(q_empty(qb), ((qi / QB) & 1) ^ 1u);
        // 64 x 64 boxes: chunk c of head slot t, query rows r*64.. -> chunk region c, tile rows t*QPT + r*64
        mbar_expect_tx(q_full(qb), nh * NCH * (QPT / 64) * 64 * 128);
        for (int t = 0; t < nh; ++t)
#pragma unroll
          for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int r = 0; r < QPT / 64; ++r)
              tma_load_2d(sQ + qb * C::Q_BYTES + c * 128 * 128 + (t * QPT + r * 64) * 128, &p.q_map, q_full(qb),
                          (h0 + t) * HD + c * 64, grp.m0 + r * 64);
      }
      int pid_base = 0, pid = pid0;  // page ids [0, 32) of the slot, prefetched
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % NST;
        const int pg0 = kb * (KB / TC_PAGE);
        const int npg = min(KB / TC_PAGE, last_key / TC_PAGE - pg0 + 1);
        if (pg0 + npg > pid_base + 32) {
          pid_base = pg0;
          pid = pid_base + lane < p.max_pages ? __ldg(pt + pid_base + lane) : 0;
        }
        if (lane == 0) {
          mbar_wait(kv_empty(s), ((g / NST) & 1) ^ 1u);
          mbar_expect_tx(kv_full(s), npg * nh * NCH * 2 * TC_PAGE * 128);
        }
        const uint32_t dK = sKV + s * C::STAGE_BYTES, dV = dK + C::KT_BYTES;
        for (int j = 0; j < npg; ++j) {
          const int page = __shfl_sync(0xffffffffu, pid, pg0 + j - pid_base);
          if (lane == 0) {
            const int rk = ((page * 2 + 0) * p.heads + h0) * TC_PAGE;  // K rows of head h0
            const int rv = rk + p.heads * TC_PAGE;
            // K: chunk c of head slot t at rows t*KB + j*16 of chunk region c (the N = HPT*KB B operand);
            // V: MN-major, 64-wide N chunk (t*NCH + c) of KB keys (LBO = KB * 128)
            for (int t = 0; t < nh; ++t)
#pragma unroll
              for (int c = 0; c < NCH; ++c) {
                tma_load_2d(dK + c * C::KCH_BYTES + (t * KB + j * TC_PAGE) * 128, &p.kv_map, kv_full(s), c * 64,
                            rk + t * TC_PAGE);
                tma_load_2d(dV + (t * NCH + c) * KB * 128 + j * TC_PAGE * 128, &p.kv_map, kv_full(s), c * 64,
                            rv + t * TC_PAGE);
              }
          }
        }
      }
      grp = ngrp;
      pid0 = npid0;
    }
  } else if (warp == 1) {  // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_f16(128, HPT * KB, H16_FMT);
      constexpr uint32_t idesc_o = idesc_f16(128, HPT * HD, H16_FMT) | (1u << 16);  // B (V) MN-major
      // Two cursors: S runs ahead of PV (across items), and whichever MMA has its inputs ready is
      // issued first - a PV never waits behind the next block's K/V load. The MMAs are small
      // (32-64 tensor cycles each), so this thread's own instruction count per block matters: ring
      // slots and barrier parities advance incrementally (no div / mod), descriptors are bases plus
      // 16-byte offsets (the start-address field is linear in the shared-memory address), and
      // each cursor holds the next item's block count, loaded when it entered the current item.
      struct Cur {
        int item, kb, nkb, nkb_next, qi;
        int s, sph;  // K/V ring stage and its phase bit
        int b, bph;  // S / P buffer and its phase bit
        int qb, qph; // Q tile and its phase bit
        int g;       // global block ordinal (S ahead of PV)
      };
      auto nkb_of = [&](int item) {
        const AttnGroup gr = load_grp(item);
        return (gr.pos0 + gr.nq - 1) / KB + 1;
      };
      Cur sc{static_cast<int>(blockIdx.x), 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      sc.nkb = nkb_of(sc.item);
      sc.nkb_next = nkb_of(sc.item + gridDim.x);
      Cur pc = sc;
      auto advance = [&](Cur& c) {
        ++c.g;
        if (++c.s == NST) { c.s = 0; c.sph ^= 1; }
        c.b ^= 1;
        if (c.b == 0) c.bph ^= 1;
        if (++c.kb == c.nkb) {
          c.kb = 0;
          c.item += gridDim.x;
          ++c.qi;
          if (++c.qb == QB) { c.qb = 0; c.qph ^= 1; }
          c.nkb = c.nkb_next;
          c.nkb_next = nkb_of(c.item + gridDim.x);
        }
      };
      const uint64_t dq0 = smem_desc_k_sw128(sQ), dk0 = smem_desc_k_sw128(sKV);
      const uint64_t dv0 = smem_desc_mn_sw128(sKV + C::KT_BYTES, KB * 128), dp0 = smem_desc_k_sw64(sP);
      while (pc.item < n_items) {
        if (sc.item < n_items && (sc.kb != 0 || mbar_test_wait(q_full(sc.qb), sc.qph)) &&
            mbar_test_wait(kv_full(sc.s), sc.sph) && mbar_test_wait(s_empty(sc.b), sc.bph ^ 1) &&
            (!PT || mbar_test_wait(p_empty(sc.b), sc.bph ^ 1))) {  // PT: P(g - 2) read from buffer b
          tc_fence_after();
          const uint32_t d = tmem + C::S_COL + sc.b * HPT * KB;
          const uint64_t aq = dq0 + (sc.qb * C::Q_BYTES >> 4), bk = dk0 + (sc.s * C::STAGE_BYTES >> 4);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off_a = ((kk / 4) * 128 * 128 + (kk % 4) * 32) >> 4;
            const uint32_t off_b = ((kk / 4) * C::KCH_BYTES + (kk % 4) * 32) >> 4;
            umma_f16(d, aq + off_a, bk + off_b, idesc_s, kk ? 1u : 0u);
          }
          umma_commit(s_full(sc.b));
          if (sc.kb + 1 == sc.nkb) umma_commit(q_empty(sc.qb));  // the item's last read of its Q tile
          advance(sc);
        }
        if (pc.g < sc.g && mbar_test_wait(p_full(pc.b), pc.bph) &&
            (pc.kb != 0 || mbar_test_wait(o_empty, (pc.qi & 1) ^ 1u))) {  // previous item's O read
          tc_fence_after();
          const uint64_t av = dv0 + (pc.s * C::STAGE_BYTES >> 4), ap = dp0 + (pc.b * C::P_BYTES >> 4);
#pragma unroll
          for (int kk = 0; kk < KB / 16; ++kk) {
            const uint32_t accum = (pc.kb > 0 || kk > 0) ? 1u : 0u;
            if constexpr (PT)
              umma_f16_ts(tmem + C::O_COL, tmem + C::S_COL + pc.b * HPT * KB + kk * 8, av + (kk * 2048 >> 4), idesc_o,
                          accum);
            else
              umma_f16(tmem + C::O_COL, ap + (kk * 32 >> 4), av + (kk * 2048 >> 4), idesc_o, accum);
          }
          umma_commit(p_empty(pc.b));
          umma_commit(kv_empty(pc.s));
          advance(pc);
        }
      }
    }
  } else {  // ------------------------------------------------------------------ softmax warps
    const int q = warp & 3;          // TMEM lane quarter
    const int row = q * 32 + lane;   // tile row = TMEM lane
    const int hs = row / QPT;        // head slot of the row (hd 64: 0 = head h0, 1 = head h0 + 1)
    const int qr = row % QPT;        // query within the group
    const int wq0 = (q % (QPT / 32)) * 32;  // the warp's first query within the group
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t o_addr = lane_base + C::O_COL + hs * HD;
    uint8_t* const prow0 = tsm + (sP - raw) + row * 64;
    const int pswz = (row >> 1) & 3;  // SWIZZLE_64B: 16-byte chunk c of row r at c ^ ((r >> 1) & 3)
    // Deferred epilogue: an item's O is read out after the NEXT item's first P block is written,
    // so the last PV of an item runs while this warpgroup already computes the next softmax.
    struct Pending {
      h16* z;      // this thread's output row (nullptr: nothing to store)
      float l;     // softmax denominator
      bool live;   // the warp's rows exist
      int g_last;  // global index of the item's last block
    };
    Pending pend{nullptr, 0.f, false, -1};
    auto finish = [&](const Pending& e) {  // wait the item's last PV, read O, release O, store z
      mbar_wait(p_empty(e.g_last & 1), (e.g_last >> 1) & 1);
      tc_fence_after();
      if (e.live) {  // O in two 32-column halves: load, normalise, store
        const float inv = e.l > 0.f ? 1.f / e.l : 0.f;
#pragma unroll
        for (int c = 0; c < HD; c += 32) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(o_addr + c, o);
          tmem_ld_wait();
          if (c + 32 == HD) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_empty);
          }
          if (e.z != nullptr) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint4 w;
              w.x = pack_h16x2(__uint_as_float(o[j + 0]) * inv, __uint_as_float(o[j + 1]) * inv);
              w.y = pack_h16x2(__uint_as_float(o[j + 2]) * inv, __uint_as_float(o[j + 3]) * inv);
              w.z = pack_h16x2(__uint_as_float(o[j + 4]) * inv, __uint_as_float(o[j + 5]) * inv);
              w.w = pack_h16x2(__uint_as_float(o[j + 6]) * inv, __uint_as_float(o[j + 7]) * inv);
              *reinterpret_cast<uint4*>(e.z + c + j) = w;
            }
          }
        }
      } else {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_empty);
      }
    };
    int g = 0;
    AttnGroup grp = load_grp(blockIdx.x);
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const AttnGroup ngrp = load_grp(item + gridDim.x);  // in flight during this item
      const int h = HPT * (item % npairs) + hs;
      const int last_key = grp.pos0 + grp.nq - 1;
      const int nkb = last_key / KB + 1;
      const int qpos = grp.pos0 + qr;
      // warp-uniform: the warp's rows exist (query in the group, head in the layer)
      const bool warp_live = wq0 < grp.nq && h < p.heads;
      const int warp_min_pos = grp.pos0 + wq0;
      const int warp_max_pos = grp.pos0 + min(grp.nq - 1, wq0 + 31);
      float m_ref = -INFINITY, l_run = 0.f;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int b = g & 1;
        const int key0 = kb * KB;
        const bool live = warp_live && key0 <= warp_max_pos;  // warp-uniform
        mbar_wait(s_full(b), (g >> 1) & 1);
        if (live) {
          tc_fence_after();
          uint32_t sr[KB];
          tmem_ld_32x32b_x32(lane_base + C::S_COL + b * HPT * KB + hs * KB, sr);
          tmem_ld_wait();
          // S(g) is in registers: release its TMEM buffer now, so S(g + 2) overlaps this softmax
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_empty(b));
          if (key0 + KB - 1 > warp_min_pos) {  // the block straddles the warp's diagonal
            const int lim = qpos - key0;       // keys key0 + i with i <= lim are visible
#pragma unroll
            for (int i = 0; i < KB; ++i)
              if (i > lim) sr[i] = __float_as_uint(-INFINITY);
          }
          float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
          for (int i = 0; i < KB; i += 2) {
            mx0 = fmaxf(mx0, __uint_as_float(sr[i]));
            mx1 = fmaxf(mx1, __uint_as_float(sr[i + 1]));
          }
          const float ms = fmaxf(mx0, mx1) * p.scale_log2;
          // reference max: set by the first block, moved only by a jump of more than HP_RESCALE
          const bool jump = m_ref != -INFINITY && ms > m_ref + HP_RESCALE;
          if (m_ref == -INFINITY) m_ref = ms;
          if (__any_sync(0xffffffffu, jump)) {  // rare: rescale this warp's O rows in TMEM
            const float f = jump ? ex2f(m_ref - ms) : 1.f;
            if (jump) {
              m_ref = ms;
              l_run *= f;
            }
            if (kb > 0) {  // O holds blocks < kb once PV(kb - 1) has landed
              mbar_wait(p_empty(b ^ 1), ((g - 1) >> 1) & 1);
              tc_fence_after();
              uint32_t r[32];
#pragma unroll
              for (int c = 0; c < HD; c += 32) {
                tmem_ld_32x32b_x32(o_addr + c, r);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
                tmem_st_32x32b_x32(o_addr + c, r);
              }
              tmem_st_wait();
            }
          }
          const float msub = m_ref == -INFINITY ? 0.f : m_ref;  // no visible key yet: p = ex2(-inf) = 0
          float ls[4] = {0.f, 0.f, 0.f, 0.f};
          uint32_t pw[KB / 2];
#pragma unroll
          for (int i = 0; i < KB; i += 2) {
            const float p0 = ex2f(fmaf(__uint_as_float(sr[i]), p.scale_log2, -msub));
            const float p1 = ex2f(fmaf(__uint_as_float(sr[i + 1]), p.scale_log2, -msub));
            ls[(i >> 1) & 3] += p0 + p1;
            pw[i >> 1] = pack_h16x2(p0, p1);
          }
          l_run += (ls[0] + ls[1]) + (ls[2] + ls[3]);
          mbar_wait(p_empty(b), ((g >> 1) & 1) ^ 1u);  // PV of block g - 2 has read this P buffer
          if constexpr (PT) {
            tmem_st_32x32b_x16(lane_base + C::S_COL + b * HPT * KB, pw);
            tmem_st_wait();
          } else {
#pragma unroll
            for (int c4 = 0; c4 < KB / 8; ++c4)
              *reinterpret_cast<uint4*>(prow0 + b * C::P_BYTES + ((c4 ^ pswz) << 4)) =
                  make_uint4(pw[4 * c4], pw[4 * c4 + 1], pw[4 * c4 + 2], pw[4 * c4 + 3]);
          }
        } else if (warp_live) {  // a block past the warp's last query: its P rows must add nothing
          mbar_wait(p_empty(b), ((g >> 1) & 1) ^ 1u);
          if constexpr (PT) {
            uint32_t z[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) z[i] = 0u;
            tmem_st_32x32b_x16(lane_base + C::S_COL + b * HPT * KB, z);
            tmem_st_wait();
          } else {
#pragma unroll
            for (int c4 = 0; c4 < KB / 8; ++c4)
              *reinterpret_cast<uint4*>(prow0 + b * C::P_BYTES + ((c4 ^ pswz) << 4)) = make_uint4(0, 0, 0, 0);
          }
        }
        if (!live) {
          // a warp that skipped this block releases S here; it too waits for PV(g - 2) before its
          // p_full arrival, so no warp's arrival for block g can land in block g - 2's phase
          __syncwarp();
          if (lane == 0) mbar_arrive(s_empty(b));
          if (!warp_live) mbar_wait(p_empty(b), ((g >> 1) & 1) ^ 1u);
        }
        tc_fence_before();
        if constexpr (!PT) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (generic) -> tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full(b));
        if (kb == 0 && pend.g_last >= 0) finish(pend);  // the previous item's O (PV(g) waits for it)
      }
      pend.z = warp_live && qr < grp.nq ? p.z + static_cast<size_t>(grp.m0 + qr) * p.ldz + h * HD : nullptr;
      pend.l = l_run;
      pend.live = warp_live;
      pend.g_last = g - 1;
      grp = ngrp;
    }
    if (pend.g_last >= 0) finish(pend);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

}  // namespace iolmk

namespace iolmh {


using namespace iolmk;

template <int HD>
static void launch_tc(const AttnParams& p, cudaStream_t st) {
  constexpr int smem = static_cast<int>(TcCfg<HD>::SMEM);
  ensure_smem(attn_prefill_tc_kernel<HD, false>, smem);
  ensure_smem(attn_prefill_tc_kernel<HD, true>, smem);
  const int sms = device_sms();
  const int items = p.n_groups * p.heads;
  const int grid = std::min(items, sms * (HD == 64 ? 2 : 1));  // persistent: every CTA walks items
  if (p.key_mask) launch_k(attn_prefill_tc_kernel<HD, true>, grid, 192, smem, st, p);
  else launch_k(attn_prefill_tc_kernel<HD, false>, grid, 192, smem, st, p);
}

// Groups must hold <= 128 queries. Returns false when hd has no tcgen05 variant (caller falls back).
bool launch_prefill_tc(const AttnParams& p, int hd, cudaStream_t st) {
  if (p.n_groups <= 0) return true;
  if (hd == 64) launch_tc<64>(p, st);
  else if (hd == 128) launch_tc<128>(p, st);
  else return false;
  CUDA_OK(cudaGetLastError());
  return true;
}

// Prompt chunks without a key mask: hd 64 as head-pair tiles over 64-query chunks (two Q tiles, three
// K/V stages: one Q tile + four stages, and an L2 prefetch of the next item's pages, were both slower,
// profiles/r02_experiments.md); hd 128 as one head x 128-query chunks (one 32 KB Q tile, three stages:
// two CTAs per SM). Returns false for other head sizes.
bool launch_prefill_hp(const AttnParams& p, int hd, cudaStream_t st) {
  if (p.n_groups <= 0) return true;
  auto go = [&](auto kern, size_t smem, int hpt) {
    ensure_smem(kern, smem);
    const int items = p.n_groups * ((p.heads + hpt - 1) / hpt);
    launch_k(kern, std::min(items, 2 * device_sms()), 192, smem, st, p);
  };
  // default: P in TMEM, PV with A from TMEM, one more K/V stage in the freed smem (C4 prefill -3%,
  // C1 neutral); IOLM_HP_PT=0 selects the shared-memory P tile (A/B measurements)
  static const bool pt = [] {
    const char* e = std::getenv("IOLM_HP_PT");
    return e == nullptr || std::string(e) != "0";
  }();
  if (hd == 64) {
    if (pt) go(attn_prefill_hp_kernel<64, 2, 4, true>, HpCfg<64, 2, 4, true>::SMEM, 2);
    else go(attn_prefill_hp_kernel<64, 2, 3, false>, HpCfg<64, 2, 3>::SMEM, 2);
  } else if (hd == 128) {
    if (pt) go(attn_prefill_hp_kernel<128, 1, 4, true>, HpCfg<128, 1, 4, true>::SMEM, 1);
    else go(attn_prefill_hp_kernel<128, 1, 3, false>, HpCfg<128, 1, 3>::SMEM, 1);
  } else {
    return false;
  }
  CUDA_OK(cudaGetLastError());
  return true;
}

}  // namespace iolmh
