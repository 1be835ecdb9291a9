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
//               online softmax in fp32 (exp2), writes P_j (bf16) into a swizzled smem tile (the A
//               operand of the PV MMA), then accumulates O = O * alpha_j + Ob_j in registers
// TMEM: S double-buffered (2 x KB columns) + Ob double-buffered (2 x hd columns).
// Keys are processed in blocks aligned to absolute positions, so a query's arithmetic never depends
// on which other queries share its tile (batch invariance, test_model.cpp:240-267).
#include <algorithm>

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
      constexpr uint32_t idesc_s = idesc_f16(128, KB, 1);
      constexpr uint32_t idesc_o = idesc_f16(128, HD, 1) | (1u << 16);  // B (V) MN-major
      // S blocks run one ahead of PV blocks, across item boundaries
      TcCursor sc{static_cast<int>(blockIdx.x), 0, 0, 0, 0};
      if (sc.item < n_items) sc.nkb = item_nkb(sc.item);
      auto issue_s = [&](const TcCursor& c) {
        const int s = c.g % NST, b = c.g & 1, qb = c.qi & 1;
        if (c.kb == 0) mbar_wait(q_full(qb), (c.qi >> 1) & 1);
        mbar_wait(kv_full(s), (c.g / NST) & 1);
        mbar_wait(s_empty(b), ((c.g >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + C::S_COL + b * KB;
        const uint32_t sK = sKV + s * C::STAGE_BYTES;
        const uint32_t sq = sQ + qb * C::Q_BYTES;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t cb = kk / 4, ko = (kk % 4) * 32;
          umma_f16(d, smem_desc_k_sw128(sq + cb * 128 * 128 + ko), smem_desc_k_sw128(sK + cb * KB * 128 + ko), idesc_s,
                   kk ? 1u : 0u);
        }
        umma_commit(s_full(b));
        if (c.kb + 1 == c.nkb) umma_commit(q_empty(qb));  // the item's last read of its Q tile
      };
      auto advance = [&](TcCursor& c) {
        ++c.g;
        if (++c.kb == c.nkb) {
          c.kb = 0;
          c.item += gridDim.x;
          ++c.qi;
          c.nkb = c.item < n_items ? item_nkb(c.item) : 0;
        }
      };
      if (sc.item < n_items) issue_s(sc);
      TcCursor pc = sc;
      advance(sc);
      while (pc.item < n_items) {
        if (sc.item < n_items) {
          issue_s(sc);
          advance(sc);
        }
        const int s = pc.g % NST, b = pc.g & 1;
        mbar_wait(p_full(b), (pc.g >> 1) & 1);
        mbar_wait(o_empty(b), ((pc.g >> 1) & 1) ^ 1u);
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
          if (lane == 0) {
            mbar_arrive(s_empty(b));
            mbar_arrive(p_full(b));
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
        // pass 2: P = exp2(s * scale - m) as bf16 into the swizzled A tile of the PV MMA
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
            w.x = pack_bf16x2(pv[g4 * 8 + 0], pv[g4 * 8 + 1]);
            w.y = pack_bf16x2(pv[g4 * 8 + 2], pv[g4 * 8 + 3]);
            w.z = pack_bf16x2(pv[g4 * 8 + 4], pv[g4 * 8 + 5]);
            w.w = pack_bf16x2(pv[g4 * 8 + 6], pv[g4 * 8 + 7]);
            *reinterpret_cast<uint4*>(prow + region * 128 * 128 + ((cg ^ (row & 7)) << 4)) = w;
          }
        }
        tc_fence_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (generic writes) -> tensor core
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(s_empty(b));
          mbar_arrive(p_full(b));
        }
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
        __nv_bfloat16* zr = p.z + static_cast<size_t>(grp.m0 + row) * p.ldz + head * HD;
#pragma unroll
        for (int c = 0; c < HD; c += 8) {
          uint4 w;
          w.x = pack_bf16x2(o[c + 0] * inv, o[c + 1] * inv);
          w.y = pack_bf16x2(o[c + 2] * inv, o[c + 3] * inv);
          w.z = pack_bf16x2(o[c + 4] * inv, o[c + 5] * inv);
          w.w = pack_bf16x2(o[c + 6] * inv, o[c + 7] * inv);
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

}  // namespace iolmh
