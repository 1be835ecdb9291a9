/*
 * iolm_oracle.c - TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference's CPU hot path, IEEE f32 with the reference's exact
 * per-element operation order, built with -ffp-contract=off like the reference core
 * (proj/src/CMakeLists.txt:25-28). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. Parity of this restatement is pinned bit-for-bit against the
 * reference compiled from /root/reference (oracle/_ref/libiolm_ref.so) and against the committed
 * golden vectors in tests/golden/ (tests/test_oracle.py).
 *
 * Restated reference functions (file:line under /root/reference/proj):
 *   Rng (xoshiro256**, splitmix64, Box-Muller)  src/rng.cpp:14-78
 *   ToyModelParams::init                        src/train.cpp:45-75
 *   matmul (ascending-k f32)                    src/numerics.cpp:56-76
 *   softmax_row                                 src/numerics.cpp:130-156
 *   layernorm_row (eps 1e-5)                    src/numerics.cpp:158-177
 *   gelu (tanh form)                            src/numerics.cpp:179-184
 *   argmax_row (ties -> lowest id)              src/numerics.cpp:190-197
 *   dot_strict + ModelRuntime::advance          src/runtime.cpp:17-21, 104-211
 *   forward / batch_decode                      src/runtime.cpp:217-309
 *   rtn_scales / quantize_one (W8A8 activations, src/quant.cpp:23-38; the reference has no
 *   activation quantization, so W8A8 semantics are pinned here and in DESIGN.md)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ Rng (src/rng.cpp) */
typedef struct {
  uint64_t s[4];
  double cached;
  int has_cached;
} orc_rng;

static uint64_t splitmix64(uint64_t* x) {
  *x += 0x9e3779b97f4a7c15ull;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&sm);
  r->cached = 0.0;
  r->has_cached = 0;
}
uint64_t orc_rng_next_u64(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}
double orc_rng_next_double(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }
uint64_t orc_rng_next_below(orc_rng* r, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t x = orc_rng_next_u64(r);
    if (x >= threshold) return x % n;
  }
}
double orc_rng_next_normal(orc_rng* r) {
  if (r->has_cached) {
    r->has_cached = 0;
    return r->cached;
  }
  const double u1 = ((double)(orc_rng_next_u64(r) >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = orc_rng_next_double(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.141592653589793238462643 * u2;
  r->cached = rad * sin(theta);
  r->has_cached = 1;
  return rad * cos(theta);
}

/* ToyModelParams::init for a dense config: fills `out` with every tensor in canonical
 * (serialization) order - tok_embed, pos_embed, per layer {attn_norm.gain, attn_norm.bias, wq,
 * wk, wv, wo, ffn_norm.gain, ffn_norm.bias, w_in, w_out}, final_norm.gain, final_norm.bias.
 * Random draws happen in the reference's order (train.cpp:53-71). Returns floats written. */
static void normal_fill(float* p, size_t n, double stddev, orc_rng* r) {
  for (size_t i = 0; i < n; ++i) p[i] = (float)(stddev * orc_rng_next_normal(r));
}
size_t orc_init_dense_params(int V, int d, int L, int H, int F, int S, uint64_t seed, float* out) {
  (void)H;
  orc_rng r;
  orc_rng_seed(&r, seed);
  const double base_std = 0.02;
  const double resid_std = base_std / sqrt(2.0 * L);
  const int kh = d; /* dense: all heads */
  float* p = out;
  normal_fill(p, (size_t)V * d, base_std, &r);
  p += (size_t)V * d;
  normal_fill(p, (size_t)S * d, base_std, &r);
  p += (size_t)S * d;
  for (int l = 0; l < L; ++l) {
    for (int i = 0; i < d; ++i) p[i] = 1.0f;
    p += d;
    memset(p, 0, sizeof(float) * d);
    p += d;
    for (int w = 0; w < 3; ++w) {
      normal_fill(p, (size_t)kh * d, base_std, &r);
      p += (size_t)kh * d;
    }
    normal_fill(p, (size_t)d * kh, resid_std, &r);
    p += (size_t)d * kh;
    for (int i = 0; i < d; ++i) p[i] = 1.0f;
    p += d;
    memset(p, 0, sizeof(float) * d);
    p += d;
    normal_fill(p, (size_t)F * d, base_std, &r);
    p += (size_t)F * d;
    normal_fill(p, (size_t)d * F, resid_std, &r);
    p += (size_t)d * F;
  }
  for (int i = 0; i < d; ++i) p[i] = 1.0f;
  p += d;
  memset(p, 0, sizeof(float) * d);
  p += d;
  return (size_t)(p - out);
}

/* ------------------------------------------------------------------ numerics (numerics.cpp) */
/* C[n x N] = A[n x K] * Wt[K x N] with Wt the transposed weight (runtime.cpp:80-85): the
 * reference's i-k-j loop, every element summed from 0 in ascending k (numerics.cpp:56-76). */
static void matmul_wt(const float* A, int n, int K, const float* Wt, int N, float* Cm) {
  for (int i = 0; i < n; ++i) {
    const float* a = A + (size_t)i * K;
    float* c = Cm + (size_t)i * N;
    for (int j = 0; j < N; ++j) c[j] = 0.0f;
    for (int k = 0; k < K; ++k) {
      const float av = a[k];
      const float* w = Wt + (size_t)k * N;
      for (int j = 0; j < N; ++j) c[j] += av * w[j];
    }
  }
}

static void layernorm_row(const float* x, int d, const float* g, const float* b, float* out) {
  float mean = 0.0f;
  for (int i = 0; i < d; ++i) mean += x[i];
  mean /= (float)d;
  float var = 0.0f;
  for (int i = 0; i < d; ++i) {
    const float t = x[i] - mean;
    var += t * t;
  }
  var /= (float)d;
  const float inv_std = 1.0f / sqrtf(var + 1e-5f);
  for (int i = 0; i < d; ++i) out[i] = (x[i] - mean) * inv_std * g[i] + b[i];
}

static float gelu(float x) {
  const float inner = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(inner));
}

static int argmax_row(const float* x, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (x[i] > x[best]) best = i;
  return best;
}

/* ------------------------------------------------------------------ model + advance */
typedef struct {
  int V, d, L, H, S, hd;
  const int* heads; /* active head count per layer */
  const int* ffn;   /* active FFN width per layer */
  const float* tok;
  const float* pos;
  const float* lnf_g;
  const float* lnf_b;
  const float* const* ln1_g;
  const float* const* ln1_b;
  const float* const* ln2_g;
  const float* const* ln2_b;
  const float* tok_t;       /* tok_embed^T [d x V] for the tied head */
  const float* const* wq;   /* transposed: [d x kh] (x * W^T form, runtime.cpp:80-85) */
  const float* const* wk;
  const float* const* wv;
  const float* const* wo;    /* [kh x d] */
  const float* const* w_in;  /* [d x f] */
  const float* const* w_out; /* [f x d] */
  /* W8A8 restatement (act_quant != 0): per linear (index layer*6 + {q,k,v,o,in,out}) the int8 weight
   * codes transposed to [K x N] and the per-output-channel scales [N]. */
  int act_quant;
  const int8_t* const* wcodes_t;
  const float* const* wscale;
  /* act_quant only: 1 = the GPU W8A8 engine's rounding points - q/k/v leave the QKV GEMM epilogue
   * as fp16 (KV pages, q operand), the attention output z and the GELU output g are fp16 before
   * they are quantized (engine.cu launch_step; kernels.cu quant_rows_kernel). fp16 = RNE of f32. */
  int gpu_points;
} orc_model;

/* f32 -> IEEE binary16 -> f32, round to nearest even (cvt.rn.f16.f32 / __float2half_rn): the GPU
 * engine's 16-bit storage type (paper_2507_04967_b200/csrc/dtype.hpp). Subnormal halves keep the
 * 2^-24 quantum; magnitudes >= 65520 become inf. */
static float h16r(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  const uint32_t sign = u & 0x80000000u, a = u & 0x7fffffffu;
  if (a >= 0x7f800000u) return x; /* inf / nan */
  float ax;
  memcpy(&ax, &a, 4);
  uint32_t r;
  if (ax >= 65520.0f) {
    r = 0x7f800000u;
  } else if (ax < 6.103515625e-05f) { /* subnormal half: multiples of 2^-24 */
    const float q = rintf(ax * 16777216.0f) * 5.9604644775390625e-08f;
    memcpy(&r, &q, 4);
  } else { /* 10 mantissa bits: round away the low 13 */
    r = (a + 0xfffu + ((a >> 13) & 1u)) & ~0x1fffu;
  }
  r |= sign;
  memcpy(&x, &r, 4);
  return x;
}
static void h16r_rows(float* p, size_t n) {
  for (size_t i = 0; i < n; ++i) p[i] = h16r(p[i]);
}

/* Capture of the int8 GEMM operands of one W8A8 forward (orc_forward_codes): per layer the codes of
 * [attn_in n x d][attn_out_in n x kh][ffn_in n x d][ffn_mid n x f] and their per-token scales
 * [4 x n]. Thread-local so concurrent decodes on one model are unaffected. */
static __thread int8_t* tl_cap_codes;
static __thread float* tl_cap_scales;
static __thread size_t tl_cap_off, tl_cap_soff;

void orc_quant_rows_s8(const float* x, int n, int d, int8_t* codes, float* scales);

/* y[n x N] = W8A8(x[n x K], linear `which`): per-token int8 x codes, exact int32 dot with the int8
 * weight codes, then (float)acc * s_x * s_w - the GPU kind::i8 GEMM epilogue's arithmetic. */
static void linear_w8a8(const orc_model* m, int li, const float* x, int n, int K, int N, float* y) {
  int8_t* xc = (int8_t*)malloc((size_t)n * K);
  float* xs = (float*)malloc(sizeof(float) * n);
  int32_t* acc = (int32_t*)malloc(sizeof(int32_t) * N);
  orc_quant_rows_s8(x, n, K, xc, xs);
  if (tl_cap_codes && li % 6 != 1 && li % 6 != 2) { /* wk / wv share wq's input */
    memcpy(tl_cap_codes + tl_cap_off, xc, (size_t)n * K);
    memcpy(tl_cap_scales + tl_cap_soff, xs, sizeof(float) * n);
    tl_cap_off += (size_t)n * K;
    tl_cap_soff += (size_t)n;
  }
  const int8_t* w = m->wcodes_t[li];
  const float* ws = m->wscale[li];
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < N; ++j) acc[j] = 0;
    for (int k = 0; k < K; ++k) {
      const int32_t a = xc[(size_t)i * K + k];
      const int8_t* wr = w + (size_t)k * N;
      for (int j = 0; j < N; ++j) acc[j] += a * (int32_t)wr[j];
    }
    for (int j = 0; j < N; ++j) y[(size_t)i * N + j] = (float)acc[j] * xs[i] * ws[j];
  }
  free(xc);
  free(xs);
  free(acc);
}

/* The GPU GEMM epilogue's GELU (ptx.cuh gelu_tanh): x * 1/(1 + 2^(inner * -2log2(e))),
 * inner = x * fma(x*x, k*0.044715, k) - the reference's tanh form rewritten as x * sigmoid(2u). */
static float gelu_gpu(float x) {
  const float k = 0.7978845608028654f, k3 = 0.7978845608028654f * 0.044715f;
  const float m2l2e = -2.0f * 1.4426950408889634f;
  const float inner = x * fmaf(x * x, k3, k);
  return x * (1.0f / (1.0f + exp2f(inner * m2l2e)));
}

/* The GPU prefill attention of one (query, head) at the W8A8 engine's rounding points
 * (kernels.cu attn_prefill_kernel for hd <= 32: 32-key blocks, exact running max; attn_tc.cu
 * attn_prefill_hp_kernel for hd 64 and 128: 32-key blocks, reference max moved only by a jump of
 * more than HP_RESCALE = 8; blocks aligned to absolute positions): online softmax in base 2 with scale_log2 = log2(e)/sqrt(hd)
 * in f32, per block ms = max_j(s_j) * scale_log2, m_new = max(m, ms) (hd >= 64: m_new = ms only when
 * m = -inf or ms > m + 8, else m), alpha = 2^(m - m_new), l = l * alpha + sum_j p_j with
 * p_j = 2^(fma(s_j, scale_log2, -m_new)) in f32, O = O * alpha + sum_j fp16(p_j) * v_j (the PV product
 * takes P as fp16), z = fp16(O * (1 / l)). Scores are f32 dots of the fp16 q / k.
 * Remaining differences to the GPU are f32 summation orders and the 2-ulp ex2.approx. */
static void flash_head_gpu(const float* qh, const float* k0, const float* v0, int ld, int hd, int span,
                           const uint8_t* valid, float* zh) {
  const int KB = 32;
  const int stale = hd >= 64; /* attn_prefill_hp_kernel's reference-max rule */
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
  float m_run = -INFINITY, l_run = 0.0f;
  float o[128], s[64];
  for (int j = 0; j < hd; ++j) o[j] = 0.0f;
  for (int key0 = 0; key0 < span; key0 += KB) {
    const int nk = span - key0 < KB ? span - key0 : KB;
    float mx = -INFINITY;
    for (int t = 0; t < nk; ++t) {
      const int key = key0 + t;
      if (!valid[key]) {
        s[t] = -INFINITY;
        continue;
      }
      const float* kr = k0 + (size_t)key * ld;
      float acc = 0.0f;
      for (int c = 0; c < hd; ++c) acc += qh[c] * kr[c];
      s[t] = acc;
      if (acc > mx) mx = acc;
    }
    const float ms = mx * scale_log2;
    float mnew = fmaxf(m_run, ms);
    if (stale) mnew = (m_run == -INFINITY || ms > m_run + 8.0f) ? ms : m_run;
    const float alpha = (mnew == -INFINITY || m_run == -INFINITY) ? 1.0f : exp2f(m_run - mnew);
    const float msub = mnew == -INFINITY ? 0.0f : mnew;
    m_run = mnew;
    l_run *= alpha;
    /* O is rescaled (only on a reference-max move for hd >= 64), then the block's P V accumulates
     * into it, as the tensor core accumulates into O in TMEM */
    for (int j = 0; j < hd; ++j) o[j] *= alpha;
    for (int t = 0; t < nk; ++t) {
      const float pv = exp2f(fmaf(s[t], scale_log2, -msub));
      l_run += pv;
      const float pb = h16r(pv);
      if (pb == 0.0f) continue;
      const float* vr = v0 + (size_t)(key0 + t) * ld;
      for (int j = 0; j < hd; ++j) o[j] = fmaf(pb, vr[j], o[j]);
    }
  }
  const float inv = l_run > 0.0f ? 1.0f / l_run : 0.0f;
  for (int j = 0; j < hd; ++j) zh[j] = h16r(o[j] * inv);
}

typedef struct {
  float** k; /* per layer [S x kh] */
  float** v;
  uint8_t* valid;
  int len;
} orc_state;

static void state_init(const orc_model* m, orc_state* st) {
  st->k = (float**)calloc((size_t)m->L, sizeof(float*));
  st->v = (float**)calloc((size_t)m->L, sizeof(float*));
  for (int l = 0; l < m->L; ++l) {
    const int kh = m->heads[l] * m->hd;
    st->k[l] = (float*)calloc((size_t)m->S * kh, sizeof(float));
    st->v[l] = (float*)calloc((size_t)m->S * kh, sizeof(float));
  }
  st->valid = (uint8_t*)calloc((size_t)m->S, 1);
  st->len = 0;
}
static void state_free(const orc_model* m, orc_state* st) {
  for (int l = 0; l < m->L; ++l) {
    free(st->k[l]);
    free(st->v[l]);
  }
  free(st->k);
  free(st->v);
  free(st->valid);
}

/* ModelRuntime::advance for n consecutive positions p0.. of ONE sequence (runtime.cpp:104-211).
 * Returns final-norm rows y[n x d]. madds accumulates exactly what the reference counter adds. */
static void advance(const orc_model* m, orc_state* st, const int* toks, const uint8_t* valid,
                    int p0, int n, float* y, uint64_t* madds) {
  const int d = m->d, hd = m->hd;
  const float inv_sqrt_hd = 1.0f / sqrtf((float)hd);
  for (int i = 0; i < n; ++i) st->valid[p0 + i] = valid ? valid[i] : 1;
  float* x = (float*)malloc(sizeof(float) * n * d);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j)
      x[(size_t)i * d + j] = m->tok[(size_t)toks[i] * d + j] + m->pos[(size_t)(p0 + i) * d + j];
  float* scores = (float*)malloc(sizeof(float) * m->S);
  float* probs = (float*)malloc(sizeof(float) * m->S);
  float* h = (float*)malloc(sizeof(float) * n * d);
  for (int l = 0; l < m->L; ++l) {
    const int kh = m->heads[l] * hd, f = m->ffn[l];
    float* q = (float*)malloc(sizeof(float) * n * kh);
    float* kn = (float*)malloc(sizeof(float) * n * kh);
    float* vn = (float*)malloc(sizeof(float) * n * kh);
    float* z = (float*)calloc((size_t)n * kh, sizeof(float));
    float* ao = (float*)malloc(sizeof(float) * n * d);
    float* g = (float*)malloc(sizeof(float) * n * f);
    for (int i = 0; i < n; ++i) layernorm_row(x + (size_t)i * d, d, m->ln1_g[l], m->ln1_b[l], h + (size_t)i * d);
    if (m->act_quant) {
      linear_w8a8(m, l * 6 + 0, h, n, d, kh, q);
      linear_w8a8(m, l * 6 + 1, h, n, d, kh, kn);
      linear_w8a8(m, l * 6 + 2, h, n, d, kh, vn);
    } else {
      matmul_wt(h, n, d, m->wq[l], kh, q);
      matmul_wt(h, n, d, m->wk[l], kh, kn);
      matmul_wt(h, n, d, m->wv[l], kh, vn);
    }
    if (m->act_quant && m->gpu_points) {
      h16r_rows(q, (size_t)n * kh);
      h16r_rows(kn, (size_t)n * kh);
      h16r_rows(vn, (size_t)n * kh);
    }
    *madds += 3ull * n * d * kh;
    for (int i = 0; i < n; ++i) {
      memcpy(st->k[l] + (size_t)(p0 + i) * kh, kn + (size_t)i * kh, sizeof(float) * kh);
      memcpy(st->v[l] + (size_t)(p0 + i) * kh, vn + (size_t)i * kh, sizeof(float) * kh);
    }
    for (int i = 0; i < n; ++i) {
      if (valid && !valid[i]) continue;
      const int span = p0 + i + 1;
      if (m->act_quant && m->gpu_points) {
        for (int hh = 0; hh < m->heads[l]; ++hh)
          flash_head_gpu(q + (size_t)i * kh + (size_t)hh * hd, st->k[l] + (size_t)hh * hd,
                         st->v[l] + (size_t)hh * hd, kh, hd, span, st->valid, z + (size_t)i * kh + (size_t)hh * hd);
        *madds += 2ull * span * hd * m->heads[l];
        continue;
      }
      for (int hh = 0; hh < m->heads[l]; ++hh) {
        const float* qh = q + (size_t)i * kh + (size_t)hh * hd;
        for (int s = 0; s < span; ++s) {
          const float* kr = st->k[l] + (size_t)s * kh + (size_t)hh * hd;
          float acc = 0.0f;
          for (int k = 0; k < hd; ++k) acc += qh[k] * kr[k];
          scores[s] = acc * inv_sqrt_hd;
        }
        *madds += (uint64_t)span * hd;
        /* softmax_row with the state's validity mask */
        float mx = 0.0f;
        int any = 0;
        for (int s = 0; s < span; ++s) {
          if (!st->valid[s]) continue;
          if (!any || scores[s] > mx) mx = scores[s];
          any = 1;
        }
        float sum = 0.0f;
        for (int s = 0; s < span; ++s) {
          probs[s] = 0.0f;
          if (!st->valid[s]) continue;
          const float e = expf(scores[s] - mx);
          probs[s] = e;
          sum += e;
        }
        for (int s = 0; s < span; ++s)
          if (st->valid[s]) probs[s] /= sum;
        float* zh = z + (size_t)i * kh + (size_t)hh * hd;
        for (int s = 0; s < span; ++s) {
          const float w = probs[s];
          const float* vr = st->v[l] + (size_t)s * kh + (size_t)hh * hd;
          for (int j = 0; j < hd; ++j) zh[j] += w * vr[j];
        }
        *madds += (uint64_t)span * hd;
      }
    }
    if (m->act_quant && m->gpu_points) h16r_rows(z, (size_t)n * kh);
    if (m->act_quant) linear_w8a8(m, l * 6 + 3, z, n, kh, d, ao);
    else matmul_wt(z, n, kh, m->wo[l], d, ao);
    *madds += (uint64_t)n * kh * d;
    for (size_t t = 0; t < (size_t)n * d; ++t) x[t] += ao[t];
    for (int i = 0; i < n; ++i) layernorm_row(x + (size_t)i * d, d, m->ln2_g[l], m->ln2_b[l], h + (size_t)i * d);
    if (m->act_quant) linear_w8a8(m, l * 6 + 4, h, n, d, f, g);
    else matmul_wt(h, n, d, m->w_in[l], f, g);
    *madds += (uint64_t)n * d * f;
    if (m->act_quant && m->gpu_points)
      for (size_t t = 0; t < (size_t)n * f; ++t) g[t] = gelu_gpu(g[t]);
    else
      for (size_t t = 0; t < (size_t)n * f; ++t) g[t] = gelu(g[t]);
    if (m->act_quant && m->gpu_points) h16r_rows(g, (size_t)n * f);
    if (m->act_quant) linear_w8a8(m, l * 6 + 5, g, n, f, d, ao);
    else matmul_wt(g, n, f, m->w_out[l], d, ao);
    *madds += (uint64_t)n * f * d;
    for (size_t t = 0; t < (size_t)n * d; ++t) x[t] += ao[t];
    free(q);
    free(kn);
    free(vn);
    free(z);
    free(ao);
    free(g);
  }
  for (int i = 0; i < n; ++i) layernorm_row(x + (size_t)i * d, d, m->lnf_g, m->lnf_b, y + (size_t)i * d);
  if (p0 + n > st->len) st->len = p0 + n;
  free(x);
  free(h);
  free(scores);
  free(probs);
}

/* logits_for: y * tok_embed^T (runtime.cpp:213-215). */
static void logits_for(const orc_model* m, const float* y, int n, float* logits, uint64_t* madds) {
  matmul_wt(y, n, m->d, m->tok_t, m->V, logits);
  *madds += (uint64_t)n * m->d * m->V;
}

/* ModelRuntime::forward (runtime.cpp:217-232). Returns 0, 1 (contract) or 2 (too long). */
int orc_forward(const orc_model* m, const int* ids, const uint8_t* mask, int n, float* logits,
                uint64_t* madds) {
  if (n <= 0) return 1;
  if (n > m->S) return 2;
  for (int i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= m->V) return 1;
  orc_state st;
  state_init(m, &st);
  float* y = (float*)malloc(sizeof(float) * n * m->d);
  uint64_t c = 0;
  advance(m, &st, ids, mask, 0, n, y, &c);
  logits_for(m, y, n, logits, &c);
  if (madds) *madds = c;
  free(y);
  state_free(m, &st);
  return 0;
}

/* W8A8 forward that also returns the int8 operand codes and scales of every linear input (layout
 * at tl_cap_codes above). Requires act_quant. */
int orc_forward_codes(const orc_model* m, const int* ids, int n, float* logits, int8_t* codes,
                      float* scales) {
  if (!m->act_quant) return 1;
  tl_cap_codes = codes;
  tl_cap_scales = scales;
  tl_cap_off = tl_cap_soff = 0;
  const int st = orc_forward(m, ids, NULL, n, logits, NULL);
  tl_cap_codes = NULL;
  tl_cap_scales = NULL;
  return st;
}

/* Greedy decode of ONE prompt (ids already [BOS]+bytes): the per-item state machine of
 * batch_decode (runtime.cpp:261-307). batch_decode(P)[i] == this(P[i]) bit-for-bit, which is the
 * reference's own batch-invariance contract (test_model.cpp:240-267). */
static void top2(const float* x, int n, float* gap, float* amax) {
  float a = -INFINITY, b = -INFINITY, mx = 0.0f;
  for (int i = 0; i < n; ++i) {
    if (x[i] > a) {
      b = a;
      a = x[i];
    } else if (x[i] > b) {
      b = x[i];
    }
    mx = fmaxf(mx, fabsf(x[i]));
  }
  *gap = a - b;
  *amax = mx;
}

/* gap / amax (optional, max_new + 1 entries each): the CPU logits' top-1 minus top-2 and max |logit| at
 * every prediction of the row - what a GPU divergence at that step is traced against (tests/parity.py). */
static int decode_row_gaps(const orc_model* m, const int* ids, int n, int max_new, int* out_ids,
                           int* out_len, uint64_t* madds, float* gap, float* amax) {
  *out_len = 0;
  if (max_new == 0) return 0;
  if (n > m->S) return 2;
  for (int i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= m->V) return 1;
  orc_state st;
  state_init(m, &st);
  float* y = (float*)malloc(sizeof(float) * n * m->d);
  float* logits = (float*)malloc(sizeof(float) * m->V);
  uint64_t c = 0;
  advance(m, &st, ids, NULL, 0, n, y, &c);
  logits_for(m, y + (size_t)(n - 1) * m->d, 1, logits, &c);
  int emitted = 0;
  for (;;) {
    if (gap) top2(logits, m->V, gap + emitted, amax + emitted);
    const int next = argmax_row(logits, m->V);
    if (next == 130 || emitted == max_new) break;
    out_ids[emitted++] = next;
    if (st.len == m->S) break;
    advance(m, &st, &next, NULL, st.len, 1, y, &c);
    logits_for(m, y, 1, logits, &c);
  }
  *out_len = emitted;
  if (madds) *madds = c;
  free(y);
  free(logits);
  state_free(m, &st);
  return 0;
}

int orc_decode_row(const orc_model* m, const int* ids, int n, int max_new, int* out_ids,
                   int* out_len, uint64_t* madds) {
  return decode_row_gaps(m, ids, n, max_new, out_ids, out_len, madds, NULL, NULL);
}

typedef struct {
  const orc_model* m;
  float* gap;
  float* amax;
  const int* ids;
  const int64_t* offsets;
  int n_rows, max_new;
  int* out_ids;
  int* out_len;
  uint64_t madds;
  int status;
  int* next;
  pthread_mutex_t* mu;
} decode_job;

static void* decode_worker(void* arg) {
  decode_job* j = (decode_job*)arg;
  for (;;) {
    pthread_mutex_lock(j->mu);
    const int r = (*j->next)++;
    pthread_mutex_unlock(j->mu);
    if (r >= j->n_rows) break;
    uint64_t c = 0;
    const size_t g = (size_t)r * (j->max_new + 1);
    const int st = decode_row_gaps(j->m, j->ids + j->offsets[r], (int)(j->offsets[r + 1] - j->offsets[r]),
                                   j->max_new, j->out_ids + (size_t)r * j->max_new, j->out_len + r, &c,
                                   j->gap ? j->gap + g : NULL, j->amax ? j->amax + g : NULL);
    if (st && !j->status) j->status = st;
    j->madds += c;
  }
  return NULL;
}

/* Rows spread over `threads` workers. */
int orc_decode_rows_gaps(const orc_model* m, const int* ids, const int64_t* offsets, int n_rows,
                         int max_new, int* out_ids, int* out_len, uint64_t* madds, int threads,
                         float* gap, float* amax) {
  if (threads < 1) threads = 1;
  int next = 0;
  pthread_mutex_t mu;
  pthread_mutex_init(&mu, NULL);
  decode_job* jobs = (decode_job*)calloc((size_t)threads, sizeof(decode_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (decode_job){m, gap, amax, ids, offsets, n_rows, max_new, out_ids, out_len, 0, 0, &next, &mu};
    if (t) pthread_create(&th[t], NULL, decode_worker, &jobs[t]);
  }
  decode_worker(&jobs[0]);
  int status = 0;
  uint64_t total = 0;
  for (int t = 0; t < threads; ++t) {
    if (t) pthread_join(th[t], NULL);
    if (jobs[t].status && !status) status = jobs[t].status;
    total += jobs[t].madds;
  }
  if (madds) *madds = total;
  free(jobs);
  free(th);
  pthread_mutex_destroy(&mu);
  return status;
}

int orc_decode_rows(const orc_model* m, const int* ids, const int64_t* offsets, int n_rows,
                    int max_new, int* out_ids, int* out_len, uint64_t* madds, int threads) {
  return orc_decode_rows_gaps(m, ids, offsets, n_rows, max_new, out_ids, out_len, madds, threads, NULL, NULL);
}

/* ------------------------------------------------------------------ W8A8 restatement */
/* Per-token symmetric int8 quantization of activation rows, modelled on the reference's RTN rule
 * (quant.cpp:23-38) applied to rows: scale = amax/127 (amax == 0 -> 1); inv = 1/scale (fp32);
 * code = clamp(nearbyint(x * inv), -127, 127) with the fp32 product (round-to-nearest-even).
 * The reference has no activation quantization; this is the rule the GPU W8A8 path
 * implements (kernels.cu quant_one), pinned here bit-for-bit. */
void orc_quant_rows_s8(const float* x, int n, int d, int8_t* codes, float* scales) {
  for (int i = 0; i < n; ++i) {
    const float* r = x + (size_t)i * d;
    float amax = 0.0f;
    for (int k = 0; k < d; ++k) amax = fmaxf(amax, fabsf(r[k]));
    const float s = amax == 0.0f ? 1.0f : amax / 127.0f;
    const float inv = 1.0f / s;
    scales[i] = s;
    for (int k = 0; k < d; ++k) {
      const float y = r[k] * inv;
      float q = nearbyintf(y);
      if (q > 127.0f) q = 127.0f;
      if (q < -127.0f) q = -127.0f;
      codes[(size_t)i * d + k] = (int8_t)q;
    }
  }
}

/* Exact int32 GEMM: C[M x N] = A[M x K] * W[N x K]^T. */
void orc_gemm_s8(const int8_t* A, const int8_t* W, int M, int N, int K, int32_t* Cm) {
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t acc = 0;
      for (int k = 0; k < K; ++k) acc += (int32_t)A[(size_t)i * K + k] * (int32_t)W[(size_t)j * K + k];
      Cm[(size_t)i * N + j] = acc;
    }
}
