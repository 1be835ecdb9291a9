/*
 * iolm_cuda.h - C ABI of the B200-native prompt() hot path.
 *
 * This is the drop-in boundary for the reference's model runtime, iolm::ModelRuntime
 * (/root/reference/proj/include/iolm/runtime.hpp:37-95, proj/src/runtime.cpp:60-345). The
 * reference has no plugin registry; every caller (PromptResolver::flush, proj/src/exec.cpp:133;
 * semantic join, exec.cpp:320-322; validate, proj/src/optimize.cpp:335-336) holds a
 * `const ModelRuntime&`. The C++ shim in include/iolm_cuda_runtime.hpp rebuilds that exact class
 * surface on top of these entry points; INTEGRATION.md shows the swap.
 *
 * Plain pointers and sizes only: no C++ or torch types cross this boundary.
 *
 * Status codes (return value of every int-returning entry point) mirror the reference's
 * exception classes (proj/include/iolm/common.hpp:16-89):
 */
#ifndef IOLM_CUDA_H_
#define IOLM_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IOLM_OK 0
#define IOLM_E_CONTRACT 1          /* iolm::ContractViolation */
#define IOLM_E_SEQ_TOO_LONG 2      /* iolm::SequenceTooLong (bad_row set) */
#define IOLM_E_UNSUPPORTED 3       /* encoding/shape this GPU build does not run */
#define IOLM_E_CUDA 4              /* CUDA runtime / launch failure */
#define IOLM_E_OOM 5               /* device memory exhausted */
#define IOLM_E_CORRUPT_HEADER 6    /* iolm::CorruptHeader */
#define IOLM_E_TRUNCATED_BLOB 7    /* iolm::TruncatedBlob */
#define IOLM_E_UNKNOWN_ENCODING 8  /* iolm::UnknownEncoding */
#define IOLM_E_STALE 9             /* device-layout image does not match the bundle hash / weight options */

/* Tokenizer constants (proj/include/iolm/tokenizer.hpp:17-20). */
#define IOLM_VOCAB 131
#define IOLM_PAD 128
#define IOLM_BOS 129
#define IOLM_EOS 130

typedef struct iolm_cuda_ctx iolm_cuda_ctx;

/* Engine options. Zero means "default" for every field. */
typedef struct iolm_cuda_opts {
  int32_t max_tokens_per_step; /* continuous-batching token budget per engine step (default: SMs/2 x 256) */
  int32_t max_slots;           /* sequences resident in the paged KV pool (default: derived) */
  int32_t page_size;           /* KV page size in tokens (default 16) */
  int32_t act_quant;           /* 1: W8A8 int8 activations for q8 / sparse24 weights (default 0) */
  int32_t prefix_sharing;      /* -1: off; 0/1: share the common prompt prefix KV (default on) */
  int32_t use_cuda_graph;      /* reserved, ignored: steps are enqueued asynchronously (programmatic dependent
                                  launch between kernels), so the host runs ahead of the device */
  int32_t kernel_timing;       /* 1: time every kernel class with CUDA events (iolm_cuda_kernel_times) */
  int32_t sparse_mma;          /* -1: expand sparse24_q8 to dense codes; 0/1: 2:4 sparse tensor cores (kind::i8 with
                                  act_quant, kind::f16 over fp16 activations without) */
  int32_t int4_mma;            /* -1: expand q4 codes to fp16 in HBM; 0/1: int4 in HBM, expanded in smem (W4A16) */
  int32_t prefill_tc;          /* prefill attention: -1 mma.sync; 0 default (tcgen05: 128-query tiles for hd 128, head-pair tiles for hd 64); 1 128-query tiles for hd 64 too */
  int32_t reserved[6];
} iolm_cuda_opts;

/* ModelConfig (proj/include/iolm/model.hpp:20-41); per-layer lists are queried separately. */
typedef struct iolm_cuda_model_config {
  int32_t vocab_size, d_model, n_layers, n_heads, d_ff, max_seq_len, head_dim;
} iolm_cuda_model_config;

/* Counters of the most recent decode/forward call. */
typedef struct iolm_cuda_stats {
  int64_t steps;          /* engine steps (one batched forward each) */
  int64_t tokens;         /* token rows pushed through the layers */
  int64_t prefill_tokens; /* of which prompt tokens */
  int64_t decode_tokens;  /* of which generated-token advances */
  int64_t prefix_tokens;  /* shared-prefix tokens computed once */
  int64_t kernel_launches;
  double device_ms;       /* device time of the call measured with CUDA events */
} iolm_cuda_stats;

/*
 * Replaces ModelRuntime::ModelRuntime(const ModelBundle&) (runtime.cpp:60-89).
 * bundle_bytes: the canonical serialize_bundle() byte stream (proj/src/model.cpp:311-346,
 * proj/docs/format.md). The weights are decoded/repacked onto `device`; the bytes may be freed
 * after the call returns.
 */
int iolm_cuda_create(const uint8_t* bundle_bytes, size_t len, int device,
                     const iolm_cuda_opts* opts, iolm_cuda_ctx** out);
void iolm_cuda_destroy(iolm_cuda_ctx* ctx);

/*
 * One context over several GPUs of a box (the table is range-partitioned, every GPU holds a
 * full replica and its own KV pool). iolm_cuda_decode on such a context splits the rows into
 * contiguous ranges of near-equal token counts, decodes them concurrently (one host thread per
 * device) and writes each range's ids / lengths straight into the caller's out_ids / out_len - the
 * output-column gather; row order is the caller's (PromptResolver's row-order guarantee,
 * proj/src/exec.cpp:139-142). madds is the sum over devices, *bad_row the batch's first too-long row
 * (all lengths are checked before any device work, runtime.cpp:264-267), and the error of the lowest
 * failing range otherwise. Outputs equal a one-device context's bit for bit (batch invariance).
 * forward / capture / codes / save_image run on devices[0]; last_stats and kernel_times of a
 * multi-device decode are summed over devices (device_ms: the slowest device).
 * iolm_cuda_decode_device_ids is single-device only (IOLM_E_UNSUPPORTED here). The same device may
 * be listed twice (tests on a 1-GPU box).
 */
int iolm_cuda_create_multi(const uint8_t* bundle_bytes, size_t len, const int32_t* devices, int32_t n_devices,
                           const iolm_cuda_opts* opts, iolm_cuda_ctx** out);
/* Number of devices (engines) of a context: 1 for iolm_cuda_create. */
int iolm_cuda_device_count(const iolm_cuda_ctx* ctx, int32_t* n);

/* ModelRuntime::bundle_hash() (runtime.hpp:42; FNV-1a over the serialized bundle, model.cpp:408). */
int iolm_cuda_bundle_hash(const iolm_cuda_ctx* ctx, uint64_t* out);
/* ModelRuntime::config() (runtime.hpp:41). */
int iolm_cuda_config(const iolm_cuda_ctx* ctx, iolm_cuda_model_config* out);
/* Per-layer pruning info: active head count and FFN width of layer l (model.hpp:30-31). */
int iolm_cuda_layer_shape(const iolm_cuda_ctx* ctx, int32_t layer, int32_t* heads, int32_t* ffn);
/* ModelConfig::active_heads[layer] (model.hpp:29): the surviving heads' ORIGINAL indices, ascending.
 * heads: capacity cap (>= n_heads always suffices); *n receives the count. */
int iolm_cuda_layer_heads(const iolm_cuda_ctx* ctx, int32_t layer, int32_t* heads, int32_t cap, int32_t* n);

/*
 * Replaces ModelRuntime::batch_decode(prompts, max_new_tokens, counter) (runtime.cpp:241-309).
 * ids/row_offsets: CSR token rows, row i = ids[row_offsets[i] .. row_offsets[i+1]) and already
 * tokenized exactly as the reference does it: [BOS] + one id per ASCII byte (runtime.cpp:262-263).
 * Host buffers. Outputs (host): out_ids[i*max_new_tokens + t] for t < out_len[i] are the emitted
 * ids (PAD/BOS included; they render nothing), out_len[i] the count. madds (optional) receives the
 * multiply-adds the reference FlopCounter would have added for the same call (runtime.cpp:311-345).
 * On IOLM_E_SEQ_TOO_LONG, *bad_row is the first offending row (runtime.cpp:264-267).
 */
int iolm_cuda_decode(iolm_cuda_ctx* ctx, const int32_t* ids, const int64_t* row_offsets,
                     int64_t n_rows, int32_t max_new_tokens, int32_t* out_ids, int32_t* out_len,
                     uint64_t* madds, int64_t* bad_row);

/* Same as iolm_cuda_decode but `d_ids` is already resident in device memory (row_offsets stay on
 * the host). Used to time the device path with inputs already in HBM. */
int iolm_cuda_decode_device_ids(iolm_cuda_ctx* ctx, const int32_t* d_ids,
                                const int64_t* row_offsets, int64_t n_rows,
                                int32_t max_new_tokens, int32_t* out_ids, int32_t* out_len,
                                uint64_t* madds, int64_t* bad_row);

/*
 * Replaces ModelRuntime::forward(ids, mask, counter) (runtime.cpp:217-232): logits for every
 * position, logits[n x 131] row-major f32. mask may be NULL (all valid); masked positions are
 * excluded as attention keys and their logits rows are unspecified (the reference says "callers
 * must not read", runtime.hpp:44-47).
 */
int iolm_cuda_forward_logits(iolm_cuda_ctx* ctx, const int32_t* ids, const uint8_t* mask,
                             int32_t n, float* logits, uint64_t* madds);

/*
 * forward with calibration capture (ModelRuntime::forward(ids, mask, counter, CaptureSink*),
 * runtime.hpp:22-28 / :48-49, used by capture_calibration, proj/src/calib.cpp:20-62): logits as in
 * iolm_cuda_forward_logits, plus the inputs every linear weight saw, as fp16 bit patterns, for ALL n
 * positions (the caller drops masked rows, as the reference records non-pad positions only).
 * Layout, layer by layer: [attn_in n x d][attn_out_in n x kh_l][ffn_in n x d][ffn_mid n x f_l]
 * (capture points "layers.<l>.attn_in" = LN1 output, "attn_out_in" = attention output, "ffn_in" =
 * LN2 output, "ffn_mid" = GELU output). capture holds n * sum_l (2 d + kh_l + f_l) elements.
 * Not available with opts.act_quant (the reference calibrates the baseline model).
 */
int iolm_cuda_forward_capture(iolm_cuda_ctx* ctx, const int32_t* ids, const uint8_t* mask, int32_t n,
                              float* logits, uint16_t* capture, uint64_t* madds);

/*
 * W8A8 parity (opts.act_quant): forward logits plus the int8 operand codes every linear layer consumed,
 * per layer [attn_in n x d][attn_out_in n x kh_l][ffn_in n x d][ffn_mid n x f_l] (the capture points of
 * iolm_cuda_forward_capture, as the per-token int8 codes of DESIGN.md's W8A8 rule), and their per-token
 * scales, per layer [4 x n] f32. Checked against the W8A8 restatement's codes (oracle/iolm_oracle.c
 * orc_forward_codes). Every projection must run W8A8, else IOLM_E_UNSUPPORTED.
 */
int iolm_cuda_forward_codes(iolm_cuda_ctx* ctx, const int32_t* ids, int32_t n, float* logits, int8_t* codes,
                            float* scales, uint64_t* madds);

/*
 * Device-layout image: the pre-tiled cache a registry keeps next to a bundle.
 * The reference rebuilds its runtime from the bundle on every load - deserialize, FNV-1a over the
 * whole serialized bundle, decode every tensor (ModelRegistry::lookup, proj/src/optimize.cpp:
 * 139-151; deserialize_bundle / ModelBundle::hash, proj/src/model.cpp:348-411; ModelRuntime ctor,
 * proj/src/runtime.cpp:60-89). An image holds the weights exactly as this engine keeps them in HBM
 * (fp16 / int8 / 2:4-compressed codes + pre-tiled metadata / packed int4, per-row scales), the model
 * config and the bundle hash, so loading is a streamed file read + H2D copy: no hashing, no decode,
 * no host repack, and half the bytes of the f32 bundle for dense models.
 *
 * save_image: writes the context's device layout to `path` (atomically: path.tmp + rename).
 * create_from_image: builds a context from an image. expected_hash != 0 must equal the image's
 * bundle hash (the registry index entry's hash), and the weight-shaping options (act_quant,
 * sparse_mma, int4_mma) must resolve as they did for the saved context; otherwise IOLM_E_STALE and
 * the caller falls back to iolm_cuda_create on the bundle. Engine-only options (token budget,
 * slots, prefix sharing, timing, prefill kernel) may differ. Bad magic / malformed header:
 * IOLM_E_CORRUPT_HEADER; short file: IOLM_E_TRUNCATED_BLOB; checksum mismatch: IOLM_E_CORRUPT_HEADER.
 * The context then behaves bit-for-bit like the one that was saved.
 * image_info: header only (no device work): the image's bundle hash and model config.
 */
int iolm_cuda_save_image(iolm_cuda_ctx* ctx, const char* path);
int iolm_cuda_create_from_image(const char* path, uint64_t expected_hash, int device,
                                const iolm_cuda_opts* opts, iolm_cuda_ctx** out);
int iolm_cuda_image_info(const char* path, uint64_t* bundle_hash, iolm_cuda_model_config* cfg);

/*
 * Calibration Gram matrix (the GPTQ / compensated-2:4 Hessian): h[cols x cols] =
 * scale * X^T X in f64 for X = x[rows x cols] f32 row-major (host buffers; device work on `device`).
 * Replaces fastmath::gram_accumulate under build_hessian (proj/src/calib.cpp:64-74,
 * proj/src/fastmath.cpp:79-100): every element is the same sequential f64 sum over samples in the
 * same order of exact f32 x f32 products, so h is BIT-IDENTICAL to the reference's. The shim's
 * iolm::cuda::build_hessian adds the damping exactly as the reference does.
 */
int iolm_cuda_gram(int device, const float* x, int64_t rows, int32_t cols, double scale, double* h);

/* Counters of the last decode/forward call on this context. */
int iolm_cuda_last_stats(const iolm_cuda_ctx* ctx, iolm_cuda_stats* out);

/* Per kernel-class device time of the last call, recorded with CUDA events on the engine stream
 * when opts.kernel_timing = 1. Classes (index): 0 embed+LN1, 1 QKV GEMM, 2 prefill attention,
 * 3 decode attention, 4 Wo GEMM, 5 LN, 6 W_in GEMM, 7 W_out GEMM, 8 head+argmax,
 * 9 int8 row quantization (W8A8).
 * ms[i]: summed launch durations; work[i]: algorithmic FLOPs (GEMMs, attention) or bytes (LN,
 * head, embed) of those launches; launches[i]: launch count. n: capacity of the arrays (>= 10). */
#define IOLM_KCLASSES 10
/* Turns the per-kernel CUDA-event timing of opts.kernel_timing on or off for subsequent calls
 * (the events cost ~3% of a step, so throughput runs leave it off and time a separate pass). */
int iolm_cuda_set_kernel_timing(iolm_cuda_ctx* ctx, int32_t on);
int iolm_cuda_kernel_times(const iolm_cuda_ctx* ctx, double* ms, double* work, int64_t* launches, int32_t n);

/* Thread-local message for the last non-OK status. */
const char* iolm_cuda_last_error(void);

/* ---- kernel-level entry points used by the parity tests (device work, host buffers) ---- */

/* C[M x N] = A[M x K] * W[N x K]^T with fp16 operands (raw uint16 bit patterns), f32 result,
 * through the production tcgen05 GEMM. epi: 0 f32 store, 2 GELU (result returned as f32 after a
 * fp16 round trip). bn: 256 = 2-SM 256x256 tiles (CTA pairs), 128 = single-CTA 128x128 tiles. */
int iolm_cuda_debug_gemm_f16(const uint16_t* A, const uint16_t* W, float* C, int32_t M, int32_t N,
                              int32_t K, int32_t bn, int32_t epi);

/* W8A8 integer GEMM: C_i32[M x N] = A_s8[M x K] * W_s8[N x K]^T through tcgen05 kind::i8.
 * Bit-exact integer accumulators. pair: 1 = 2-SM 256x256 tiles, 0 = single-CTA tiles. */
int iolm_cuda_debug_gemm_s8(const int8_t* A, const int8_t* W, int32_t* C, int32_t M, int32_t N,
                            int32_t K, int32_t pair);

/* Device-only GEMM timing (kernel tuning): mean ms per launch of `iters` launches on synthetic
 * operands. epi: 0 f32, 1 fp16, 2 gelu, 3 residual-add, 5 s32 (i8 only), 6 none (mainloop only).
 * i8: 0 fp16 x fp16, 1 s8 x s8 (W8A8), 2 fp16 x int4 (W4A16, K % 32 == 0). */
int iolm_cuda_debug_gemm_time(int32_t M, int32_t N, int32_t K, int32_t epi, int32_t pair, int32_t i8,
                              int32_t iters, float* ms_out);

/* Per-token int8 activation quantization (the W8A8 rule) of fp16 rows [n x d] on the
 * device: codes [n x d] and one f32 scale per row. */
/* 2:4 sparse W8A8 GEMM on the sparse tensor cores (tcgen05.mma.sp kind::i8): X_s8 [T x K] times a
 * sparse24_q8 tensor payload W [N x K] exactly as stored in a bundle (proj/src/model.cpp:255-290).
 * epi 5: raw int32 accumulators -> out_s32 [T x N] (bit-exact); epi 0: acc * a_scale[t] * w_scale[n]
 * -> out_f32 (w_scale = the payload's per-row scales). K % 16 == 0. */
int iolm_cuda_debug_gemm_sp24(const int8_t* X, const uint8_t* payload, int32_t T, int32_t N, int32_t K,
                              int32_t epi, const float* a_scale, int32_t* out_s32, float* out_f32);
/* W4A16 GEMM: C[M x N] = A_f16[M x K] * (codes(W) * scale)^T with W a q4_perchannel tensor payload
 * exactly as stored in a bundle (nibble rows + per-row f32 scales, proj/src/model.cpp:164-176); the
 * int4 codes are expanded to fp16 inside the kernel. epi 0: f32 out. pair as in debug_gemm_s8. */
int iolm_cuda_debug_gemm_w4(const uint16_t* A, const uint8_t* payload, float* C, int32_t M, int32_t N, int32_t K,
                            int32_t pair);
/* 2:4 sparse fp16 GEMM (tcgen05.mma.sp kind::f16): X fp16 [T x K] (raw uint16) times a sparse24_q8
 * payload's kept codes as exact fp16 integers, out_f32 [T x N] = acc * payload scale[n]. K % 16 == 0. */
int iolm_cuda_debug_gemm_sp24_f16(const uint16_t* X, const uint8_t* payload, int32_t T, int32_t N, int32_t K,
                                   float* out_f32);
/* Device-only timing of the sparse GEMM: mean ms per launch (epi as in debug_gemm_time). */
int iolm_cuda_debug_gemm_sp24_time(int32_t T, int32_t N, int32_t K, int32_t epi, int32_t iters, float* ms_out);
/* The same for the fp16 (kind::f16) sparse kernel. */
int iolm_cuda_debug_gemm_sp24_f16_time(int32_t T, int32_t N, int32_t K, int32_t epi, int32_t iters, float* ms_out);

/* The multi-device row split (host only, no device work): cut[0..*n_cut) with cut[0] = 0 and
 * cut[last] = n_rows; range i = rows [cut[i], cut[i+1]). cut needs shards + 1 entries. */
int iolm_cuda_debug_partition(const int64_t* row_offsets, int64_t n_rows, int32_t shards, int64_t* cut,
                              int32_t* n_cut);

int iolm_cuda_debug_quant_rows_f16(const uint16_t* x, int32_t n, int32_t d, int8_t* codes, float* scales);

#ifdef __cplusplus
}
#endif
#endif /* IOLM_CUDA_H_ */
