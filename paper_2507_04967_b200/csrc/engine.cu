// The B200 model runtime behind the C ABI (include/iolm_cuda.h).
//
// Replaces iolm::ModelRuntime (proj/src/runtime.cpp:60-345):
//   * construction: the bundle is parsed/validated like the reference (bundle.cu), every linear
//     weight is decoded ONCE on the device into the GEMM operand layout (fp16, K-major = the
//     bundle's own [out x in] layout, so no transpose), norms/embeddings stay fp32;
//   * batch_decode: a continuous-batching scheduler. Each engine step is ONE batched forward over
//     a token list mixing (a) one generated token for every live sequence and (b) the prompt tokens
//     of newly admitted rows, so every GEMM runs at M = thousands of rows. The common prompt prefix
//     of the call is prefilled once into shared KV pages that every row's page table references.
//   * K/V live in a paged fp16 pool (16-token pages); attention reads through per-slot page tables.
//   * steps are pipelined: whether a row keeps decoding is decided by its emitted count and its
//     length alone, except for EOS, so step k+1 is planned and launched before step k's tokens are
//     read back. A row that hits EOS gets one speculative token in the next step; it is discarded.
//     Generated token ids stay on the device (per-slot register written by the argmax kernel).
// Output semantics follow batch_decode exactly (runtime.cpp:280-307): argmax (ties -> lowest id),
// stop on EOS / budget before emitting, stop on a full context after emitting; the FlopCounter
// contribution is the reference's closed form (runtime.cpp:311-345).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "bundle.hpp"
#include "capi_util.hpp"
#include "kernels.cuh"
#include "launch.hpp"
#include "sparse24.hpp"
#include "tma_host.hpp"

namespace iolmh {

using iolmk::AttnGroup;
using iolmk::AttnParams;
using iolmk::GemmEpi;

void launch_ln(const float* x, int M, int d, const float* g, const float* b, h16* h, int ldh,
               cudaStream_t st, int8_t* q8, float* qscale);
void launch_embed_ln(const int32_t* ids, const int64_t* tok_src, const int* tok_slot, const int* tok_pos,
                     const int32_t* last_tok, int M, int d, const float* tok_embed, const float* pos_embed, float* x,
                     const float* g, const float* b, h16* h, int ldh, cudaStream_t st, int8_t* q8,
                     float* qscale);
void launch_quant_rows(const h16* src, int lds, int M, int cols, int8_t* dst, int ldd, float* scale,
                       cudaStream_t st);
void launch_decode_codes(const void* payload, int enc, int rows, int cols, void* dst, bool int8, int ld,
                         float* scales, cudaStream_t st);
void launch_attention(const AttnParams& prefill, const AttnParams& decode, int hd, cudaStream_t st);
bool launch_prefill_tc(const AttnParams& prefill, int hd, cudaStream_t st);
bool launch_prefill_hp(const AttnParams& prefill, int hd, cudaStream_t st);
int decode_heads_per_cta(int heads, int hd);
void launch_head(const float* x, int d, const int* rows, int n_rows, const float* g, const float* b,
                 const float* embed_t, int V, const int* row_slot, int32_t* next_tok, int32_t* last_tok,
                 float* logits_out, cudaStream_t st);
void launch_gather_head_rows(const float* x, int d, const h16* z, int ldz, int kh, const int* rows, int n_rows,
                             float* xc, h16* zc, int ldzc, cudaStream_t st);
void launch_lcp(const int32_t* ids, const int64_t* offsets, int64_t n_rows, int limit, int* out, cudaStream_t st);
void launch_check_ids(const int32_t* ids, int64_t n, int V, int* bad, cudaStream_t st);
void launch_decode_weight(const void* payload, int enc, int rows, int cols, h16* dst, int ld,
                          cudaStream_t st);
void launch_transpose(const float* src, int rows, int cols, float* dst, cudaStream_t st);

namespace {

constexpr int PAGE = 16;
constexpr int QCHUNK = 64;

template <typename T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  DevArray() = default;
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  ~DevArray() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    CUDA_OK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
};

template <typename T>
struct PinnedArray {
  T* p = nullptr;
  size_t n = 0;
  PinnedArray() = default;
  PinnedArray(const PinnedArray&) = delete;
  ~PinnedArray() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    CUDA_OK(cudaMallocHost(&p, std::max<size_t>(count, 1) * sizeof(T)));
    n = count;
  }
};

int round_up(int x, int m) { return (x + m - 1) / m * m; }
size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

// Weights of one GEMM ([N x K], K-major as stored in the bundle) in one of three forms:
//   VALUES : fp16(value)                       dense_f32 tensors (or mixed-encoding groups)
//   CODES  : fp16(code) + f32 scale per row    q8 / q4 / sparse24 without activation quant (W8A16,
//            W4A16): integer codes are exact in fp16, the scale is applied in the GEMM epilogue
//   INT8   : int8 code + f32 scale per row     q8 / sparse24 with act_quant (W8A8, kind::i8)
//   SP24   : kept int8 codes [N x K/2] + 2:4 metadata + f32 scale per row: sparse24_q8 with
//            act_quant on the sparse tensor cores (tcgen05.mma.sp kind::i8, gemm_sp_sm100.cuh)
//   INT4   : packed q4 nibbles [N x ceil(K/2)] + f32 scale per row: W4A16, the codes are expanded
//            to fp16 inside the GEMM (shared memory), never in HBM
//   SP24F  : kept codes as exact fp16 [N x K/2] + 2:4 metadata + f32 scale per row: sparse24_q8
//            WITHOUT act_quant on the sparse tensor cores (tcgen05.mma.sp kind::f16, fp16 activations)
enum WMode : int { W_VALUES = 0, W_CODES = 1, W_INT8 = 2, W_SP24 = 3, W_INT4 = 4, W_SP24F = 5 };
struct GemmW {
  int mode = W_VALUES;
  DevArray<h16> wb;
  DevArray<int8_t> w8;
  DevArray<float> scale;
  CUtensorMap tm;
  // W_SP24 (metadata) / W_INT4 (packed nibbles)
  DevArray<uint8_t> w4;
  DevArray<uint8_t> meta;
  Sp24Layout sl;
  CUtensorMap tm_e;
  bool int8() const { return mode == W_INT8 || mode == W_SP24; }
};

size_t w4_pitch(int K) { return (static_cast<size_t>(K + 1) / 2 + 15) / 16 * 16; }

// TMA descriptors of one weight group once its arrays are resident (bundle or image load).
void weight_maps(GemmW& w, int N, int K, int ld) {
  switch (w.mode) {
    case W_SP24:
      w.tm = sp24_codes_map(w.sl, w.w8.p);
      w.tm_e = sp24_meta_map(w.sl, w.meta.p);
      break;
    case W_SP24F:
      w.tm = sp24_codes_map(w.sl, w.wb.p);
      w.tm_e = sp24_meta_map(w.sl, w.meta.p);
      break;
    case W_INT4:
      w.tm = make_w4_map(w.w4.p, static_cast<uint64_t>(K), static_cast<uint64_t>(N), w4_pitch(K));
      break;
    case W_INT8:
      w.tm = make_kmajor_map(w.w8.p, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, K, N, static_cast<uint64_t>(ld), 128);
      break;
    default:
      w.tm = make_kmajor_map(w.wb.p, H16_TMA, 2, K, N, 2ull * ld, 128);
  }
}

struct Layer {
  int heads = 0, kh = 0, f = 0;
  DevArray<float> ln1_g, ln1_b, ln2_g, ln2_b;
  GemmW qkv, o, in, out;
  CUtensorMap tm_z, tm_g;    // fp16 A operands with this layer's K extent
  CUtensorMap tm_z8, tm_g8;  // int8 A operands (W8A8)
  CUtensorMap tm_z8s, tm_g8s;  // the same in the sparse kernel's 112-row boxes
  CUtensorMap tm_zs, tm_gs;    // fp16 z / g in the sparse kernel's 112-row boxes (W_SP24F)
  CUtensorMap tm_g_out;        // g as the W_in GEMM's TMA store target (fp16 32 x 32 boxes)
  DevArray<h16> kv;  // paged pool [pages][K|V][heads][PAGE][hd]
  CUtensorMap tm_kv, tm_kvg;     // the pool as rows of hd (prefill / decode attention TMA boxes)
};

GemmW& weight_group(Layer& ly, int g) { return g == 0 ? ly.qkv : g == 1 ? ly.o : g == 2 ? ly.in : ly.out; }

// 2-SM 256x256 tiles once both M and N fill at least one pair tile. IOLM_GEMM_TILES=single|pair
// overrides (A/B measurements).
bool use_pair(int M, int N) {
  static const int mode = [] {
    const char* e = std::getenv("IOLM_GEMM_TILES");
    if (!e) return 0;
    return std::string(e) == "single" ? 1 : (std::string(e) == "pair" ? 2 : 0);
  }();
  if (mode == 1) return false;
  if (mode == 2) return true;
  return M >= 256 && N >= 256;
}

// Host-side description of one engine step.
struct Step {
  std::vector<int64_t> tok_src;  // >= 0: index into the id table; -1: slot's last generated token
  std::vector<int> tok_slot, tok_pos;
  std::vector<AttnGroup> pre, dec;
  std::vector<int> head_rows, head_slot;
  std::vector<int64_t> head_owner;  // caller row index per head row (host only)
  void clear() {
    tok_src.clear();
    tok_slot.clear();
    tok_pos.clear();
    pre.clear();
    dec.clear();
    head_rows.clear();
    head_slot.clear();
    head_owner.clear();
  }
  int T() const { return static_cast<int>(tok_src.size()); }
};

// Device + pinned-host buffers of one in-flight step (double-buffered by step parity).
struct StepBuffers {
  PinnedArray<uint8_t> h_meta;  // packed metadata staging
  DevArray<uint8_t> d_meta;
  DevArray<int32_t> d_next;
  PinnedArray<int32_t> h_next;
  cudaEvent_t done = nullptr;
  // device views into d_meta for the current step
  const int64_t* tok_src = nullptr;
  const int *tok_slot = nullptr, *tok_pos = nullptr, *head_rows = nullptr, *head_slot = nullptr;
  const int* head_iota = nullptr;  // 0 .. R-1: the head rows of the compacted last layer
  const AttnGroup *pre = nullptr, *dec = nullptr;
  Step step;
  ~StepBuffers() {
    if (done) cudaEventDestroy(done);
  }
};

// ------------------------------------------------ device-layout image I/O (iolm_cuda_save_image)
// File: "IOLMDL02" | u64 header words | int64 header words | per weight array: u64 bytes + bytes |
// u64 checksum. The checksum combines one ImageSum per section (header, each array). Version 02:
// 16-bit arrays hold fp16 (version 01 held bf16 and is rejected as a bad magic).
constexpr char kImageMagic[8] = {'I', 'O', 'L', 'M', 'D', 'L', '0', '2'};
constexpr size_t kImageChunk = 32ull << 20;  // pinned staging chunk (2 in flight)
constexpr uint64_t kSumPrime = 0x100000001B3ull;

// 4-lane multiplicative word hash: (h ^ w) * odd is a bijection of h, so any single corrupted word
// changes the result; 4 independent lanes run at memory speed. Restartable across chunks whose
// sizes are multiples of 32 bytes.
struct ImageSum {
  uint64_t h[4] = {0x9E3779B97F4A7C15ull, 0xC2B2AE3D27D4EB4Full, 0x165667B19E3779F9ull, 0x27D4EB2F165667C5ull};
  uint64_t n = 0;
  void add(const uint8_t* p, size_t len) {
    size_t i = 0;
    for (; i + 32 <= len; i += 32) {
      uint64_t w[4];
      std::memcpy(w, p + i, 32);
      for (int k = 0; k < 4; ++k) h[k] = (h[k] ^ w[k]) * kSumPrime;
    }
    for (; i < len; ++i) h[0] = (h[0] ^ p[i]) * kSumPrime;
    n += len;
  }
  uint64_t value() const {
    uint64_t r = n * 0x9E3779B97F4A7C15ull;
    for (int k = 0; k < 4; ++k) r = (r ^ h[k]) * kSumPrime;
    return r;
  }
  void combine(uint64_t section) { h[0] = (h[0] ^ section) * kSumPrime, ++n; }
};

struct ImageHeader {
  uint64_t hash = 0;
  ModelConfig cfg;
  int act_quant = 0, sparse_mma = 0, int4_mma = 0;
  std::vector<int> modes;  // 4 per layer: qkv, o, in, out
};

struct ImageFile {
  FILE* f = nullptr;
  ImageFile(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {
    if (!f) throw ContractViolation("device-layout image: cannot open " + path);
  }
  ~ImageFile() {
    if (f) std::fclose(f);
  }
  void read(void* p, size_t n) const {
    if (std::fread(p, 1, n, f) != n) throw TruncatedBlob("device-layout image: file ends early");
  }
  void write(const void* p, size_t n) const {
    if (std::fwrite(p, 1, n, f) != n) throw ContractViolation("device-layout image: write failed");
  }
};

ImageHeader read_image_header(const ImageFile& f, ImageSum& total) {
  char magic[8];
  f.read(magic, 8);
  if (std::memcmp(magic, kImageMagic, 8) != 0) throw CorruptHeader("device-layout image: bad magic");
  uint64_t nw = 0;
  f.read(&nw, 8);
  if (nw < 10 || nw > (1u << 24)) throw CorruptHeader("device-layout image: bad header length");
  std::vector<int64_t> w(nw);
  f.read(w.data(), nw * 8);
  ImageSum hs;
  hs.add(reinterpret_cast<const uint8_t*>(w.data()), nw * 8);
  total.combine(hs.value());
  size_t at = 0;
  auto next = [&]() -> int64_t {
    if (at >= w.size()) throw CorruptHeader("device-layout image: header too short");
    return w[at++];
  };
  auto next_int = [&](int64_t lo, int64_t hi) -> int {
    const int64_t v = next();
    if (v < lo || v > hi) throw CorruptHeader("device-layout image: header field out of range");
    return static_cast<int>(v);
  };
  ImageHeader h;
  h.hash = static_cast<uint64_t>(next());
  h.cfg.vocab_size = next_int(1, 1 << 20);
  h.cfg.d_model = next_int(1, 1 << 16);
  h.cfg.n_layers = next_int(1, 1 << 12);
  h.cfg.n_heads = next_int(1, 1 << 12);
  h.cfg.d_ff = next_int(1, 1 << 20);
  h.cfg.max_seq_len = next_int(1, 1 << 20);
  h.act_quant = next_int(0, 1);
  h.sparse_mma = next_int(0, 1);
  h.int4_mma = next_int(0, 1);
  for (int l = 0; l < h.cfg.n_layers; ++l) {
    std::vector<int> heads(next_int(1, h.cfg.n_heads));
    for (int& x : heads) x = next_int(0, h.cfg.n_heads - 1);
    h.cfg.active_heads.push_back(std::move(heads));
  }
  for (int l = 0; l < h.cfg.n_layers; ++l) h.cfg.active_ffn.push_back(next_int(1, h.cfg.d_ff));
  for (int i = 0; i < 4 * h.cfg.n_layers; ++i) h.modes.push_back(next_int(W_VALUES, W_INT4));
  if (at != w.size()) throw CorruptHeader("device-layout image: trailing header words");
  try {
    h.cfg.validate();
  } catch (const EngineError& e) {
    throw CorruptHeader(std::string("device-layout image: ") + e.what());
  }
  return h;
}

// Pinned double-buffered staging between the image file and HBM.
class ImageStager {
 public:
  ~ImageStager() {
    for (auto e : ev_)
      if (e) {
        cudaEventSynchronize(e);
        cudaEventDestroy(e);
      }
  }
  // file -> device: the read of chunk i+1 overlaps the H2D copy of chunk i
  void to_device(const ImageFile& f, void* dst, size_t n, cudaStream_t st, ImageSum& sum) {
    for (size_t off = 0; off < n; off += kImageChunk) {
      const size_t c = std::min(kImageChunk, n - off);
      uint8_t* b = slot();
      f.read(b, c);
      sum.add(b, c);
      CUDA_OK(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, b, c, cudaMemcpyHostToDevice, st));
      CUDA_OK(cudaEventRecord(ev_[k_], st));
      k_ ^= 1;
    }
  }
  void from_device(const ImageFile& f, const void* src, size_t n, cudaStream_t st, ImageSum& sum) {
    for (size_t off = 0; off < n; off += kImageChunk) {
      const size_t c = std::min(kImageChunk, n - off);
      uint8_t* b = slot();
      CUDA_OK(cudaMemcpyAsync(b, static_cast<const uint8_t*>(src) + off, c, cudaMemcpyDeviceToHost, st));
      CUDA_OK(cudaStreamSynchronize(st));
      sum.add(b, c);
      f.write(b, c);
    }
  }

 private:
  uint8_t* slot() {
    if (!ev_[k_]) {
      buf_[k_].ensure(kImageChunk);
      CUDA_OK(cudaEventCreateWithFlags(&ev_[k_], cudaEventDisableTiming));
    } else {
      CUDA_OK(cudaEventSynchronize(ev_[k_]));  // the copy that last used this buffer is done
    }
    return buf_[k_].p;
  }
  PinnedArray<uint8_t> buf_[2];
  cudaEvent_t ev_[2] = {nullptr, nullptr};
  int k_ = 0;
};

}  // namespace

class Engine {
 public:
  Engine(const uint8_t* bytes, size_t len, int device, const iolm_cuda_opts* opts);
  // From a device-layout image written by save_image (iolm_cuda_create_from_image).
  Engine(const std::string& image_path, uint64_t expected_hash, int device, const iolm_cuda_opts* opts);
  void save_image(const std::string& path);

  const ModelConfig& config() const { return cfg_; }
  uint64_t bundle_hash() const { return hash_; }
  const iolm_cuda_stats& stats() const { return stats_; }

  void decode(const int32_t* ids, bool ids_on_device, const int64_t* offsets, int64_t n_rows, int max_new,
              int32_t* out_ids, int32_t* out_len, uint64_t* madds, int64_t* bad_row);
  void forward(const int32_t* ids, const uint8_t* mask, int n, float* logits, uint64_t* madds,
               uint16_t* capture = nullptr, int8_t* codes = nullptr, float* code_scales = nullptr);

  std::mutex mu;
  void set_kernel_timing(bool on) { ktime_ = on; }
  double kms_[IOLM_KCLASSES] = {}, kwork_[IOLM_KCLASSES] = {};
  int64_t kcount_[IOLM_KCLASSES] = {};

 private:
  void reset_counters();
  void setup(int device, const iolm_cuda_opts* opts);
  void finish_setup();
  // [N x K] (row pitch ld elements) of weight group g (0 qkv, 1 o, 2 in, 3 out) of a layer
  void group_dims(const Layer& ly, int g, int& N, int& K, int& ld) const;
  template <typename F>
  void visit_weights(F&& f);
  void upload_weights(const BundleView& b);
  void alloc_runtime();
  void set_prefix_pages(int prefix_pages);
  void setup_l2_persistence();
  void add_prefill(Step& s, int slot, int64_t src_base, int p_begin, int p_end, bool want_head,
                   int64_t owner) const;
  void launch_step(StepBuffers& sb, const int32_t* d_ids, const uint8_t* d_key_mask, float* d_logits);
  void gemm(int epi, bool i8, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K, const GemmEpi& ep);
  // one projection: dense (A = activations, B = weights) or 2:4 sparse (weights are the MMA's A)
  void gemm_w(int epi, const GemmW& w, const CUtensorMap& act, const CUtensorMap& act_sp, int M, int N, int K,
              const GemmEpi& ep, const CUtensorMap* out_map = nullptr);
  void load_gemm_weights(const BundleView& b, GemmW& w, const std::vector<std::string>& names, int K, int ld);
  uint64_t ref_madds_row(int s0, int advances) const;
  template <typename F>
  void timed(int cat, double work, F&& f);
  void collect_times(int64_t upto_step);

  ModelConfig cfg_;
  uint64_t hash_ = 0;
  int device_ = 0, sms_ = 148;
  int d_ = 0, L_ = 0, V_ = 0, S_ = 0, hd_ = 0, kh_max_ = 0, f_ld_max_ = 0;
  int T_max_ = 0, max_slots_ = 0, pps_ = 0, prefix_slot_ = 0;
  int cur_prefix_pages_ = -1;
  bool auto_budget_ = false;
  bool prefix_sharing_ = true;
  bool act_quant_ = false;
  bool sparse_mma_ = true;
  bool int4_mma_ = true;
  bool prefill_tc_ = true;  // 128-query tcgen05 prefill kernel (hd 128: masked forward; forced by prefill_tc = 1)
  bool prefill_tc_force_ = false;
  bool prefill_hp_ = true;  // hd 64 / 128: attn_tc.cu attn_prefill_hp_kernel (head-pair / one-head tiles)
  // TMA-store epilogue of the W_in GEMM (IOLM_GEMM_TMA_EPI=0 disables, for A/B measurements):
  // measured 3% faster than the warp's coalesced stores at the C1 shape
  bool tma_epi_ = std::getenv("IOLM_GEMM_TMA_EPI") == nullptr || std::string(std::getenv("IOLM_GEMM_TMA_EPI")) != "0";
  uint64_t madds_A_ = 0, madds_B_ = 0;  // sum_l (4*d*kh + 2*d*f), sum_l kh
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  iolm_cuda_stats stats_{};
  int64_t step_seq_ = 0;  // steps launched on this engine (kernel-timing bookkeeping)

  // kernel-class timing (opts.kernel_timing)
  bool ktime_ = false;
  std::vector<cudaEvent_t> kev_;
  // Destroys the raw stream / event handles above, also when a constructor throws after creating
  // them (members are unwound then, the destructor body is not run).
  struct HandleGuard {
    Engine* e;
    ~HandleGuard() {
      for (auto ev : e->kev_) cudaEventDestroy(ev);
      if (e->stream_) cudaStreamDestroy(e->stream_);
      if (e->ev0_) cudaEventDestroy(e->ev0_);
      if (e->ev1_) cudaEventDestroy(e->ev1_);
    }
  } handle_guard_{this};
  std::vector<int> kev_free_;
  struct KPending {
    int cat, ev0, ev1;
    double work;
    int64_t step;
  };
  std::vector<KPending> kpend_;

  std::vector<int> iota_;  // host 0, 1, 2, ... (head_iota staging)
  std::vector<std::unique_ptr<Layer>> layers_;
  DevArray<float> tok_embed_, tok_embed_t_, pos_embed_, lnf_g_, lnf_b_;
  DevArray<float> x_;
  DevArray<h16> h_, q_, z_, g_;
  CUtensorMap tm_h_, tm_q_;
  DevArray<int8_t> h8_, z8_, g8_;  // W8A8 operands + per-token scales
  DevArray<float> hs_, zs_, gs_;
  CUtensorMap tm_h8_, tm_h8s_;
  CUtensorMap tm_hs_;  // fp16 h in the sparse kernel's 112-row boxes (W_SP24F)
  CUtensorMap tm_x_resid_;  // x as the 2:4 GEMM's TMA reduce-add target (32 x 8 boxes)
  // Last-layer head-row compaction: after the last layer's QKV GEMM (which still writes K/V for every
  // token) and attention, only the tokens whose logits are read (the step's head rows) go through
  // Wo / LN2 / W_in / W_out: their x and z rows are gathered into xc_ / zc_ (rows 0 .. R-1) and the
  // head reads xc_. Every op after the gather is row-wise, so outputs are bitwise those of the
  // uncompacted path. Off for forward() (all positions' logits) and the calibration capture, and
  // with IOLM_LAST_COMPACT=0 (A/B measurements).
  bool last_compact_ = std::getenv("IOLM_LAST_COMPACT") == nullptr || std::string(std::getenv("IOLM_LAST_COMPACT")) != "0";
  DevArray<float> xc_;
  DevArray<h16> zc_;
  CUtensorMap tm_zc_, tm_zcs_, tm_xc_resid_;
  // dense residual GEMMs: x += acc through TMA reduce-add (32 x 32 fp32 boxes, fp32 RN add in L2:
  // bitwise equal) instead of the warps' coalesced read-modify-write: C2-W8A8 Wo 182 -> 148 ms,
  // C1 +0.6% (profiles/r02_experiments.md). IOLM_RESID_TMA=0 restores the RMW (A/B). Not for the
  // W4A16 kernel: with it the C2-W4A16 bench's two passes over the same rows disagreed (unexplained,
  // so the converter-warp kernel keeps the RMW epilogue).
  bool resid_tma_ = std::getenv("IOLM_RESID_TMA") == nullptr || std::string(std::getenv("IOLM_RESID_TMA")) != "0";
  CUtensorMap tm_x_out_, tm_xc_out_;
  bool any_int8_ = false;
  DevArray<int> page_table_;
  StepBuffers sbuf_[2];
  DevArray<int32_t> d_last_tok_, d_ids_;
  DevArray<int64_t> d_offsets_;
  DevArray<int> d_scalar_;
  DevArray<float> d_logits_;
  DevArray<uint8_t> d_mask_;
  // calibration capture (forward with a CaptureSink, runtime.hpp:22-28): per layer the four linear
  // inputs [attn_in n x d][attn_out_in n x kh][ffn_in n x d][ffn_mid n x f] as fp16, back to back
  DevArray<h16> d_cap_;
  h16* cap_ = nullptr;  // non-null while a capturing forward is being launched
  size_t cap_off_ = 0;
  // W8A8 capture (iolm_cuda_forward_codes): the int8 operand codes of the same four points and their
  // per-token scales [4 x n] per layer
  DevArray<int8_t> d_cap8_;
  DevArray<float> d_capsc_;
  int8_t* cap8_ = nullptr;
  float* capsc_ = nullptr;
  size_t capsc_off_ = 0;
  // point: 0 attn_in (LN1 out), 1 attn_out_in (attention out), 2 ffn_in (LN2 out), 3 ffn_mid (GELU out)
  void capture_point(int point, int T, int cols);
};

Engine::Engine(const uint8_t* bytes, size_t len, int device, const iolm_cuda_opts* opts) {
  if (!bytes || len == 0) throw ContractViolation("iolm_cuda_create: empty bundle");
  BundleView b = parse_bundle(bytes, len);
  cfg_ = b.config;
  setup(device, opts);
  // The FNV-1a hash of the serialized bundle is inherently sequential; overlap it with the upload.
  std::thread hasher([&] { hash_ = fnv1a64(bytes, len); });
  try {
    upload_weights(b);
    finish_setup();
  } catch (...) {
    hasher.join();
    throw;
  }
  hasher.join();
}

// Everything that depends on the model config and the options only (shared by the bundle and the
// device-layout image constructors).
void Engine::setup(int device, const iolm_cuda_opts* opts) {
  d_ = cfg_.d_model;
  L_ = cfg_.n_layers;
  V_ = cfg_.vocab_size;
  S_ = cfg_.max_seq_len;
  hd_ = cfg_.head_dim();
  if (V_ != IOLM_VOCAB) throw Unsupported("vocab_size must be 131 (tokenizer.hpp:17)");
  if (d_ % 8 != 0) throw Unsupported("d_model must be a multiple of 8 for the GPU layout");
  if (hd_ != 16 && hd_ != 32 && hd_ != 64 && hd_ != 128)
    throw Unsupported("head_dim must be 16, 32, 64 or 128 on the GPU path");

  if (d_ > 4096) throw Unsupported("d_model > 4096");
  device_ = device;
  CUDA_OK(cudaSetDevice(device_));
  CUDA_OK(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device_));
  CUDA_OK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  CUDA_OK(cudaEventCreate(&ev0_));
  CUDA_OK(cudaEventCreate(&ev1_));
  if (opts) {
    if (opts->max_tokens_per_step > 0) T_max_ = opts->max_tokens_per_step;
    if (opts->max_slots > 0) max_slots_ = opts->max_slots;
    if (opts->page_size != 0 && opts->page_size != PAGE) throw Unsupported("page_size must be 16");
    act_quant_ = opts->act_quant != 0;
    if (opts->prefix_sharing < 0) prefix_sharing_ = false;
    ktime_ = opts->kernel_timing != 0;
    if (opts->sparse_mma < 0) sparse_mma_ = false;
    if (opts->int4_mma < 0) int4_mma_ = false;
    if (opts->prefill_tc < 0) prefill_tc_ = prefill_hp_ = false;
    prefill_tc_force_ = opts->prefill_tc > 0;
  }
  // default: attn_prefill_hp_kernel (hd 64: 64-query chunks as head-pair tiles; hd 128: 128-query
  // chunks); prefill_tc = 1 selects the round-1 128-query tcgen05 kernel, -1 the mma.sync kernel
  prefill_hp_ = prefill_hp_ && (hd_ == 64 || hd_ == 128) && !prefill_tc_force_;
  // the round-1 128-query kernel (attn_prefill_tc_kernel): when forced (hd 64 / 128), and for hd 128
  // forward() calls with a key mask (the head-pair kernel has no masked variant; both use 128-query
  // chunks at hd 128, so the chunking never depends on the mask)
  prefill_tc_ = prefill_tc_ && (hd_ == 128 || (hd_ == 64 && prefill_tc_force_));
  // Default token budget: one 256-row GEMM M-tile per SM pair (74 x 256 = 18944 on a 148-SM B200),
  // so every projection's tile count is a whole number of waves of the persistent GEMM grid.
  auto_budget_ = T_max_ <= 0;
  if (auto_budget_) T_max_ = std::max(1, sms_ / 2) * 256;
  T_max_ = std::max(round_up(T_max_, 128), round_up(S_, 128));
  for (int l = 0; l < L_; ++l) {
    const uint64_t kh = static_cast<uint64_t>(cfg_.layer_heads(l)) * hd_;
    madds_A_ += 4ull * d_ * kh + 2ull * d_ * cfg_.layer_ffn(l);
    madds_B_ += kh;
  }
}

void Engine::finish_setup() {
  // All projections on the 2:4 sparse kernel (224-token pair tiles): whole waves of that grid.
  bool all_sp = true;
  for (const auto& ly : layers_)
    for (int g = 0; g < 4; ++g) {
      const int m = weight_group(*ly, g).mode;
      all_sp = all_sp && (m == W_SP24 || m == W_SP24F);
    }
  if (auto_budget_ && all_sp) T_max_ = std::max(std::max(1, sms_ / 2) * 224, round_up(S_, 32));
  alloc_runtime();
}

void Engine::group_dims(const Layer& ly, int g, int& N, int& K, int& ld) const {
  switch (g) {
    case 0: N = 3 * ly.kh, K = d_, ld = d_; break;          // wq | wk | wv  [3 kh x d]
    case 1: N = d_, K = ly.kh, ld = ly.kh; break;           // wo            [d x kh]
    case 2: N = ly.f, K = d_, ld = d_; break;               // w_in          [f x d]
    default: N = d_, K = ly.f, ld = round_up(ly.f, 16);     // w_out         [d x f]
  }
}

// Every resident weight array, in image order, with the element count its weight form implies
// (derived from config + form, so the image loader validates sizes before allocating).
template <typename F>
void Engine::visit_weights(F&& f) {
  const size_t d = static_cast<size_t>(d_);
  f(tok_embed_, static_cast<size_t>(V_) * d);
  f(pos_embed_, static_cast<size_t>(S_) * d);
  f(lnf_g_, d);
  f(lnf_b_, d);
  for (auto& ly : layers_) {
    f(ly->ln1_g, d);
    f(ly->ln1_b, d);
    f(ly->ln2_g, d);
    f(ly->ln2_b, d);
    for (int g = 0; g < 4; ++g) {
      GemmW& w = weight_group(*ly, g);
      int N, K, ld;
      group_dims(*ly, g, N, K, ld);
      const size_t nl = static_cast<size_t>(N) * ld;
      switch (w.mode) {
        case W_VALUES: f(w.wb, nl); break;
        case W_CODES: f(w.wb, nl), f(w.scale, static_cast<size_t>(N)); break;
        case W_INT8: f(w.w8, nl), f(w.scale, static_cast<size_t>(N)); break;
        case W_SP24:
          f(w.w8, w.sl.code_bytes()), f(w.meta, w.sl.meta_bytes()), f(w.scale, static_cast<size_t>(N));
          break;
        case W_SP24F:
          f(w.wb, w.sl.code_bytes() / 2), f(w.meta, w.sl.meta_bytes()), f(w.scale, static_cast<size_t>(N));
          break;
        case W_INT4: f(w.w4, static_cast<size_t>(N) * w4_pitch(K)), f(w.scale, static_cast<size_t>(N)); break;
      }
    }
  }
}

void Engine::save_image(const std::string& path) {
  CUDA_OK(cudaSetDevice(device_));
  CUDA_OK(cudaStreamSynchronize(stream_));
  std::vector<int64_t> hw = {static_cast<int64_t>(hash_), cfg_.vocab_size, cfg_.d_model, cfg_.n_layers,
                             cfg_.n_heads, cfg_.d_ff, cfg_.max_seq_len, act_quant_, sparse_mma_, int4_mma_};
  for (const auto& heads : cfg_.active_heads) {
    hw.push_back(static_cast<int64_t>(heads.size()));
    hw.insert(hw.end(), heads.begin(), heads.end());
  }
  hw.insert(hw.end(), cfg_.active_ffn.begin(), cfg_.active_ffn.end());
  for (auto& ly : layers_)
    for (int g = 0; g < 4; ++g) hw.push_back(weight_group(*ly, g).mode);
  const std::string tmp = path + ".tmp";
  try {
    ImageFile f(tmp, "wb");
    ImageSum total, hs;
    f.write(kImageMagic, 8);
    const uint64_t nw = hw.size();
    f.write(&nw, 8);
    f.write(hw.data(), nw * 8);
    hs.add(reinterpret_cast<const uint8_t*>(hw.data()), nw * 8);
    total.combine(hs.value());
    ImageStager stager;
    visit_weights([&](auto& arr, size_t count) {
      using T = std::remove_pointer_t<decltype(arr.p)>;
      if (arr.n != count) throw ContractViolation("save_image: internal size mismatch");
      const uint64_t nb = count * sizeof(T);
      f.write(&nb, 8);
      ImageSum s;
      stager.from_device(f, arr.p, nb, stream_, s);
      total.combine(s.value());
    });
    const uint64_t sum = total.value();
    f.write(&sum, 8);
    if (std::fflush(f.f) != 0) throw ContractViolation("save_image: write failed");
  } catch (...) {
    std::remove(tmp.c_str());
    throw;
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    throw ContractViolation("save_image: cannot rename " + tmp + " to " + path);
  }
}

Engine::Engine(const std::string& image_path, uint64_t expected_hash, int device, const iolm_cuda_opts* opts) {
  ImageFile f(image_path, "rb");
  ImageSum total;
  const ImageHeader h = read_image_header(f, total);
  if (expected_hash != 0 && h.hash != expected_hash)
    throw StaleImage("device-layout image was built from another bundle (hash mismatch)");
  cfg_ = h.cfg;
  setup(device, opts);
  if (act_quant_ != (h.act_quant != 0) || sparse_mma_ != (h.sparse_mma != 0) || int4_mma_ != (h.int4_mma != 0))
    throw StaleImage("device-layout image was built with other weight options (act_quant/sparse_mma/int4_mma)");
  hash_ = h.hash;
  for (int l = 0; l < L_; ++l) {
    auto ly = std::make_unique<Layer>();
    ly->heads = cfg_.layer_heads(l);
    ly->kh = ly->heads * hd_;
    ly->f = cfg_.layer_ffn(l);
    for (int g = 0; g < 4; ++g) {
      GemmW& w = weight_group(*ly, g);
      w.mode = h.modes[4 * l + g];
      // the forms the bundle loader can produce under these options
      const bool ok = act_quant_ ? (w.mode == W_INT8 || (w.mode == W_SP24 && sparse_mma_))
                                 : (w.mode == W_VALUES || w.mode == W_CODES || (w.mode == W_INT4 && int4_mma_) ||
                                    (w.mode == W_SP24F && sparse_mma_));
      if (!ok) throw CorruptHeader("device-layout image: weight form inconsistent with its options");
      int N, K, ld;
      group_dims(*ly, g, N, K, ld);
      if (w.mode == W_SP24 || w.mode == W_SP24F) {
        if (K % 4 != 0) throw CorruptHeader("device-layout image: 2:4 form needs K % 4 == 0");
        w.sl = sp24_layout(N, K, w.mode == W_SP24F);
      }
    }
    any_int8_ = any_int8_ || ly->qkv.int8() || ly->o.int8() || ly->in.int8() || ly->out.int8();
    kh_max_ = std::max(kh_max_, ly->kh);
    f_ld_max_ = std::max(f_ld_max_, round_up(ly->f, 16));
    layers_.push_back(std::move(ly));
  }
  {
    ImageStager stager;
    visit_weights([&](auto& arr, size_t count) {
      using T = std::remove_pointer_t<decltype(arr.p)>;
      uint64_t nb = 0;
      f.read(&nb, 8);
      if (nb != count * sizeof(T)) throw CorruptHeader("device-layout image: array size does not match the config");
      arr.alloc(count);
      ImageSum s;
      stager.to_device(f, arr.p, nb, stream_, s);
      total.combine(s.value());
    });
    CUDA_OK(cudaStreamSynchronize(stream_));
  }
  uint64_t sum = 0;
  f.read(&sum, 8);
  if (sum != total.value()) throw CorruptHeader("device-layout image: checksum mismatch");
  if (std::fgetc(f.f) != EOF) throw CorruptHeader("device-layout image: trailing bytes");
  tok_embed_t_.alloc(static_cast<size_t>(V_) * d_);
  launch_transpose(tok_embed_.p, V_, d_, tok_embed_t_.p, stream_);
  for (auto& ly : layers_)
    for (int g = 0; g < 4; ++g) {
      int N, K, ld;
      group_dims(*ly, g, N, K, ld);
      weight_maps(weight_group(*ly, g), N, K, ld);
    }
  CUDA_OK(cudaStreamSynchronize(stream_));
  finish_setup();
}

void Engine::upload_weights(const BundleView& b) {
  auto upload_f32 = [&](const std::string& name, DevArray<float>& dst) {
    const auto& t = b.tensor(name);
    dst.alloc(static_cast<size_t>(t.rows) * t.cols);
    CUDA_OK(cudaMemcpy(dst.p, b.payload(t), t.length, cudaMemcpyHostToDevice));
  };
  upload_f32("tok_embed", tok_embed_);
  upload_f32("pos_embed", pos_embed_);
  upload_f32("final_norm.gain", lnf_g_);
  upload_f32("final_norm.bias", lnf_b_);
  tok_embed_t_.alloc(static_cast<size_t>(V_) * d_);
  launch_transpose(tok_embed_.p, V_, d_, tok_embed_t_.p, stream_);

  for (int l = 0; l < L_; ++l) {
    auto ly = std::make_unique<Layer>();
    const std::string p = "layers." + std::to_string(l) + ".";
    ly->heads = cfg_.layer_heads(l);
    ly->kh = ly->heads * hd_;
    ly->f = cfg_.layer_ffn(l);
    upload_f32(p + "attn_norm.gain", ly->ln1_g);
    upload_f32(p + "attn_norm.bias", ly->ln1_b);
    upload_f32(p + "ffn_norm.gain", ly->ln2_g);
    upload_f32(p + "ffn_norm.bias", ly->ln2_b);
    const int kh = ly->kh, f = ly->f, f_ld = round_up(f, 16);
    load_gemm_weights(b, ly->qkv, {p + "attn.wq", p + "attn.wk", p + "attn.wv"}, d_, d_);
    load_gemm_weights(b, ly->o, {p + "attn.wo"}, kh, kh);
    load_gemm_weights(b, ly->in, {p + "ffn.w_in"}, d_, d_);
    load_gemm_weights(b, ly->out, {p + "ffn.w_out"}, f, f_ld);
    any_int8_ = any_int8_ || ly->qkv.int8() || ly->o.int8() || ly->in.int8() || ly->out.int8();
    kh_max_ = std::max(kh_max_, kh);
    f_ld_max_ = std::max(f_ld_max_, f_ld);
    layers_.push_back(std::move(ly));
  }
  CUDA_OK(cudaStreamSynchronize(stream_));
}

// L2 residency of the fp32 residual stream x (T x d): every layer reads it in two LayerNorms and
// read-modify-writes it in two residual GEMM epilogues, so keeping it in the 126 MB L2 turns those
// passes from HBM- into L2-bandwidth work. An access-policy window on the engine stream marks x's
// lines persisting (hitRatio = the persisting set-aside / window when x does not fit).
// IOLM_L2_PERSIST=<MB of set-aside> (0: off) - A/B switch, see DESIGN.md.
void Engine::setup_l2_persistence() {
  const char* e = std::getenv("IOLM_L2_PERSIST");
  if (!e) return;
  const double mb = std::atof(e);
  if (mb <= 0) return;
  int maxp = 0, maxw = 0;
  CUDA_OK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device_));
  CUDA_OK(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, device_));
  const size_t xb = static_cast<size_t>(T_max_) * d_ * sizeof(float);
  const size_t win = std::min<size_t>(xb, static_cast<size_t>(maxw));
  const size_t persist = std::min<size_t>(static_cast<size_t>(mb * 1048576.0), static_cast<size_t>(maxp));
  CUDA_OK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist));
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.base_ptr = x_.p;
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = static_cast<float>(std::min(1.0, static_cast<double>(persist) / win));
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  CUDA_OK(cudaStreamSetAttribute(stream_, cudaStreamAttributeAccessPolicyWindow, &v));
  if (std::getenv("IOLM_L2_VERBOSE"))
    std::fprintf(stderr, "L2 persist: max set-aside %d B, max window %d B, x %zu B, window %zu, set-aside %zu, hit %.3f\n",
                 maxp, maxw, xb, win, persist, v.accessPolicyWindow.hitRatio);
}

// Decodes the tensors of one GEMM (stacked along N, e.g. wq|wk|wv) into the chosen weight form.
void Engine::load_gemm_weights(const BundleView& b, GemmW& w, const std::vector<std::string>& names, int K,
                               int ld) {
  std::vector<const TensorRecord*> ts;
  int N = 0;
  bool all_dense = true, all_quant = true, int8_ok = true, sp_ok = sparse_mma_;
  bool q4_ok = !act_quant_ && int4_mma_;
  for (const auto& n : names) {
    ts.push_back(&b.tensor(n));
    N += ts.back()->rows;
    all_dense = all_dense && ts.back()->encoding == ENC_DENSE_F32;
    all_quant = all_quant && ts.back()->encoding != ENC_DENSE_F32;
    int8_ok = int8_ok && (ts.back()->encoding == ENC_Q8 || ts.back()->encoding == ENC_SPARSE24_Q8);
    q4_ok = q4_ok && ts.back()->encoding == ENC_Q4;
    sp_ok = sp_ok && ts.back()->encoding == ENC_SPARSE24_Q8 &&
            sp24_check(b.payload(*ts.back()), ts.back()->rows, ts.back()->cols);
  }
  w.mode = all_quant ? (act_quant_ && int8_ok ? W_INT8 : W_CODES) : W_VALUES;
  if ((w.mode == W_INT8 || w.mode == W_CODES) && sp_ok) {
    // 2:4 sparse tensor cores: the bundle's kept codes and position nibbles are repacked on the host;
    // W8A8 keeps the codes as int8 (kind::i8), fp16 activations take them as exact fp16 (kind::f16)
    const bool f16 = w.mode == W_CODES;
    w.mode = f16 ? W_SP24F : W_SP24;
    w.sl = sp24_layout(N, K, f16);
    std::vector<uint8_t> codes(w.sl.code_bytes(), 0);
    std::vector<uint8_t> meta(w.sl.meta_bytes(), 0x44);
    std::vector<float> scales(N);
    int row0 = 0;
    for (auto* t : ts) {
      sp24_append(w.sl, b.payload(*t), t->rows, t->cols, row0, codes.data(), meta.data(), scales.data());
      row0 += t->rows;
    }
    sp24_finalize(w.sl, meta.data());
    if (f16) w.wb.alloc(codes.size() / 2);
    else w.w8.alloc(codes.size());
    w.meta.alloc(meta.size());
    w.scale.alloc(N);
    CUDA_OK(cudaMemcpy(f16 ? static_cast<void*>(w.wb.p) : static_cast<void*>(w.w8.p), codes.data(), codes.size(),
                       cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(w.meta.p, meta.data(), meta.size(), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(w.scale.p, scales.data(), sizeof(float) * N, cudaMemcpyHostToDevice));
    weight_maps(w, N, K, ld);
    return;
  }
  if (w.mode == W_CODES && q4_ok) {
    // W4A16: the bundle's nibble rows (ceil(K/2) bytes, low nibble = even column) re-pitched to 16 B
    w.mode = W_INT4;
    const size_t rb = static_cast<size_t>(K + 1) / 2, ld4 = w4_pitch(K);
    w.w4.alloc(static_cast<size_t>(N) * ld4);
    w.scale.alloc(N);
    CUDA_OK(cudaMemset(w.w4.p, 0x88, static_cast<size_t>(N) * ld4));  // pad bytes: codes 0
    int row0 = 0;
    for (auto* t : ts) {
      const uint8_t* pl = b.payload(*t);
      CUDA_OK(cudaMemcpy2D(w.w4.p + static_cast<size_t>(row0) * ld4, ld4, pl, rb, rb, t->rows, cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(w.scale.p + row0, pl + static_cast<size_t>(t->rows) * rb, sizeof(float) * t->rows,
                         cudaMemcpyHostToDevice));
      row0 += t->rows;
    }
    weight_maps(w, N, K, ld);
    return;
  }
  if (act_quant_ && w.mode != W_INT8)
    throw Unsupported("act_quant (W8A8) needs q8 or sparse24_q8 encodings for every linear weight; " + names[0] +
                      " is " + (all_dense ? "dense_f32" : "q4 or mixed"));
  size_t max_payload = 0;
  for (auto* t : ts) max_payload = std::max<size_t>(max_payload, t->length);
  DevArray<uint8_t> scratch;
  scratch.alloc(max_payload + 16);
  if (w.mode == W_INT8) w.w8.alloc(static_cast<size_t>(N) * ld);
  else w.wb.alloc(static_cast<size_t>(N) * ld);
  if (w.mode != W_VALUES) w.scale.alloc(N);
  int row0 = 0;
  for (auto* t : ts) {
    CUDA_OK(cudaMemcpyAsync(scratch.p, b.payload(*t), t->length, cudaMemcpyHostToDevice, stream_));
    const size_t off = static_cast<size_t>(row0) * ld;
    if (w.mode == W_VALUES)
      launch_decode_weight(scratch.p, t->encoding, t->rows, t->cols, w.wb.p + off, ld, stream_);
    else if (w.mode == W_CODES)
      launch_decode_codes(scratch.p, t->encoding, t->rows, t->cols, w.wb.p + off, false, ld, w.scale.p + row0,
                          stream_);
    else
      launch_decode_codes(scratch.p, t->encoding, t->rows, t->cols, w.w8.p + off, true, ld, w.scale.p + row0,
                          stream_);
    CUDA_OK(cudaStreamSynchronize(stream_));  // scratch is reused by the next tensor
    row0 += t->rows;
  }
  weight_maps(w, N, K, ld);
}

void Engine::alloc_runtime() {
  const size_t T = T_max_;
  x_.alloc(T * d_);
  setup_l2_persistence();
  h_.alloc(T * d_);
  q_.alloc(T * kh_max_);
  z_.alloc(T * kh_max_);
  g_.alloc(T * f_ld_max_);
  CUDA_OK(cudaMemset(z_.p, 0, T * kh_max_ * sizeof(h16)));
  if (last_compact_ && L_ > 0) {
    xc_.alloc(T * d_);
    zc_.alloc(T * kh_max_);
    CUDA_OK(cudaMemset(zc_.p, 0, T * kh_max_ * sizeof(h16)));
  }
  const auto BF = H16_TMA;
  tm_h_ = make_kmajor_map(h_.p, BF, 2, d_, T, 2ull * d_, 128);
  tm_q_ = make_rows_map_h16(q_.p, kh_max_, T, 2ull * kh_max_, std::min(hd_, 64), 64);
  for (auto& ly : layers_) {
    ly->tm_z = make_kmajor_map(z_.p, BF, 2, ly->kh, T, 2ull * kh_max_, 128);
    ly->tm_g = make_kmajor_map(g_.p, BF, 2, ly->f, T, 2ull * f_ld_max_, 128);
    ly->tm_g_out = make_out_map(g_.p, false, ly->f, T, 2ull * f_ld_max_);
    ly->tm_zs = sp24_act_map_h16(z_.p, ly->kh, static_cast<int>(T), kh_max_);
    ly->tm_gs = sp24_act_map_h16(g_.p, ly->f, static_cast<int>(T), f_ld_max_);
  }
  tm_hs_ = sp24_act_map_h16(h_.p, d_, static_cast<int>(T), d_);
  tm_x_resid_ = make_resid_map(x_.p, d_, T, 4ull * d_);
  if (resid_tma_) tm_x_out_ = make_out_map(x_.p, true, d_, T, 4ull * d_);
  if (last_compact_ && L_ > 0) {
    const int khl = layers_.back()->kh;
    tm_zc_ = make_kmajor_map(zc_.p, BF, 2, khl, T, 2ull * kh_max_, 128);
    tm_zcs_ = sp24_act_map_h16(zc_.p, khl, static_cast<int>(T), kh_max_);
    tm_xc_resid_ = make_resid_map(xc_.p, d_, T, 4ull * d_);
    if (resid_tma_) tm_xc_out_ = make_out_map(xc_.p, true, d_, T, 4ull * d_);
  }
  if (any_int8_) {
    const auto U8 = CU_TENSOR_MAP_DATA_TYPE_UINT8;
    h8_.alloc(T * d_);
    z8_.alloc(T * kh_max_);
    g8_.alloc(T * f_ld_max_);
    hs_.alloc(T);
    zs_.alloc(T);
    gs_.alloc(T);
    tm_h8_ = make_kmajor_map(h8_.p, U8, 1, d_, T, static_cast<uint64_t>(d_), 128);
    tm_h8s_ = sp24_act_map(h8_.p, d_, static_cast<int>(T), d_);
    for (auto& ly : layers_) {
      ly->tm_z8 = make_kmajor_map(z8_.p, U8, 1, ly->kh, T, static_cast<uint64_t>(kh_max_), 128);
      ly->tm_g8 = make_kmajor_map(g8_.p, U8, 1, ly->f, T, static_cast<uint64_t>(f_ld_max_), 128);
      ly->tm_z8s = sp24_act_map(z8_.p, ly->kh, static_cast<int>(T), kh_max_);
      ly->tm_g8s = sp24_act_map(g8_.p, ly->f, static_cast<int>(T), f_ld_max_);
    }
  }
  // packed step metadata: tok_src i64[T], tok_slot/pos i32[T], groups 2 x [T], head rows/slots i32[T]
  const size_t meta_bytes = align16(T * 8) + 2 * align16(T * 4) + 2 * align16(T * sizeof(AttnGroup)) +
                            3 * align16(T * 4) + 64;
  for (auto& sb : sbuf_) {
    sb.h_meta.ensure(meta_bytes);
    sb.d_meta.alloc(meta_bytes);
    sb.d_next.alloc(T);
    sb.h_next.ensure(T);
    CUDA_OK(cudaEventCreateWithFlags(&sb.done, cudaEventDisableTiming));
  }
  d_logits_.alloc(T * V_);
  d_mask_.alloc(S_);
  d_scalar_.alloc(4);

  // Paged KV pool: one fixed run of pps_ pages per slot plus one prefix slot.
  pps_ = (S_ + PAGE - 1) / PAGE;
  size_t bytes_per_slot = 0;
  for (auto& ly : layers_) bytes_per_slot += static_cast<size_t>(pps_) * 2 * ly->heads * PAGE * hd_ * 2;
  size_t free_b = 0, total_b = 0;
  CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
  const size_t cap = static_cast<size_t>(0.7 * static_cast<double>(free_b)) / std::max<size_t>(bytes_per_slot, 1);
  if (max_slots_ <= 0) max_slots_ = 2560;
  max_slots_ = static_cast<int>(std::min<size_t>(max_slots_, cap > 1 ? cap - 1 : 0));
  if (max_slots_ < 1) throw OutOfMemory("KV pool: not enough device memory for one sequence");
  prefix_slot_ = max_slots_;
  const size_t pages = static_cast<size_t>(max_slots_ + 1) * pps_;
  for (auto& ly : layers_) {
    const size_t elems = pages * 2 * ly->heads * PAGE * hd_;
    ly->kv.alloc(elems);
    CUDA_OK(cudaMemset(ly->kv.p, 0, elems * sizeof(h16)));
    ly->tm_kv = make_rows_map_h16(ly->kv.p, hd_, pages * 2 * ly->heads * PAGE, 2ull * hd_,
                                   std::min(hd_, 64), PAGE);
    ly->tm_kvg = make_rows_map_h16(ly->kv.p, hd_, pages * 2 * ly->heads * PAGE, 2ull * hd_, std::min(hd_, 64),
                                    decode_heads_per_cta(ly->heads, hd_) * PAGE);
  }
  page_table_.alloc(static_cast<size_t>(max_slots_ + 1) * pps_);
  d_last_tok_.alloc(max_slots_ + 1);
  CUDA_OK(cudaMemset(d_last_tok_.p, 0, (max_slots_ + 1) * sizeof(int32_t)));
}

// Page table: slot s owns pages [s*pps, (s+1)*pps); positions below the shared prefix map to the
// prefix slot's pages instead.
void Engine::set_prefix_pages(int prefix_pages) {
  if (prefix_pages == cur_prefix_pages_) return;
  std::vector<int> pt(static_cast<size_t>(max_slots_ + 1) * pps_);
  for (int s = 0; s <= max_slots_; ++s)
    for (int i = 0; i < pps_; ++i)
      pt[static_cast<size_t>(s) * pps_ + i] =
          (s != prefix_slot_ && i < prefix_pages) ? prefix_slot_ * pps_ + i : s * pps_ + i;
  CUDA_OK(cudaMemcpyAsync(page_table_.p, pt.data(), pt.size() * sizeof(int), cudaMemcpyHostToDevice, stream_));
  CUDA_OK(cudaStreamSynchronize(stream_));
  cur_prefix_pages_ = prefix_pages;
}

void Engine::add_prefill(Step& s, int slot, int64_t src_base, int p_begin, int p_end, bool want_head,
                         int64_t owner) const {
  const int m0 = s.T();
  for (int p = p_begin; p < p_end; ++p) {
    s.tok_src.push_back(src_base + p);
    s.tok_slot.push_back(slot);
    s.tok_pos.push_back(p);
  }
  const int qc = prefill_tc_ ? 2 * QCHUNK : QCHUNK;  // tcgen05 kernel: 128-query tiles
  for (int c = p_begin; c < p_end; c += qc)
    s.pre.push_back(AttnGroup{slot, m0 + (c - p_begin), std::min(qc, p_end - c), c});
  if (want_head) {
    s.head_rows.push_back(m0 + (p_end - p_begin) - 1);
    s.head_slot.push_back(slot);
    s.head_owner.push_back(owner);
  }
}

void Engine::gemm(int epi, bool i8, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                  const GemmEpi& ep) {
  launch_gemm(use_pair(M, N), i8, epi, A, B, M, N, K, ep, stream_, sms_);
  ++stats_.kernel_launches;
}

void Engine::gemm_w(int epi, const GemmW& w, const CUtensorMap& act, const CUtensorMap& act_sp, int M, int N, int K,
                    const GemmEpi& ep, const CUtensorMap* out_map) {
  if (w.mode == W_SP24 || w.mode == W_SP24F) {
    launch_gemm_sp(epi, w.tm, act_sp, w.tm_e, K, w.sl.katoms_pad, ep, stream_, sms_, w.mode == W_SP24F,
                   epi != iolmk::EPI_RESID_F32 ? nullptr
                   : ep.out == x_.p     ? &tm_x_resid_
                   : ep.out == xc_.p    ? &tm_xc_resid_
                                        : nullptr);
    ++stats_.kernel_launches;
  } else if (w.mode == W_INT4) {
    launch_gemm_w4(use_pair(M, N), epi, act, w.tm, M, N, K, ep, stream_, sms_, out_map);
    ++stats_.kernel_launches;
  } else {
    launch_gemm(use_pair(M, N), w.mode == W_INT8, epi, act, w.tm, M, N, K, ep, stream_, sms_, out_map);
    ++stats_.kernel_launches;
  }
}

template <typename F>
void Engine::timed(int cat, double work, F&& f) {
  if (!ktime_) {
    f();
    return;
  }
  auto get_ev = [&] {
    if (kev_free_.empty()) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreate(&e));
      kev_.push_back(e);
      kev_free_.push_back(static_cast<int>(kev_.size()) - 1);
    }
    const int i = kev_free_.back();
    kev_free_.pop_back();
    return i;
  };
  const int a = get_ev(), b = get_ev();
  CUDA_OK(cudaEventRecord(kev_[a], stream_));
  f();
  CUDA_OK(cudaEventRecord(kev_[b], stream_));
  kpend_.push_back({cat, a, b, work, step_seq_});
}

// Accumulates the durations of every timed launch of steps <= upto_step (already complete).
void Engine::collect_times(int64_t upto_step) {
  if (!ktime_ || kpend_.empty()) return;
  std::vector<KPending> keep;
  for (const auto& k : kpend_) {
    if (k.step > upto_step) {
      keep.push_back(k);
      continue;
    }
    float ms = 0.f;
    CUDA_OK(cudaEventSynchronize(kev_[k.ev1]));
    CUDA_OK(cudaEventElapsedTime(&ms, kev_[k.ev0], kev_[k.ev1]));
    kms_[k.cat] += ms;
    kwork_[k.cat] += k.work;
    kcount_[k.cat] += 1;
    kev_free_.push_back(k.ev0);
    kev_free_.push_back(k.ev1);
  }
  kpend_.swap(keep);
}

// Packs the step's metadata into the pinned staging buffer, copies it with ONE async H2D, runs
// the layer stack, the head + argmax, copies the generated ids back (async) and records sb.done.
void Engine::launch_step(StepBuffers& sb, const int32_t* d_ids, const uint8_t* d_key_mask, float* d_logits) {
  const Step& s = sb.step;
  const int T = s.T();
  const int R = static_cast<int>(s.head_rows.size());
  // The previous step on these buffers may still be reading h_meta (its H2D copy is async): e.g. the
  // shared-prefix step, whose buffers are reused by the decode loop's second step without a
  // process(). A never-recorded or already-processed event returns at once.
  CUDA_OK(cudaEventSynchronize(sb.done));
  uint8_t* h = sb.h_meta.p;
  uint8_t* d = sb.d_meta.p;
  size_t off = 0;
  auto put = [&](const void* src, size_t bytes) {
    if (bytes) std::memcpy(h + off, src, bytes);
    const uint8_t* dev = d + off;
    off = align16(off + bytes);
    return dev;
  };
  sb.tok_src = reinterpret_cast<const int64_t*>(put(s.tok_src.data(), T * sizeof(int64_t)));
  sb.tok_slot = reinterpret_cast<const int*>(put(s.tok_slot.data(), T * sizeof(int)));
  sb.tok_pos = reinterpret_cast<const int*>(put(s.tok_pos.data(), T * sizeof(int)));
  sb.pre = reinterpret_cast<const AttnGroup*>(put(s.pre.data(), s.pre.size() * sizeof(AttnGroup)));
  sb.dec = reinterpret_cast<const AttnGroup*>(put(s.dec.data(), s.dec.size() * sizeof(AttnGroup)));
  sb.head_rows = reinterpret_cast<const int*>(put(s.head_rows.data(), R * sizeof(int)));
  sb.head_slot = reinterpret_cast<const int*>(put(s.head_slot.data(), R * sizeof(int)));
  // last-layer compaction (see last_compact_): only when the step computes fewer head rows than
  // tokens, and never for forward() logits or a calibration capture (they read every position)
  const bool compact = last_compact_ && d_logits == nullptr && cap_ == nullptr && cap8_ == nullptr && R < T;
  if (compact) {
    if (iota_.size() < static_cast<size_t>(R)) {
      const size_t n0 = iota_.size();
      iota_.resize(R);
      for (size_t i = n0; i < iota_.size(); ++i) iota_[i] = static_cast<int>(i);
    }
    sb.head_iota = reinterpret_cast<const int*>(put(iota_.data(), R * sizeof(int)));
  }
  CUDA_OK(cudaMemcpyAsync(d, h, off, cudaMemcpyHostToDevice, stream_));

  const double dT = static_cast<double>(T);
  const bool q8_first = layers_[0]->qkv.int8();
  timed(0, dT * d_ * 14.0, [&] {
    launch_embed_ln(d_ids, sb.tok_src, sb.tok_slot, sb.tok_pos, d_last_tok_.p, T, d_, tok_embed_.p, pos_embed_.p,
                    x_.p, layers_[0]->ln1_g.p, layers_[0]->ln1_b.p, h_.p, d_, stream_, q8_first ? h8_.p : nullptr,
                    hs_.p);
  });
  ++stats_.kernel_launches;
  capture_point(0, T, d_);  // layers.0.attn_in
  // algorithmic attention work of this step (per head): prefill FLOPs 4*hd*sum(pos+1),
  // decode K+V bytes 2*2*hd*(pos+1)
  double pre_keys = 0, dec_keys = 0;
  if (ktime_) {
    for (const auto& g : s.pre)
      for (int i = 0; i < g.nq; ++i) pre_keys += g.pos0 + i + 1;
    for (const auto& g : s.dec) dec_keys += g.pos0 + 1;
  }
  const float scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(hd_));
  // weight scale (CODES / INT8) and activation scale (INT8) of one GEMM
  auto scales = [](GemmEpi& e, const GemmW& w, const float* a_scale) {
    e.w_scale = w.mode == W_VALUES ? nullptr : w.scale.p;
    e.a_scale = w.int8() ? a_scale : nullptr;
  };
  for (int l = 0; l < L_; ++l) {
    Layer& ly = *layers_[l];
    const bool i8_qkv = ly.qkv.int8(), i8_o = ly.o.int8();
    const bool i8_in = ly.in.int8(), i8_out = ly.out.int8();
    GemmEpi ep;
    ep.M = T;
    // QKV projection; K/V scattered into the paged pool by the epilogue.
    ep.N = 3 * ly.kh;
    ep.out = q_.p;
    ep.ldo = kh_max_;
    ep.kv_layer = ly.kv.p;
    ep.tok_slot = sb.tok_slot;
    ep.tok_pos = sb.tok_pos;
    ep.page_table = page_table_.p;
    ep.max_pages = pps_;
    ep.kh = ly.kh;
    ep.hd = hd_;
    ep.hd_shift = hd_ == 16 ? 4 : hd_ == 32 ? 5 : hd_ == 64 ? 6 : 7;
    ep.heads = ly.heads;
    ep.page_size = PAGE;
    scales(ep, ly.qkv, hs_.p);
    timed(1, 2.0 * dT * 3 * ly.kh * d_, [&] {
      gemm_w(iolmk::EPI_QKV, ly.qkv, i8_qkv ? tm_h8_ : tm_h_, ly.qkv.mode == W_SP24F ? tm_hs_ : tm_h8s_, T, 3 * ly.kh,
             d_, ep);
    });
    if (compact && R == 0 && l + 1 == L_) break;  // K/V-only step (shared prefix): nothing reads the rest
    AttnParams ap{};
    ap.q_map = tm_q_;
    ap.kv_map = ly.tm_kv;
    ap.kvg_map = ly.tm_kvg;
    ap.q = q_.p;
    ap.ldq = kh_max_;
    ap.z = z_.p;
    ap.ldz = kh_max_;
    ap.kv = ly.kv.p;
    ap.page_table = page_table_.p;
    ap.max_pages = pps_;
    ap.heads = ly.heads;
    ap.key_mask = d_key_mask;
    ap.scale_log2 = scale_log2;
    AttnParams pre = ap, dec = ap, none = ap;
    pre.groups = sb.pre;
    pre.n_groups = static_cast<int>(s.pre.size());
    dec.groups = sb.dec;
    dec.n_groups = static_cast<int>(s.dec.size());
    none.n_groups = 0;
    if (pre.n_groups) {
      timed(2, 4.0 * hd_ * ly.heads * pre_keys, [&] {
        if (prefill_hp_ && d_key_mask == nullptr) launch_prefill_hp(pre, hd_, stream_);
        else if (prefill_tc_) launch_prefill_tc(pre, hd_, stream_);
        else launch_attention(pre, none, hd_, stream_);
      });
      ++stats_.kernel_launches;
    }
    if (dec.n_groups) {
      timed(3, 4.0 * hd_ * ly.heads * dec_keys, [&] { launch_attention(none, dec, hd_, stream_); });
      ++stats_.kernel_launches;
    }
    // last layer, compacted: only the R head rows continue (x / z rows gathered into xc_ / zc_)
    const bool cl = compact && l + 1 == L_;
    const int Tl = cl ? R : T;
    const double dTl = static_cast<double>(Tl);
    float* const xl = cl ? xc_.p : x_.p;
    const h16* const zl = cl ? zc_.p : z_.p;
    if (cl) {
      timed(8, static_cast<double>(R) * (8.0 * d_ + 4.0 * ly.kh), [&] {
        launch_gather_head_rows(x_.p, d_, z_.p, kh_max_, ly.kh, sb.head_rows, R, xc_.p, zc_.p, kh_max_, stream_);
      });
      ++stats_.kernel_launches;
    }
    // x += z * Wo^T
    if (i8_o) {
      timed(9, dTl * ly.kh * 3.0, [&] { launch_quant_rows(zl, kh_max_, Tl, ly.kh, z8_.p, kh_max_, zs_.p, stream_); });
      ++stats_.kernel_launches;
    }
    capture_point(1, Tl, ly.kh);  // layers.l.attn_out_in
    GemmEpi eo;
    eo.M = Tl;
    eo.N = d_;
    eo.out = xl;
    eo.ldo = d_;
    scales(eo, ly.o, zs_.p);
    timed(4, 2.0 * dTl * d_ * ly.kh, [&] {
      gemm_w(iolmk::EPI_RESID_F32, ly.o, i8_o ? ly.tm_z8 : cl ? tm_zc_ : ly.tm_z, ly.o.mode == W_SP24F ? (cl ? tm_zcs_ : ly.tm_zs) : ly.tm_z8s, Tl, d_,
             ly.kh, eo, resid_tma_ && d_ % 8 == 0 && ly.o.mode != W_INT4 ? (cl ? &tm_xc_out_ : &tm_x_out_) : nullptr);
    });
    // h = LN2(x)
    timed(5, dTl * d_ * 6.0, [&] {
      launch_ln(xl, Tl, d_, ly.ln2_g.p, ly.ln2_b.p, h_.p, d_, stream_, i8_in ? h8_.p : nullptr, hs_.p);
    });
    ++stats_.kernel_launches;
    capture_point(2, Tl, d_);  // layers.l.ffn_in
    // g = gelu(h * Win^T)
    GemmEpi ei;
    ei.M = Tl;
    ei.N = ly.f;
    ei.out = g_.p;
    ei.ldo = f_ld_max_;
    scales(ei, ly.in, hs_.p);
    timed(6, 2.0 * dTl * ly.f * d_, [&] {
      gemm_w(iolmk::EPI_GELU_H16, ly.in, i8_in ? tm_h8_ : tm_h_, ly.in.mode == W_SP24F ? tm_hs_ : tm_h8s_, Tl, ly.f, d_,
             ei,
             tma_epi_ ? &ly.tm_g_out : nullptr);
    });
    // x += g * Wout^T
    if (i8_out) {
      timed(9, dTl * ly.f * 3.0, [&] { launch_quant_rows(g_.p, f_ld_max_, Tl, ly.f, g8_.p, f_ld_max_, gs_.p, stream_); });
      ++stats_.kernel_launches;
    }
    capture_point(3, Tl, ly.f);  // layers.l.ffn_mid (post-GELU)
    GemmEpi eo2 = eo;
    scales(eo2, ly.out, gs_.p);
    timed(7, 2.0 * dTl * d_ * ly.f, [&] {
      gemm_w(iolmk::EPI_RESID_F32, ly.out, i8_out ? ly.tm_g8 : ly.tm_g, ly.out.mode == W_SP24F ? ly.tm_gs : ly.tm_g8s, Tl,
             d_, ly.f, eo2, resid_tma_ && d_ % 8 == 0 && ly.out.mode != W_INT4 ? (cl ? &tm_xc_out_ : &tm_x_out_) : nullptr);
    });
    if (l + 1 < L_) {
      const bool q8_next = layers_[l + 1]->qkv.int8();
      timed(5, dT * d_ * 6.0, [&] {
        launch_ln(x_.p, T, d_, layers_[l + 1]->ln1_g.p, layers_[l + 1]->ln1_b.p, h_.p, d_, stream_,
                  q8_next ? h8_.p : nullptr, hs_.p);
      });
      ++stats_.kernel_launches;
      capture_point(0, T, d_);  // layers.l+1.attn_in
    }
  }
  if (R > 0) {
    timed(8, static_cast<double>(R) * d_ * 4.0 + static_cast<double>(V_) * d_ * 4.0, [&] {
      launch_head(compact ? xc_.p : x_.p, d_, compact ? sb.head_iota : sb.head_rows, R, lnf_g_.p, lnf_b_.p, tok_embed_t_.p, V_, sb.head_slot, sb.d_next.p,
                  d_last_tok_.p, d_logits, stream_);
    });
    ++stats_.kernel_launches;
    CUDA_OK(cudaMemcpyAsync(sb.h_next.p, sb.d_next.p, R * sizeof(int32_t), cudaMemcpyDeviceToHost, stream_));
  }
  CUDA_OK(cudaEventRecord(sb.done, stream_));
  ++stats_.steps;
  stats_.tokens += T;
  ++step_seq_;
}

uint64_t Engine::ref_madds_row(int s0, int advances) const {
  const uint64_t dv = static_cast<uint64_t>(d_) * V_;
  const uint64_t S0 = static_cast<uint64_t>(s0);
  uint64_t t = S0 * madds_A_ + madds_B_ * S0 * (S0 + 1) + dv;
  for (int i = 1; i <= advances; ++i) t += madds_A_ + 2 * madds_B_ * (S0 + static_cast<uint64_t>(i)) + dv;
  return t;
}

void Engine::reset_counters() {
  stats_ = iolm_cuda_stats{};
  for (int i = 0; i < IOLM_KCLASSES; ++i) {
    kms_[i] = kwork_[i] = 0;
    kcount_[i] = 0;
  }
}

void Engine::decode(const int32_t* ids, bool ids_on_device, const int64_t* offsets, int64_t n_rows, int max_new,
                    int32_t* out_ids, int32_t* out_len, uint64_t* madds, int64_t* bad_row) {
  CUDA_OK(cudaSetDevice(device_));
  reset_counters();
  if (bad_row) *bad_row = -1;
  if (n_rows <= 0) throw ContractViolation("batch_decode: batch size must be >= 1");
  if (max_new < 0) throw ContractViolation("batch_decode: max_new_tokens must be >= 0");
  if (!offsets || !out_len || (max_new > 0 && !out_ids)) throw ContractViolation("batch_decode: null buffer");
  for (int64_t i = 0; i < n_rows; ++i) out_len[i] = 0;
  if (madds) *madds = 0;
  if (max_new == 0) return;  // runtime.cpp:249 - no encode, no compute
  int min_len = INT32_MAX;
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t len = offsets[i + 1] - offsets[i];
    if (len <= 0) throw ContractViolation("batch_decode: empty token row " + std::to_string(i));
    if (len > S_) {
      if (bad_row) *bad_row = i;
      throw SequenceTooLong("batch_decode: prompt " + std::to_string(i) + " needs " + std::to_string(len) +
                            " tokens, max_seq_len is " + std::to_string(S_));
    }
    min_len = std::min<int>(min_len, static_cast<int>(len));
  }
  CUDA_OK(cudaEventRecord(ev0_, stream_));
  const int64_t total = offsets[n_rows] - offsets[0];
  const int32_t* d_ids;
  const int64_t base = offsets[0];
  if (ids_on_device) {
    d_ids = ids;
  } else {
    d_ids_.ensure(total + 1);
    CUDA_OK(cudaMemcpyAsync(d_ids_.p, ids + base, total * sizeof(int32_t), cudaMemcpyHostToDevice, stream_));
    d_ids = d_ids_.p - base;  // keep absolute offsets valid
  }
  // id range check + longest common prefix, on the device
  d_offsets_.ensure(n_rows + 1);
  CUDA_OK(cudaMemcpyAsync(d_offsets_.p, offsets, (n_rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream_));
  int init[2] = {1, min_len - 1};
  CUDA_OK(cudaMemcpyAsync(d_scalar_.p, init, sizeof(init), cudaMemcpyHostToDevice, stream_));
  launch_check_ids(d_ids + base, total, V_, d_scalar_.p, stream_);
  if (prefix_sharing_) launch_lcp(d_ids, d_offsets_.p, n_rows, min_len - 1, d_scalar_.p + 1, stream_);
  int res[2];
  CUDA_OK(cudaMemcpyAsync(res, d_scalar_.p, sizeof(res), cudaMemcpyDeviceToHost, stream_));
  CUDA_OK(cudaStreamSynchronize(stream_));
  if (res[0] == 0) throw ContractViolation("forward: token id out of range");
  const int prefix_pages = prefix_sharing_ ? std::max(0, res[1]) / PAGE : 0;
  const int P = prefix_pages * PAGE;
  set_prefix_pages(prefix_pages);

  int parity = 0;
  if (P > 0) {  // shared prefix: K/V only, computed once per call
    StepBuffers& sb = sbuf_[parity];
    sb.step.clear();
    add_prefill(sb.step, prefix_slot_, offsets[0], 0, P, false, -1);
    launch_step(sb, d_ids, nullptr, nullptr);
    stats_.prefix_tokens += P;
    parity ^= 1;
  }

  struct RowState {
    int slot = -1, s0 = 0;
    int cur_plan = 0;    // sequence length after every planned step
    int heads_plan = 0;  // token predictions planned
    int emitted = 0;     // tokens confirmed and emitted
    bool done = false;
  };
  std::vector<RowState> rows(n_rows);
  std::vector<int> free_slots;
  for (int sl = max_slots_ - 1; sl >= 0; --sl) free_slots.push_back(sl);
  std::vector<int64_t> live;  // rows with a token prediction in the last planned step
  std::vector<int64_t> next_live;
  int64_t next_row = 0;
  uint64_t madd_total = 0;
  StepBuffers* inflight = nullptr;

  // Results of one completed step: emit tokens, finish rows (EOS / budget / full context).
  auto process = [&](StepBuffers& sb) {
    CUDA_OK(cudaEventSynchronize(sb.done));
    const Step& st = sb.step;
    for (size_t i = 0; i < st.head_owner.size(); ++i) {
      const int64_t ri = st.head_owner[i];
      RowState& r = rows[ri];
      if (r.done) continue;  // speculative token after an EOS
      const int nxt = sb.h_next.p[i];
      int advances = -1;
      if (nxt == IOLM_EOS || r.emitted == max_new) {
        advances = r.emitted;  // stop before emitting (runtime.cpp:287-290)
      } else {
        out_ids[static_cast<size_t>(ri) * max_new + r.emitted] = nxt;
        ++r.emitted;
        if (r.s0 + r.emitted - 1 == S_) advances = r.emitted - 1;  // full context (runtime.cpp:293-296)
        else if (r.emitted == max_new) advances = r.emitted;     // reference advances once more
      }
      if (advances >= 0) {
        r.done = true;
        out_len[ri] = r.emitted;
        madd_total += ref_madds_row(r.s0, advances);
      }
    }
  };

  while (next_row < n_rows || !live.empty()) {
    StepBuffers& sb = sbuf_[parity];
    Step& s = sb.step;
    s.clear();
    // (a) one generated token for every row whose previous prediction will be emitted and fed
    //     back; rows that stop here release their slot (stream order protects its pages)
    next_live.clear();
    for (int64_t ri : live) {
      RowState& r = rows[ri];
      if (r.done || r.heads_plan >= max_new || r.cur_plan >= S_) {
        free_slots.push_back(r.slot);
        r.slot = -1;
        continue;
      }
      const int m = s.T();
      s.tok_src.push_back(-1);  // token from the slot's last argmax (device register)
      s.tok_slot.push_back(r.slot);
      s.tok_pos.push_back(r.cur_plan);
      s.dec.push_back(AttnGroup{r.slot, m, 1, r.cur_plan});
      s.head_rows.push_back(m);
      s.head_slot.push_back(r.slot);
      s.head_owner.push_back(ri);
      ++r.cur_plan;
      ++r.heads_plan;
      next_live.push_back(ri);
    }
    stats_.decode_tokens += s.T();
    // (b) admit new rows while slots and the token budget allow
    while (next_row < n_rows && !free_slots.empty()) {
      const int len = static_cast<int>(offsets[next_row + 1] - offsets[next_row]);
      if (s.T() + (len - P) > T_max_) break;
      RowState& r = rows[next_row];
      r.slot = free_slots.back();
      free_slots.pop_back();
      r.s0 = len;
      r.cur_plan = len;
      r.heads_plan = 1;
      add_prefill(s, r.slot, offsets[next_row], P, len, true, next_row);
      stats_.prefill_tokens += len - P;
      next_live.push_back(next_row);
      ++next_row;
    }
    live.swap(next_live);
    if (s.T() == 0) {
      if (inflight) {  // only finished rows left in flight
        process(*inflight);
        inflight = nullptr;
        continue;
      }
      throw CudaError("scheduler stalled (no slot or token budget)");
    }
    launch_step(sb, d_ids, nullptr, nullptr);
    if (inflight) {
      process(*inflight);
      collect_times(step_seq_ - 2);
    }
    inflight = &sb;
    parity ^= 1;
  }
  if (inflight) process(*inflight);
  collect_times(step_seq_);
  if (madds) *madds = madd_total;
  CUDA_OK(cudaEventRecord(ev1_, stream_));
  CUDA_OK(cudaEventSynchronize(ev1_));
  float ms = 0.f;
  CUDA_OK(cudaEventElapsedTime(&ms, ev0_, ev1_));
  stats_.device_ms = ms;
}

void Engine::capture_point(int point, int T, int cols) {
  if (cap_) {
    const h16* src = point == 1 ? z_.p : point == 3 ? g_.p : h_.p;
    const int ld = point == 1 ? kh_max_ : point == 3 ? f_ld_max_ : d_;
    CUDA_OK(cudaMemcpy2DAsync(cap_ + cap_off_, static_cast<size_t>(cols) * 2, src, static_cast<size_t>(ld) * 2,
                              static_cast<size_t>(cols) * 2, T, cudaMemcpyDeviceToDevice, stream_));
    cap_off_ += static_cast<size_t>(T) * cols;
  }
  if (cap8_) {
    const int8_t* src = point == 1 ? z8_.p : point == 3 ? g8_.p : h8_.p;
    const float* sc = point == 1 ? zs_.p : point == 3 ? gs_.p : hs_.p;
    const int ld = point == 1 ? kh_max_ : point == 3 ? f_ld_max_ : d_;
    CUDA_OK(cudaMemcpy2DAsync(cap8_ + cap_off_, static_cast<size_t>(cols), src, static_cast<size_t>(ld),
                              static_cast<size_t>(cols), T, cudaMemcpyDeviceToDevice, stream_));
    CUDA_OK(cudaMemcpyAsync(capsc_ + capsc_off_, sc, sizeof(float) * T, cudaMemcpyDeviceToDevice, stream_));
    cap_off_ += static_cast<size_t>(T) * cols;
    capsc_off_ += static_cast<size_t>(T);
  }
}

void Engine::forward(const int32_t* ids, const uint8_t* mask, int n, float* logits, uint64_t* madds,
                     uint16_t* capture, int8_t* codes, float* code_scales) {
  CUDA_OK(cudaSetDevice(device_));
  reset_counters();
  if (n <= 0 || !ids) throw ContractViolation("forward: empty sequence");
  if (n > S_)
    throw SequenceTooLong("forward: sequence length " + std::to_string(n) + " exceeds max_seq_len " +
                          std::to_string(S_));
  for (int i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= V_) throw ContractViolation("forward: token id out of range");
  CUDA_OK(cudaEventRecord(ev0_, stream_));
  d_ids_.ensure(n);
  CUDA_OK(cudaMemcpyAsync(d_ids_.p, ids, n * sizeof(int32_t), cudaMemcpyHostToDevice, stream_));
  const uint8_t* dmask = nullptr;
  if (mask) {
    CUDA_OK(cudaMemcpyAsync(d_mask_.p, mask, n, cudaMemcpyHostToDevice, stream_));
    dmask = d_mask_.p;
  }
  set_prefix_pages(0);
  StepBuffers& sb = sbuf_[0];
  sb.step.clear();
  add_prefill(sb.step, 0, 0, 0, n, false, -1);
  for (int i = 0; i < n; ++i) {
    sb.step.head_rows.push_back(i);
    sb.step.head_slot.push_back(0);
    sb.step.head_owner.push_back(0);
  }
  size_t cap_elems = 0;
  if (capture) {
    if (act_quant_) throw Unsupported("forward capture: not available with act_quant (capture the baseline model)");
    for (const auto& ly : layers_) cap_elems += static_cast<size_t>(n) * (2 * d_ + ly->kh + ly->f);
    d_cap_.ensure(cap_elems);
    cap_ = d_cap_.p;
    cap_off_ = 0;
  }
  if (codes) {
    if (!act_quant_ || !any_int8_) throw Unsupported("forward_codes: needs act_quant (W8A8) weights");
    for (const auto& ly : layers_) {
      if (!(ly->qkv.int8() && ly->o.int8() && ly->in.int8() && ly->out.int8()))
        throw Unsupported("forward_codes: every projection must run W8A8");
      cap_elems += static_cast<size_t>(n) * (2 * d_ + ly->kh + ly->f);
    }
    d_cap8_.ensure(cap_elems);
    d_capsc_.ensure(static_cast<size_t>(4) * n * L_);
    cap8_ = d_cap8_.p;
    capsc_ = d_capsc_.p;
    cap_off_ = capsc_off_ = 0;
  }
  try {
    launch_step(sb, d_ids_.p, dmask, d_logits_.p);
  } catch (...) {
    cap_ = nullptr;
    cap8_ = nullptr;
    capsc_ = nullptr;
    throw;
  }
  cap_ = nullptr;
  cap8_ = nullptr;
  capsc_ = nullptr;
  if (capture)
    CUDA_OK(cudaMemcpyAsync(capture, d_cap_.p, cap_elems * sizeof(h16), cudaMemcpyDeviceToHost, stream_));
  if (codes) {
    CUDA_OK(cudaMemcpyAsync(codes, d_cap8_.p, cap_elems, cudaMemcpyDeviceToHost, stream_));
    CUDA_OK(cudaMemcpyAsync(code_scales, d_capsc_.p, sizeof(float) * 4 * n * L_, cudaMemcpyDeviceToHost, stream_));
  }
  CUDA_OK(cudaMemcpyAsync(logits, d_logits_.p, sizeof(float) * n * V_, cudaMemcpyDeviceToHost, stream_));
  CUDA_OK(cudaEventRecord(ev1_, stream_));
  CUDA_OK(cudaEventSynchronize(ev1_));
  collect_times(step_seq_);
  float ms = 0.f;
  CUDA_OK(cudaEventElapsedTime(&ms, ev0_, ev1_));
  stats_.device_ms = ms;
  stats_.prefill_tokens = n;
  if (madds) {
    // full_forward_flops with the reference's attention count for a masked sequence
    uint64_t t = 0;
    const uint64_t dv = static_cast<uint64_t>(d_) * V_;
    for (int i = 0; i < n; ++i) {
      t += madds_A_ + dv;
      if (!mask || mask[i]) t += 2 * madds_B_ * static_cast<uint64_t>(i + 1);
    }
    *madds = t;
  }
}

}  // namespace iolmh

// ====================================================================== C ABI
using iolmh::Engine;
using iolmh::guarded;

// A context is one Engine per device. One device: the plain runtime. Several (iolm_cuda_create_multi):
// every Engine holds a full replica and its own KV pool; batch_decode range-partitions the rows over
// them (SURVEY §8e / BASELINE north_star: rows are independent, exec.cpp:139-142), one host thread
// per device, each writing its rows' generated ids straight into the caller's output buffers - that
// write IS the output-column gather; no collective and no device-to-device traffic. Single-sequence
// calls (forward, capture, codes, image) run on the first device.
struct iolm_cuda_ctx {
  std::unique_ptr<Engine> eng;                 // == shards[0].get() owner for the first device
  std::vector<std::unique_ptr<Engine>> extra;  // devices 1..n-1
  iolm_cuda_stats agg{};                       // last multi-device decode, summed over shards
  bool multi_last = false;
  int n_shards() const { return 1 + static_cast<int>(extra.size()); }
  Engine& shard(int i) const { return i == 0 ? *eng : *extra[i - 1]; }
};

namespace iolmh {
// Contiguous row ranges [cut[i], cut[i+1]) with near-equal token counts (prefill dominates a row's
// cost; every row then generates the same budget), at most one shard per row.
std::vector<int64_t> partition_rows(const int64_t* offsets, int64_t n_rows, int shards) {
  std::vector<int64_t> cut{0};
  const int s = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(shards, n_rows)));
  const double total = static_cast<double>(offsets[n_rows] - offsets[0]);
  int64_t r = 0;
  for (int i = 1; i < s; ++i) {
    const double target = total * i / s;
    while (r < n_rows && static_cast<double>(offsets[r] - offsets[0]) < target) ++r;
    r = std::max<int64_t>(r, cut.back() + 1);  // non-empty shard
    r = std::min<int64_t>(r, n_rows - (s - i));  // leave >= 1 row per remaining shard
    cut.push_back(r);
  }
  cut.push_back(n_rows);
  return cut;
}

// batch_decode over every shard of ctx (host ids). Lengths are checked for the WHOLE batch first, in
// row order, so SequenceTooLong names the first offending row exactly as runtime.cpp:264-267 does;
// any other shard failure is re-thrown from the lowest failing shard (the earliest rows).
void multi_decode(iolm_cuda_ctx& ctx, const int32_t* ids, bool on_device, const int64_t* offsets, int64_t n_rows,
                  int max_new, int32_t* out_ids, int32_t* out_len, uint64_t* madds, int64_t* bad_row) {
  if (bad_row) *bad_row = -1;
  if (n_rows <= 0) throw ContractViolation("batch_decode: batch size must be >= 1");
  if (max_new < 0) throw ContractViolation("batch_decode: max_new_tokens must be >= 0");
  if (!offsets || !out_len || (max_new > 0 && !out_ids)) throw ContractViolation("batch_decode: null buffer");
  if (on_device) throw Unsupported("multi-device context: device-resident ids are per device; pass host ids");
  const int S = ctx.eng->config().max_seq_len;
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t len = offsets[i + 1] - offsets[i];
    if (len <= 0) throw ContractViolation("batch_decode: empty token row " + std::to_string(i));
    if (len > S) {
      if (bad_row) *bad_row = i;
      throw SequenceTooLong("batch_decode: prompt " + std::to_string(i) + " needs " + std::to_string(len) +
                            " tokens, max_seq_len is " + std::to_string(S));
    }
  }
  const std::vector<int64_t> cut = partition_rows(offsets, n_rows, ctx.n_shards());
  const int used = static_cast<int>(cut.size()) - 1;
  std::vector<uint64_t> m(used, 0);
  std::vector<std::exception_ptr> err(used);
  auto run = [&](int i) {
    try {
      Engine& e = ctx.shard(i);
      std::lock_guard<std::mutex> lk(e.mu);
      int64_t bad = -1;
      e.decode(ids, false, offsets + cut[i], cut[i + 1] - cut[i], max_new,
               max_new > 0 ? out_ids + static_cast<size_t>(cut[i]) * max_new : out_ids, out_len + cut[i], &m[i], &bad);
    } catch (...) {
      err[i] = std::current_exception();
    }
  };
  std::vector<std::thread> th;
  for (int i = 1; i < used; ++i) th.emplace_back(run, i);
  run(0);
  for (auto& t : th) t.join();
  for (int i = 0; i < used; ++i)
    if (err[i]) std::rethrow_exception(err[i]);
  iolm_cuda_stats a{};
  for (int i = 0; i < used; ++i) {
    const iolm_cuda_stats& s = ctx.shard(i).stats();
    a.steps += s.steps;
    a.tokens += s.tokens;
    a.prefill_tokens += s.prefill_tokens;
    a.decode_tokens += s.decode_tokens;
    a.prefix_tokens += s.prefix_tokens;
    a.kernel_launches += s.kernel_launches;
    a.device_ms = std::max(a.device_ms, s.device_ms);  // shards run concurrently
  }
  ctx.agg = a;
  ctx.multi_last = true;
  if (madds) {
    uint64_t t = 0;
    for (uint64_t x : m) t += x;
    *madds = t;
  }
}
}  // namespace iolmh

extern "C" int iolm_cuda_create(const uint8_t* bundle_bytes, size_t len, int device, const iolm_cuda_opts* opts,
                                iolm_cuda_ctx** out) {
  return guarded([&] {
    if (!out) throw iolmh::ContractViolation("iolm_cuda_create: null out");
    *out = nullptr;
    auto ctx = std::make_unique<iolm_cuda_ctx>();
    ctx->eng = std::make_unique<Engine>(bundle_bytes, len, device, opts);
    *out = ctx.release();
  });
}

extern "C" int iolm_cuda_create_multi(const uint8_t* bundle_bytes, size_t len, const int32_t* devices,
                                      int32_t n_devices, const iolm_cuda_opts* opts, iolm_cuda_ctx** out) {
  return guarded([&] {
    if (!out || !devices || n_devices < 1) throw iolmh::ContractViolation("iolm_cuda_create_multi: bad arguments");
    *out = nullptr;
    auto ctx = std::make_unique<iolm_cuda_ctx>();
    std::vector<std::unique_ptr<Engine>> engs(n_devices);
    std::vector<std::exception_ptr> err(n_devices);
    std::vector<std::thread> th;  // weights decode / upload on every device at once
    for (int i = 0; i < n_devices; ++i)
      th.emplace_back([&, i] {
        try {
          engs[i] = std::make_unique<Engine>(bundle_bytes, len, devices[i], opts);
        } catch (...) {
          err[i] = std::current_exception();
        }
      });
    for (auto& t : th) t.join();
    for (int i = 0; i < n_devices; ++i)
      if (err[i]) std::rethrow_exception(err[i]);
    ctx->eng = std::move(engs[0]);
    for (int i = 1; i < n_devices; ++i) ctx->extra.push_back(std::move(engs[i]));
    *out = ctx.release();
  });
}

extern "C" int iolm_cuda_device_count(const iolm_cuda_ctx* ctx, int32_t* n) {
  return guarded([&] {
    if (!ctx || !n) throw iolmh::ContractViolation("null argument");
    *n = ctx->n_shards();
  });
}

extern "C" int iolm_cuda_debug_partition(const int64_t* row_offsets, int64_t n_rows, int32_t shards, int64_t* cut,
                                         int32_t* n_cut) {
  return guarded([&] {
    if (!row_offsets || !cut || !n_cut || n_rows <= 0 || shards < 1)
      throw iolmh::ContractViolation("debug_partition: bad arguments");
    const auto c = iolmh::partition_rows(row_offsets, n_rows, shards);
    *n_cut = static_cast<int32_t>(c.size());
    for (size_t i = 0; i < c.size(); ++i) cut[i] = c[i];
  });
}

extern "C" void iolm_cuda_destroy(iolm_cuda_ctx* ctx) { delete ctx; }

extern "C" int iolm_cuda_save_image(iolm_cuda_ctx* ctx, const char* path) {
  return guarded([&] {
    if (!ctx || !path) throw iolmh::ContractViolation("null argument");
    std::lock_guard<std::mutex> lock(ctx->eng->mu);
    ctx->eng->save_image(path);
  });
}

extern "C" int iolm_cuda_create_from_image(const char* path, uint64_t expected_hash, int device,
                                           const iolm_cuda_opts* opts, iolm_cuda_ctx** out) {
  return guarded([&] {
    if (!out || !path) throw iolmh::ContractViolation("iolm_cuda_create_from_image: null argument");
    *out = nullptr;
    auto ctx = std::make_unique<iolm_cuda_ctx>();
    ctx->eng = std::make_unique<Engine>(std::string(path), expected_hash, device, opts);
    *out = ctx.release();
  });
}

extern "C" int iolm_cuda_image_info(const char* path, uint64_t* bundle_hash, iolm_cuda_model_config* cfg) {
  return guarded([&] {
    if (!path || !bundle_hash || !cfg) throw iolmh::ContractViolation("null argument");
    iolmh::ImageFile f(path, "rb");
    iolmh::ImageSum total;
    const iolmh::ImageHeader h = iolmh::read_image_header(f, total);
    *bundle_hash = h.hash;
    const auto& c = h.cfg;
    *cfg = iolm_cuda_model_config{c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.d_ff, c.max_seq_len,
                                  c.head_dim()};
  });
}

extern "C" int iolm_cuda_bundle_hash(const iolm_cuda_ctx* ctx, uint64_t* out) {
  return guarded([&] {
    if (!ctx || !out) throw iolmh::ContractViolation("null argument");
    *out = ctx->eng->bundle_hash();
  });
}

extern "C" int iolm_cuda_config(const iolm_cuda_ctx* ctx, iolm_cuda_model_config* out) {
  return guarded([&] {
    if (!ctx || !out) throw iolmh::ContractViolation("null argument");
    const auto& c = ctx->eng->config();
    *out = iolm_cuda_model_config{c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.d_ff, c.max_seq_len,
                                  c.head_dim()};
  });
}

extern "C" int iolm_cuda_layer_shape(const iolm_cuda_ctx* ctx, int32_t layer, int32_t* heads, int32_t* ffn) {
  return guarded([&] {
    if (!ctx || !heads || !ffn) throw iolmh::ContractViolation("null argument");
    const auto& c = ctx->eng->config();
    if (layer < 0 || layer >= c.n_layers) throw iolmh::ContractViolation("layer index out of range");
    *heads = c.layer_heads(layer);
    *ffn = c.layer_ffn(layer);
  });
}

extern "C" int iolm_cuda_layer_heads(const iolm_cuda_ctx* ctx, int32_t layer, int32_t* heads, int32_t cap,
                                     int32_t* n) {
  return guarded([&] {
    if (!ctx || !n) throw iolmh::ContractViolation("null argument");
    const auto& c = ctx->eng->config();
    if (layer < 0 || layer >= c.n_layers) throw iolmh::ContractViolation("layer index out of range");
    const auto& h = c.active_heads[layer];
    *n = static_cast<int32_t>(h.size());
    if (cap < *n || (*n > 0 && !heads)) throw iolmh::ContractViolation("layer_heads: buffer too small");
    for (size_t i = 0; i < h.size(); ++i) heads[i] = h[i];
  });
}

extern "C" int iolm_cuda_decode(iolm_cuda_ctx* ctx, const int32_t* ids, const int64_t* row_offsets, int64_t n_rows,
                                int32_t max_new_tokens, int32_t* out_ids, int32_t* out_len, uint64_t* madds,
                                int64_t* bad_row) {
  return guarded([&] {
    if (!ctx) throw iolmh::ContractViolation("null context");
    if (ctx->n_shards() > 1) {
      iolmh::multi_decode(*ctx, ids, false, row_offsets, n_rows, max_new_tokens, out_ids, out_len, madds, bad_row);
      return;
    }
    ctx->multi_last = false;
    std::lock_guard<std::mutex> lock(ctx->eng->mu);
    ctx->eng->decode(ids, false, row_offsets, n_rows, max_new_tokens, out_ids, out_len, madds, bad_row);
  });
}

extern "C" int iolm_cuda_decode_device_ids(iolm_cuda_ctx* ctx, const int32_t* d_ids, const int64_t* row_offsets,
                                           int64_t n_rows, int32_t max_new_tokens, int32_t* out_ids,
                                           int32_t* out_len, uint64_t* madds, int64_t* bad_row) {
  return guarded([&] {
    if (!ctx) throw iolmh::ContractViolation("null context");
    if (ctx->n_shards() > 1) {
      iolmh::multi_decode(*ctx, d_ids, true, row_offsets, n_rows, max_new_tokens, out_ids, out_len, madds, bad_row);
      return;
    }
    ctx->multi_last = false;
    std::lock_guard<std::mutex> lock(ctx->eng->mu);
    ctx->eng->decode(d_ids, true, row_offsets, n_rows, max_new_tokens, out_ids, out_len, madds, bad_row);
  });
}

extern "C" int iolm_cuda_forward_logits(iolm_cuda_ctx* ctx, const int32_t* ids, const uint8_t* mask, int32_t n,
                                        float* logits, uint64_t* madds) {
  return guarded([&] {
    if (!ctx || !logits) throw iolmh::ContractViolation("null argument");
    std::lock_guard<std::mutex> lock(ctx->eng->mu);
    ctx->multi_last = false;
    ctx->eng->forward(ids, mask, n, logits, madds);
  });
}

extern "C" int iolm_cuda_last_stats(const iolm_cuda_ctx* ctx, iolm_cuda_stats* out) {
  return guarded([&] {
    if (!ctx || !out) throw iolmh::ContractViolation("null argument");
    *out = ctx->multi_last ? ctx->agg : ctx->eng->stats();
  });
}

extern "C" int iolm_cuda_set_kernel_timing(iolm_cuda_ctx* ctx, int32_t on) {
  return guarded([&] {
    if (!ctx) throw iolmh::ContractViolation("null argument");
    for (int i = 0; i < ctx->n_shards(); ++i) {
      std::lock_guard<std::mutex> lk(ctx->shard(i).mu);
      ctx->shard(i).set_kernel_timing(on != 0);
    }
  });
}

extern "C" int iolm_cuda_forward_capture(iolm_cuda_ctx* ctx, const int32_t* ids, const uint8_t* mask, int32_t n,
                                         float* logits, uint16_t* capture, uint64_t* madds) {
  return guarded([&] {
    if (!ctx || !logits || !capture) throw iolmh::ContractViolation("null argument");
    std::lock_guard<std::mutex> lock(ctx->eng->mu);
    ctx->multi_last = false;
    ctx->eng->forward(ids, mask, n, logits, madds, capture);
  });
}

extern "C" int iolm_cuda_forward_codes(iolm_cuda_ctx* ctx, const int32_t* ids, int32_t n, float* logits,
                                       int8_t* codes, float* scales, uint64_t* madds) {
  return guarded([&] {
    if (!ctx || !logits || !codes || !scales) throw iolmh::ContractViolation("null argument");
    std::lock_guard<std::mutex> lock(ctx->eng->mu);
    ctx->multi_last = false;
    ctx->eng->forward(ids, nullptr, n, logits, madds, nullptr, codes, scales);
  });
}

extern "C" int iolm_cuda_kernel_times(const iolm_cuda_ctx* ctx, double* ms, double* work, int64_t* launches,
                                      int32_t n) {
  return guarded([&] {
    if (!ctx || !ms || !work || !launches) throw iolmh::ContractViolation("null argument");
    if (n < IOLM_KCLASSES) throw iolmh::ContractViolation("kernel_times: array too small");
    for (int i = 0; i < IOLM_KCLASSES; ++i) {  // summed over the shards of the last decode
      ms[i] = work[i] = 0;
      launches[i] = 0;
      for (int k = 0; k < (ctx->multi_last ? ctx->n_shards() : 1); ++k) {
        ms[i] += ctx->shard(k).kms_[i];
        work[i] += ctx->shard(k).kwork_[i];
        launches[i] += ctx->shard(k).kcount_[i];
      }
    }
  });
}
