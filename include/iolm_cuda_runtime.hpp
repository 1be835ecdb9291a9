// iolm_cuda_runtime.hpp - header-only C++ shim: the public surface of iolm::ModelRuntime
// (/root/reference/proj/include/iolm/runtime.hpp:37-60) on top of the C ABI in iolm_cuda.h.
//
//   iolm::cuda::ModelRuntime rt(serialized_bundle_bytes);        // ModelRuntime(bundle)
//   rt.config(); rt.bundle_hash();                                // runtime.hpp:41-42
//   rt.forward(ids, mask, counter);                               // runtime.hpp:48-49
//   rt.greedy_decode(prompt, n, counter);                         // runtime.hpp:54-55
//   rt.batch_decode(prompts, n, counter);                         // runtime.hpp:59-60
//
// Tokenization (BOS + one id per ASCII byte), the per-prompt length check, rendering of emitted ids
// and the error classes follow the reference (runtime.cpp:241-309, tokenizer.cpp:10-36,
// common.hpp:16-89). Define IOLM_CUDA_WITH_REFERENCE_TYPES before including this header (with the
// reference's include/ on the path) to get a constructor from iolm::ModelBundle, results as
// iolm::Matrix and errors thrown as the reference's own exception classes - see INTEGRATION.md.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "iolm_cuda.h"

#ifdef IOLM_CUDA_WITH_REFERENCE_TYPES
#include "iolm/common.hpp"
#include "iolm/matrix.hpp"
#include "iolm/model.hpp"
#include "iolm/runtime.hpp"  // iolm::CaptureSink
#endif

namespace iolm::cuda {

#ifdef IOLM_CUDA_WITH_REFERENCE_TYPES
using Error = iolm::Error;
using ContractViolation = iolm::ContractViolation;
using SequenceTooLong = iolm::SequenceTooLong;
using CorruptHeader = iolm::CorruptHeader;
using TruncatedBlob = iolm::TruncatedBlob;
using UnknownEncoding = iolm::UnknownEncoding;
using FlopCounter = iolm::FlopCounter;
#else
struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct ContractViolation : Error {
  using Error::Error;
};
struct SequenceTooLong : Error {
  using Error::Error;
};
struct CorruptHeader : Error {
  using Error::Error;
};
struct TruncatedBlob : Error {
  using Error::Error;
};
struct UnknownEncoding : Error {
  using Error::Error;
};
class FlopCounter {
 public:
  void add(uint64_t m) { t_ += m; }
  uint64_t total() const { return t_; }
  void reset() { t_ = 0; }

 private:
  uint64_t t_ = 0;
};
#endif
// GPU-side failures have no reference counterpart (the reference is CPU-only).
struct GpuError : Error {
  explicit GpuError(const std::string& w) : Error(w) {}
};
// A device-layout image that no longer matches its bundle / the requested weight options: the
// caller rebuilds from the bundle (what ModelRegistry::lookup does for a stale entry, optimize.cpp:145).
struct StaleImage : Error {
  explicit StaleImage(const std::string& w) : Error(w) {}
};

inline void check(int st) {
  if (st == IOLM_OK) return;
  const std::string msg = iolm_cuda_last_error();
  switch (st) {
    case IOLM_E_CONTRACT: throw ContractViolation(msg);
    case IOLM_E_SEQ_TOO_LONG: throw SequenceTooLong(msg);
    case IOLM_E_CORRUPT_HEADER: throw CorruptHeader(msg);
    case IOLM_E_TRUNCATED_BLOB: throw TruncatedBlob(msg);
    case IOLM_E_UNKNOWN_ENCODING: throw UnknownEncoding(msg);
    case IOLM_E_STALE: throw StaleImage(msg);
    default: throw GpuError(msg);
  }
}

#ifdef IOLM_CUDA_WITH_REFERENCE_TYPES
using Config = iolm::ModelConfig;  // config() returns the reference's own type (runtime.hpp:41)
using Logits = iolm::Matrix;       // forward() returns the reference's own type (runtime.hpp:48)
#else
// Mirror of iolm::ModelConfig (proj/include/iolm/model.hpp:20-41): same fields and accessors.
struct Config {
  int vocab_size = 131, d_model = 0, n_layers = 0, n_heads = 0, d_ff = 0, max_seq_len = 0;
  std::vector<std::vector<int>> active_heads;  // per layer, original head indices, ascending
  std::vector<int> active_ffn;                 // per layer
  int head_dim() const { return d_model / n_heads; }
  int layer_heads(int layer) const { return static_cast<int>(active_heads[layer].size()); }
  int layer_ffn(int layer) const { return active_ffn[layer]; }
};
// Mirror of iolm::Matrix (proj/include/iolm/matrix.hpp:28-46): row-major f32 rows x cols.
struct Logits {
  int rows = 0;
  int cols = 0;
  std::vector<float> data;
  Logits() = default;
  Logits(int r, int c, std::vector<float> v) : rows(r), cols(c), data(std::move(v)) {}
  float at(int r, int c) const { return data[static_cast<size_t>(r) * cols + c]; }
  const float* row(int r) const { return data.data() + static_cast<size_t>(r) * cols; }
};
#endif

// ModelConfig of a context through the C ABI (iolm_cuda_config / layer_shape / layer_heads).
inline Config read_config(const iolm_cuda_ctx* ctx) {
  iolm_cuda_model_config c{};
  check(iolm_cuda_config(ctx, &c));
  Config cfg;
  cfg.vocab_size = c.vocab_size;
  cfg.d_model = c.d_model;
  cfg.n_layers = c.n_layers;
  cfg.n_heads = c.n_heads;
  cfg.d_ff = c.d_ff;
  cfg.max_seq_len = c.max_seq_len;
  cfg.active_heads.resize(c.n_layers);
  cfg.active_ffn.resize(c.n_layers);
  for (int l = 0; l < c.n_layers; ++l) {
    int32_t heads = 0, ffn = 0, n = 0;
    check(iolm_cuda_layer_shape(ctx, l, &heads, &ffn));
    std::vector<int32_t> idx(static_cast<size_t>(c.n_heads));
    check(iolm_cuda_layer_heads(ctx, l, idx.data(), c.n_heads, &n));
    cfg.active_heads[l].assign(idx.begin(), idx.begin() + n);
    cfg.active_ffn[l] = ffn;
  }
  return cfg;
}

// IEEE binary16 bit pattern -> f32 (exact; the engine's captured activations are fp16).
inline float f16_to_f32(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu, bits;
  if (e == 0x1F) bits = sign | 0x7F800000u | (m << 13);  // inf / nan
  else if (e != 0) bits = sign | ((e + 112u) << 23) | (m << 13);
  else if (m == 0) bits = sign;
  else {  // subnormal: renormalise
    e = 113;
    while (!(m & 0x400u)) { m <<= 1; --e; }
    bits = sign | (e << 23) | ((m & 0x3FFu) << 13);
  }
  float f;
  std::memcpy(&f, &bits, 4);
  return f;
}

class ModelRuntime {
 public:
  explicit ModelRuntime(std::span<const uint8_t> bundle_bytes, int device = 0, const iolm_cuda_opts* opts = nullptr) {
    check(iolm_cuda_create(bundle_bytes.data(), bundle_bytes.size(), device, opts, &ctx_));
    try {
      cfg_ = read_config(ctx_);
    } catch (...) {
      iolm_cuda_destroy(ctx_);
      throw;
    }
  }
#ifdef IOLM_CUDA_WITH_REFERENCE_TYPES
  // Drop-in for ModelRuntime(const ModelBundle&): the bundle is handed over in its canonical
  // serialized form (model.cpp:311-346), so bundle_hash() is the reference's exactly.
  explicit ModelRuntime(const iolm::ModelBundle& bundle, int device = 0, const iolm_cuda_opts* opts = nullptr)
      : ModelRuntime(std::span<const uint8_t>(iolm::serialize_bundle(bundle)), device, opts) {}

  // What the reference-side patch (oracle/reference_gpu.patch) calls from
  // iolm::ModelRuntime's constructor: a B200 runtime for `bundle` when the environment names a device
  // (IOLM_CUDA_DEVICE=<index>; IOLM_CUDA_ACT_QUANT=1 runs q8 / sparse24_q8 bundles as W8A8), else null
  // and the reference keeps its CPU path.
  // IOLM_CUDA_DEVICE may list several devices ("0,1,2,3"): one multi-device runtime over them.
  static std::shared_ptr<const ModelRuntime> from_env(const iolm::ModelBundle& bundle) {
    const char* dev = std::getenv("IOLM_CUDA_DEVICE");
    if (!dev || !*dev) return nullptr;
    iolm_cuda_opts o{};
    if (const char* aq = std::getenv("IOLM_CUDA_ACT_QUANT")) o.act_quant = std::atoi(aq) > 0 ? 1 : 0;
    std::vector<int> devs;
    for (const char* p = dev; *p;) {
      devs.push_back(std::atoi(p));
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
    if (devs.size() == 1) return std::make_shared<const ModelRuntime>(bundle, devs[0], &o);
    const std::vector<uint8_t> bytes = iolm::serialize_bundle(bundle);
    return std::make_shared<const ModelRuntime>(std::span<const uint8_t>(bytes), std::span<const int>(devs), &o);
  }
#endif
  // One runtime over several GPUs (iolm_cuda_create_multi): batch_decode range-partitions the rows
  // over full per-GPU replicas, one host thread per device, outputs in row order (the multi-GPU
  // deployment of SURVEY §8e behind the same surface).
  ModelRuntime(std::span<const uint8_t> bundle_bytes, std::span<const int> devices, const iolm_cuda_opts* opts = nullptr) {
    std::vector<int32_t> d(devices.begin(), devices.end());
    check(iolm_cuda_create_multi(bundle_bytes.data(), bundle_bytes.size(), d.data(), static_cast<int32_t>(d.size()),
                                 opts, &ctx_));
    try {
      cfg_ = read_config(ctx_);
    } catch (...) {
      iolm_cuda_destroy(ctx_);
      throw;
    }
  }
  int device_count() const {
    int32_t n = 0;
    check(iolm_cuda_device_count(ctx_, &n));
    return n;
  }
  ModelRuntime(const ModelRuntime&) = delete;
  ModelRuntime& operator=(const ModelRuntime&) = delete;
  ~ModelRuntime() { iolm_cuda_destroy(ctx_); }

  // From a device-layout image (iolm_cuda_create_from_image); expected_hash = the registry entry's
  // bundle hash (0: unchecked). Throws StaleImage when the image must be rebuilt from the bundle.
  static std::unique_ptr<ModelRuntime> from_image(const std::string& path, uint64_t expected_hash, int device = 0,
                                                  const iolm_cuda_opts* opts = nullptr) {
    iolm_cuda_ctx* ctx = nullptr;
    check(iolm_cuda_create_from_image(path.c_str(), expected_hash, device, opts, &ctx));
    return std::unique_ptr<ModelRuntime>(new ModelRuntime(ctx));
  }
  // Writes this runtime's device layout next to its bundle (iolm_cuda_save_image).
  void save_image(const std::string& path) const { check(iolm_cuda_save_image(ctx_, path.c_str())); }

  const Config& config() const { return cfg_; }
  uint64_t bundle_hash() const {
    uint64_t h = 0;
    check(iolm_cuda_bundle_hash(ctx_, &h));
    return h;
  }

  // forward(ids, mask, counter, capture) (runtime.hpp:48-49): logits for every position, a
  // [ids.size() x 131] matrix (iolm::Matrix with the reference types). Masked positions' rows are
  // "not to be read" (runtime.hpp:44-47); they come back as zeros so the Matrix stays finite.
  // With a CaptureSink, the inputs of every linear weight at the non-pad positions are recorded
  // under the reference's capture-point names (capture_calibration, calib.cpp:44-51), captured on
  // the GPU as fp16 and widened to f32.
#ifdef IOLM_CUDA_WITH_REFERENCE_TYPES
  Logits forward(std::span<const int> ids, std::span<const uint8_t> mask, FlopCounter& counter,
                 iolm::CaptureSink* capture = nullptr) const {
#else
  Logits forward(std::span<const int> ids, std::span<const uint8_t> mask, FlopCounter& counter) const {
    void* capture = nullptr;
#endif
    if (ids.empty()) throw ContractViolation("forward: empty sequence");
    if (!mask.empty() && mask.size() != ids.size()) throw ContractViolation("forward: mask length mismatch");
    if (static_cast<int>(ids.size()) > cfg_.max_seq_len)
      throw SequenceTooLong("forward: sequence length " + std::to_string(ids.size()) + " exceeds max_seq_len " +
                            std::to_string(cfg_.max_seq_len));
    const int n = static_cast<int>(ids.size());
    std::vector<int32_t> v(ids.begin(), ids.end());
    std::vector<float> out(static_cast<size_t>(n) * cfg_.vocab_size);
    uint64_t madds = 0;
    const uint8_t* m = mask.empty() ? nullptr : mask.data();
    if (!capture) {
      check(iolm_cuda_forward_logits(ctx_, v.data(), m, n, out.data(), &madds));
    } else {
#ifdef IOLM_CUDA_WITH_REFERENCE_TYPES
      std::vector<int> kh(cfg_.n_layers), f(cfg_.n_layers);
      size_t total = 0;
      for (int l = 0; l < cfg_.n_layers; ++l) {
        kh[l] = cfg_.layer_heads(l) * cfg_.head_dim();
        f[l] = cfg_.layer_ffn(l);
        total += static_cast<size_t>(n) * (2 * cfg_.d_model + kh[l] + f[l]);
      }
      std::vector<uint16_t> cap(total);
      check(iolm_cuda_forward_capture(ctx_, v.data(), m, n, out.data(), cap.data(), &madds));
      size_t off = 0;
      std::vector<float> row;
      auto take = [&](const std::string& point, int cols) {
        for (int t = 0; t < n; ++t) {
          if (mask.empty() || mask[t]) {
            row.resize(cols);
            for (int c = 0; c < cols; ++c) row[c] = f16_to_f32(cap[off + static_cast<size_t>(t) * cols + c]);
            capture->add_row(point, row);
          }
        }
        off += static_cast<size_t>(n) * cols;
      };
      for (int l = 0; l < cfg_.n_layers; ++l) {
        const std::string p = "layers." + std::to_string(l) + ".";
        take(p + "attn_in", cfg_.d_model);
        take(p + "attn_out_in", kh[l]);
        take(p + "ffn_in", cfg_.d_model);
        take(p + "ffn_mid", f[l]);
      }
#endif
    }
    counter.add(madds);
    if (m)
      for (int t = 0; t < n; ++t)
        if (!m[t]) std::fill_n(out.begin() + static_cast<size_t>(t) * cfg_.vocab_size, cfg_.vocab_size, 0.0f);
    return Logits(n, cfg_.vocab_size, std::move(out));
  }

  std::string greedy_decode(std::string_view prompt, int max_new_tokens, FlopCounter& counter) const {
    const std::string p(prompt);
    return batch_decode(std::span<const std::string>(&p, 1), max_new_tokens, counter)[0];
  }

  std::vector<std::string> batch_decode(std::span<const std::string> prompts, int max_new_tokens,
                                        FlopCounter& counter) const {
    if (prompts.empty()) throw ContractViolation("batch_decode: batch size must be >= 1");
    if (max_new_tokens < 0) throw ContractViolation("batch_decode: max_new_tokens must be >= 0");
    std::vector<std::string> out(prompts.size());
    if (max_new_tokens == 0) return out;
    std::vector<int32_t> ids;
    std::vector<int64_t> offsets{0};
    for (size_t i = 0; i < prompts.size(); ++i) {  // encode + length check in prompt order
      ids.push_back(IOLM_BOS);
      for (size_t j = 0; j < prompts[i].size(); ++j) {
        const auto b = static_cast<unsigned char>(prompts[i][j]);
        if (b > 127)
          throw ContractViolation("Tokenizer: non-ASCII byte " + std::to_string(b) + " at offset " + std::to_string(j));
        ids.push_back(b);
      }
      const int64_t len = static_cast<int64_t>(ids.size()) - offsets.back();
      if (len > cfg_.max_seq_len)
        throw SequenceTooLong("batch_decode: prompt " + std::to_string(i) + " needs " + std::to_string(len) +
                              " tokens, max_seq_len is " + std::to_string(cfg_.max_seq_len));
      offsets.push_back(static_cast<int64_t>(ids.size()));
    }
    const size_t n = prompts.size();
    std::vector<int32_t> gen(n * static_cast<size_t>(max_new_tokens)), len(n);
    uint64_t madds = 0;
    int64_t bad = -1;
    check(iolm_cuda_decode(ctx_, ids.data(), offsets.data(), static_cast<int64_t>(n), max_new_tokens, gen.data(),
                           len.data(), &madds, &bad));
    counter.add(madds);
    for (size_t i = 0; i < n; ++i)
      for (int t = 0; t < len[i]; ++t) {
        const int32_t id = gen[i * max_new_tokens + t];
        if (id >= 0 && id <= 127) out[i].push_back(static_cast<char>(id));  // PAD/BOS render nothing
      }
    return out;
  }

  iolm_cuda_ctx* handle() const { return ctx_; }

 private:
  explicit ModelRuntime(iolm_cuda_ctx* ctx) : ctx_(ctx) {
    try {
      cfg_ = read_config(ctx_);
    } catch (...) {
      iolm_cuda_destroy(ctx_);
      throw;
    }
  }
  iolm_cuda_ctx* ctx_ = nullptr;
  Config cfg_{};
};

#ifdef IOLM_CUDA_WITH_REFERENCE_TYPES
// build_hessian (proj/src/calib.cpp:64-74) with the Gram matrix on the GPU (iolm_cuda_gram): H =
// 2 X^T X + lambda I, lambda = lambda_rel * mean(diag(2 X^T X)) - bit-identical to the reference's.
inline iolm::MatrixD build_hessian(const iolm::Matrix& x, double lambda_rel, int device = 0) {
  if (x.rows < 1) throw iolm::EmptyCalibration("build_hessian: no calibration samples");
  iolm::MatrixD h(x.cols, x.cols);
  check(iolm_cuda_gram(device, x.data.data(), x.rows, x.cols, 2.0, h.data.data()));
  double diag_mean = 0.0;
  for (int i = 0; i < h.rows; ++i) diag_mean += h.at(i, i);
  diag_mean /= h.rows;
  const double lambda = lambda_rel * diag_mean;
  for (int i = 0; i < h.rows; ++i) h.at(i, i) += lambda;
  return h;
}

// The device the reference-side patch uses for calibration work: the first of IOLM_CUDA_DEVICE, or -1.
inline int env_device() {
  const char* dev = std::getenv("IOLM_CUDA_DEVICE");
  return dev && *dev ? std::atoi(dev) : -1;
}
#endif

}  // namespace iolm::cuda
