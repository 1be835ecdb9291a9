// Model bundle reader: the "IOLM" header + blob format of proj/docs/format.md, parsed and validated
// with the same error classes as the reference (deserialize_bundle, model.cpp:348-406;
// ModelBundle::validate, model.cpp:292-309; ModelConfig::validate, model.cpp:35-56).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace iolmh {

enum Encoding : int { ENC_DENSE_F32 = 0, ENC_Q8 = 1, ENC_Q4 = 2, ENC_SPARSE24_Q8 = 3 };

struct ModelConfig {
  int vocab_size = 131, d_model = 0, n_layers = 0, n_heads = 0, d_ff = 0, max_seq_len = 0;
  std::vector<std::vector<int>> active_heads;
  std::vector<int> active_ffn;
  int head_dim() const { return d_model / n_heads; }
  int layer_heads(int l) const { return static_cast<int>(active_heads[l].size()); }
  int layer_ffn(int l) const { return active_ffn[l]; }
  void validate() const;
};

struct TensorRecord {
  std::string name;
  int rows = 0, cols = 0, encoding = 0;
  uint64_t offset = 0, length = 0;
  static uint64_t payload_bytes(int rows, int cols, int enc);
};

struct BundleView {
  ModelConfig config;
  std::vector<TensorRecord> tensors;
  const uint8_t* blob = nullptr;
  size_t blob_len = 0;
  uint64_t hash = 0;  // FNV-1a over the whole serialized bundle (model.cpp:408-411)

  const TensorRecord& tensor(const std::string& name) const;
  const uint8_t* payload(const TensorRecord& t) const { return blob + t.offset; }
  void validate() const;
};

// Parses + fully validates; throws the engine errors (CorruptHeader, TruncatedBlob,
// UnknownEncoding, ContractViolation). The view borrows `bytes`.
BundleView parse_bundle(const uint8_t* bytes, size_t len);

uint64_t fnv1a64(const uint8_t* p, size_t n);

}  // namespace iolmh
