// Host-only: bundle header parsing and validation (see bundle.hpp).
#include <cctype>
#include <cstring>
#include <map>
#include <memory>

#include "bundle.hpp"
#include "launch.hpp"

namespace iolmh {

uint64_t fnv1a64(const uint8_t* p, size_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

namespace {

// ---- minimal JSON reader for the bundle header (objects, arrays, strings, integers)
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0;
  bool is_int = false;
  long long ival = 0;
  unsigned long long uval = 0;
  bool b = false;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const char* p;
  const char* end;
  [[noreturn]] void fail(const std::string& what) {
    throw CorruptHeader("bundle: header is not valid JSON: " + what);
  }
  void ws() {
    while (p < end && std::isspace(static_cast<unsigned char>(*p))) ++p;
  }
  JVal parse() {
    ws();
    if (p >= end) fail("unexpected end");
    JVal v;
    const char c = *p;
    if (c == '{') {
      v.kind = JVal::Obj;
      ++p;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return v;
      }
      for (;;) {
        ws();
        if (p >= end || *p != '"') fail("expected key");
        std::string k = parse_string();
        ws();
        if (p >= end || *p != ':') fail("expected ':'");
        ++p;
        v.obj.emplace_back(std::move(k), parse());
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JVal::Arr;
      ++p;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return v;
      }
      for (;;) {
        v.arr.push_back(parse());
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      v.str = parse_string();
      return v;
    }
    if (c == 't' && end - p >= 4 && std::memcmp(p, "true", 4) == 0) {
      p += 4;
      v.kind = JVal::Bool;
      v.b = true;
      return v;
    }
    if (c == 'f' && end - p >= 5 && std::memcmp(p, "false", 5) == 0) {
      p += 5;
      v.kind = JVal::Bool;
      return v;
    }
    if (c == 'n' && end - p >= 4 && std::memcmp(p, "null", 4) == 0) {
      p += 4;
      return v;
    }
    if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) {
      const char* s = p;
      bool neg = false;
      if (*p == '-') {
        neg = true;
        ++p;
      }
      bool integral = true;
      unsigned long long u = 0;
      bool overflow = false;
      while (p < end && std::isdigit(static_cast<unsigned char>(*p))) {
        const unsigned d = static_cast<unsigned>(*p - '0');
        if (u > (~0ull - d) / 10) overflow = true;
        u = u * 10 + d;
        ++p;
      }
      if (p < end && (*p == '.' || *p == 'e' || *p == 'E')) {
        integral = false;
        while (p < end && (std::isdigit(static_cast<unsigned char>(*p)) || *p == '.' || *p == 'e' ||
                           *p == 'E' || *p == '+' || *p == '-'))
          ++p;
      }
      v.kind = JVal::Num;
      v.num = std::strtod(std::string(s, p).c_str(), nullptr);
      v.is_int = integral && !overflow;
      v.uval = u;
      v.ival = neg ? -static_cast<long long>(u) : static_cast<long long>(u);
      if (neg && u == 0 && integral) v.uval = 0;
      if (neg) v.uval = 0;
      return v;
    }
    fail(std::string("unexpected character '") + c + "'");
  }
  std::string parse_string() {
    ++p;
    std::string out;
    while (p < end && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (p >= end) fail("bad escape");
        switch (*p) {
          case '"': out.push_back('"'); break;
          case '\\': out.push_back('\\'); break;
          case '/': out.push_back('/'); break;
          case 'b': out.push_back('\b'); break;
          case 'f': out.push_back('\f'); break;
          case 'n': out.push_back('\n'); break;
          case 'r': out.push_back('\r'); break;
          case 't': out.push_back('\t'); break;
          case 'u': {
            if (end - p < 5) fail("bad \\u escape");
            const unsigned cp = std::stoul(std::string(p + 1, p + 5), nullptr, 16);
            if (cp < 0x80) out.push_back(static_cast<char>(cp));
            else if (cp < 0x800) {
              out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
              out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
            } else {
              out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
              out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
              out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
            }
            p += 4;
            break;
          }
          default: fail("bad escape");
        }
        ++p;
      } else {
        out.push_back(*p++);
      }
    }
    if (p >= end) fail("unterminated string");
    ++p;
    return out;
  }
};

[[noreturn]] void malformed(const std::string& what) {
  throw CorruptHeader("bundle: malformed header fields: " + what);
}
const JVal& need(const JVal& o, const std::string& k) {
  if (o.kind != JVal::Obj) malformed("expected object for '" + k + "'");
  const JVal* v = o.get(k);
  if (!v) malformed("missing key '" + k + "'");
  return *v;
}
int as_int(const JVal& v, const std::string& what) {
  if (v.kind != JVal::Num || !v.is_int || v.ival < INT32_MIN || v.ival > INT32_MAX)
    malformed(what + " must be an integer");
  return static_cast<int>(v.ival);
}
uint64_t as_u64(const JVal& v, const std::string& what) {
  if (v.kind != JVal::Num || !v.is_int || v.ival < 0) malformed(what + " must be an unsigned integer");
  return v.uval;
}
std::string as_str(const JVal& v, const std::string& what) {
  if (v.kind != JVal::Str) malformed(what + " must be a string");
  return v.str;
}

bool is_weight_tensor(const std::string& name) {
  return name.find(".attn.w") != std::string::npos || name.find(".ffn.w") != std::string::npos;
}

std::vector<std::string> required_tensor_names(const ModelConfig& c) {
  std::vector<std::string> names = {"tok_embed", "pos_embed"};
  for (int l = 0; l < c.n_layers; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    for (const char* s : {"attn_norm.gain", "attn_norm.bias", "attn.wq", "attn.wk", "attn.wv", "attn.wo",
                          "ffn_norm.gain", "ffn_norm.bias", "ffn.w_in", "ffn.w_out"})
      names.push_back(p + s);
  }
  names.push_back("final_norm.gain");
  names.push_back("final_norm.bias");
  return names;
}

std::pair<int, int> tensor_shape(const ModelConfig& c, const std::string& name) {
  if (name == "tok_embed") return {c.vocab_size, c.d_model};
  if (name == "pos_embed") return {c.max_seq_len, c.d_model};
  if (name == "final_norm.gain" || name == "final_norm.bias") return {1, c.d_model};
  const size_t dot = name.find('.', 7);
  const int layer = std::stoi(name.substr(7, dot - 7));
  const std::string field = name.substr(dot + 1);
  const int kh = c.layer_heads(layer) * c.head_dim();
  const int f = c.layer_ffn(layer);
  if (field == "attn.wq" || field == "attn.wk" || field == "attn.wv") return {kh, c.d_model};
  if (field == "attn.wo") return {c.d_model, kh};
  if (field == "ffn.w_in") return {f, c.d_model};
  if (field == "ffn.w_out") return {c.d_model, f};
  return {1, c.d_model};
}

}  // namespace

void ModelConfig::validate() const {
  if (vocab_size <= 0 || d_model <= 0 || n_layers <= 0 || n_heads <= 0 || d_ff <= 0 || max_seq_len <= 0)
    throw ContractViolation("ModelConfig: all dimensions must be positive");
  if (d_model % n_heads != 0) throw ContractViolation("ModelConfig: d_model not divisible by n_heads");
  if (static_cast<int>(active_heads.size()) != n_layers || static_cast<int>(active_ffn.size()) != n_layers)
    throw ContractViolation("ModelConfig: per-layer lists must have n_layers entries");
  for (int l = 0; l < n_layers; ++l) {
    if (active_heads[l].empty())
      throw ContractViolation("ModelConfig: layer " + std::to_string(l) + " has no active heads");
    int prev = -1;
    for (int h : active_heads[l]) {
      if (h <= prev || h >= n_heads)
        throw ContractViolation("ModelConfig: active head list must be ascending and in range");
      prev = h;
    }
    if (active_ffn[l] < 1 || active_ffn[l] > d_ff)
      throw ContractViolation("ModelConfig: active FFN count out of range");
  }
}

uint64_t TensorRecord::payload_bytes(int rows, int cols, int enc) {
  const uint64_t r = static_cast<uint64_t>(rows), c = static_cast<uint64_t>(cols);
  switch (enc) {
    case ENC_DENSE_F32: return r * c * 4;
    case ENC_Q8: return r * c + r * 4;
    case ENC_Q4: return r * ((c + 1) / 2) + r * 4;
    case ENC_SPARSE24_Q8: {
      const uint64_t groups = c / 4;
      return r * (c / 2) + r * ((groups + 1) / 2) + r * 4;
    }
  }
  throw UnknownEncoding("payload_bytes: unknown encoding tag");
}

const TensorRecord& BundleView::tensor(const std::string& name) const {
  for (const auto& t : tensors)
    if (t.name == name) return t;
  throw ContractViolation("ModelBundle: missing tensor " + name);
}

void BundleView::validate() const {
  config.validate();
  for (const std::string& name : required_tensor_names(config)) {
    const TensorRecord* rec = nullptr;
    for (const auto& t : tensors)
      if (t.name == name) {
        rec = &t;
        break;
      }
    if (!rec) throw ContractViolation("ModelBundle: missing tensor " + name);
    const auto [r, c] = tensor_shape(config, name);
    if (rec->rows != r || rec->cols != c)
      throw ContractViolation("ModelBundle: tensor " + name + " has shape " + std::to_string(rec->rows) + "x" +
                              std::to_string(rec->cols) + ", expected " + std::to_string(r) + "x" +
                              std::to_string(c));
    if (!is_weight_tensor(name) && rec->encoding != ENC_DENSE_F32)
      throw ContractViolation("ModelBundle: tensor " + name + " must be dense_f32");
    if (rec->length != TensorRecord::payload_bytes(rec->rows, rec->cols, rec->encoding))
      throw ContractViolation("ModelBundle: tensor " + name + " payload length mismatch");
    if (rec->offset + rec->length > blob_len)
      throw TruncatedBlob("ModelBundle: tensor " + name + " extends past end of blob");
  }
}

BundleView parse_bundle(const uint8_t* bytes, size_t len) {
  if (len < 10 || std::memcmp(bytes, "IOLM", 4) != 0) throw CorruptHeader("bundle: bad magic");
  const uint16_t version = static_cast<uint16_t>(bytes[4] | (bytes[5] << 8));
  if (version != 1) throw CorruptHeader("bundle: unsupported format version " + std::to_string(version));
  uint32_t hl = 0;
  for (int i = 0; i < 4; ++i) hl |= static_cast<uint32_t>(bytes[6 + i]) << (8 * i);
  if (10 + static_cast<size_t>(hl) > len) throw CorruptHeader("bundle: header length exceeds file size");
  JParser jp{reinterpret_cast<const char*>(bytes) + 10, reinterpret_cast<const char*>(bytes) + 10 + hl};
  JVal root = jp.parse();
  jp.ws();
  if (jp.p != jp.end) throw CorruptHeader("bundle: header is not valid JSON: trailing characters");

  BundleView b;
  const JVal& cfg = need(root, "config");
  ModelConfig& c = b.config;
  c.vocab_size = as_int(need(cfg, "vocab_size"), "vocab_size");
  c.d_model = as_int(need(cfg, "d_model"), "d_model");
  c.n_layers = as_int(need(cfg, "n_layers"), "n_layers");
  c.n_heads = as_int(need(cfg, "n_heads"), "n_heads");
  c.d_ff = as_int(need(cfg, "d_ff"), "d_ff");
  c.max_seq_len = as_int(need(cfg, "max_seq_len"), "max_seq_len");
  const JVal& ah = need(cfg, "active_heads");
  if (ah.kind != JVal::Arr) malformed("active_heads must be an array");
  for (const auto& l : ah.arr) {
    if (l.kind != JVal::Arr) malformed("active_heads entries must be arrays");
    std::vector<int> hs;
    for (const auto& h : l.arr) hs.push_back(as_int(h, "active head"));
    c.active_heads.push_back(std::move(hs));
  }
  const JVal& af = need(cfg, "active_ffn");
  if (af.kind != JVal::Arr) malformed("active_ffn must be an array");
  for (const auto& f : af.arr) c.active_ffn.push_back(as_int(f, "active_ffn"));

  const JVal& ts = need(root, "tensors");
  if (ts.kind != JVal::Arr) malformed("tensors must be an array");
  for (const auto& t : ts.arr) {
    TensorRecord r;
    r.name = as_str(need(t, "name"), "name");
    r.rows = as_int(need(t, "rows"), "rows");
    r.cols = as_int(need(t, "cols"), "cols");
    const int enc = as_int(need(t, "encoding"), "encoding");
    if (enc < 0 || enc > 3)
      throw UnknownEncoding("bundle: unknown encoding tag " + std::to_string(enc) + " for tensor " + r.name);
    r.encoding = enc;
    r.offset = as_u64(need(t, "offset"), "offset");
    r.length = as_u64(need(t, "length"), "length");
    b.tensors.push_back(std::move(r));
  }
  const JVal& prov = need(root, "provenance");
  as_str(need(prov, "recipe_id"), "recipe_id");
  as_str(need(prov, "parent_hash"), "parent_hash");

  b.blob = bytes + 10 + hl;
  b.blob_len = len - 10 - hl;
  for (const auto& t : b.tensors) {
    if (t.rows < 0 || t.cols < 0 || t.length != TensorRecord::payload_bytes(t.rows, t.cols, t.encoding))
      throw CorruptHeader("bundle: tensor " + t.name + " length inconsistent with shape");
    if (t.offset + t.length > b.blob_len)
      throw TruncatedBlob("bundle: tensor " + t.name + " extends past end of blob");
  }
  b.validate();
  return b;
}

}  // namespace iolmh
