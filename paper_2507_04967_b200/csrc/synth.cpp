// libiolm_synth: workload generator for the throughput harness (bench.py) and the tests.
//
// Produces byte-identical inputs to what the reference's own generators would give, so the CPU
// reference arm and the GPU arm see the same table and the same model:
//   * random-init weights: ToyModelParams::init (proj/src/train.cpp:45-75) drawn from iolm::Rng
//     (xoshiro256** + Box-Muller, proj/src/rng.cpp:26-78), serialized exactly like
//     serialize_bundle (proj/src/model.cpp:311-346) so bundle_hash() matches the reference's;
//   * synthetic table rows: instruction literal + R printable chars where char j of
//     row r is 32 + Rng(0x5EED0000 ^ r).next_below(95);
//   * RTN compression twins (quantize_rtn, proj/src/quant.cpp:23-38,79-92; magnitude 2:4,
//     quant.cpp:181-200) for the compressed configs, encoded per proj/docs/format.md.
// This is harness code: the engine never links it.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

struct Rng {
  uint64_t s[4];
  double cached = 0.0;
  bool has_cached = false;
  static uint64_t splitmix64(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  explicit Rng(uint64_t seed) {
    uint64_t sm = seed;
    for (auto& v : s) v = splitmix64(sm);
  }
  uint64_t next_u64() {
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
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  uint64_t next_below(uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
      const uint64_t r = next_u64();
      if (r >= threshold) return r % n;
    }
  }
  double next_normal() {
    if (has_cached) {
      has_cached = false;
      return cached;
    }
    const double u1 = (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = next_double();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.141592653589793238462643 * u2;
    cached = r * std::sin(theta);
    has_cached = true;
    return r * std::cos(theta);
  }
};

// Batched, multi-threaded view of Rng::next_normal() * stddev cast to float.
class NormalStream {
 public:
  explicit NormalStream(uint64_t seed) : rng_(seed) {}
  void fill(float* out, size_t n, double sd) {
    size_t i = 0;
    if (has_cached_ && n > 0) {
      out[i++] = static_cast<float>(sd * cached_);
      has_cached_ = false;
    }
    while (i < n) {
      const size_t pairs = std::min<size_t>((n - i + 1) / 2, kChunkPairs);
      draws_.resize(2 * pairs);
      for (size_t j = 0; j < 2 * pairs; ++j) draws_[j] = rng_.next_u64();
      normals_.resize(2 * pairs);
      const size_t take = std::min(n - i, 2 * pairs);
      transform(pairs, out + i, take, sd);
      i += take;
      if (take < 2 * pairs) {  // odd tail: keep the sin half for the next request
        cached_ = normals_[take];
        has_cached_ = true;
      }
    }
  }

 private:
  static constexpr size_t kChunkPairs = 1u << 22;
  void transform(size_t pairs, float* out, size_t take, double sd) {
    auto work = [&](size_t lo, size_t hi) {
      for (size_t j = lo; j < hi; ++j) {
        const double u1 = (static_cast<double>(draws_[2 * j] >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(draws_[2 * j + 1] >> 11) * 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.141592653589793238462643 * u2;
        normals_[2 * j] = r * std::cos(theta);
        normals_[2 * j + 1] = r * std::sin(theta);
        if (2 * j < take) out[2 * j] = static_cast<float>(sd * normals_[2 * j]);
        if (2 * j + 1 < take) out[2 * j + 1] = static_cast<float>(sd * normals_[2 * j + 1]);
      }
    };
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    if (pairs < 65536 || hw == 1) {
      work(0, pairs);
      return;
    }
    std::vector<std::thread> pool;
    const size_t chunk = (pairs + hw - 1) / hw;
    for (unsigned t = 0; t < hw; ++t) {
      const size_t lo = t * chunk, hi = std::min(pairs, lo + chunk);
      if (lo < hi) pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
  }
  Rng rng_;
  std::vector<uint64_t> draws_;
  std::vector<double> normals_;
  double cached_ = 0.0;
  bool has_cached_ = false;
};

struct Tensor {
  std::string name;
  int rows, cols, enc;
  uint64_t offset, length;
};

struct Cfg {
  int V = 131, d, L, H, F, S;
  std::vector<std::vector<int>> heads;
  std::vector<int> ffn;
};

std::string config_json(const Cfg& c) {
  std::string s = "{\"vocab_size\":" + std::to_string(c.V) + ",\"d_model\":" + std::to_string(c.d) +
                  ",\"n_layers\":" + std::to_string(c.L) + ",\"n_heads\":" + std::to_string(c.H) +
                  ",\"d_ff\":" + std::to_string(c.F) + ",\"max_seq_len\":" + std::to_string(c.S) +
                  ",\"active_heads\":[";
  for (size_t l = 0; l < c.heads.size(); ++l) {
    if (l) s += ",";
    s += "[";
    for (size_t i = 0; i < c.heads[l].size(); ++i) {
      if (i) s += ",";
      s += std::to_string(c.heads[l][i]);
    }
    s += "]";
  }
  s += "],\"active_ffn\":[";
  for (size_t l = 0; l < c.ffn.size(); ++l) {
    if (l) s += ",";
    s += std::to_string(c.ffn[l]);
  }
  return s + "]}";
}

// serialize_bundle (model.cpp:311-346): magic, u16 version 1, u32 header length, compact JSON
// header with fixed key order, blob.
std::vector<uint8_t> serialize(const Cfg& c, const std::vector<Tensor>& ts, const std::vector<uint8_t>& blob,
                               const std::string& recipe_id, const std::string& parent_hash) {
  std::string h = "{\"config\":" + config_json(c) + ",\"tensors\":[";
  for (size_t i = 0; i < ts.size(); ++i) {
    if (i) h += ",";
    h += "{\"name\":\"" + ts[i].name + "\",\"rows\":" + std::to_string(ts[i].rows) +
         ",\"cols\":" + std::to_string(ts[i].cols) + ",\"encoding\":" + std::to_string(ts[i].enc) +
         ",\"offset\":" + std::to_string(ts[i].offset) + ",\"length\":" + std::to_string(ts[i].length) + "}";
  }
  h += "],\"provenance\":{\"recipe_id\":\"" + recipe_id + "\",\"parent_hash\":\"" + parent_hash + "\"}}";
  std::vector<uint8_t> out;
  out.reserve(10 + h.size() + blob.size());
  out.insert(out.end(), {'I', 'O', 'L', 'M', 1, 0});
  const uint32_t hl = static_cast<uint32_t>(h.size());
  for (int i = 0; i < 4; ++i) out.push_back(static_cast<uint8_t>((hl >> (8 * i)) & 0xff));
  out.insert(out.end(), h.begin(), h.end());
  out.insert(out.end(), blob.begin(), blob.end());
  return out;
}

uint64_t fnv1a(const uint8_t* p, size_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

std::string hex16(uint64_t v) {
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(v));
  return buf;
}

bool is_weight(const std::string& n) {
  return n.find(".attn.w") != std::string::npos || n.find(".ffn.w") != std::string::npos;
}

// --- RTN (quant.cpp:23-38)
void rtn(const float* w, int rows, int cols, int qmax, std::vector<int8_t>& codes, std::vector<float>& scales) {
  codes.resize(static_cast<size_t>(rows) * cols);
  scales.resize(rows);
  for (int r = 0; r < rows; ++r) {
    float amax = 0.0f;
    for (int c = 0; c < cols; ++c) amax = std::max(amax, std::fabs(w[static_cast<size_t>(r) * cols + c]));
    scales[r] = amax == 0.0f ? 1.0f : amax / static_cast<float>(qmax);
    const double s = scales[r];
    for (int c = 0; c < cols; ++c) {
      const double q = std::nearbyint(w[static_cast<size_t>(r) * cols + c] / s);
      codes[static_cast<size_t>(r) * cols + c] =
          static_cast<int8_t>(std::min(static_cast<double>(qmax), std::max(-static_cast<double>(qmax), q)));
    }
  }
}

// magnitude two_of_four (quant.cpp:181-200): keep the 2 largest |w| per aligned group, ties keep
// the lower index.
void magnitude24(std::vector<float>& w, int rows, int cols, std::vector<uint8_t>& mask) {
  mask.assign(w.size(), 1);
  for (int r = 0; r < rows; ++r)
    for (int g = 0; g < cols / 4; ++g) {
      float* p = &w[static_cast<size_t>(r) * cols + g * 4];
      int order[4] = {0, 1, 2, 3};
      double sc[4];
      for (int j = 0; j < 4; ++j) sc[j] = std::fabs(p[j]);
      // stable sort by score desc, index asc
      for (int a = 1; a < 4; ++a)
        for (int b = a; b > 0; --b) {
          const int x = order[b - 1], y = order[b];
          if (sc[y] > sc[x] || (sc[y] == sc[x] && y < x)) std::swap(order[b - 1], order[b]);
        }
      for (int j = 2; j < 4; ++j) {
        p[order[j]] = 0.0f;
        mask[static_cast<size_t>(r) * cols + g * 4 + order[j]] = 0;
      }
    }
}

}  // namespace

extern "C" {

void synth_free(void* p) { std::free(p); }

uint64_t synth_fnv1a(const uint8_t* p, size_t n) { return fnv1a(p, n); }

// ToyModelParams::init(ModelConfig::dense(d,L,H,F,S), Rng(seed)).to_bundle() + serialize_bundle.
// quant: 0 dense f32; 8 -> q8 RTN; 4 -> q4 RTN; 24 -> magnitude 2:4 then q8 (sparse24_q8).
// prune_heads/prune_ffn (optional, may be NULL): per-layer active head count / ffn width; the
// surviving heads are the first `prune_heads[l]` heads and the first `prune_ffn[l]` channels (a
// structural shape for irregular-GEMM benchmarks; the reference chooses survivors by importance,
// prune.cpp:52-145, which changes values but not shapes).
int synth_toy_bundle(int d, int L, int H, int F, int S, uint64_t seed, int quant, const int* prune_heads,
                     const int* prune_ffn, uint8_t** out, size_t* out_len) {
  Cfg c;
  c.d = d;
  c.L = L;
  c.H = H;
  c.F = F;
  c.S = S;
  const int hd = d / H;
  c.heads.resize(L);
  c.ffn.resize(L);
  for (int l = 0; l < L; ++l) {
    const int nh = prune_heads ? prune_heads[l] : H;
    for (int h = 0; h < nh; ++h) c.heads[l].push_back(h);
    c.ffn[l] = prune_ffn ? prune_ffn[l] : F;
  }
  // The reference draws every normal from one Rng stream (train.cpp:21-25): pair j of the
  // Box-Muller stream consumes u64 draws 2j and 2j+1 and yields normals 2j (cos) and 2j+1 (sin)
  // (rng.cpp:60-73). Drawing the u64s is cheap and sequential; the transcendental transform is
  // done in parallel over chunks, giving the identical float stream. Tensors are planned first so
  // the serialized bundle is written once, in place.
  NormalStream ns(seed);
  const double base_std = 0.02;
  const double resid_std = base_std / std::sqrt(2.0 * L);
  struct Plan {
    std::string name;
    int rows, cols;
    double sd;     // > 0: normal(sd); else constant
    float value;   // constant fill
  };
  std::vector<Plan> plan;
  plan.push_back({"tok_embed", c.V, d, base_std, 0.f});
  plan.push_back({"pos_embed", S, d, base_std, 0.f});
  for (int l = 0; l < L; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    const int kh = static_cast<int>(c.heads[l].size()) * hd, f = c.ffn[l];
    plan.push_back({p + "attn_norm.gain", 1, d, 0.0, 1.f});
    plan.push_back({p + "attn_norm.bias", 1, d, 0.0, 0.f});
    plan.push_back({p + "attn.wq", kh, d, base_std, 0.f});
    plan.push_back({p + "attn.wk", kh, d, base_std, 0.f});
    plan.push_back({p + "attn.wv", kh, d, base_std, 0.f});
    plan.push_back({p + "attn.wo", d, kh, resid_std, 0.f});
    plan.push_back({p + "ffn_norm.gain", 1, d, 0.0, 1.f});
    plan.push_back({p + "ffn_norm.bias", 1, d, 0.0, 0.f});
    plan.push_back({p + "ffn.w_in", f, d, base_std, 0.f});
    plan.push_back({p + "ffn.w_out", d, f, resid_std, 0.f});
  }
  plan.push_back({"final_norm.gain", 1, d, 0.0, 1.f});
  plan.push_back({"final_norm.bias", 1, d, 0.0, 0.f});

  auto enc_of = [&](const Plan& t) {
    if (!is_weight(t.name) || quant == 0) return 0;
    if (quant == 8) return 1;
    if (quant == 4) return 2;
    return 3;
  };
  auto payload_bytes = [](int rows, int cols, int enc) -> uint64_t {
    const uint64_t r = rows, cc = cols;
    if (enc == 0) return r * cc * 4;
    if (enc == 1) return r * cc + r * 4;
    if (enc == 2) return r * ((cc + 1) / 2) + r * 4;
    const uint64_t g = cc / 4;
    return r * (cc / 2) + r * ((g + 1) / 2) + r * 4;
  };
  std::vector<Tensor> ts;
  uint64_t total = 0;
  for (const auto& t : plan) {
    const int enc = enc_of(t);
    if (enc == 3 && t.cols % 4 != 0) return 1;
    const uint64_t n = payload_bytes(t.rows, t.cols, enc);
    ts.push_back(Tensor{t.name, t.rows, t.cols, enc, total, n});
    total += n;
  }
  std::vector<uint8_t> empty;
  const std::vector<uint8_t> head = serialize(c, ts, empty, "", "");
  uint8_t* buf = static_cast<uint8_t*>(std::malloc(head.size() + total));
  if (!buf) return 2;
  std::memcpy(buf, head.data(), head.size());
  uint8_t* blob = buf + head.size();
  std::vector<float> w;
  for (size_t i = 0; i < plan.size(); ++i) {
    const Plan& t = plan[i];
    const Tensor& rec = ts[i];
    const size_t n = static_cast<size_t>(t.rows) * t.cols;
    w.resize(n);
    if (t.sd > 0) ns.fill(w.data(), n, t.sd);
    else std::fill(w.begin(), w.end(), t.value);
    uint8_t* dst = blob + rec.offset;
    if (rec.enc == 0) {
      std::memcpy(dst, w.data(), n * 4);
      continue;
    }
    std::vector<int8_t> codes;
    std::vector<float> scales;
    if (rec.enc == 1 || rec.enc == 2) {
      rtn(w.data(), t.rows, t.cols, rec.enc == 1 ? 127 : 7, codes, scales);
      size_t o = 0;
      if (rec.enc == 1) {
        std::memcpy(dst, codes.data(), codes.size());
        o = codes.size();
      } else {
        const size_t rb = (static_cast<size_t>(t.cols) + 1) / 2;
        std::memset(dst, 0, t.rows * rb);
        for (int r = 0; r < t.rows; ++r)
          for (int j = 0; j < t.cols; ++j) {
            const auto nib = static_cast<uint8_t>(codes[static_cast<size_t>(r) * t.cols + j] + 8);
            dst[r * rb + j / 2] |= (j % 2 == 0) ? nib : static_cast<uint8_t>(nib << 4);
          }
        o = t.rows * rb;
      }
      std::memcpy(dst + o, scales.data(), scales.size() * 4);
      continue;
    }
    // sparse24_q8: magnitude 2:4 then RTN q8 on the sparsified weights (compress.cpp:86-136)
    std::vector<uint8_t> mask;
    magnitude24(w, t.rows, t.cols, mask);
    rtn(w.data(), t.rows, t.cols, 127, codes, scales);
    const size_t groups = t.cols / 4, irb = (groups + 1) / 2;
    int8_t* kept = reinterpret_cast<int8_t*>(dst);
    uint8_t* idx = dst + static_cast<size_t>(t.rows) * groups * 2;
    std::memset(idx, 0, t.rows * irb);
    for (int r = 0; r < t.rows; ++r)
      for (size_t g = 0; g < groups; ++g) {
        int found = 0;
        uint8_t pos[2] = {0, 0};
        for (int j = 0; j < 4 && found < 2; ++j) {
          const size_t e = static_cast<size_t>(r) * t.cols + g * 4 + j;
          if (mask[e]) {
            kept[(static_cast<size_t>(r) * groups + g) * 2 + found] = codes[e];
            pos[found++] = static_cast<uint8_t>(j);
          }
        }
        const auto nib = static_cast<uint8_t>(pos[0] | (pos[1] << 2));
        idx[r * irb + g / 2] |= (g % 2 == 0) ? nib : static_cast<uint8_t>(nib << 4);
      }
    std::memcpy(idx + t.rows * irb, scales.data(), scales.size() * 4);
  }
  *out = buf;
  *out_len = head.size() + total;
  return 0;
}

// Synthetic table rows as token ids ([BOS] + instruction + row chars), CSR layout.
// Row r (global index first_row + i) draws its R chars from Rng(0x5EED0000 ^ r).
void synth_rows(const char* instruction, int64_t first_row, int64_t n_rows, int row_chars, int32_t* ids,
                int64_t* offsets) {
  const int il = static_cast<int>(std::strlen(instruction));
  const int per = 1 + il + row_chars;
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      int32_t* p = ids + i * per;
      p[0] = 129;
      for (int j = 0; j < il; ++j) p[1 + j] = static_cast<unsigned char>(instruction[j]);
      Rng rng(0x5EED0000ull ^ static_cast<uint64_t>(first_row + i));
      for (int j = 0; j < row_chars; ++j) p[1 + il + j] = 32 + static_cast<int32_t>(rng.next_below(95));
    }
  };
  const int threads = n_rows > 4096 ? 8 : 1;
  std::vector<std::thread> pool;
  const int64_t chunk = (n_rows + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n_rows, lo + chunk);
    if (lo < hi) pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
  for (int64_t i = 0; i <= n_rows; ++i) offsets[i] = i * per;
}

}  // extern "C"
