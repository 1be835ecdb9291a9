// TEST INFRASTRUCTURE ONLY - never linked into or called by the product path.
//
// C-ABI wrapper around the UNMODIFIED reference implementation, compiled from the read-only
// sources under /root/reference/proj/src by oracle/Makefile into oracle/_ref/libiolm_ref.so.
// It lets the Python tests (and bench.py's reference arm / cpu_baseline leg) drive the
// reference's own public API: ToyModelParams::init + to_bundle (train.cpp:45-75,128-134),
// serialize/deserialize_bundle (model.cpp:311-406), ModelRuntime::forward/batch_decode
// (runtime.cpp:217-309), capture_calibration + apply_recipe (calib.cpp:20-62, compress.cpp:52-146).
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "iolm/calib.hpp"
#include "iolm/common.hpp"
#include "iolm/compress.hpp"
#include "iolm/model.hpp"
#include "iolm/recipe.hpp"
#include "iolm/rng.hpp"
#include "iolm/runtime.hpp"
#include "iolm/train.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const iolm::SequenceTooLong& e) {
    g_err = e.what();
    return 2;
  } catch (const iolm::ContractViolation& e) {
    g_err = e.what();
    return 1;
  } catch (const iolm::CorruptHeader& e) {
    g_err = e.what();
    return 6;
  } catch (const iolm::TruncatedBlob& e) {
    g_err = e.what();
    return 7;
  } catch (const iolm::UnknownEncoding& e) {
    g_err = e.what();
    return 8;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

void emit(const std::vector<uint8_t>& bytes, uint8_t** out, size_t* len) {
  *out = static_cast<uint8_t*>(std::malloc(bytes.size()));
  std::memcpy(*out, bytes.data(), bytes.size());
  *len = bytes.size();
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// ToyModelParams::init(ModelConfig::dense(d, L, H, F, S), Rng(seed)).to_bundle(), serialized.
int ref_toy_bundle(int d, int L, int H, int F, int S, uint64_t seed, uint8_t** out, size_t* len) {
  return guard([&] {
    iolm::Rng rng(seed);
    auto params = iolm::ToyModelParams::init(iolm::ModelConfig::dense(d, L, H, F, S), rng);
    emit(iolm::serialize_bundle(params.to_bundle()), out, len);
  });
}

// apply_recipe(bundle, recipe, capture_calibration(runtime, prompts)) - the reference's own
// compression pipeline; returns the compressed bundle bytes.
int ref_compress(const uint8_t* bytes, size_t len, const char* recipe_json, const char* chars,
                 const int64_t* offsets, int n_prompts, uint64_t calib_seed, uint8_t** out,
                 size_t* out_len) {
  return guard([&] {
    auto bundle = iolm::deserialize_bundle({bytes, len});
    auto recipe = iolm::CompressionRecipe::from_json(nlohmann::json::parse(recipe_json));
    std::vector<std::string> prompts;
    for (int i = 0; i < n_prompts; ++i)
      prompts.emplace_back(chars + offsets[i], chars + offsets[i + 1]);
    iolm::ModelRuntime rt(bundle);
    iolm::Rng rng(calib_seed);
    auto calib = iolm::capture_calibration(rt, prompts, n_prompts, rng);
    emit(iolm::serialize_bundle(iolm::apply_recipe(bundle, recipe, calib)), out, out_len);
  });
}

void* ref_runtime_create(const uint8_t* bytes, size_t len) {
  iolm::ModelRuntime* rt = nullptr;
  int st = guard([&] { rt = new iolm::ModelRuntime(iolm::deserialize_bundle({bytes, len})); });
  return st == 0 ? rt : nullptr;
}

void ref_runtime_destroy(void* rt) { delete static_cast<iolm::ModelRuntime*>(rt); }

uint64_t ref_runtime_hash(void* rt) { return static_cast<iolm::ModelRuntime*>(rt)->bundle_hash(); }

int ref_forward(void* rt, const int* ids, const uint8_t* mask, int n, float* logits,
                uint64_t* madds) {
  return guard([&] {
    iolm::FlopCounter counter;
    std::span<const uint8_t> m;
    if (mask) m = {mask, static_cast<size_t>(n)};
    auto out = static_cast<iolm::ModelRuntime*>(rt)->forward({ids, static_cast<size_t>(n)}, m,
                                                              counter);
    std::memcpy(logits, out.data.data(), sizeof(float) * out.data.size());
    if (madds) *madds = counter.total();
  });
}

// ModelRuntime::batch_decode over chunks of `batch_size` prompts (the executor's flush window,
// exec.hpp:70-74), chunks spread over `threads` host threads (the runtime is const and
// thread-safe). out: n * max_new chars, out_len: rendered lengths.
int ref_batch_decode(void* rtp, const char* chars, const int64_t* offsets, int n, int max_new,
                     char* out, int* out_len, uint64_t* madds, int threads, int batch_size) {
  auto* rt = static_cast<iolm::ModelRuntime*>(rtp);
  if (threads < 1) threads = 1;
  if (batch_size < 1) batch_size = 1;
  const int chunks = (n + batch_size - 1) / batch_size;
  std::atomic<int> next{0};
  std::atomic<uint64_t> total{0};
  std::vector<int> status(threads, 0);
  std::vector<std::string> errs(threads);
  auto worker = [&](int t) {
    iolm::FlopCounter counter;
    status[t] = guard([&] {
      for (int c = next++; c < chunks; c = next++) {
        const int lo = c * batch_size, hi = std::min(n, lo + batch_size);
        std::vector<std::string> prompts;
        for (int i = lo; i < hi; ++i) prompts.emplace_back(chars + offsets[i], chars + offsets[i + 1]);
        auto res = rt->batch_decode(prompts, max_new, counter);
        for (int i = lo; i < hi; ++i) {
          const auto& s = res[i - lo];
          std::memcpy(out + static_cast<size_t>(i) * max_new, s.data(), s.size());
          out_len[i] = static_cast<int>(s.size());
        }
      }
    });
    if (status[t]) errs[t] = g_err;
    total += counter.total();
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  for (int t = 0; t < threads; ++t)
    if (status[t]) {
      g_err = errs[t];
      return status[t];
    }
  if (madds) *madds = total.load();
  return 0;
}

}  // extern "C"
