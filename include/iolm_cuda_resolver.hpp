// iolm_cuda_resolver.hpp - streaming replacement for the reference's prompt() operator resolver
// (PromptResolver + PromptCache, /root/reference/proj/src/exec.cpp:14-46 and :84-159,
// proj/include/iolm/exec.hpp:25-85), header-only C++20.
//
// The reference resolver renders every row's prompt, looks it up in an LRU PromptCache keyed by
// (bundle_hash, max_new_tokens, prompt), de-duplicates misses inside a "flush window" and calls
// ModelRuntime::batch_decode every `batch_size` (16) distinct prompts. On a B200 a 16-prompt call is
// all launch overhead. This resolver keeps the reference's observable behaviour exactly - outputs in
// row order, the cache contents / LRU order / hit and miss counts, and the invocation-count law
// (ExecStats::model_invocations = the distinct prompts of each reference flush window) - while
// submitting many closed windows to the model in ONE call of up to `device_batch` prompts:
//
//   * windows are closed exactly when the reference would flush them; at that point every prompt of
//     the window is inserted into the cache in the reference's order, as a *pending* entry whose
//     value is filled when the device batch it rides in completes;
//   * a later lookup that finds a pending entry is a cache hit (the reference had already decoded
//     it), and the row is bound to that pending slot;
//   * batch_decode results are independent of batch composition (proj/tests/test_model.cpp:240-267,
//     kept bitwise by the GPU runtime), so merging windows cannot change any output.
//
// Streaming: push() takes rows one at a time (no need to materialise the table's prompts), and
// take_ready() hands back the finished prefix of the output column in row order.
//
// `Model` is any type with the reference ModelRuntime's `batch_decode(span<const string>, int,
// FlopCounter&) const` and `bundle_hash() const` - iolm::cuda::ModelRuntime (the B200 runtime) or
// iolm::ModelRuntime itself (used by the CPU tests to prove equivalence with the reference).
#pragma once

#include <cstdint>
#include <list>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "iolm_cuda_runtime.hpp"  // error classes (the reference's own with IOLM_CUDA_WITH_REFERENCE_TYPES)

namespace iolm::cuda {

// Counters of the reference's ExecStats (exec.hpp:76-85) that the resolver maintains.
struct ResolverStats {
  uint64_t model_invocations = 0;  // prompts decoded through the model (reference accounting)
  uint64_t cache_hits = 0;
  uint64_t cache_misses = 0;
  uint64_t device_calls = 0;       // batch_decode calls actually issued (GPU-side accounting)
};

// LRU prompt cache with the semantics of iolm::PromptCache (exec.cpp:14-46): exact-key lookups
// refresh recency, inserts of an existing key overwrite and refresh, capacity 0 disables caching.
// Values may be pending (bound to a slot of an in-flight device batch).
class PromptCache {
 public:
  struct Key {
    uint64_t bundle_hash = 0;
    int max_new_tokens = 0;
    std::string prompt;
    bool operator==(const Key&) const = default;
  };
  struct Value {
    std::string text;
    int64_t slot = -1;  // >= 0: pending, the value is the output of resolver slot `slot`
  };

  explicit PromptCache(size_t capacity) : capacity_(capacity) {}
  bool enabled() const { return capacity_ > 0; }
  size_t size() const { return lru_.size(); }
  uint64_t hits() const { return hits_; }
  uint64_t misses() const { return misses_; }

  const Value* lookup(const Key& key) {
    auto it = index_.find(key);
    if (it == index_.end()) {
      ++misses_;
      return nullptr;
    }
    ++hits_;
    lru_.splice(lru_.begin(), lru_, it->second);
    return &it->second->value;
  }
  void insert(const Key& key, Value value) {
    if (capacity_ == 0) return;
    auto it = index_.find(key);
    if (it != index_.end()) {
      it->second->value = std::move(value);
      lru_.splice(lru_.begin(), lru_, it->second);
      return;
    }
    lru_.push_front(Entry{key, std::move(value)});
    index_[key] = lru_.begin();
    if (lru_.size() > capacity_) {
      index_.erase(lru_.back().key);
      lru_.pop_back();
    }
  }
  // Fills a pending entry (no recency change: the reference inserted the value at window close).
  void resolve_pending(const Key& key, int64_t slot, const std::string& text) {
    auto it = index_.find(key);
    if (it != index_.end() && it->second->value.slot == slot) it->second->value = Value{text, -1};
  }

 private:
  struct Entry {
    Key key;
    Value value;
  };
  struct KeyHash {
    size_t operator()(const Key& k) const {
      uint64_t h = 1469598103934665603ull;  // FNV-1a (the reference hashes the same fields)
      auto mix = [&](const void* p, size_t n) {
        const auto* b = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
      };
      mix(k.prompt.data(), k.prompt.size());
      mix(&k.bundle_hash, sizeof k.bundle_hash);
      mix(&k.max_new_tokens, sizeof k.max_new_tokens);
      return static_cast<size_t>(h);
    }
  };
  size_t capacity_;
  std::list<Entry> lru_;
  std::unordered_map<Key, typename std::list<Entry>::iterator, KeyHash> index_;
  uint64_t hits_ = 0, misses_ = 0;
};

template <typename Model, typename Counter>
class StreamingPromptResolver {
 public:
  // batch_size: the reference's ExecOptions::batch_size (flush-window size, accounting only);
  // device_batch: distinct prompts per model call (one GPU continuous-batching decode).
  StreamingPromptResolver(const Model& model, PromptCache& cache, int batch_size, int max_new_tokens,
                          ResolverStats& stats, Counter& counter, size_t device_batch = 32768)
      : model_(model), cache_(cache), batch_size_(batch_size < 1 ? 1 : batch_size), max_new_(max_new_tokens),
        stats_(stats), counter_(counter), device_batch_(device_batch < 1 ? 1 : device_batch),
        hash_(model.bundle_hash()) {}

  // Next table row's rendered prompt.
  void push(std::string_view prompt_sv) {
    std::string prompt(prompt_sv);
    const int64_t row = static_cast<int64_t>(row_slot_.size());
    if (cache_.enabled()) {
      if (const PromptCache::Value* hit = cache_.lookup(key(prompt))) {
        ++stats_.cache_hits;
        if (hit->slot >= 0) {
          row_slot_.push_back(hit->slot);
        } else {
          row_slot_.push_back(static_cast<int64_t>(slots_.size()));
          slots_.push_back(Slot{std::string(), hit->text, true, row});
        }
        return;
      }
      ++stats_.cache_misses;
    }
    auto it = window_index_.find(prompt);
    if (it != window_index_.end()) {
      row_slot_.push_back(it->second);
      return;
    }
    const int64_t slot = static_cast<int64_t>(slots_.size());
    if (window_first_row_ < 0) window_first_row_ = row;
    slots_.push_back(Slot{prompt, std::string(), false, window_first_row_});
    window_index_.emplace(std::move(prompt), slot);
    window_.push_back(slot);
    row_slot_.push_back(slot);
    if (static_cast<int>(window_.size()) == batch_size_) close_window();
  }

  // End of input: closes the last window and decodes everything still queued.
  void finish() {
    close_window();
    run_device();
  }

  // Output column entries for rows [taken, first unfinished row), in row order.
  std::vector<std::string> take_ready() {
    std::vector<std::string> out;
    while (taken_ < row_slot_.size() && slots_[row_slot_[taken_]].done) {
      out.push_back(slots_[row_slot_[taken_]].text);
      ++taken_;
    }
    return out;
  }

  // One-shot API with the reference PromptResolver::resolve signature (exec.cpp:95-122).
  std::vector<std::string> resolve(const std::vector<std::string>& prompts) {
    for (const auto& p : prompts) push(p);
    finish();
    return take_ready();
  }

 private:
  struct Slot {
    std::string prompt;
    std::string text;
    bool done = false;
    int64_t first_row = -1;  // first row of the reference flush window (error messages)
  };

  PromptCache::Key key(const std::string& p) const { return {hash_, max_new_, p}; }

  // The reference's flush(): the window's distinct prompts count as model invocations and enter the
  // cache (pending) in window order; the prompts join the device queue.
  void close_window() {
    if (window_.empty()) return;
    stats_.model_invocations += window_.size();
    for (int64_t s : window_) {
      cache_.insert(key(slots_[s].prompt), PromptCache::Value{std::string(), s});
      queue_.push_back(s);
    }
    window_.clear();
    window_index_.clear();
    window_first_row_ = -1;
    if (queue_.size() >= device_batch_) run_device();
  }

  void run_device() {
    size_t i = 0;
    while (i < queue_.size()) {
      const size_t n = std::min(device_batch_, queue_.size() - i);
      std::vector<std::string> prompts;
      prompts.reserve(n);
      for (size_t j = 0; j < n; ++j) prompts.push_back(slots_[queue_[i + j]].prompt);
      std::vector<std::string> decoded;
      try {
        decoded = model_.batch_decode(std::span<const std::string>(prompts), max_new_, counter_);
      } catch (const SequenceTooLong&) {
        replay_windows(i, n);  // reproduces the reference's failure point exactly, then throws
      }
      ++stats_.device_calls;
      fill(i, n, decoded);
      i += n;
    }
    queue_.clear();
  }

  void fill(size_t i, size_t n, std::vector<std::string>& decoded) {
    for (size_t j = 0; j < n; ++j) {
      Slot& s = slots_[queue_[i + j]];
      s.text = std::move(decoded[j]);
      s.done = true;
      cache_.resolve_pending(key(s.prompt), queue_[i + j], s.text);
    }
  }

  // Error path: decode the device batch window by window, as the reference would have, so the
  // windows before the failing one complete (and stay cached) and SequenceTooLong carries the
  // reference's " (row N)" suffix, N = first row of the failing flush window (exec.cpp:134-137).
  [[noreturn]] void replay_windows(size_t i, size_t n) {
    size_t a = i;
    while (a < i + n) {
      size_t b = a;
      while (b < i + n && slots_[queue_[b]].first_row == slots_[queue_[a]].first_row) ++b;
      std::vector<std::string> prompts;
      for (size_t j = a; j < b; ++j) prompts.push_back(slots_[queue_[j]].prompt);
      std::vector<std::string> decoded;
      try {
        decoded = model_.batch_decode(std::span<const std::string>(prompts), max_new_, counter_);
      } catch (const SequenceTooLong& e) {
        throw SequenceTooLong(std::string(e.what()) + " (row " + std::to_string(slots_[queue_[a]].first_row) + ")");
      }
      ++stats_.device_calls;
      fill(a, b - a, decoded);
      a = b;
    }
    throw SequenceTooLong("StreamingPromptResolver: device batch failed but no flush window did");
  }

  const Model& model_;
  PromptCache& cache_;
  int batch_size_;
  int max_new_;
  ResolverStats& stats_;
  Counter& counter_;
  size_t device_batch_;
  uint64_t hash_;
  std::vector<Slot> slots_;
  std::vector<int64_t> row_slot_;
  size_t taken_ = 0;
  std::vector<int64_t> window_;
  std::map<std::string, int64_t> window_index_;
  int64_t window_first_row_ = -1;
  std::vector<int64_t> queue_;
};

}  // namespace iolm::cuda
