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
// take_ready() hands back the finished prefix of the output column in row order; rows and decoded
// slots are released once handed back, so host memory is bounded by the rows in flight (about
// device_batch x batch_size), not by the table.
//
// Errors: everything since the last completed device call is one transaction. If a device call
// throws (SequenceTooLong, ContractViolation, GpuError, ...), the cache (contents, LRU order, hit /
// miss counters) and the stats are rolled back to the transaction start and the transaction's rows
// are replayed exactly as the reference executes them - lookup, window, synchronous batch_decode per
// flush window - so the exception, its " (row N)" suffix, the cache and the stats are the reference's
// at its failure point (exec.cpp:95-146): earlier windows decoded and cached, the failing window
// neither counted nor cached, later rows never looked up. No pending entry survives a failure.
//
// `Model` is any type with the reference ModelRuntime's `batch_decode(span<const string>, int,
// FlopCounter&) const` and `bundle_hash() const` - iolm::cuda::ModelRuntime (the B200 runtime) or
// iolm::ModelRuntime itself (used by the CPU tests to prove equivalence with the reference).
#pragma once

#include <cstdint>
#include <deque>
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
// Values may be pending (bound to a slot of an in-flight device batch of one resolver). Mutations can
// be journaled (begin / commit / rollback) so a failed device batch leaves no trace.
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
    int64_t slot = -1;            // >= 0: pending, the value is the output of resolver slot `slot`
    const void* owner = nullptr;  // the resolver whose slot it is
  };

  explicit PromptCache(size_t capacity) : capacity_(capacity) {}
  PromptCache(const PromptCache&) = delete;
  PromptCache& operator=(const PromptCache&) = delete;
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
    to_front(it->second);
    return &it->second->value;
  }
  void insert(const Key& key, Value value) {
    if (capacity_ == 0) return;
    auto it = index_.find(key);
    if (it != index_.end()) {
      if (journaling_) log_.push_back(Op{Op::SET, it->second, it->second->value});
      it->second->value = std::move(value);
      to_front(it->second);
      return;
    }
    lru_.push_front(Entry{key, std::move(value)});
    index_[key] = lru_.begin();
    if (journaling_) log_.push_back(Op{Op::INSERT, lru_.begin(), {}});
    if (lru_.size() > capacity_) {
      auto last = std::prev(lru_.end());
      index_.erase(last->key);
      if (journaling_) {  // keep the node itself so a rollback restores it in place
        graveyard_.splice(graveyard_.end(), lru_, last);
        log_.push_back(Op{Op::EVICT, last, {}});
      } else {
        lru_.pop_back();
      }
    }
  }
  // Fills a pending entry (no recency change: the reference inserted the value at window close).
  void resolve_pending(const Key& key, const void* owner, int64_t slot, const std::string& text) {
    auto it = index_.find(key);
    if (it == index_.end() || it->second->value.slot != slot || it->second->value.owner != owner) return;
    if (journaling_) log_.push_back(Op{Op::SET, it->second, it->second->value});
    it->second->value = Value{text, -1, nullptr};
  }

  // Journal of every mutation (and the counters) from begin() until commit() / rollback().
  void begin() {
    log_.clear();
    graveyard_.clear();
    journaling_ = true;
    saved_hits_ = hits_;
    saved_misses_ = misses_;
  }
  void commit() {
    log_.clear();
    graveyard_.clear();
    journaling_ = false;
  }
  void rollback() {
    for (auto op = log_.rbegin(); op != log_.rend(); ++op) {
      switch (op->kind) {
        case Op::MOVE: lru_.splice(op->next, lru_, op->it); break;
        case Op::SET: op->it->value = op->old; break;
        case Op::INSERT:
          index_.erase(op->it->key);
          lru_.erase(op->it);
          break;
        case Op::EVICT:
          lru_.splice(lru_.end(), graveyard_, op->it);
          index_[op->it->key] = op->it;
          break;
      }
    }
    hits_ = saved_hits_;
    misses_ = saved_misses_;
    commit();
  }

 private:
  struct Entry {
    Key key;
    Value value;
  };
  using Iter = typename std::list<Entry>::iterator;
  struct Op {
    enum Kind { MOVE, SET, INSERT, EVICT } kind;
    Iter it;
    Value old;
    Iter next{};  // MOVE: the node that followed `it` before it moved to the front
  };
  void to_front(Iter it) {
    if (it == lru_.begin()) return;
    if (journaling_) log_.push_back(Op{Op::MOVE, it, {}, std::next(it)});
    lru_.splice(lru_.begin(), lru_, it);
  }
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
  std::unordered_map<Key, Iter, KeyHash> index_;
  uint64_t hits_ = 0, misses_ = 0;
  bool journaling_ = false;
  std::vector<Op> log_;
  std::list<Entry> graveyard_;
  uint64_t saved_hits_ = 0, saved_misses_ = 0;
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
  StreamingPromptResolver(const StreamingPromptResolver&) = delete;
  StreamingPromptResolver& operator=(const StreamingPromptResolver&) = delete;
  ~StreamingPromptResolver() {
    if (in_txn_) cache_.rollback();  // abandoned mid-transaction: no pending entry may outlive us
  }

  // Next table row's rendered prompt.
  void push(std::string_view prompt_sv) {
    if (failed_) throw ContractViolation("StreamingPromptResolver: a previous device batch failed");
    if (!in_txn_) begin_txn();
    txn_prompts_.emplace_back(prompt_sv);
    process_row(txn_prompts_.back());
    if (window_.empty() && queue_.empty()) commit_txn();  // nothing in flight: rows are final
  }

  // End of input: closes the last window and decodes everything still queued.
  void finish() {
    if (failed_) throw ContractViolation("StreamingPromptResolver: a previous device batch failed");
    if (!in_txn_) return;
    close_window();
    run_device();
  }

  // Output column entries for rows [taken, first unfinished row), in row order (rows of completed
  // transactions only), released from the resolver as they are handed back.
  std::vector<std::string> take_ready() {
    std::vector<std::string> out;
    const int64_t limit = in_txn_ ? txn_row0_ : n_rows_;
    while (row_base_ < limit) {
      Row& r = rows_.front();
      if (r.slot >= 0) {
        const Slot& s = slot(r.slot);
        if (!s.done) break;
        out.push_back(s.text);
      } else {
        out.push_back(std::move(r.text));
      }
      rows_.pop_front();
      ++row_base_;
    }
    // a slot is referenced only by rows up to its last binding; once those are handed back and the
    // slot is decoded (its cache entry resolved), nothing refers to it any more
    while (!slots_.empty() && slots_.front().done && slots_.front().last_row < row_base_) {
      slots_.pop_front();
      ++slot_base_;
    }
    return out;
  }

  // One-shot API with the reference PromptResolver::resolve signature (exec.cpp:95-122).
  std::vector<std::string> resolve(const std::vector<std::string>& prompts) {
    for (const auto& p : prompts) push(p);
    finish();
    return take_ready();
  }

  // Rows / decoded slots currently held (memory accounting for the streaming tests).
  size_t rows_held() const { return rows_.size(); }
  size_t slots_held() const { return slots_.size(); }

 private:
  struct Slot {
    std::string prompt;
    std::string text;
    bool done = false;
    int64_t first_row = -1;  // first row of the reference flush window (error messages)
    int64_t last_row = -1;   // last row bound to this slot
  };
  struct Row {
    int64_t slot = -1;  // >= 0: the row's output is that slot's; < 0: `text` is final (cache hit)
    std::string text;
  };

  PromptCache::Key key(const std::string& p) const { return {hash_, max_new_, p}; }
  Slot& slot(int64_t id) { return slots_[static_cast<size_t>(id - slot_base_)]; }
  int64_t next_slot_id() const { return slot_base_ + static_cast<int64_t>(slots_.size()); }

  void process_row(const std::string& prompt) {
    const int64_t row = n_rows_++;
    if (cache_.enabled()) {
      if (const PromptCache::Value* hit = cache_.lookup(key(prompt))) {
        ++stats_.cache_hits;
        if (hit->slot >= 0) {
          if (hit->owner != this) throw ContractViolation("PromptCache: entry pending in another resolver");
          slot(hit->slot).last_row = row;
          rows_.push_back(Row{hit->slot, {}});
        } else {
          rows_.push_back(Row{-1, hit->text});
        }
        return;
      }
      ++stats_.cache_misses;
    }
    auto it = window_index_.find(prompt);
    if (it != window_index_.end()) {
      slot(it->second).last_row = row;
      rows_.push_back(Row{it->second, {}});
      return;
    }
    const int64_t s = next_slot_id();
    if (window_first_row_ < 0) window_first_row_ = row;
    slots_.push_back(Slot{prompt, std::string(), false, window_first_row_, row});
    window_index_.emplace(prompt, s);
    window_.push_back(s);
    rows_.push_back(Row{s, {}});
    if (static_cast<int>(window_.size()) == batch_size_) close_window();
  }

  // The reference's flush(): the window's distinct prompts count as model invocations and enter the
  // cache (pending) in window order; the prompts join the device queue.
  void close_window() {
    if (window_.empty()) return;
    stats_.model_invocations += window_.size();
    for (int64_t s : window_) {
      cache_.insert(key(slot(s).prompt), PromptCache::Value{std::string(), s, this});
      queue_.push_back(s);
    }
    window_.clear();
    window_index_.clear();
    window_first_row_ = -1;
    if (queue_.size() >= device_batch_) run_device();
  }

  void run_device() {
    try {
      size_t i = 0;
      while (i < queue_.size()) {
        const size_t n = std::min(device_batch_, queue_.size() - i);
        std::vector<std::string> prompts;
        prompts.reserve(n);
        for (size_t j = 0; j < n; ++j) prompts.push_back(slot(queue_[i + j]).prompt);
        std::vector<std::string> decoded = model_.batch_decode(std::span<const std::string>(prompts), max_new_, counter_);
        ++stats_.device_calls;
        for (size_t j = 0; j < n; ++j) {
          Slot& s = slot(queue_[i + j]);
          s.text = std::move(decoded[j]);
          s.done = true;
          cache_.resolve_pending(key(s.prompt), this, queue_[i + j], s.text);
          std::string().swap(s.prompt);  // only the pending cache key needed it
        }
        i += n;
      }
    } catch (...) {
      rollback_and_replay();  // throws the reference's exception (or returns after a transient error)
      return;
    }
    queue_.clear();
    commit_txn();
  }

  void begin_txn() {
    cache_.begin();
    in_txn_ = true;
    txn_stats_ = stats_;
    txn_row0_ = n_rows_;
    txn_slot0_ = next_slot_id();
    txn_prompts_.clear();
  }
  void commit_txn() {
    cache_.commit();
    in_txn_ = false;
    txn_prompts_.clear();
  }

  // Undo the transaction and run its rows as the reference does: lookup per row, synchronous
  // batch_decode per flush window, cache inserts after each successful window (exec.cpp:95-146).
  void rollback_and_replay() {
    cache_.rollback();
    in_txn_ = false;
    stats_ = txn_stats_;
    rows_.resize(static_cast<size_t>(txn_row0_ - row_base_));
    slots_.resize(static_cast<size_t>(txn_slot0_ - slot_base_));
    n_rows_ = txn_row0_;
    window_.clear();
    window_index_.clear();
    window_first_row_ = -1;
    queue_.clear();
    std::vector<std::string> prompts = std::move(txn_prompts_);
    txn_prompts_.clear();
    failed_ = true;  // until the replay completes
    std::vector<int64_t> win;
    std::map<std::string, int64_t> win_index;
    auto flush = [&] {
      if (win.empty()) return;
      std::vector<std::string> ps;
      for (int64_t s : win) ps.push_back(slot(s).prompt);
      std::vector<std::string> decoded;
      try {
        decoded = model_.batch_decode(std::span<const std::string>(ps), max_new_, counter_);
      } catch (const SequenceTooLong& e) {
        throw SequenceTooLong(std::string(e.what()) + " (row " + std::to_string(slot(win.front()).first_row) + ")");
      }
      ++stats_.device_calls;
      stats_.model_invocations += win.size();
      for (size_t j = 0; j < win.size(); ++j) {
        Slot& s = slot(win[j]);
        s.text = std::move(decoded[j]);
        s.done = true;
        cache_.insert(key(s.prompt), PromptCache::Value{s.text, -1, nullptr});
      }
      win.clear();
      win_index.clear();
    };
    for (const std::string& prompt : prompts) {
      const int64_t row = n_rows_++;
      if (cache_.enabled()) {
        if (const PromptCache::Value* hit = cache_.lookup(key(prompt))) {
          ++stats_.cache_hits;
          rows_.push_back(Row{-1, hit->text});
          continue;
        }
        ++stats_.cache_misses;
      }
      auto it = win_index.find(prompt);
      if (it != win_index.end()) {
        slot(it->second).last_row = row;
        rows_.push_back(Row{it->second, {}});
        continue;
      }
      const int64_t s = next_slot_id();
      slots_.push_back(Slot{prompt, std::string(), false, win.empty() ? row : slot(win.front()).first_row, row});
      win_index.emplace(prompt, s);
      win.push_back(s);
      rows_.push_back(Row{s, {}});
      if (static_cast<int>(win.size()) == batch_size_) flush();
    }
    flush();
    failed_ = false;  // the failure did not reproduce (transient): the rows are decoded and final
  }

  const Model& model_;
  PromptCache& cache_;
  int batch_size_;
  int max_new_;
  ResolverStats& stats_;
  Counter& counter_;
  size_t device_batch_;
  uint64_t hash_;
  std::deque<Slot> slots_;
  int64_t slot_base_ = 0;  // id of slots_.front()
  std::deque<Row> rows_;
  int64_t row_base_ = 0;  // index of rows_.front() = rows handed back so far
  int64_t n_rows_ = 0;
  std::vector<int64_t> window_;
  std::map<std::string, int64_t> window_index_;
  int64_t window_first_row_ = -1;
  std::vector<int64_t> queue_;
  // transaction: everything since the last completed device call
  bool in_txn_ = false, failed_ = false;
  ResolverStats txn_stats_{};
  int64_t txn_row0_ = 0, txn_slot0_ = 0;
  std::vector<std::string> txn_prompts_;
};

}  // namespace iolm::cuda
