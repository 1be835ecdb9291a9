// Streaming prompt() resolver (include/iolm_cuda_resolver.hpp) against the reference executor
// (iolm::execute -> PromptResolver, /root/reference/proj/src/exec.cpp:84-159, :353-370).
//
// CPU build (default): the resolver drives the reference's own iolm::ModelRuntime, so every output
// must be IDENTICAL to iolm::execute's, and so must the ExecStats it maintains (model_invocations,
// cache_hits, cache_misses) for every batch size, cache capacity (incl. eviction) and device batch
// size - the scenarios of proj/tests/test_query.cpp:375-431 plus streaming take_ready().
// GPU build (-DWITH_GPU): the same scenarios with iolm::cuda::ModelRuntime (B200) as the model;
// stats must still match the reference exactly, outputs must equal the GPU's own batch_decode of
// the distinct prompts (batch invariance) and agree with the CPU reference on >= 99% of rows.
// Built by oracle/Makefile (targets resolver / resolver_gpu) - test only.
#define IOLM_CUDA_WITH_REFERENCE_TYPES
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <set>
#include <string>
#include <vector>

#include "iolm/exec.hpp"
#include "iolm/rng.hpp"
#include "iolm/sql.hpp"
#include "iolm/table.hpp"
#include "iolm/train.hpp"
#include "iolm_cuda_join.hpp"
#include "iolm_cuda_resolver.hpp"

static int fails = 0;
#define EXPECT(c, msg)                                      \
  do {                                                      \
    if (!(c)) {                                             \
      std::printf("FAIL %s (line %d)\n", msg, __LINE__);    \
      ++fails;                                              \
    }                                                       \
  } while (0)

namespace {

iolm::Table words_table(int n, uint64_t seed) {
  iolm::Table t;
  t.name = "t";
  iolm::Column c;
  c.name = "w";
  c.type = iolm::ColumnType::text;
  iolm::Rng rng(seed);
  for (int i = 0; i < n; ++i) {
    std::string s;
    for (int j = 0; j < 1 + static_cast<int>(rng.next_below(10)); ++j)
      s.push_back(static_cast<char>('a' + rng.next_below(26)));
    if (i % 2 == 1) s = c.texts[rng.next_below(c.texts.size())];  // ~50% duplicates
    c.texts.push_back(s);
  }
  t.columns.push_back(c);
  t.row_count = static_cast<size_t>(n);
  return t;
}

struct RefRun {
  std::vector<std::string> out;
  iolm::ExecStats stats;
};

RefRun run_reference(const iolm::ModelRuntime& cpu, const iolm::Table& t, int batch, size_t capacity, int max_new) {
  const iolm::QueryPlan plan = iolm::parse_query("SELECT prompt('echo ' || w) AS r FROM t");
  iolm::PromptCache cache(capacity);
  iolm::ExecOptions opts;
  opts.batch_size = batch;
  opts.max_new_tokens = max_new;
  opts.cache_capacity = capacity;
  RefRun r;
  iolm::FlopCounter fc;
  const iolm::Table out = iolm::execute(plan, {{"t", t}}, cpu, cache, opts, r.stats, fc);
  r.out = out.columns[0].texts;
  return r;
}

std::vector<std::string> run_reference_on(const iolm::ModelRuntime& cpu, const iolm::Table& t, int batch,
                                          iolm::PromptCache& cache, iolm::ExecStats& stats, int max_new) {
  const iolm::QueryPlan plan = iolm::parse_query("SELECT prompt('echo ' || w) AS r FROM t");
  iolm::ExecOptions opts;
  opts.batch_size = batch;
  opts.max_new_tokens = max_new;
  iolm::FlopCounter fc;
  return iolm::execute(plan, {{"t", t}}, cpu, cache, opts, stats, fc).columns[0].texts;
}

}  // namespace

int main() {
  iolm::Rng wrng(21);
  const auto bundle = iolm::ToyModelParams::init(iolm::ModelConfig::dense(32, 2, 2, 64, 96), wrng).to_bundle();
  const iolm::ModelRuntime cpu(bundle);
#ifdef WITH_GPU
  const iolm::cuda::ModelRuntime model(bundle);
#else
  const iolm::ModelRuntime& model = cpu;
#endif
  using Resolver = iolm::cuda::StreamingPromptResolver<std::remove_cv_t<std::remove_reference_t<decltype(model)>>,
                                                       iolm::FlopCounter>;
  const iolm::Table t = words_table(40, 5);
  std::vector<std::string> prompts;
  for (const auto& w : t.columns[0].texts) prompts.push_back("echo " + w);
  const size_t distinct = std::set<std::string>(prompts.begin(), prompts.end()).size();

  int scenarios = 0;
  size_t agree = 0, total = 0;
  for (int batch : {1, 4, 16, 64})
    for (size_t capacity : {size_t{0}, size_t{3}, size_t{1024}})
      for (size_t device_batch : {size_t{1}, size_t{7}, size_t{100000}}) {
        const RefRun ref = run_reference(cpu, t, batch, capacity, 6);
        iolm::cuda::PromptCache cache(capacity);
        iolm::cuda::ResolverStats st;
        iolm::FlopCounter fc;
        Resolver res(model, cache, batch, 6, st, fc, device_batch);
        const auto out = res.resolve(prompts);
        ++scenarios;
        EXPECT(out.size() == ref.out.size(), "row count");
        EXPECT(st.model_invocations == ref.stats.model_invocations, "model_invocations");
        EXPECT(st.cache_hits == ref.stats.cache_hits, "cache_hits");
        EXPECT(st.cache_misses == ref.stats.cache_misses, "cache_misses");
        if (capacity == 1024) EXPECT(st.model_invocations == distinct, "invocation law: distinct prompts");
#ifdef WITH_GPU
        // outputs = the GPU's own decode of each distinct prompt (batch invariance), rows aligned
        const std::set<std::string> uset(prompts.begin(), prompts.end());
        const std::vector<std::string> uniq(uset.begin(), uset.end());
        iolm::FlopCounter f2;
        const auto solo = model.batch_decode(std::span<const std::string>(uniq), 6, f2);
        for (size_t i = 0; i < prompts.size(); ++i) {
          const size_t k = std::lower_bound(uniq.begin(), uniq.end(), prompts[i]) - uniq.begin();
          EXPECT(out[i] == solo[k], "gpu output = gpu batch_decode of the distinct prompt");
          agree += out[i] == ref.out[i];
          ++total;
        }
#else
        EXPECT(out == ref.out, "outputs identical to iolm::execute");
#endif
      }

  // streaming: rows pushed one at a time, outputs drained as they complete
  {
    const RefRun ref = run_reference(cpu, t, 16, 1024, 6);
    iolm::cuda::PromptCache cache(1024);
    iolm::cuda::ResolverStats st;
    iolm::FlopCounter fc;
    Resolver res(model, cache, 16, 6, st, fc, 5);
    std::vector<std::string> got;
    for (const auto& p : prompts) {
      res.push(p);
      for (auto& s : res.take_ready()) got.push_back(std::move(s));
    }
    res.finish();
    for (auto& s : res.take_ready()) got.push_back(std::move(s));
    EXPECT(got.size() == prompts.size(), "streaming row count");
    EXPECT(st.model_invocations == ref.stats.model_invocations && st.cache_hits == ref.stats.cache_hits,
           "streaming stats");
#ifndef WITH_GPU
    EXPECT(got == ref.out, "streaming outputs");
#endif
    // the same cache serves a second identical query entirely from hits
    iolm::cuda::ResolverStats st2;
    Resolver res2(model, cache, 16, 6, st2, fc, 5);
    const auto again = res2.resolve(prompts);
    EXPECT(st2.model_invocations == 0 && st2.cache_hits == prompts.size(), "second query all hits");
    EXPECT(again == got, "second query outputs");
  }

  // SequenceTooLong carries the first row of the failing reference flush window
  {
    iolm::Table t2 = t;
    t2.columns[0].texts.resize(20);
    t2.columns[0].texts[17] = std::string(200, 'x');  // "echo " + 200 chars > max_seq_len 96
    t2.row_count = 20;
    std::string ref_msg, got_msg;
    try {
      run_reference(cpu, t2, 2, 0, 6);
    } catch (const iolm::SequenceTooLong& e) {
      ref_msg = e.what();
    }
    std::vector<std::string> p3;
    for (const auto& w : t2.columns[0].texts) p3.push_back("echo " + w);
    iolm::cuda::PromptCache cache(0);
    iolm::cuda::ResolverStats st;
    iolm::FlopCounter fc;
    Resolver res(model, cache, 2, 6, st, fc, 100000);
    try {
      res.resolve(p3);
    } catch (const iolm::SequenceTooLong& e) {
      got_msg = e.what();
    }
    const auto tail = [](const std::string& s) { return s.substr(s.rfind(" (row ") == std::string::npos ? 0 : s.rfind(" (row ")); };
    EXPECT(!ref_msg.empty() && !got_msg.empty(), "SequenceTooLong raised by both");
    std::printf("SequenceTooLong: reference \"%s\" / resolver \"%s\"\n", ref_msg.c_str(), got_msg.c_str());
    EXPECT(tail(ref_msg) == tail(got_msg), "SequenceTooLong row suffix");
  }

  // A failing query on a SHARED cache (SequenceTooLong / non-ASCII ContractViolation at row 25):
  // the cache contents, LRU order and counters and the ExecStats must be the reference's at its
  // failure point (earlier flush windows decoded and cached, the failing one not, later rows never
  // looked up), and the same cache must then serve the next query exactly like the reference's.
  for (int kind = 0; kind < 2; ++kind)
    for (int batch : {2, 16})
      for (size_t capacity : {size_t{0}, size_t{5}, size_t{1024}})
        for (size_t device_batch : {size_t{1}, size_t{7}, size_t{100000}}) {
          iolm::Table bad = words_table(40, 9);
          bad.columns[0].texts[25] = kind == 0 ? std::string(200, 'x') : std::string("caf\xe9");
          std::vector<std::string> pb;
          for (const auto& w : bad.columns[0].texts) pb.push_back("echo " + w);
          iolm::PromptCache rcache(capacity);
          iolm::ExecStats rs;
          std::string rmsg = "none", gmsg = "none";
          int rkind = -1, gkind = -1;
          try {
            run_reference_on(cpu, bad, batch, rcache, rs, 6);
          } catch (const iolm::SequenceTooLong& e) {
            rkind = 0, rmsg = e.what();
          } catch (const iolm::ContractViolation& e) {
            rkind = 1, rmsg = e.what();
          }
          iolm::cuda::PromptCache cache(capacity);
          iolm::cuda::ResolverStats st;
          iolm::FlopCounter fc;
          {
            Resolver res(model, cache, batch, 6, st, fc, device_batch);
            try {
              for (const auto& p : pb) {
                res.push(p);
                res.take_ready();
              }
              res.finish();
            } catch (const iolm::SequenceTooLong& e) {
              gkind = 0, gmsg = e.what();
            } catch (const iolm::ContractViolation& e) {
              gkind = 1, gmsg = e.what();
            }
          }
          const auto tail = [](const std::string& m) { return m.substr(m.rfind(" (row ") == std::string::npos ? m.size() : m.rfind(" (row ")); };
          EXPECT(rkind == kind && gkind == kind, "failing query raises the reference's exception class");
          EXPECT(tail(rmsg) == tail(gmsg), "failing query: row suffix");
          EXPECT(st.model_invocations == rs.model_invocations && st.cache_hits == rs.cache_hits &&
                     st.cache_misses == rs.cache_misses,
                 "failing query: stats at the failure point");
          EXPECT(cache.size() == rcache.size() && cache.hits() == rcache.hits() && cache.misses() == rcache.misses(),
                 "failing query: cache size and counters");
          // the next query through the same cache: identical stats (LRU contents and order) and outputs
          iolm::ExecStats rs2;
          const auto rout = run_reference_on(cpu, t, batch, rcache, rs2, 6);
          iolm::cuda::ResolverStats st2;
          Resolver res2(model, cache, batch, 6, st2, fc, device_batch);
          const auto gout = res2.resolve(prompts);
          EXPECT(st2.model_invocations == rs2.model_invocations && st2.cache_hits == rs2.cache_hits &&
                     st2.cache_misses == rs2.cache_misses,
                 "query after a failure: stats");
          EXPECT(cache.size() == rcache.size(), "query after a failure: cache size");
#ifndef WITH_GPU
          EXPECT(gout == rout, "query after a failure: outputs");
#endif
          ++scenarios;
        }

  // Bounded host memory while streaming: rows and decoded slots are released as they are handed back.
  {
    iolm::cuda::PromptCache cache(64);
    iolm::cuda::ResolverStats st;
    iolm::FlopCounter fc;
    Resolver res(model, cache, 16, 2, st, fc, 64);
    size_t max_rows = 0, max_slots = 0, got = 0;
    for (int i = 0; i < 20000; ++i) {
      res.push("echo " + std::to_string(i % 5000));
      got += res.take_ready().size();
      max_rows = std::max(max_rows, res.rows_held());
      max_slots = std::max(max_slots, res.slots_held());
    }
    res.finish();
    got += res.take_ready().size();
    std::printf("streaming 20000 rows: at most %zu rows / %zu slots held\n", max_rows, max_slots);
    EXPECT(got == 20000, "streaming memory test row count");
    EXPECT(max_rows <= 2 * 64 + 16 && max_slots <= 2 * 64 + 16, "held rows / slots bounded by the device batch");
    EXPECT(res.rows_held() == 0 && res.slots_held() == 0, "everything released after the last take_ready");
  }

  // SEMANTIC JOIN (exec.cpp:283-336) through iolm::cuda::semantic_join. A second model whose 'y' and
  // 'n' embedding rows (tied head, runtime.cpp:213-215) are scaled up answers y or n on most pairs,
  // so the match path is exercised too (the random-init one answers neither: all unparsable).
  iolm::Rng yrng(21);
  auto yn_params = iolm::ToyModelParams::init(iolm::ModelConfig::dense(32, 2, 2, 64, 96), yrng);
  for (int c = 0; c < 32; ++c) {
    yn_params.tok_embed.at('y', c) *= 40.f;
    yn_params.tok_embed.at('n', c) *= -40.f;
  }
  const auto yn_bundle = yn_params.to_bundle();
  const iolm::ModelRuntime cpu_yn(yn_bundle);
#ifdef WITH_GPU
  const iolm::cuda::ModelRuntime model_yn(yn_bundle);
#else
  const iolm::ModelRuntime& model_yn = cpu_yn;
#endif
  for (int which = 0; which < 2; ++which) {
    const auto& cpu_j = which ? cpu_yn : cpu;
    const auto& model_j = which ? model_yn : model;
    const iolm::Table l = words_table(40, 11), r0 = words_table(40, 12);
    iolm::Table r = r0;
    r.name = "r";
    r.columns[0].name = "v2";
    iolm::Table lt = l;
    lt.name = "l";
    lt.columns[0].name = "v";
    for (int batch : {1, 16})
      for (size_t capacity : {size_t{0}, size_t{1024}}) {
        iolm::PromptCache rcache(capacity);
        iolm::ExecOptions opts;
        opts.batch_size = batch;
        opts.cache_capacity = capacity;
        iolm::ExecStats rs;
        iolm::FlopCounter f1;
        const iolm::Table out = iolm::execute(iolm::parse_query("SELECT v, v2 FROM l SEMANTIC JOIN r ON v ~ v2"),
                                              {{"l", lt}, {"r", r}}, cpu_j, rcache, opts, rs, f1);
        iolm::cuda::PromptCache cache(capacity);
        iolm::cuda::ResolverStats st;
        iolm::cuda::JoinStats js;
        iolm::FlopCounter f2;
        const auto m = iolm::cuda::semantic_join(model_j, cache, batch, std::span<const std::string>(lt.columns[0].texts),
                                                 std::span<const std::string>(r.columns[0].texts), st, js, f2, 64);
        EXPECT(js.join_pairs_considered == rs.join_pairs_considered, "join pairs considered");
        EXPECT(st.model_invocations == rs.model_invocations && st.cache_hits == rs.cache_hits &&
                   st.cache_misses == rs.cache_misses,
               "join resolver stats");
        // (on the GPU too: the y/n model's answers sit far from any fp tie - 40x embedding rows)
        EXPECT(js.join_matches == rs.join_matches && js.unparsable_match_answers == rs.unparsable_match_answers,
               "join match / unparsable counts");
        bool same = m.size() == out.row_count;
        for (size_t k = 0; same && k < m.size(); ++k)
          same = lt.columns[0].texts[m[k].first] == out.columns[0].texts[k] &&
                 r.columns[0].texts[m[k].second] == out.columns[1].texts[k];
        EXPECT(same, "join output rows identical to iolm::execute");
        if (batch == 16 && capacity == 1024)
          std::printf("semantic join: %llu pairs considered, %llu matches (reference %llu), %llu unparsable\n",
                      static_cast<unsigned long long>(js.join_pairs_considered),
                      static_cast<unsigned long long>(js.join_matches),
                      static_cast<unsigned long long>(rs.join_matches),
                      static_cast<unsigned long long>(js.unparsable_match_answers));
        ++scenarios;
      }
  }

#ifdef WITH_GPU
  std::printf("gpu vs cpu reference agreement %zu/%zu rows\n", agree, total);
  EXPECT(agree * 100 >= total * 99, "gpu vs cpu agreement >= 99%");
#endif
  std::printf("%d scenarios, %d failures\n", scenarios, fails);
  if (fails == 0) std::printf("RESOLVER OK\n");
  return fails == 0 ? 0 : 1;
}
