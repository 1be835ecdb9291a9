// The reference itself, patched (oracle/reference_gpu.patch) and rebuilt against the B200 runtime,
// driven through its UNCHANGED callers (GPU box).
//
// oracle/Makefile target `patched` copies /root/reference/proj/{include,src} to a scratch tree,
// applies the patch (runtime.hpp / runtime.cpp / CMakeLists.txt: 3 files, 30 lines), and compiles
// every reference source with -DIOLM_WITH_CUDA into oracle/_ref/patched/libiolm_ref_gpu.so, linked
// to paper_2507_04967_b200/libiolm_cuda.so. In this ONE library, iolm::ModelRuntime runs on the CPU
// when IOLM_CUDA_DEVICE is unset at construction and on the B200 when it names a device, so both
// are built side by side here and handed to the reference's own code:
//   * iolm::execute - prompt() over a table (PromptResolver::flush -> batch_decode, exec.cpp:84-159)
//     and SEMANTIC JOIN (exec.cpp:283-336): outputs, ExecStats, join match counts;
//   * capture_calibration (calib.cpp:20-62) - forward(ids, mask, counter, CaptureSink*);
//   * validate (optimize.cpp:331-351) and specialize (optimize.cpp:358-470), which construct their
//     own ModelRuntimes from bundles (baseline, compressed candidates) inside the reference;
//   * forward (Matrix), greedy_decode, config() and bundle_hash(), and the error classes.
// Divergent rows must be fp near-ties of the CPU logits (tests/parity.py's rule).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "iolm/calib.hpp"
#include "iolm/exec.hpp"
#include "iolm/optimize.hpp"
#include "iolm/rng.hpp"
#include "iolm/runtime.hpp"
#include "iolm/sql.hpp"
#include "iolm/table.hpp"
#include "iolm/tokenizer.hpp"
#include "iolm/train.hpp"

static int fails = 0;
#define EXPECT(c, msg)                                   \
  do {                                                   \
    if (!(c)) {                                          \
      std::printf("FAIL %s (line %d)\n", msg, __LINE__); \
      ++fails;                                           \
    }                                                    \
  } while (0)

namespace {

// The runtime a caller gets from the reference's own constructor with / without a device named.
iolm::ModelRuntime make_runtime(const iolm::ModelBundle& b, bool gpu) {
  if (gpu) setenv("IOLM_CUDA_DEVICE", "0", 1);
  else unsetenv("IOLM_CUDA_DEVICE");
  iolm::ModelRuntime rt(b);
  unsetenv("IOLM_CUDA_DEVICE");
  return rt;
}

iolm::Table words_table(const std::string& name, const std::string& col, int n, uint64_t seed) {
  iolm::Table t;
  t.name = name;
  iolm::Column c;
  c.name = col;
  c.type = iolm::ColumnType::text;
  iolm::Rng rng(seed);
  for (int i = 0; i < n; ++i) {
    std::string s;
    for (int j = 0; j < 1 + static_cast<int>(rng.next_below(12)); ++j)
      s.push_back(static_cast<char>('a' + rng.next_below(26)));
    if (i % 3 == 2) s = c.texts[rng.next_below(c.texts.size())];  // duplicates: cache traffic
    c.texts.push_back(s);
  }
  t.columns.push_back(c);
  t.row_count = static_cast<size_t>(n);
  return t;
}

// CPU top-2 logit gap after prompt + the common output prefix: a divergence is accepted only as an
// fp near-tie (gap < 0.05 + 4e-3 * max|logit|, tests/parity.py).
bool is_tie(const iolm::ModelRuntime& cpu, const std::string& prompt, const std::string& a, const std::string& b,
            double* gap_out) {
  size_t k = 0;
  while (k < a.size() && k < b.size() && a[k] == b[k]) ++k;
  std::vector<int> ids{iolm::Tokenizer::kBos};
  for (int id : iolm::Tokenizer::encode(prompt + a.substr(0, k))) ids.push_back(id);
  if (static_cast<int>(ids.size()) > cpu.config().max_seq_len) return false;
  iolm::FlopCounter fc;
  const iolm::Matrix lg = cpu.forward(ids, {}, fc);
  std::vector<float> row(lg.row(lg.rows - 1), lg.row(lg.rows - 1) + lg.cols);
  float amax = 0;
  for (float v : row) amax = std::max(amax, std::fabs(v));
  std::partial_sort(row.begin(), row.begin() + 2, row.end(), std::greater<float>());
  *gap_out = row[0] - row[1];
  return *gap_out < 0.05 + 4e-3 * amax;
}

// >= 99% identical rows, every other one an fp tie.
void check_rows(const iolm::ModelRuntime& cpu, const std::vector<std::string>& prompts,
                const std::vector<std::string>& ref, const std::vector<std::string>& got, const char* what) {
  EXPECT(ref.size() == got.size(), what);
  if (ref.size() != got.size()) return;
  size_t same = 0, ties = 0;
  for (size_t i = 0; i < ref.size(); ++i) {
    if (ref[i] == got[i]) {
      ++same;
      continue;
    }
    double gap = 0;
    const bool tie = is_tie(cpu, prompts[i], ref[i], got[i], &gap);
    ties += tie;
    if (!tie) std::printf("  %s row %zu: \"%s\" vs \"%s\", CPU top-2 gap %.4g (not a tie)\n", what, i,
                          ref[i].c_str(), got[i].c_str(), gap);
  }
  std::printf("%s: %zu/%zu identical, %zu tie-traced divergences\n", what, same, ref.size(), ties);
  EXPECT(same * 100 >= ref.size() * 99, what);
  EXPECT(same + ties == ref.size(), what);
}

struct Run {
  iolm::Table out;
  iolm::ExecStats stats;
  uint64_t cache_size = 0;
};

Run run_query(const std::string& sql, const std::map<std::string, iolm::Table>& tables, const iolm::ModelRuntime& m,
              int batch, size_t capacity, int max_new) {
  iolm::PromptCache cache(capacity);
  iolm::ExecOptions opts;
  opts.batch_size = batch;
  opts.cache_capacity = capacity;
  opts.max_new_tokens = max_new;
  Run r;
  iolm::FlopCounter fc;
  r.out = iolm::execute(iolm::parse_query(sql), tables, m, cache, opts, r.stats, fc);
  r.cache_size = cache.size();
  return r;
}

}  // namespace

int main() {
  iolm::Rng wrng(21);
  const auto bundle = iolm::ToyModelParams::init(iolm::ModelConfig::reference(), wrng).to_bundle();
  const iolm::ModelRuntime cpu = make_runtime(bundle, false);
  const iolm::ModelRuntime gpu = make_runtime(bundle, true);

  // surface: config() (incl. active_heads / active_ffn), bundle_hash(), forward -> Matrix
  EXPECT(gpu.config() == cpu.config(), "config() equal (ModelConfig::operator==)");
  EXPECT(gpu.bundle_hash() == cpu.bundle_hash(), "bundle_hash");
  {
    std::vector<int> ids{iolm::Tokenizer::kBos};
    for (int id : iolm::Tokenizer::encode("the quick brown fox jumps over the lazy dog")) ids.push_back(id);
    std::vector<uint8_t> mask(ids.size(), 1);
    mask[3] = 0;
    iolm::FlopCounter f1, f2;
    const iolm::Matrix a = cpu.forward(ids, mask, f1), b = gpu.forward(ids, mask, f2);
    EXPECT(a.rows == b.rows && a.cols == b.cols, "forward Matrix shape");
    double worst = 0;
    for (int t = 0; t < a.rows; ++t) {
      if (!mask[t]) continue;
      double num = 0, den = 0;
      for (int v = 0; v < a.cols; ++v) {
        num += (a.at(t, v) - b.at(t, v)) * (a.at(t, v) - b.at(t, v));
        den += static_cast<double>(a.at(t, v)) * a.at(t, v);
      }
      worst = std::max(worst, std::sqrt(num / den));
    }
    std::printf("forward (masked): worst rel-L2 %.3e, madds %llu vs %llu\n", worst,
                static_cast<unsigned long long>(f1.total()), static_cast<unsigned long long>(f2.total()));
    EXPECT(worst <= 1e-2, "forward logits rel-L2 <= 1e-2");
    EXPECT(f1.total() == f2.total(), "forward madds");
    iolm::FlopCounter g1, g2;
    const std::string p = "translate to french: good morning";
    const std::string ga = cpu.greedy_decode(p, 12, g1), gb = gpu.greedy_decode(p, 12, g2);
    double gap = 0;
    EXPECT(ga == gb || is_tie(cpu, p, ga, gb, &gap), "greedy_decode");
    EXPECT(ga != gb || g1.total() == g2.total(), "greedy_decode madds");
    bool threw = false;
    try {
      gpu.batch_decode(std::vector<std::string>{"ok", std::string(300, 'x')}, 4, g2);
    } catch (const iolm::SequenceTooLong&) {
      threw = true;
    }
    EXPECT(threw, "SequenceTooLong from the GPU path");
    threw = false;
    try {
      gpu.batch_decode(std::vector<std::string>{"caf\xc3\xa9"}, 4, g2);
    } catch (const iolm::ContractViolation&) {
      threw = true;
    }
    EXPECT(threw, "ContractViolation (non-ASCII) from the GPU path");
  }

  // iolm::execute: prompt() over a table, reference batch sizes and cache capacities
  const iolm::Table t = words_table("t", "w", 300, 5);
  std::vector<std::string> prompts;
  for (const auto& w : t.columns[0].texts) prompts.push_back("describe " + w);
  for (int batch : {1, 16, 512})
    for (size_t capacity : {size_t{0}, size_t{65536}}) {
      const std::string sql = "SELECT w, prompt('describe ' || w) AS r FROM t";
      const Run a = run_query(sql, {{"t", t}}, cpu, batch, capacity, 10);
      const Run b = run_query(sql, {{"t", t}}, gpu, batch, capacity, 10);
      EXPECT(a.stats.model_invocations == b.stats.model_invocations && a.stats.cache_hits == b.stats.cache_hits &&
                 a.stats.cache_misses == b.stats.cache_misses && a.stats.rows_out == b.stats.rows_out,
             "execute prompt(): ExecStats");
      EXPECT(a.cache_size == b.cache_size, "execute prompt(): cache size");
      EXPECT(a.out.columns[0].texts == b.out.columns[0].texts, "execute prompt(): passthrough column");
      const std::string label = "execute prompt() batch " + std::to_string(batch) + " cache " + std::to_string(capacity);
      check_rows(cpu, prompts, a.out.columns[1].texts, b.out.columns[1].texts, label.c_str());
    }

  // IOLM_CUDA_DEVICE="0,0": the reference's ModelRuntime over a multi-device context (two replicas,
  // rows range-partitioned); identical outputs and stats to the one-device GPU runtime
  {
    setenv("IOLM_CUDA_DEVICE", "0,0", 1);
    const iolm::ModelRuntime multi(bundle);
    unsetenv("IOLM_CUDA_DEVICE");
    const std::string sql = "SELECT w, prompt('describe ' || w) AS r FROM t";
    const Run a = run_query(sql, {{"t", t}}, gpu, 512, 65536, 10);
    const Run b = run_query(sql, {{"t", t}}, multi, 512, 65536, 10);
    EXPECT(a.out.columns[1].texts == b.out.columns[1].texts, "multi-device execute: outputs identical");
    EXPECT(a.stats.model_invocations == b.stats.model_invocations && a.stats.cache_hits == b.stats.cache_hits,
           "multi-device execute: stats");
    std::printf("multi-device (IOLM_CUDA_DEVICE=0,0) execute prompt(): outputs %s\n",
                a.out.columns[1].texts == b.out.columns[1].texts ? "identical" : "DIFFER");
  }

  // SEMANTIC JOIN through iolm::execute with a model whose 'y' / 'n' rows (tied head) are scaled so
  // that most 1-token answers are y or n. Answers that differ must be fp ties of the CPU logits, and
  // the match / unparsable counts may differ by exactly those rows.
  {
    iolm::Rng yrng(21);
    auto yn = iolm::ToyModelParams::init(iolm::ModelConfig::reference(), yrng);
    for (int c = 0; c < yn.tok_embed.cols; ++c) {
      yn.tok_embed.at('y', c) *= -30.f;
      yn.tok_embed.at('n', c) *= -60.f;
    }
    const auto ynb = yn.to_bundle();
    const iolm::ModelRuntime cpu_yn = make_runtime(ynb, false), gpu_yn = make_runtime(ynb, true);
    iolm::Table l = words_table("l", "v", 60, 11), r = words_table("r", "v2", 60, 12);
    const std::string sql = "SELECT v, v2 FROM l SEMANTIC JOIN r ON v ~ v2";
    const Run a = run_query(sql, {{"l", l}, {"r", r}}, cpu_yn, 16, 65536, 48);
    const Run b = run_query(sql, {{"l", l}, {"r", r}}, gpu_yn, 16, 65536, 48);
    std::printf("semantic join: %llu pairs, %llu matches (CPU %llu), %llu unparsable (CPU %llu)\n",
                static_cast<unsigned long long>(b.stats.join_pairs_considered),
                static_cast<unsigned long long>(b.stats.join_matches),
                static_cast<unsigned long long>(a.stats.join_matches),
                static_cast<unsigned long long>(b.stats.unparsable_match_answers),
                static_cast<unsigned long long>(a.stats.unparsable_match_answers));
    EXPECT(a.stats.join_pairs_considered == b.stats.join_pairs_considered, "join pairs considered");
    EXPECT(a.stats.model_invocations == b.stats.model_invocations, "join model invocations");
    EXPECT(a.stats.join_matches > 0 && a.stats.join_matches < a.stats.join_pairs_considered, "join exercises y and n");
    // the candidate prompts exactly as run_semantic_join renders them (exec.cpp:308-317)
    std::vector<std::string> jp;
    for (const auto& lv : l.columns[0].texts)
      for (const auto& rv : r.columns[0].texts)
        if (iolm::blocking_pass(lv, rv)) jp.push_back(iolm::semantic_match_prompt(lv, rv));
    EXPECT(jp.size() == a.stats.join_pairs_considered, "join candidate count");
    iolm::FlopCounter f1, f2;
    const auto ja = cpu_yn.batch_decode(jp, 1, f1), jb = gpu_yn.batch_decode(jp, 1, f2);
    check_rows(cpu_yn, jp, ja, jb, "semantic join answers");
    uint64_t diff = 0;
    for (size_t k = 0; k < ja.size(); ++k) diff += ja[k] != jb[k];
    const auto absd = [](uint64_t x, uint64_t y) { return x > y ? x - y : y - x; };
    EXPECT(absd(a.stats.join_matches, b.stats.join_matches) + absd(a.stats.unparsable_match_answers,
                                                                     b.stats.unparsable_match_answers) <= 2 * diff,
           "join counts differ only by tie-traced answers");
    if (diff == 0)
      EXPECT(a.out.columns[0].texts == b.out.columns[0].texts && a.out.columns[1].texts == b.out.columns[1].texts,
             "join output rows");
  }

  // capture_calibration through forward(..., CaptureSink*)
  {
    std::vector<std::string> cal(prompts.begin(), prompts.begin() + 24);
    iolm::Rng r1(3), r2(3);
    const iolm::CalibrationSet a = iolm::capture_calibration(cpu, cal, 16, r1);
    const iolm::CalibrationSet b = iolm::capture_calibration(gpu, cal, 16, r2);
    EXPECT(a.prompts == b.prompts && a.sample_count == b.sample_count, "calibration sample");
    EXPECT(a.fingerprint == b.fingerprint, "calibration fingerprint");
    EXPECT(a.inputs.size() == b.inputs.size(), "capture point count");
    double worst = 0;
    for (const auto& [point, m] : a.inputs) {
      auto it = b.inputs.find(point);
      EXPECT(it != b.inputs.end() && it->second.rows == m.rows && it->second.cols == m.cols, "capture point shape");
      if (it == b.inputs.end() || it->second.rows != m.rows || it->second.cols != m.cols) continue;
      double num = 0, den = 0;
      for (size_t i = 0; i < m.data.size(); ++i) {
        num += (m.data[i] - it->second.data[i]) * (m.data[i] - it->second.data[i]);
        den += static_cast<double>(m.data[i]) * m.data[i];
      }
      worst = std::max(worst, std::sqrt(num / std::max(den, 1e-30)));
    }
    std::printf("capture_calibration: %zu points, worst rel-L2 %.3e\n", a.inputs.size(), worst);
    EXPECT(worst <= 1e-2, "capture rel-L2 <= 1e-2");
  }

  // build_hessian (calib.cpp:64-74) with IOLM_CUDA_DEVICE set: the Gram matrix runs on the GPU and
  // must be BIT-identical; so GPTQ (quant.cpp:51) through apply_recipe yields the identical bundle
  {
    std::vector<std::string> cal(prompts.begin(), prompts.begin() + 32);
    iolm::Rng r1(5);
    const iolm::CalibrationSet calib = iolm::capture_calibration(cpu, cal, 32, r1);
    size_t checked = 0, identical = 0;
    for (const auto& [point, m] : calib.inputs) {
      unsetenv("IOLM_CUDA_DEVICE");
      const iolm::MatrixD hc = iolm::build_hessian(m, 0.01);
      setenv("IOLM_CUDA_DEVICE", "0", 1);
      const iolm::MatrixD hg = iolm::build_hessian(m, 0.01);
      unsetenv("IOLM_CUDA_DEVICE");
      ++checked;
      identical += hc.rows == hg.rows && hc.cols == hg.cols &&
                   std::memcmp(hc.data.data(), hg.data.data(), hc.data.size() * sizeof(double)) == 0;
    }
    std::printf("build_hessian on the GPU: %zu/%zu capture points bit-identical (%d x %d samples x features at attn_in)\n",
                identical, checked, calib.inputs.begin()->second.rows, calib.inputs.begin()->second.cols);
    EXPECT(checked > 0 && identical == checked, "build_hessian bit-identical");
    iolm::CompressionRecipe gptq;
    gptq.quantize = iolm::CompressionRecipe::QuantizeStep{8, iolm::CompressionRecipe::QuantizeStep::Method::gptq};
    unsetenv("IOLM_CUDA_DEVICE");
    const auto bc = iolm::apply_recipe(bundle, gptq, calib);
    setenv("IOLM_CUDA_DEVICE", "0", 1);
    const auto bg = iolm::apply_recipe(bundle, gptq, calib);
    unsetenv("IOLM_CUDA_DEVICE");
    std::printf("apply_recipe(gptq 8-bit) with the GPU Hessian: bundle hash %s\n",
                bc.hash() == bg.hash() ? "identical" : "DIFFERENT");
    EXPECT(bc.hash() == bg.hash(), "GPTQ bundle identical with the GPU Hessian");
  }

  // validate(candidate, baseline): an 8-bit RTN candidate against the baseline, both on the GPU
  {
    auto recipe = iolm::CompressionRecipe{};
    recipe.quantize = iolm::CompressionRecipe::QuantizeStep{};
    std::vector<std::string> cal(prompts.begin(), prompts.begin() + 16);
    iolm::Rng r1(4);
    const iolm::CalibrationSet calib = iolm::capture_calibration(cpu, cal, 16, r1);
    const auto q8 = iolm::apply_recipe(bundle, recipe, calib);
    const iolm::ModelRuntime cq = make_runtime(q8, false), gq = make_runtime(q8, true);
    const std::vector<std::string> holdout(prompts.begin() + 100, prompts.begin() + 164);
    iolm::FlopCounter f1, f2;
    const auto ra = iolm::validate(cq, cpu, holdout, 0.9, 12, f1);
    const auto rb = iolm::validate(gq, gpu, holdout, 0.9, 12, f2);
    size_t same_rows = 0;
    for (size_t i = 0; i < ra.per_row.size(); ++i) same_rows += ra.per_row[i] == rb.per_row[i];
    std::printf("validate (q8 RTN vs baseline): CPU score %.4f exact %.4f, GPU score %.4f exact %.4f, %zu/%zu rows equal\n",
                ra.score, ra.exact_match, rb.score, rb.exact_match, same_rows, ra.per_row.size());
    EXPECT(ra.per_row.size() == rb.per_row.size(), "validate rows");
    EXPECT(std::fabs(ra.score - rb.score) <= 0.05, "validate score within 0.05");
    EXPECT(ra.pass == rb.pass || std::fabs(ra.score - 0.9) < 0.05, "validate pass decision");
    EXPECT(f1.total() == f2.total() || same_rows != ra.per_row.size(), "validate madds");
  }

  // specialize("perf"): the reference builds the baseline and candidate runtimes itself
  {
    iolm::Rng srng(1), grng(1);
    const iolm::QueryPlan plan = iolm::parse_query("SELECT prompt('describe ' || w) AS r FROM t");
    const std::map<std::string, iolm::Table> tables{{"t", t}};
    iolm::FlopCounter f1, f2;
    unsetenv("IOLM_CUDA_DEVICE");
    const auto a = iolm::specialize(bundle, tables, plan, iolm::OptimizationProfile::perf(), nullptr, srng, 8, f1);
    setenv("IOLM_CUDA_DEVICE", "0", 1);
    const auto b = iolm::specialize(bundle, tables, plan, iolm::OptimizationProfile::perf(), nullptr, grng, 8, f2);
    unsetenv("IOLM_CUDA_DEVICE");
    std::printf("specialize(perf): CPU -> %s (score %.4f, %zu attempts), GPU -> %s (score %.4f, %zu attempts)\n",
                a.profile_used.c_str(), a.validation_score, a.attempts.size(), b.profile_used.c_str(),
                b.validation_score, b.attempts.size());
    for (size_t i = 0; i < a.attempts.size() && i < b.attempts.size(); ++i)
      std::printf("  attempt %s: CPU score %.4f pass %d / GPU score %.4f pass %d\n", a.attempts[i].profile.c_str(),
                  a.attempts[i].score, a.attempts[i].passed, b.attempts[i].score, b.attempts[i].passed);
    bool decisive = true;
    for (const auto& at : a.attempts)
      if (at.profile != "baseline" && std::fabs(at.score - (at.profile == "perf" ? 0.85 : 0.95)) < 0.05) decisive = false;
    EXPECT(!decisive || a.profile_used == b.profile_used, "specialize: same profile chosen");
    const iolm::ModelRuntime chosen = make_runtime(b.bundle, true);  // the GPU-specialized bundle runs
    iolm::FlopCounter f3;
    EXPECT(chosen.batch_decode(std::vector<std::string>{"describe abc"}, 4, f3).size() == 1, "specialized bundle runs");
  }

  std::printf(fails ? "PATCHED REFERENCE FAIL (%d)\n" : "PATCHED REFERENCE OK\n", fails);
  return fails ? 1 : 0;
}
