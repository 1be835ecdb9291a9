// iolm_cuda_join.hpp - the reference's SEMANTIC JOIN operator (/root/reference/proj/src/exec.cpp:283-336)
// on the streaming resolver: candidate pairs that survive the deterministic blocking filter
// (exec.cpp:48-76) are asked the fixed 1-token yes/no prompt (tasks.cpp:130-132) through
// StreamingPromptResolver with max_new_tokens = 1, i.e. a prefill + head-argmax workload on the B200
// (the paper's fuzzy-join workload). Semantics kept from the reference: candidates in (left, right)
// order, a pair matches iff the answer starts with 'y', answers starting with neither 'y' nor 'n'
// are counted as unparsable, and all cache / dedup / invocation accounting is the reference's.
// Difference (performance only): each string is normalised once instead of once per pair.
#pragma once

#include <cctype>
#include <cstdlib>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "iolm_cuda_resolver.hpp"

namespace iolm::cuda {

// exec.cpp:48-62: lowercase alphanumerics, every run of other characters becomes one space
// (none leading or trailing).
inline std::string engine_normalize(const std::string& s) {
  std::string out;
  bool pending_space = false;
  for (char c : s) {
    const auto u = static_cast<unsigned char>(c);
    if (std::isalnum(u)) {
      if (pending_space && !out.empty()) out.push_back(' ');
      pending_space = false;
      out.push_back(static_cast<char>(std::tolower(u)));
    } else {
      pending_space = true;
    }
  }
  return out;
}

// exec.cpp:64-72 on pre-normalised strings: same first character, or lengths within 2.
inline bool blocking_pass_normalized(const std::string& na, const std::string& nb) {
  const char fa = na.empty() ? '\0' : na[0];
  const char fb = nb.empty() ? '\0' : nb[0];
  if (fa == fb) return true;
  return std::labs(static_cast<long>(na.size()) - static_cast<long>(nb.size())) <= 2;
}

inline std::string semantic_match_prompt(const std::string& a, const std::string& b) {
  return "same: " + a + " | " + b + " ->";  // render_match_prompt, tasks.cpp:130-132
}

struct JoinStats {  // the join counters of ExecStats (exec.hpp:76-85)
  uint64_t join_pairs_considered = 0;
  uint64_t join_matches = 0;
  uint64_t unparsable_match_answers = 0;
};

// Returns the matching (left row, right row) pairs in the reference's output order.
template <typename Model, typename Counter>
std::vector<std::pair<size_t, size_t>> semantic_join(const Model& model, PromptCache& cache, int batch_size,
                                                     std::span<const std::string> left,
                                                     std::span<const std::string> right, ResolverStats& rstats,
                                                     JoinStats& jstats, Counter& counter,
                                                     size_t device_batch = 32768) {
  std::vector<std::string> nl, nr;
  nl.reserve(left.size());
  nr.reserve(right.size());
  for (const auto& s : left) nl.push_back(engine_normalize(s));
  for (const auto& s : right) nr.push_back(engine_normalize(s));
  StreamingPromptResolver<Model, Counter> resolver(model, cache, batch_size, 1, rstats, counter, device_batch);
  std::vector<std::pair<size_t, size_t>> candidates, matches;
  // candidate enumeration streams into the resolver; answers are collected at the end in order
  for (size_t i = 0; i < left.size(); ++i)
    for (size_t j = 0; j < right.size(); ++j)
      if (blocking_pass_normalized(nl[i], nr[j])) {
        candidates.emplace_back(i, j);
        resolver.push(semantic_match_prompt(left[i], right[j]));
      }
  jstats.join_pairs_considered += candidates.size();
  resolver.finish();
  const auto answers = resolver.take_ready();
  for (size_t k = 0; k < candidates.size(); ++k) {
    const std::string& ans = answers[k];
    const char first = ans.empty() ? '\0' : ans[0];
    if (first != 'y' && first != 'n') ++jstats.unparsable_match_answers;
    if (first != 'y') continue;
    ++jstats.join_matches;
    matches.push_back(candidates[k]);
  }
  return matches;
}

}  // namespace iolm::cuda
