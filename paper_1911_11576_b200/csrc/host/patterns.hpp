// Candidate fusion-pattern generation (paper §4.2): substitution fusion over
// escalating partition sets (Alg. 1 + the multi-step heuristic) and
// exploratory producer/consumer growth from seeds (Alg. 2). Same API and
// results as the reference's proj/include/stitch/pattern_gen.hpp; the hot
// loops run on GraphIndex ranks instead of string sets.
#pragma once

#include <cstdint>
#include <set>
#include <string>
#include <vector>

#include "ir.hpp"

namespace stitch {

struct PartitionSet {
  std::set<std::string> op_ids;
  int stage = 0;
};

struct SeedConfig {
  int max_operands = 10;
  int64_t min_tensor_bytes = 1 << 20;
  int exploration_budget = 512;
};

struct MultiStepConfig {
  int64_t large_dot_flops = int64_t{1} << 24;
};

enum class Strategy { kSubstitution, kExploratory, kBoth };

std::vector<FusionPattern> substitution_fusion(const Graph& g, const PartitionSet& parts);
std::vector<FusionPattern> multi_step_patterns(const Graph& g, const MultiStepConfig& cfg = {});
std::vector<FusionPattern> exploratory_fusion(const Graph& g, const FusionPattern& seed,
                                              const SeedConfig& cfg);
std::vector<FusionPattern> select_seeds(const Graph& g, const SeedConfig& cfg);
std::vector<FusionPattern> generate_patterns(const Graph& g, Strategy strategy,
                                             const SeedConfig& seed_cfg = {},
                                             const MultiStepConfig& ms_cfg = {});

// --- rank-level engine (shared with the pipeline) ---------------------------
using RankSet = std::vector<int>;  // sorted lexicographic node ranks

class PatternEngine {
 public:
  explicit PatternEngine(const GraphIndex& ix);

  std::vector<RankSet> substitution(const std::vector<char>& is_partition) const;
  std::vector<RankSet> multi_step(const MultiStepConfig& cfg) const;
  std::vector<RankSet> exploratory(const RankSet& seed, const SeedConfig& cfg) const;
  std::vector<RankSet> seeds(const SeedConfig& cfg) const;
  std::vector<RankSet> generate(Strategy s, const SeedConfig& sc, const MultiStepConfig& mc) const;

  // True when contracting the single pattern creates a cycle.
  bool contraction_cyclic(const RankSet& p) const;
  bool connected(const RankSet& p) const;
  static void sort_unique(std::vector<RankSet>& ps);
  std::vector<FusionPattern> to_patterns(const std::vector<RankSet>& ps, bool assign_ids) const;

 private:
  const GraphIndex& ix_;
  mutable std::vector<int> mark_;   // scratch stamps
  mutable std::vector<int> seen_;
  mutable int stamp_ = 0;
};

}  // namespace stitch
