// Fusion-pattern scoring (paper §4.3) and the shared-memory transfer analysis
// behind its feasibility gate (paper §5.3/§5.4, Alg. 4). Public API mirrors
// the reference's proj/include/stitch/cost_model.hpp plus the analysis half of
// emitter.hpp (requests, post-dominance, reuse planning). Scores are computed
// with the reference's exact floating-point expression order, so candidate
// scores -- and therefore ILP selections -- are bit-identical.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "ir.hpp"
#include "patterns.hpp"

namespace stitch {

struct BandwidthModel {
  struct Point {
    int64_t bytes;
    double bytes_per_sec;
  };
  std::vector<Point> points;

  static BandwidthModel from_csv_text(const std::string& text);
  static BandwidthModel from_csv_file(const std::string& path);
  static BandwidthModel default_model();
  double bandwidth_at(int64_t bytes) const;
};

enum class CostMode { kModelBased, kExecutionBased, kHybrid };

struct CostConfig {
  double phi_us = 8.0;
  int64_t shared_limit_bytes = 49152;
  CostMode mode = CostMode::kHybrid;
};

struct PatternScore {
  int pattern_id = -1;
  double score_us = 0.0;
  bool feasible = true;
  int64_t saved_bytes = 0;
};

struct ExecSample {
  std::vector<double> per_op_us;
  std::optional<double> fused_us;
};

class ExecutionEvaluator {
 public:
  virtual ~ExecutionEvaluator() = default;
  virtual std::optional<ExecSample> measure(const Graph& g, const FusionPattern& p) = 0;
};

int64_t saved_bytes(const Graph& g, const FusionPattern& p);
double m_of_v(const BandwidthModel& bm, int64_t v);
std::pair<bool, int64_t> shared_feasible(const Graph& g, const FusionPattern& p, const CostConfig& cfg);
PatternScore score_model_based(const Graph& g, const FusionPattern& p, const BandwidthModel& bm,
                               const CostConfig& cfg);
PatternScore score_execution_based(const FusionPattern& p, const std::vector<double>& per_op_us,
                                   std::optional<double> fused_us, const CostConfig& cfg);
bool is_complex_pattern(const Graph& g, const FusionPattern& p);
PatternScore score_pattern(const Graph& g, const FusionPattern& p, const BandwidthModel& bm,
                           const CostConfig& cfg, ExecutionEvaluator* evaluator = nullptr);

// --- shared-memory transfer analysis ----------------------------------------

enum class SharedReason { kReduceTransfer, kDotTransfer, kElemwiseStage };
std::string to_string(SharedReason r);

struct SharedRequest {
  std::string op_id;  // "<op>__tree" names a block-reduction scratch
  int64_t bytes = 0;
  SharedReason reason = SharedReason::kElemwiseStage;
};

struct AllocEntry {
  std::string op_id;
  int64_t offset = 0;
  int64_t size = 0;
  std::optional<std::string> reused_from;
};

struct AllocMap {
  std::vector<AllocEntry> entries;
  int64_t total = 0;
  const AllocEntry* find(const std::string& op_id) const;
  int64_t requested() const;
};

class PostDominance {
 public:
  PostDominance(const Graph& g, const FusionPattern& p);
  bool dominates(const std::string& a, const std::string& b) const;

 private:
  std::map<std::string, std::set<std::string>> pdom_;
};

std::set<std::string> pattern_outputs(const Graph& g, const FusionPattern& p);
std::vector<SharedRequest> canonical_shared_requests(const Graph& g, const FusionPattern& p);
AllocMap shared_planning(const Graph& g, const FusionPattern& p, const std::vector<SharedRequest>& requests);

// --- rank-level analysis used by the pipeline's scoring loop -----------------

// One pattern's members with the per-pattern facts every analysis needs.
struct PatternView {
  PatternView(const GraphIndex& ix, const RankSet& ranks);
  const GraphIndex& ix;
  std::vector<int> topo;                 // member node indices, graph topo order
  std::vector<std::vector<int>> inside;  // per topo position: in-pattern consumer positions (unique)
  std::vector<char> output;              // per topo position: value escapes the pattern
  int pos(int node) const;               // topo position of a member, -1 outside
  bool member(int node) const { return pos(node) >= 0; }
  const OpNode& op(int p) const { return ix.g.nodes[topo[p]]; }

 private:
  std::vector<std::pair<int, int>> by_node_;  // (node index, topo position), sorted
};

struct RankRequest {
  int pos;  // requesting op, position in PatternView::topo
  std::string op_id;
  int64_t bytes;
  SharedReason reason;
};

std::vector<RankRequest> canonical_requests(const PatternView& pv);
AllocMap plan_shared(const PatternView& pv, const std::vector<RankRequest>& reqs);
int64_t saved_bytes(const PatternView& pv);
bool is_complex(const PatternView& pv);

}  // namespace stitch
