// Fusion-plan selection (paper §4.1): maximise sum_j X_j f(P_j) subject to
// X_u + X_v <= 1 for overlapping patterns, iterated with cycle constraints
// until the contracted graph is acyclic. Same API and same answers as the
// reference's proj/include/stitch/ilp_solver.hpp: the optimum is the largest
// "canonical" total (scores summed in ascending variable order) and ties go to
// the lexicographically smallest index set. The search itself is ours: a
// clique-cover bound (patterns sharing a graph node are mutually exclusive)
// and witness-guided extraction replace the reference's additive bound, which
// takes minutes on a few thousand candidates.
#pragma once

#include <vector>

#include "ir.hpp"

namespace stitch {

struct PairConstraint {
  int u = 0;
  int v = 0;
};

struct CycleConstraint {
  std::vector<int> pattern_indices;
};

struct IlpInstance {
  int num_vars = 0;
  std::vector<double> scores;
  std::vector<PairConstraint> pairs;
  std::vector<CycleConstraint> cycles;
  // Optional: for each variable, a clique id -- variables sharing an id must
  // conflict pairwise. Supplied by the planner (one clique per graph node);
  // left empty, the solver derives cliques from the pair list.
  std::vector<int> clique_hint;
  // Optional: for each variable, the graph nodes its pattern covers (dense
  // node indices). Variables sharing a node conflict. Enables the
  // fractional node-price bound (an LP-dual bound of the set-packing
  // relaxation): any feasible selection totals at most
  // sum_x max_{P covers x} s_P / |P|.
  std::vector<std::vector<int>> node_sets;
  int num_nodes = 0;
};

struct FusionPlan {
  std::vector<int> selected;
  double total_score = 0.0;
};

std::vector<PairConstraint> build_conflicts(const std::vector<FusionPattern>& patterns);
FusionPlan solve(const IlpInstance& inst);
FusionPlan solve_with_cycle_elimination(const Graph& g, const std::vector<FusionPattern>& patterns,
                                        const std::vector<double>& scores);

// Statistics of the last solve on this thread (search nodes, rounds).
struct SolveStats {
  long long nodes = 0;
  int queries = 0;
  int rounds = 0;
  // Components whose exact search hit the node budget (the LP relaxation was
  // fractional and the gap could not be closed in time): their incumbent is
  // used, and `lp_gap` (sum of LP bound - incumbent) certifies how far the
  // plan can be from the optimum. 0 = every component solved exactly.
  int truncated = 0;
  double lp_gap = 0.0;
};

// Per-component search-node budget of the decomposed solver (default 300k;
// STITCH_ILP_NODE_BUDGET overrides). Instances the reference planner can
// solve stay far below it.
long long ilp_node_budget();
// Per-thread override (plan option "ilp_node_budget"; < 0 restores the default).
void set_ilp_node_budget(long long nodes);
const SolveStats& last_solve_stats();

}  // namespace stitch
