// Exact 0/1 selection with cycle elimination.
//
// Answer contract (reference proj/src/ilp_solver.cpp:139 solve):
//   optimum  = max over feasible selections S of canonical(S), where
//              canonical(S) sums scores in ascending variable order;
//   selected = lexicographically smallest feasible S with canonical(S) ==
//              optimum, built index by index preferring "stop here", then
//              "include", then "exclude" (ilp_solver.cpp:153-167).
// Cycle elimination (ilp_solver.cpp:175) adds sum_{i in witness} X_i <= |S|-1
// for the patterns on contract_plan's witness cycle and re-solves.
#include "ilp.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <numeric>

namespace stitch {

namespace {

thread_local SolveStats g_stats;
constexpr double kNegInf = -std::numeric_limits<double>::infinity();

class Search {
 public:
  explicit Search(const IlpInstance& inst) : in_(inst), n_(inst.num_vars) {
    adj_.resize(n_);
    for (const PairConstraint& pc : inst.pairs) {
      adj_[pc.u].push_back(pc.v);
      adj_[pc.v].push_back(pc.u);
    }
    limit_.resize(inst.cycles.size());
    cycles_of_.resize(n_);
    for (size_t c = 0; c < inst.cycles.size(); ++c) {
      limit_[c] = static_cast<int>(inst.cycles[c].pattern_indices.size()) - 1;
      for (int v : inst.cycles[c].pattern_indices) cycles_of_[v].push_back(static_cast<int>(c));
    }
    order_.resize(n_);
    std::iota(order_.begin(), order_.end(), 0);
    std::stable_sort(order_.begin(), order_.end(), [&](int a, int b) { return in_.scores[a] > in_.scores[b]; });
    build_cliques();
    words_ = (n_ + 63) / 64;
    double total = 0.0;
    for (double s : inst.scores) total += s;
    // Relative slack covering the rounding of any partial sum of <= n terms.
    slack_ = 4.0 * (n_ + 2) * std::numeric_limits<double>::epsilon();
    (void)total;
  }

  // Best canonical total consistent with `fixed` (-1 free, 0 out, 1 in);
  // -inf when the fixed-in set is itself infeasible. With `target`, stops at
  // the first selection reaching it. The witness is kept in best_bits().
  double query(const std::vector<signed char>& fixed, double target = std::numeric_limits<double>::quiet_NaN()) {
    ++g_stats.queries;
    chosen_.assign(words_, 0);
    block_.assign(n_, 0);
    ccount_.assign(limit_.size(), 0);
    approx_ = 0.0;
    for (int v = 0; v < n_; ++v) {
      if (fixed[v] != 1) continue;
      if (!takeable(v)) return kNegInf;
      take(v);
    }
    free_.clear();
    for (int v : order_)
      if (fixed[v] == -1) free_.push_back(v);
    best_ = kNegInf;
    target_ = target;
    done_ = false;
    best_bits_ = chosen_;
    cm_.assign(nclique_, 0.0);
    cm_stamp_.assign(nclique_, 0);
    stamp_ = 0;
    dfs(0);
    return best_;
  }

  bool in_best(int v) const { return (best_bits_[v >> 6] >> (v & 63)) & 1; }

 private:
  void build_cliques() {
    clique_.assign(n_, -1);
    if (static_cast<int>(in_.clique_hint.size()) == n_) {
      clique_ = in_.clique_hint;
    } else {
      // Greedy clique cover from the pair list (small instances only).
      std::vector<std::vector<int>> members;
      if (n_ <= 4096) {
        std::vector<std::vector<char>> conflict(n_, std::vector<char>(n_, 0));
        for (int v = 0; v < n_; ++v)
          for (int w : adj_[v]) conflict[v][w] = 1;
        for (int v : order_) {
          int home = -1;
          for (size_t c = 0; c < members.size() && home < 0; ++c) {
            bool all = true;
            for (int w : members[c]) all = all && conflict[v][w];
            if (all) home = static_cast<int>(c);
          }
          if (home < 0) {
            home = static_cast<int>(members.size());
            members.emplace_back();
          }
          members[home].push_back(v);
          clique_[v] = home;
        }
      } else {
        std::iota(clique_.begin(), clique_.end(), 0);
      }
    }
    nclique_ = 0;
    for (int c : clique_) nclique_ = std::max(nclique_, c + 1);
  }

  bool takeable(int v) const {
    if (block_[v]) return false;
    for (int c : cycles_of_[v])
      if (ccount_[c] + 1 > limit_[c]) return false;
    return true;
  }
  void take(int v) {
    chosen_[v >> 6] |= uint64_t{1} << (v & 63);
    for (int w : adj_[v]) ++block_[w];
    for (int c : cycles_of_[v]) ++ccount_[c];
    approx_ += in_.scores[v];
  }
  void drop(int v, double saved) {
    chosen_[v >> 6] &= ~(uint64_t{1} << (v & 63));
    for (int w : adj_[v]) --block_[w];
    for (int c : cycles_of_[v]) --ccount_[c];
    approx_ = saved;
  }
  double canonical() const {
    double t = 0.0;
    for (int wi = 0; wi < words_; ++wi) {
      uint64_t m = chosen_[wi];
      while (m) {
        int b = __builtin_ctzll(m);
        t += in_.scores[wi * 64 + b];
        m &= m - 1;
      }
    }
    return t;
  }

  void dfs(size_t pos) {
    if (done_) return;
    ++g_stats.nodes;
    // The current selection is feasible on its own (everything after `pos`
    // excluded): score it exactly when it can matter.
    if (approx_ * (1.0 + slack_) >= best_ || best_ == kNegInf) {
      double c = canonical();
      if (c > best_) {
        best_ = c;
        best_bits_ = chosen_;
        if (c == target_) {
          done_ = true;
          return;
        }
      }
    }
    // Clique-cover bound over the still-takeable free variables.
    ++stamp_;
    double extra = 0.0;
    size_t first = free_.size();
    for (size_t i = pos; i < free_.size(); ++i) {
      int v = free_[i];
      if (!takeable(v)) continue;
      if (first == free_.size()) first = i;
      int c = clique_[v];
      double s = in_.scores[v];
      if (cm_stamp_[c] != stamp_) {
        cm_stamp_[c] = stamp_;
        cm_[c] = s;
        extra += s;
      } else if (s > cm_[c]) {
        extra += s - cm_[c];
        cm_[c] = s;
      }
    }
    if (first == free_.size()) return;
    double bound = (approx_ + extra) * (1.0 + slack_);
    if (std::isnan(target_) ? bound <= best_ : bound < target_) return;
    int v = free_[first];
    double saved = approx_;
    take(v);
    dfs(first + 1);
    drop(v, saved);
    dfs(first + 1);
  }

  const IlpInstance& in_;
  int n_;
  std::vector<std::vector<int>> adj_;
  std::vector<int> limit_;
  std::vector<std::vector<int>> cycles_of_;
  std::vector<int> order_, clique_, free_;
  int nclique_ = 0, words_ = 0;
  double slack_ = 0.0;

  std::vector<uint64_t> chosen_, best_bits_;
  std::vector<int> block_, ccount_;
  double approx_ = 0.0, best_ = kNegInf, target_ = 0.0;
  bool done_ = false;
  std::vector<double> cm_;
  std::vector<unsigned> cm_stamp_;
  unsigned stamp_ = 0;
};

}  // namespace

const SolveStats& last_solve_stats() { return g_stats; }

std::vector<PairConstraint> build_conflicts(const std::vector<FusionPattern>& patterns) {
  std::map<std::string, std::vector<int>> holders;
  for (size_t i = 0; i < patterns.size(); ++i)
    for (const std::string& id : patterns[i].node_ids) holders[id].push_back(static_cast<int>(i));
  std::vector<std::pair<int, int>> pairs;
  for (const auto& [id, hs] : holders)
    for (size_t a = 0; a < hs.size(); ++a)
      for (size_t b = a + 1; b < hs.size(); ++b) pairs.push_back({hs[a], hs[b]});
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  std::vector<PairConstraint> out;
  out.reserve(pairs.size());
  for (auto [u, v] : pairs) out.push_back({u, v});
  return out;
}

FusionPlan solve(const IlpInstance& inst) {
  if (static_cast<int>(inst.scores.size()) != inst.num_vars)
    throw GraphError("ILP instance: one score per variable required");
  for (double s : inst.scores)
    if (s < 0) throw GraphError("ILP instance requires non-negative scores");
  const int n = inst.num_vars;
  Search search(inst);
  std::vector<signed char> fixed(n, -1);
  const double optimum = search.query(fixed);
  std::vector<char> witness(n, 0);
  for (int v = 0; v < n; ++v) witness[v] = search.in_best(v);

  FusionPlan plan;
  double prefix = 0.0;
  for (int v = 0; v < n; ++v) {
    if (prefix == optimum) break;  // stopping here is lexicographically smallest
    fixed[v] = 1;
    bool keep = witness[v];
    if (!keep && search.query(fixed, optimum) == optimum) {
      keep = true;
      for (int w = 0; w < n; ++w) witness[w] = search.in_best(w);
    }
    if (keep) {
      plan.selected.push_back(v);
      prefix = 0.0;
      for (int w : plan.selected) prefix += inst.scores[w];
    } else {
      fixed[v] = 0;
    }
  }
  plan.total_score = prefix;
  return plan;
}

FusionPlan solve_with_cycle_elimination(const Graph& g, const std::vector<FusionPattern>& patterns,
                                        const std::vector<double>& scores) {
  IlpInstance inst;
  inst.num_vars = static_cast<int>(patterns.size());
  inst.scores = scores;
  inst.pairs = build_conflicts(patterns);
  // Clique hint: each pattern joins the clique of its most-shared node.
  std::map<std::string, int> holders;
  for (const FusionPattern& p : patterns)
    for (const std::string& id : p.node_ids) ++holders[id];
  std::map<std::string, int> clique_id;
  inst.clique_hint.resize(patterns.size());
  for (size_t i = 0; i < patterns.size(); ++i) {
    const std::string* home = nullptr;
    for (const std::string& id : patterns[i].node_ids)
      if (!home || holders[id] > holders[*home]) home = &id;
    if (!home) {
      inst.clique_hint[i] = -1;
      continue;
    }
    auto it = clique_id.emplace(*home, static_cast<int>(clique_id.size())).first;
    inst.clique_hint[i] = it->second;
  }
  int next = static_cast<int>(clique_id.size());
  for (int& c : inst.clique_hint)
    if (c < 0) c = next++;

  SolveStats total;
  for (int round = 0; round < 10000; ++round) {
    g_stats = SolveStats{};
    FusionPlan plan = solve(inst);
    total.nodes += g_stats.nodes;
    total.queries += g_stats.queries;
    total.rounds = round + 1;
    std::vector<FusionPattern> chosen;
    for (int idx : plan.selected) {
      FusionPattern p = patterns[idx];
      p.pattern_id = idx;
      chosen.push_back(std::move(p));
    }
    ContractResult r = contract_plan(g, chosen);
    if (!r.cycle) {
      g_stats = total;
      return plan;
    }
    if (r.cycle->pattern_ids.empty()) throw InternalError("contraction cycle without any pattern on it");
    inst.cycles.push_back({r.cycle->pattern_ids});
  }
  throw GraphError("cycle elimination did not converge within 10000 rounds");
}

}  // namespace stitch
