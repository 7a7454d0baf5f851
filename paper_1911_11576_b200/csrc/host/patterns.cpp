// Pattern generation; behaviour follows reference proj/src/pattern_gen.cpp:
//   substitution_fusion  pattern_gen.cpp:49   (maximal runs between partition ops)
//   multi_step_patterns  pattern_gen.cpp:75   (large dot -> bdot -> column -> scalar)
//   exploratory_fusion   pattern_gen.cpp:117  (stack worklist, sorted candidates,
//                                               budget on emitted patterns)
//   select_seeds         pattern_gen.cpp:175
//   generate_patterns    pattern_gen.cpp:197
#include "patterns.hpp"

#include <algorithm>
#include <limits>
#include <unordered_set>

namespace stitch {

namespace {

bool grows_by_exploration(const OpNode& op) {
  return op.type == OpType::kElementwise || op.type == OpType::kBatchedDot || op.type == OpType::kReduce;
}

struct RankSetHash {
  size_t operator()(const RankSet& v) const {
    uint64_t h = 1469598103934665603ull;
    for (int x : v) h = (h ^ static_cast<uint64_t>(x)) * 1099511628211ull;
    return static_cast<size_t>(h);
  }
};

}  // namespace

PatternEngine::PatternEngine(const GraphIndex& ix) : ix_(ix), mark_(ix.n, 0), seen_(ix.n, 0) {}

void PatternEngine::sort_unique(std::vector<RankSet>& ps) {
  std::sort(ps.begin(), ps.end());
  ps.erase(std::unique(ps.begin(), ps.end()), ps.end());
}

bool PatternEngine::connected(const RankSet& p) const {
  if (p.empty()) return false;
  const int s = ++stamp_;
  for (int r : p) mark_[ix_.node_of[r]] = s;
  std::vector<int> stack{ix_.node_of[p[0]]};
  seen_[stack[0]] = s;
  size_t reached = 0;
  while (!stack.empty()) {
    int v = stack.back();
    stack.pop_back();
    ++reached;
    auto visit = [&](int w) {
      if (mark_[w] == s && seen_[w] != s) {
        seen_[w] = s;
        stack.push_back(w);
      }
    };
    for (int w : ix_.operands[v]) visit(w);
    for (int w : ix_.consumers[v]) visit(w);
  }
  return reached == p.size();
}

bool PatternEngine::contraction_cyclic(const RankSet& p) const {
  // A single contracted pattern is cyclic iff some value leaves the pattern
  // and flows back into it. Such a path only visits nodes topologically
  // before the last member, which bounds the search.
  const int s = ++stamp_;
  int last = -1;
  for (int r : p) {
    int v = ix_.node_of[r];
    mark_[v] = s;
    last = std::max(last, ix_.topo_pos[v]);
  }
  std::vector<int> frontier;
  auto push = [&](int w) {
    if (mark_[w] != s && seen_[w] != s && ix_.topo_pos[w] < last) {
      seen_[w] = s;
      frontier.push_back(w);
    }
  };
  for (int r : p)
    for (int w : ix_.consumers[ix_.node_of[r]]) push(w);
  while (!frontier.empty()) {
    int w = frontier.back();
    frontier.pop_back();
    for (int x : ix_.consumers[w]) {
      if (mark_[x] == s) return true;
      push(x);
    }
  }
  return false;
}

std::vector<RankSet> PatternEngine::substitution(const std::vector<char>& is_partition) const {
  std::vector<RankSet> out;
  RankSet run;
  auto flush = [&]() {
    if (run.empty()) return;
    std::sort(run.begin(), run.end());
    out.push_back(std::move(run));
    run.clear();
  };
  for (int v : ix_.topo) {
    if (!ix_.fusible[v] || !ix_.live[v]) continue;  // transparent to runs
    if (is_partition[v]) {
      flush();
      continue;
    }
    run.push_back(ix_.rank_of[v]);
  }
  flush();
  return out;
}

std::vector<RankSet> PatternEngine::multi_step(const MultiStepConfig& cfg) const {
  const Graph& g = ix_.g;
  std::vector<char> part(ix_.n, 0);
  size_t count = 0, last_run = std::numeric_limits<size_t>::max();
  std::vector<RankSet> all;
  for (int step = 0; step < 4; ++step) {
    for (int v = 0; v < ix_.n; ++v) {
      const OpNode& op = g.nodes[v];
      bool add = false;
      if (step == 0) add = op.type == OpType::kDot && dot_flops(g, op) >= cfg.large_dot_flops;
      if (step == 1) add = op.type == OpType::kBatchedDot;
      if (step == 2) add = op.type == OpType::kReduce && reduce_kind(g, op) == ReduceKind::kColumn;
      if (step == 3) add = op.type == OpType::kReduce && reduce_kind(g, op) == ReduceKind::kScalar;
      if (add && !part[v]) {
        part[v] = 1;
        ++count;
      }
    }
    if (step > 0 && count == last_run) continue;  // same partition set: same runs
    last_run = count;
    for (RankSet& p : substitution(part)) all.push_back(std::move(p));
  }
  sort_unique(all);
  return all;
}

std::vector<RankSet> PatternEngine::exploratory(const RankSet& seed, const SeedConfig& cfg) const {
  if (seed.empty()) return {};
  for (int r : seed)
    if (!grows_by_exploration(ix_.g.nodes[ix_.node_of[r]]))
      throw GraphError("exploratory seed contains unfusible op: " + ix_.id(ix_.node_of[r]));
  std::unordered_set<RankSet, RankSetHash> visited{seed};
  std::vector<RankSet> emitted;
  std::vector<RankSet> work{seed};
  const size_t budget = static_cast<size_t>(std::max(0, cfg.exploration_budget));
  std::vector<int> cand;
  while (!work.empty() && emitted.size() < budget) {
    RankSet cur = std::move(work.back());
    work.pop_back();
    cand.clear();
    auto consider = [&](int w) {
      int r = ix_.rank_of[w];
      if (ix_.live[w] && grows_by_exploration(ix_.g.nodes[w]) &&
          !std::binary_search(cur.begin(), cur.end(), r))
        cand.push_back(r);
    };
    for (int r : cur) {
      int v = ix_.node_of[r];
      for (int w : ix_.operands[v]) consider(w);
      for (int w : ix_.consumers[v]) consider(w);
    }
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    for (int c : cand) {
      if (emitted.size() >= budget) break;
      RankSet grown;
      grown.reserve(cur.size() + 1);
      auto at = std::lower_bound(cur.begin(), cur.end(), c);
      grown.insert(grown.end(), cur.begin(), at);
      grown.push_back(c);
      grown.insert(grown.end(), at, cur.end());
      if (visited.count(grown)) continue;
      if (contraction_cyclic(grown)) continue;
      visited.insert(grown);
      emitted.push_back(grown);
      work.push_back(std::move(grown));
    }
  }
  sort_unique(emitted);
  return emitted;
}

std::vector<RankSet> PatternEngine::seeds(const SeedConfig& cfg) const {
  const Graph& g = ix_.g;
  std::vector<RankSet> out;
  for (int v = 0; v < ix_.n; ++v) {
    const OpNode& op = g.nodes[v];
    if (!grows_by_exploration(op) || !ix_.live[v]) continue;
    if (static_cast<int>(op.operands.size()) > cfg.max_operands) continue;
    int64_t largest = op.shape.byte_count();
    for (int o : ix_.operands[v]) largest = std::max(largest, g.nodes[o].shape.byte_count());
    if (largest < cfg.min_tensor_bytes) continue;
    out.push_back({ix_.rank_of[v]});
  }
  sort_unique(out);
  return out;
}

std::vector<RankSet> PatternEngine::generate(Strategy s, const SeedConfig& sc,
                                             const MultiStepConfig& mc) const {
  std::vector<RankSet> all;
  if (s != Strategy::kExploratory) all = multi_step(mc);
  if (s != Strategy::kSubstitution)
    for (const RankSet& seed : seeds(sc))
      for (RankSet& p : exploratory(seed, sc)) all.push_back(std::move(p));
  sort_unique(all);
  return all;
}

std::vector<FusionPattern> PatternEngine::to_patterns(const std::vector<RankSet>& ps, bool assign_ids) const {
  std::vector<FusionPattern> out;
  out.reserve(ps.size());
  for (size_t i = 0; i < ps.size(); ++i) {
    FusionPattern p;
    p.node_ids = ix_.ids_of(ps[i]);
    p.pattern_id = assign_ids ? static_cast<int>(i) : -1;
    p.packing = !connected(ps[i]);
    out.push_back(std::move(p));
  }
  return out;
}

// --- public API ---------------------------------------------------------------

std::vector<FusionPattern> substitution_fusion(const Graph& g, const PartitionSet& parts) {
  GraphIndex ix(g);
  PatternEngine e(ix);
  std::vector<char> part(ix.n, 0);
  for (const std::string& id : parts.op_ids) {
    int v = g.index_of(id);
    if (v >= 0) part[v] = 1;
  }
  return e.to_patterns(e.substitution(part), false);
}

std::vector<FusionPattern> multi_step_patterns(const Graph& g, const MultiStepConfig& cfg) {
  GraphIndex ix(g);
  PatternEngine e(ix);
  return e.to_patterns(e.multi_step(cfg), true);
}

std::vector<FusionPattern> exploratory_fusion(const Graph& g, const FusionPattern& seed,
                                              const SeedConfig& cfg) {
  GraphIndex ix(g);
  PatternEngine e(ix);
  for (const std::string& id : seed.node_ids) g.at(id);  // unknown ids throw
  return e.to_patterns(e.exploratory(ix.ranks_of(seed.node_ids), cfg), true);
}

std::vector<FusionPattern> select_seeds(const Graph& g, const SeedConfig& cfg) {
  GraphIndex ix(g);
  PatternEngine e(ix);
  return e.to_patterns(e.seeds(cfg), true);
}

std::vector<FusionPattern> generate_patterns(const Graph& g, Strategy strategy,
                                             const SeedConfig& seed_cfg, const MultiStepConfig& ms_cfg) {
  GraphIndex ix(g);
  PatternEngine e(ix);
  return e.to_patterns(e.generate(strategy, seed_cfg, ms_cfg), true);
}

}  // namespace stitch
