// Scoring and shared-memory analysis. Reference anchors:
//   BandwidthModel::bandwidth_at   cost_model.cpp:101  (log-space interpolation)
//   m_of_v                         cost_model.cpp:117
//   saved_bytes                    cost_model.cpp:122
//   shared_feasible / scores       cost_model.cpp:144-200
//   canonical_shared_requests      emitter.cpp:186
//   PostDominance                  emitter.cpp:146
//   shared_planning (Alg. 4)       emitter.cpp:330
#include "cost.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>

namespace stitch {

// --- bandwidth model -----------------------------------------------------------

BandwidthModel BandwidthModel::from_csv_text(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line)) throw ParseError("bandwidth model: empty file");
  if (line.rfind("\xEF\xBB\xBF", 0) == 0) line.erase(0, 3);
  if (!line.empty() && line.back() == '\r') line.pop_back();
  if (line != "bytes,bandwidth_bytes_per_sec")
    throw ParseError("bandwidth model: expected header 'bytes,bandwidth_bytes_per_sec', got '" + line + "'");
  BandwidthModel bm;
  for (int lineno = 2; std::getline(in, line); ++lineno) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    size_t comma = line.find(',');
    if (comma == std::string::npos)
      throw ParseError("bandwidth model line " + std::to_string(lineno) + ": expected 'bytes,bandwidth'");
    try {
      bm.points.push_back({std::stoll(line.substr(0, comma)), std::stod(line.substr(comma + 1))});
    } catch (const std::exception&) {
      throw ParseError("bandwidth model line " + std::to_string(lineno) + ": malformed number");
    }
  }
  if (bm.points.size() < 2) throw ParseError("bandwidth model: need at least two sample points");
  for (size_t i = 0; i < bm.points.size(); ++i) {
    if (bm.points[i].bytes_per_sec <= 0) throw ParseError("bandwidth model: bandwidths must be positive");
    if (i && bm.points[i].bytes <= bm.points[i - 1].bytes)
      throw ParseError("bandwidth model: byte sizes must be strictly increasing");
    if (i && bm.points[i].bytes_per_sec < bm.points[i - 1].bytes_per_sec)
      throw ParseError("bandwidth model: bandwidth must be non-decreasing");
  }
  return bm;
}

BandwidthModel BandwidthModel::from_csv_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open bandwidth model: " + path);
  std::stringstream buf;
  buf << in.rdbuf();
  return from_csv_text(buf.str());
}

BandwidthModel BandwidthModel::default_model() {
  // The reference's synthetic saturating curve (data/bandwidth_model.csv).
  BandwidthModel bm;
  const int64_t kib = 1024;
  bm.points = {{4 * kib, 40e9},          {16 * kib, 80e9},           {64 * kib, 160e9},
               {256 * kib, 320e9},       {1024 * kib, 480e9},        {4096 * kib, 640e9},
               {16384 * kib, 780e9},     {65536 * kib, 850e9},       {262144 * kib, 880e9},
               {1048576 * kib, 890e9}};
  return bm;
}

double BandwidthModel::bandwidth_at(int64_t bytes) const {
  if (bytes <= points.front().bytes) return points.front().bytes_per_sec;
  if (bytes >= points.back().bytes) return points.back().bytes_per_sec;
  size_t i = 1;
  while (bytes > points[i].bytes) ++i;
  const Point& a = points[i - 1];
  const Point& b = points[i];
  // Same operation order as the reference, for bit-identical scores.
  double lo = std::log(static_cast<double>(a.bytes));
  double hi = std::log(static_cast<double>(b.bytes));
  double t = (std::log(static_cast<double>(bytes)) - lo) / (hi - lo);
  return a.bytes_per_sec + t * (b.bytes_per_sec - a.bytes_per_sec);
}

double m_of_v(const BandwidthModel& bm, int64_t v) {
  if (v <= 0) return 0.0;
  return static_cast<double>(v) / bm.bandwidth_at(v) * 1e6;
}

std::string to_string(SharedReason r) {
  switch (r) {
    case SharedReason::kReduceTransfer: return "reduce_transfer";
    case SharedReason::kDotTransfer: return "dot_transfer";
    default: return "elemwise_stage";
  }
}

const AllocEntry* AllocMap::find(const std::string& op_id) const {
  for (const AllocEntry& e : entries)
    if (e.op_id == op_id) return &e;
  return nullptr;
}

int64_t AllocMap::requested() const {
  int64_t s = 0;
  for (const AllocEntry& e : entries) s += e.size;
  return s;
}

// --- PatternView ------------------------------------------------------------------

PatternView::PatternView(const GraphIndex& index, const RankSet& ranks) : ix(index) {
  topo.reserve(ranks.size());
  for (int r : ranks) topo.push_back(ix.node_of[r]);
  std::sort(topo.begin(), topo.end(), [&](int a, int b) { return ix.topo_pos[a] < ix.topo_pos[b]; });
  by_node_.reserve(topo.size());
  for (int p = 0; p < static_cast<int>(topo.size()); ++p) by_node_.push_back({topo[p], p});
  std::sort(by_node_.begin(), by_node_.end());
  inside.resize(topo.size());
  output.assign(topo.size(), 0);
  for (int p = 0; p < static_cast<int>(topo.size()); ++p) {
    const int v = topo[p];
    bool escapes = ix.is_output[v];
    for (int c : ix.consumers[v]) {
      int cp = pos(c);
      if (cp >= 0)
        inside[p].push_back(cp);
      else
        escapes = true;
    }
    std::sort(inside[p].begin(), inside[p].end());
    inside[p].erase(std::unique(inside[p].begin(), inside[p].end()), inside[p].end());
    output[p] = escapes;
  }
}

int PatternView::pos(int node) const {
  auto it = std::lower_bound(by_node_.begin(), by_node_.end(), std::make_pair(node, -1));
  return (it != by_node_.end() && it->first == node) ? it->second : -1;
}

namespace {

bool dot_like(const OpNode& op) { return op.type == OpType::kDot || op.type == OpType::kBatchedDot; }

// Does the value at position p reach a gemm or reduction through in-pattern
// elementwise ops (reference emitter.cpp:109 reaches_heavy)?
bool reaches_heavy(const PatternView& pv, int p) {
  std::vector<int> stack(pv.inside[p].begin(), pv.inside[p].end());
  std::vector<char> seen(pv.topo.size(), 0);
  while (!stack.empty()) {
    int q = stack.back();
    stack.pop_back();
    if (seen[q]) continue;
    seen[q] = 1;
    const OpNode& op = pv.op(q);
    if (op.type == OpType::kReduce || dot_like(op)) return true;
    if (op.type == OpType::kElementwise) stack.insert(stack.end(), pv.inside[q].begin(), pv.inside[q].end());
  }
  return false;
}

// Post-dominator sets over pattern positions; position P (= size) is the
// virtual sink behind every escaping value.
std::vector<std::vector<int>> post_dominators(const PatternView& pv) {
  const int P = static_cast<int>(pv.topo.size());
  std::vector<std::vector<int>> pdom(P + 1);
  pdom[P] = {P};
  for (int p = P - 1; p >= 0; --p) {
    std::vector<int> succ = pv.inside[p];
    if (pv.output[p]) succ.push_back(P);
    std::vector<int> meet;
    for (size_t i = 0; i < succ.size(); ++i) {
      if (i == 0) {
        meet = pdom[succ[0]];
        continue;
      }
      std::vector<int> next;
      std::set_intersection(meet.begin(), meet.end(), pdom[succ[i]].begin(), pdom[succ[i]].end(),
                            std::back_inserter(next));
      meet.swap(next);
    }
    meet.insert(std::lower_bound(meet.begin(), meet.end(), p), p);
    pdom[p] = std::move(meet);
  }
  return pdom;
}

bool pdominates(const std::vector<std::vector<int>>& pdom, int a, int b) {
  return a != b && std::binary_search(pdom[b].begin(), pdom[b].end(), a);
}

}  // namespace

std::vector<RankRequest> canonical_requests(const PatternView& pv) {
  std::vector<RankRequest> reqs;
  std::vector<char> claimed(pv.topo.size(), 0);
  for (int p = 0; p < static_cast<int>(pv.topo.size()); ++p) {
    const OpNode& op = pv.op(p);
    const auto& inside = pv.inside[p];
    if (dot_like(op)) {
      if (reaches_heavy(pv, p)) reqs.push_back({p, op.id, op.shape.byte_count(), SharedReason::kDotTransfer});
    } else if (op.type == OpType::kElementwise) {
      bool feeds_dot = std::any_of(inside.begin(), inside.end(), [&](int q) { return dot_like(pv.op(q)); });
      if (feeds_dot) reqs.push_back({p, op.id, op.shape.byte_count(), SharedReason::kElemwiseStage});
    } else if (op.type == OpType::kReduce && !inside.empty()) {
      // Warp-mergeable when every in-pattern consumer is an unclaimed
      // elementwise pattern output shaped like the reduction's kept dims.
      bool mergeable = std::all_of(inside.begin(), inside.end(), [&](int q) {
        const OpNode& c = pv.op(q);
        return c.type == OpType::kElementwise && pv.output[q] && c.shape.dims == op.shape.dims && !claimed[q];
      });
      if (mergeable) {
        for (int q : inside) claimed[q] = 1;
      } else {
        reqs.push_back({p, op.id, op.shape.byte_count(), SharedReason::kReduceTransfer});
      }
    }
  }
  return reqs;
}

AllocMap plan_shared(const PatternView& pv, const std::vector<RankRequest>& reqs) {
  const int P = static_cast<int>(pv.topo.size());
  std::vector<std::vector<int>> pdom = post_dominators(pv);
  std::vector<std::vector<const RankRequest*>> req_at(P);
  for (const RankRequest& r : reqs) req_at[r.pos].push_back(&r);

  struct Slot {
    int64_t offset, size;
    int occupant;  // entry index, -1 free
  };
  AllocMap out;
  std::vector<Slot> slots;
  std::vector<int> entry_pos;              // entry -> requesting op position
  std::vector<std::vector<int>> flows(P);  // op position -> live entries reaching it (sorted)

  auto occupant_slot = [&](int e) -> Slot* {
    for (Slot& s : slots)
      if (s.occupant == e) return &s;
    return nullptr;
  };
  auto fresh = [&](const RankRequest& r) {
    int e = static_cast<int>(out.entries.size());
    entry_pos.push_back(r.pos);
    for (Slot& s : slots)
      if (s.occupant < 0 && s.size >= r.bytes) {  // first fit into reclaimed space
        s.occupant = e;
        out.entries.push_back({r.op_id, s.offset, r.bytes, std::nullopt});
        return e;
      }
    slots.push_back({out.total, r.bytes, e});
    out.entries.push_back({r.op_id, out.total, r.bytes, std::nullopt});
    out.total += r.bytes;
    return e;
  };

  for (int p = 0; p < P; ++p) {
    // Allocation info carried in by operands (propagated or produced).
    std::vector<int> incoming;
    for (int o : pv.ix.operands[pv.topo[p]]) {
      int q = pv.pos(o);
      if (q >= 0) incoming.insert(incoming.end(), flows[q].begin(), flows[q].end());
    }
    std::sort(incoming.begin(), incoming.end());
    incoming.erase(std::unique(incoming.begin(), incoming.end()), incoming.end());
    if (req_at[p].empty()) {
      flows[p] = std::move(incoming);
      continue;
    }
    std::stable_sort(incoming.begin(), incoming.end(),
                     [&](int a, int b) { return entry_pos[a] < entry_pos[b]; });
    std::vector<int> own;
    for (const RankRequest* r : req_at[p]) {
      const bool scratch = r->op_id != pv.op(p).id;
      bool placed = false;
      if (!scratch) {
        for (int prev : incoming) {
          Slot* s = occupant_slot(prev);
          if (!s || !pdominates(pdom, p, entry_pos[prev]) || s->size < r->bytes) continue;
          if (!placed) {  // take over the first dominated predecessor's slot
            int e = static_cast<int>(out.entries.size());
            out.entries.push_back({r->op_id, s->offset, r->bytes, out.entries[prev].op_id});
            entry_pos.push_back(p);
            s->occupant = e;
            own.push_back(e);
            placed = true;
          } else {
            s->occupant = -1;  // further dominated predecessors are dead: reclaim
          }
        }
      }
      if (!placed) own.push_back(fresh(*r));
    }
    std::vector<int> flow;
    for (int e : own)
      if (out.entries[e].op_id == pv.op(p).id) flow.push_back(e);
    std::sort(flow.begin(), flow.end());
    flows[p] = std::move(flow);
  }
  return out;
}

int64_t saved_bytes(const PatternView& pv) {
  int64_t v = 0;
  for (int p = 0; p < static_cast<int>(pv.topo.size()); ++p) {
    const int node = pv.topo[p];
    const int64_t bytes = pv.op(p).shape.byte_count();
    const int64_t reads = static_cast<int64_t>(pv.inside[p].size());
    bool outside = false;
    for (int c : pv.ix.consumers[node]) outside = outside || !pv.member(c);
    v += bytes * reads;
    if (!outside && !pv.ix.is_output[node] && reads > 0) v += bytes;
  }
  return v;
}

bool is_complex(const PatternView& pv) {
  bool row = false, col_or_scalar = false, reduce = false, dot = false;
  for (int p = 0; p < static_cast<int>(pv.topo.size()); ++p) {
    const OpNode& op = pv.op(p);
    if (op.type == OpType::kReduce) {
      reduce = true;
      (reduce_kind(pv.ix.g, op) == ReduceKind::kRow ? row : col_or_scalar) = true;
    }
    dot = dot || dot_like(op);
  }
  return (row && col_or_scalar) || (dot && reduce);
}

// --- public API -------------------------------------------------------------------

namespace {

struct Bound {
  GraphIndex ix;
  PatternView pv;
  Bound(const Graph& g, const FusionPattern& p) : ix(g), pv(ix, checked_ranks(ix, p)) {}
  static RankSet checked_ranks(const GraphIndex& ix, const FusionPattern& p) {
    for (const std::string& id : p.node_ids) ix.g.at(id);
    return ix.ranks_of(p.node_ids);
  }
};

}  // namespace

int64_t saved_bytes(const Graph& g, const FusionPattern& p) { return saved_bytes(Bound(g, p).pv); }

bool is_complex_pattern(const Graph& g, const FusionPattern& p) { return is_complex(Bound(g, p).pv); }

std::set<std::string> pattern_outputs(const Graph& g, const FusionPattern& p) {
  Bound b(g, p);
  std::set<std::string> outs;
  for (int q = 0; q < static_cast<int>(b.pv.topo.size()); ++q)
    if (b.pv.output[q]) outs.insert(b.pv.op(q).id);
  return outs;
}

std::vector<SharedRequest> canonical_shared_requests(const Graph& g, const FusionPattern& p) {
  Bound b(g, p);
  std::vector<SharedRequest> out;
  for (const RankRequest& r : canonical_requests(b.pv)) out.push_back({r.op_id, r.bytes, r.reason});
  return out;
}

AllocMap shared_planning(const Graph& g, const FusionPattern& p, const std::vector<SharedRequest>& requests) {
  Bound b(g, p);
  std::vector<RankRequest> reqs;
  for (const SharedRequest& r : requests) {
    std::string base = r.op_id;
    const std::string suffix = "__tree";
    if (base.size() > suffix.size() && base.compare(base.size() - suffix.size(), suffix.size(), suffix) == 0)
      base.erase(base.size() - suffix.size());
    int node = g.index_of(base);
    int q = node >= 0 ? b.pv.pos(node) : -1;
    if (q < 0) throw GraphError("shared request names op outside pattern: " + r.op_id);
    reqs.push_back({q, r.op_id, r.bytes, r.reason});
  }
  // Requests of one op keep their given order; ops are visited in topo order.
  std::stable_sort(reqs.begin(), reqs.end(), [](const RankRequest& a, const RankRequest& c) { return a.pos < c.pos; });
  return plan_shared(b.pv, reqs);
}

PostDominance::PostDominance(const Graph& g, const FusionPattern& p) {
  Bound b(g, p);
  std::vector<std::vector<int>> pd = post_dominators(b.pv);
  for (int q = 0; q < static_cast<int>(b.pv.topo.size()); ++q) {
    std::set<std::string>& s = pdom_[b.pv.op(q).id];
    for (int x : pd[q]) s.insert(x == static_cast<int>(b.pv.topo.size()) ? "__sink" : b.pv.op(x).id);
  }
}

bool PostDominance::dominates(const std::string& a, const std::string& b) const {
  if (a == b) return false;
  auto it = pdom_.find(b);
  return it != pdom_.end() && it->second.count(a) > 0;
}

std::pair<bool, int64_t> shared_feasible(const Graph& g, const FusionPattern& p, const CostConfig& cfg) {
  Bound b(g, p);
  std::vector<RankRequest> reqs = canonical_requests(b.pv);
  if (reqs.empty()) return {true, 0};
  int64_t requested = 0;
  for (const RankRequest& r : reqs) requested += r.bytes;
  return {plan_shared(b.pv, reqs).total <= cfg.shared_limit_bytes, requested};
}

PatternScore score_model_based(const Graph& g, const FusionPattern& p, const BandwidthModel& bm,
                               const CostConfig& cfg) {
  PatternScore s;
  s.pattern_id = p.pattern_id;
  if (!shared_feasible(g, p, cfg).first) {
    s.feasible = false;
    s.score_us = -1.0;
    return s;
  }
  s.saved_bytes = saved_bytes(g, p);
  const int n = static_cast<int>(p.node_ids.size());
  s.score_us = m_of_v(bm, s.saved_bytes) + (n - 1) * cfg.phi_us;
  return s;
}

PatternScore score_execution_based(const FusionPattern& p, const std::vector<double>& per_op_us,
                                   std::optional<double> fused_us, const CostConfig& cfg) {
  if (per_op_us.size() != p.node_ids.size())
    throw GraphError("execution-based score: expected one kernel time per op");
  PatternScore s;
  s.pattern_id = p.pattern_id;
  if (!fused_us) {
    s.feasible = false;
    s.score_us = -1.0;
    return s;
  }
  double sum = 0.0;
  for (double k : per_op_us) sum += k;
  const int n = static_cast<int>(p.node_ids.size());
  s.score_us = sum + (n - 1) * cfg.phi_us - *fused_us;
  s.feasible = s.score_us >= 0.0;
  return s;
}

PatternScore score_pattern(const Graph& g, const FusionPattern& p, const BandwidthModel& bm,
                           const CostConfig& cfg, ExecutionEvaluator* evaluator) {
  bool execution = cfg.mode == CostMode::kExecutionBased ||
                   (cfg.mode == CostMode::kHybrid && is_complex_pattern(g, p));
  if (execution && evaluator)
    if (std::optional<ExecSample> s = evaluator->measure(g, p))
      return score_execution_based(p, s->per_op_us, s->fused_us, cfg);
  return score_model_based(g, p, bm, cfg);
}

}  // namespace stitch
