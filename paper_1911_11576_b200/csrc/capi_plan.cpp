// C ABI, planning half (declared in include/stitch_b200.h). Strings cross the
// boundary as UTF-8 JSON; returned strings are malloc'd and released with
// stitch_free. Errors: return code != 0 and stitch_last_error() describes it.
#include <cstdlib>
#include <cstring>
#include <optional>
#include <string>

#include "host/pipeline.hpp"
#include "capi_common.hpp"
#include "stitch_b200.h"

using namespace stitch;

namespace {

#define g_error capi_last_error()

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

json::Value patterns_json(const std::vector<FusionPattern>& ps) {
  json::Value out = json::Value::array();
  for (const FusionPattern& p : ps) {
    json::Value e = json::Value::object();
    e.set("nodes", json::Value::array_of(std::vector<std::string>(p.node_ids.begin(), p.node_ids.end())));
    e.set("id", p.pattern_id);
    e.set("packing", p.packing);
    out.push(e);
  }
  return out;
}

FusionPattern pattern_of(const json::Value& ids, int id = 0) {
  FusionPattern p;
  for (const auto& s : ids.items()) p.node_ids.insert(s.as_string());
  p.pattern_id = id;
  return p;
}

SeedConfig seed_cfg(const json::Value& a) {
  SeedConfig c;
  if (a.has("max_operands")) c.max_operands = static_cast<int>(a.at("max_operands").as_int());
  if (a.has("seed_min_bytes")) c.min_tensor_bytes = a.at("seed_min_bytes").as_int();
  if (a.has("exploration_budget")) c.exploration_budget = static_cast<int>(a.at("exploration_budget").as_int());
  return c;
}

MultiStepConfig ms_cfg(const json::Value& a) {
  MultiStepConfig c;
  if (a.has("large_dot_flops")) c.large_dot_flops = a.at("large_dot_flops").as_int();
  return c;
}

CostConfig cost_cfg(const json::Value& a) {
  CostConfig c;
  if (a.has("phi_us")) c.phi_us = a.at("phi_us").as_real();
  if (a.has("shared_limit_bytes")) c.shared_limit_bytes = a.at("shared_limit_bytes").as_int();
  if (a.has("mode")) {
    const std::string& m = a.at("mode").as_string();
    c.mode = m == "model" ? CostMode::kModelBased : m == "execution" ? CostMode::kExecutionBased : CostMode::kHybrid;
  }
  return c;
}

Strategy strategy_of(const json::Value& a) {
  std::string s = a.has("strategy") ? a.at("strategy").as_string() : "both";
  return s == "substitution" ? Strategy::kSubstitution : s == "exploratory" ? Strategy::kExploratory : Strategy::kBoth;
}

BandwidthModel bm_of(const json::Value& a) {
  return a.has("bandwidth_csv") ? BandwidthModel::from_csv_text(a.at("bandwidth_csv").as_string())
                                : BandwidthModel::default_model();
}

PlanOptions plan_options(const json::Value& a) {
  PlanOptions o;
  o.strategy = strategy_of(a);
  o.seed_cfg = seed_cfg(a);
  o.ms_cfg = ms_cfg(a);
  o.cost_cfg = cost_cfg(a);
  if (a.has("seed")) o.seed = static_cast<uint64_t>(a.at("seed").as_int());
  if (a.has("threads")) o.threads = static_cast<int>(a.at("threads").as_int());
  if (a.has("ilp_node_budget")) o.ilp_node_budget = a.at("ilp_node_budget").as_int();
  return o;
}

json::Value alloc_json(const AllocMap& m) {
  json::Value es = json::Value::array();
  for (const AllocEntry& e : m.entries) {
    json::Value j = json::Value::object();
    j.set("op", e.op_id);
    j.set("offset", e.offset);
    j.set("size", e.size);
    if (e.reused_from) j.set("reused_from", *e.reused_from);
    es.push(j);
  }
  json::Value out = json::Value::object();
  out.set("entries", es);
  out.set("total", m.total);
  return out;
}

json::Value plan_result_json(const Graph& g, const PlanResult& r) {
  (void)g;
  json::Value out = json::Value::object();
  out.set("plan", json::parse(plan_to_json(r)));
  out.set("fused", graph_to_json(r.fused));
  out.set("report_text", report_to_text(r.report));
  json::Value t = json::Value::object();
  t.set("generate_ms", r.timings.generate_ms);
  t.set("score_ms", r.timings.score_ms);
  t.set("solve_ms", r.timings.solve_ms);
  t.set("rewrite_ms", r.timings.rewrite_ms);
  t.set("search_nodes", static_cast<int64_t>(r.timings.search_nodes));
  t.set("ilp_rounds", r.timings.ilp_rounds);
  t.set("ilp_truncated", r.timings.ilp_truncated);
  t.set("ilp_lp_gap", r.timings.ilp_lp_gap);
  out.set("timings", t);
  return out;
}

// run_plan with the options object; "kernel_times_csv" (name,kernel_us rows:
// op ids and '+'-joined pattern op ids) plugs in the CSV execution
// evaluator, which the executor's measured kernel times feed
// (paper_1911_11576_b200/tuning.py; reference pipeline.cpp
// CsvExecutionEvaluator).
json::Value run_plan_json(const Graph& g, const json::Value& a) {
  std::optional<CsvExecutionEvaluator> ev;
  if (a.has("kernel_times_csv")) ev = CsvExecutionEvaluator::from_csv_text(a.at("kernel_times_csv").as_string());
  return plan_result_json(g, run_plan(g, bm_of(a), plan_options(a), ev ? &*ev : nullptr));
}

// Same function names and JSON shapes as oracle/ref_driver.cpp, so parity
// tests can call both sides with one argument object.
json::Value dispatch(const std::string& fn, const json::Value& a) {
  if (fn == "parse") return graph_to_json(parse_graph(a.at("text").as_string()));
  if (fn == "validate") {
    json::Value out = json::Value::object();
    try {
      Graph g = parse_graph(a.at("graph").dump());
      json::Value d = json::Value::array();
      for (const Diagnostic& x : validate(g)) {
        json::Value e = json::Value::object();
        e.set("node", x.node_id);
        e.set("rule", x.rule);
        e.set("warning", x.warning);
        d.push(e);
      }
      out.set("ok", true);
      out.set("diags", d);
    } catch (const std::exception& e) {
      out.set("ok", false);
      out.set("error", e.what());
    }
    return out;
  }
  Graph g = a.has("graph") ? parse_graph(a.at("graph").dump()) : Graph{};
  if (fn == "topo") return json::Value::array_of(topological_sort(g));
  if (fn == "contract") {
    std::vector<FusionPattern> plan;
    int i = 0;
    for (const auto& ids : a.at("plan").items()) plan.push_back(pattern_of(ids, i++));
    ContractResult r = contract_plan(g, plan);
    json::Value out = json::Value::object();
    if (r.cycle) {
      json::Value c = json::Value::object();
      c.set("patterns", json::Value::array_of(r.cycle->pattern_ids));
      c.set("nodes", json::Value::array_of(r.cycle->node_ids));
      out.set("cycle", c);
    } else {
      out.set("graph", graph_to_json(*r.graph));
    }
    return out;
  }
  if (fn == "substitution") {
    PartitionSet ps;
    for (const auto& s : a.at("parts").items()) ps.op_ids.insert(s.as_string());
    return patterns_json(substitution_fusion(g, ps));
  }
  if (fn == "multi_step") return patterns_json(multi_step_patterns(g, ms_cfg(a)));
  if (fn == "exploratory") return patterns_json(exploratory_fusion(g, pattern_of(a.at("seed")), seed_cfg(a)));
  if (fn == "seeds") return patterns_json(select_seeds(g, seed_cfg(a)));
  if (fn == "generate_patterns") return patterns_json(generate_patterns(g, strategy_of(a), seed_cfg(a), ms_cfg(a)));
  if (fn == "pattern_info") {
    FusionPattern p = pattern_of(a.at("nodes"));
    CostConfig cc = cost_cfg(a);
    auto [feasible, requested] = shared_feasible(g, p, cc);
    std::vector<SharedRequest> reqs = canonical_shared_requests(g, p);
    PatternScore sc = score_model_based(g, p, bm_of(a), cc);
    json::Value rq = json::Value::array();
    for (const SharedRequest& r : reqs) {
      json::Value e = json::Value::object();
      e.set("op", r.op_id);
      e.set("bytes", r.bytes);
      e.set("reason", to_string(r.reason));
      rq.push(e);
    }
    std::set<std::string> outs = pattern_outputs(g, p);
    json::Value out = json::Value::object();
    out.set("saved_bytes", saved_bytes(g, p));
    out.set("feasible", feasible);
    out.set("requested", requested);
    out.set("requests", rq);
    out.set("alloc", alloc_json(shared_planning(g, p, reqs)));
    out.set("score", sc.score_us);
    out.set("score_feasible", sc.feasible);
    out.set("complex", is_complex_pattern(g, p));
    out.set("category", to_string(classify(g, p)));
    out.set("connected", pattern_is_connected(g, p));
    out.set("outputs", json::Value::array_of(std::vector<std::string>(outs.begin(), outs.end())));
    return out;
  }
  if (fn == "shared_planning") {
    FusionPattern p = pattern_of(a.at("nodes"));
    std::vector<SharedRequest> reqs;
    for (const auto& r : a.at("requests").items())
      reqs.push_back({r.at("op").as_string(), r.at("bytes").as_int(), SharedReason::kElemwiseStage});
    return alloc_json(shared_planning(g, p, reqs));
  }
  if (fn == "postdom") {
    FusionPattern p = pattern_of(a.at("nodes"));
    PostDominance pd(g, p);
    json::Value out = json::Value::array();
    for (const auto& x : p.node_ids)
      for (const auto& y : p.node_ids)
        if (pd.dominates(x, y)) {
          json::Value pr = json::Value::array();
          pr.push(x);
          pr.push(y);
          out.push(pr);
        }
    return out;
  }
  if (fn == "m_of_v") {
    BandwidthModel bm = bm_of(a);
    json::Value out = json::Value::array();
    for (const auto& v : a.at("v").items()) {
      json::Value pr = json::Value::array();
      pr.push(m_of_v(bm, v.as_int()));
      pr.push(bm.bandwidth_at(v.as_int()));
      out.push(pr);
    }
    return out;
  }
  if (fn == "score_execution") {
    FusionPattern p = pattern_of(a.at("nodes"));
    std::optional<double> fused;
    if (!a.at("fused_us").is_null()) fused = a.at("fused_us").as_real();
    std::vector<double> per;
    for (const auto& x : a.at("per_op_us").items()) per.push_back(x.as_real());
    PatternScore s = score_execution_based(p, per, fused, cost_cfg(a));
    json::Value out = json::Value::object();
    out.set("score", s.score_us);
    out.set("feasible", s.feasible);
    return out;
  }
  if (fn == "solve" || fn == "solve_cycle") {
    FusionPlan pl;
    if (fn == "solve") {
      IlpInstance inst;
      inst.num_vars = static_cast<int>(a.at("num_vars").as_int());
      for (const auto& s : a.at("scores").items()) inst.scores.push_back(s.as_real());
      for (const auto& pr : a.at("pairs").items())
        inst.pairs.push_back({static_cast<int>(pr[0].as_int()), static_cast<int>(pr[1].as_int())});
      if (a.has("cycles"))
        for (const auto& c : a.at("cycles").items()) {
          CycleConstraint cc;
          for (const auto& v : c.items()) cc.pattern_indices.push_back(static_cast<int>(v.as_int()));
          inst.cycles.push_back(cc);
        }
      pl = solve(inst);
    } else {
      std::vector<FusionPattern> ps;
      int i = 0;
      for (const auto& ids : a.at("patterns").items()) ps.push_back(pattern_of(ids, i++));
      std::vector<double> scores;
      for (const auto& s : a.at("scores").items()) scores.push_back(s.as_real());
      pl = solve_with_cycle_elimination(g, ps, scores);
    }
    json::Value out = json::Value::object();
    out.set("selected", json::Value::array_of(pl.selected));
    out.set("total", pl.total_score);
    return out;
  }
  if (fn == "apply_plan") {
    std::vector<FusionPattern> ps;
    int i = 0;
    for (const auto& ids : a.at("patterns").items()) ps.push_back(pattern_of(ids, i++));
    FusionPlan pl;
    for (const auto& s : a.at("selected").items()) pl.selected.push_back(static_cast<int>(s.as_int()));
    Graph f = apply_plan(g, pl, ps);
    json::Value out = json::Value::object();
    out.set("graph", graph_to_json(f));
    out.set("compression", compression_ratio(g, f));
    out.set("edges_equal", dependence_edges(f) == dependence_edges(g));
    return out;
  }
  if (fn == "plan") return run_plan_json(g, a);
  throw GraphError("unknown function: " + fn);
}

}  // namespace

extern "C" {

const char* stitch_last_error(void) { return g_error.c_str(); }

void stitch_free(char* p) { std::free(p); }

char* stitch_debug_call(const char* fn, const char* args_json) {
  json::Value out = json::Value::object();
  try {
    json::Value r = dispatch(fn, json::parse(args_json));
    out.set("ok", true);
    out.set("result", r);
  } catch (const std::exception& e) {
    out.set("ok", false);
    out.set("error", e.what());
  }
  return dup(out.dump());
}

int stitch_plan_graph(const char* graph_json, const char* options_json, char** result_json) {
  try {
    json::Value opts = options_json && *options_json ? json::parse(options_json) : json::Value::object();
    Graph g = parse_graph(graph_json);
    *result_json = dup(run_plan_json(g, opts).dump());
    return 0;
  } catch (const InternalError& e) {
    g_error = std::string("internal error: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

}  // extern "C"
