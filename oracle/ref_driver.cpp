// Test infrastructure (oracle) -- NOT part of the product.
//
// A JSON-in / JSON-out dispatcher over the UNMODIFIED reference planner
// (/root/reference/proj, compiled by oracle/Makefile into oracle/_ref/). The
// parity tests call `stitch_ref_call(fn, args)` here and the product's
// `stitch_debug_call(fn, args)` with identical arguments and compare results
// bit for bit. Every entry below names the reference function it exercises.

#include <cstdlib>
#include <cstring>
#include <optional>
#include <string>

#include "json.hpp"
#include "stitch/pipeline.hpp"

using nlohmann::ordered_json;
using namespace stitch;

namespace {

Graph graph_arg(const ordered_json& a) { return parse_graph(a.at("graph").dump()); }

FusionPattern pattern_arg(const ordered_json& ids, int id = 0) {
  FusionPattern p;
  for (const auto& s : ids) p.node_ids.insert(s.get<std::string>());
  p.pattern_id = id;
  return p;
}

ordered_json patterns_json(const std::vector<FusionPattern>& ps) {
  ordered_json out = ordered_json::array();
  for (const auto& p : ps) {
    out.push_back({{"nodes", std::vector<std::string>(p.node_ids.begin(), p.node_ids.end())},
                   {"id", p.pattern_id},
                   {"packing", p.packing}});
  }
  return out;
}

SeedConfig seed_cfg(const ordered_json& a) {
  SeedConfig c;
  if (a.contains("max_operands")) c.max_operands = a["max_operands"].get<int>();
  if (a.contains("seed_min_bytes")) c.min_tensor_bytes = a["seed_min_bytes"].get<int64_t>();
  if (a.contains("exploration_budget")) c.exploration_budget = a["exploration_budget"].get<int>();
  return c;
}

MultiStepConfig ms_cfg(const ordered_json& a) {
  MultiStepConfig c;
  if (a.contains("large_dot_flops")) c.large_dot_flops = a["large_dot_flops"].get<int64_t>();
  return c;
}

CostConfig cost_cfg(const ordered_json& a) {
  CostConfig c;
  if (a.contains("phi_us")) c.phi_us = a["phi_us"].get<double>();
  if (a.contains("shared_limit_bytes")) c.shared_limit_bytes = a["shared_limit_bytes"].get<int64_t>();
  if (a.contains("mode")) {
    std::string m = a["mode"].get<std::string>();
    c.mode = m == "model" ? CostMode::kModelBased
             : m == "execution" ? CostMode::kExecutionBased : CostMode::kHybrid;
  }
  return c;
}

Strategy strategy_arg(const ordered_json& a) {
  std::string s = a.value("strategy", std::string("both"));
  if (s == "substitution") return Strategy::kSubstitution;
  if (s == "exploratory") return Strategy::kExploratory;
  return Strategy::kBoth;
}

BandwidthModel bm_arg(const ordered_json& a) {
  if (a.contains("bandwidth_csv")) return BandwidthModel::from_csv_text(a["bandwidth_csv"].get<std::string>());
  return BandwidthModel::default_model();
}

ordered_json alloc_json(const AllocMap& m) {
  ordered_json e = ordered_json::array();
  for (const auto& x : m.entries) {
    ordered_json j{{"op", x.op_id}, {"offset", x.offset}, {"size", x.size}};
    if (x.reused_from) j["reused_from"] = *x.reused_from;
    e.push_back(j);
  }
  return {{"entries", e}, {"total", m.total}};
}

ordered_json requests_json(const std::vector<SharedRequest>& rs) {
  ordered_json out = ordered_json::array();
  for (const auto& r : rs) out.push_back({{"op", r.op_id}, {"bytes", r.bytes}, {"reason", to_string(r.reason)}});
  return out;
}

ordered_json dispatch(const std::string& fn, const ordered_json& a) {
  if (fn == "parse") {  // graph.cpp parse_graph + print_graph
    Graph g = parse_graph(a.at("text").get<std::string>());
    return ordered_json::parse(print_graph(g));
  }
  if (fn == "validate") {  // graph.cpp validate (parsing without the throw)
    try {
      Graph g = parse_graph(a.at("graph").dump());
      ordered_json d = ordered_json::array();
      for (const auto& x : validate(g))
        d.push_back({{"node", x.node_id}, {"rule", x.rule}, {"warning", x.warning}});
      return {{"ok", true}, {"diags", d}};
    } catch (const std::exception& e) {
      return {{"ok", false}, {"error", e.what()}};
    }
  }
  Graph g = a.contains("graph") ? graph_arg(a) : Graph{};
  if (fn == "topo") return topological_sort(g);  // graph.cpp topological_sort
  if (fn == "contract") {                        // graph.cpp contract_plan
    std::vector<FusionPattern> plan;
    int i = 0;
    for (const auto& ids : a.at("plan")) plan.push_back(pattern_arg(ids, i++));
    ContractResult r = contract_plan(g, plan);
    if (r.cycle) return {{"cycle", {{"patterns", r.cycle->pattern_ids}, {"nodes", r.cycle->node_ids}}}};
    return {{"graph", ordered_json::parse(print_graph(*r.graph))}};
  }
  if (fn == "substitution") {  // pattern_gen.cpp substitution_fusion
    PartitionSet ps;
    for (const auto& s : a.at("parts")) ps.op_ids.insert(s.get<std::string>());
    return patterns_json(substitution_fusion(g, ps));
  }
  if (fn == "multi_step") return patterns_json(multi_step_patterns(g, ms_cfg(a)));
  if (fn == "exploratory")
    return patterns_json(exploratory_fusion(g, pattern_arg(a.at("seed")), seed_cfg(a)));
  if (fn == "seeds") return patterns_json(select_seeds(g, seed_cfg(a)));
  if (fn == "generate_patterns")
    return patterns_json(generate_patterns(g, strategy_arg(a), seed_cfg(a), ms_cfg(a)));
  if (fn == "pattern_info") {  // cost_model.cpp + emitter.cpp analyses
    FusionPattern p = pattern_arg(a.at("nodes"));
    CostConfig cc = cost_cfg(a);
    auto [feasible, requested] = shared_feasible(g, p, cc);
    auto reqs = canonical_shared_requests(g, p);
    PatternScore sc = score_model_based(g, p, bm_arg(a), cc);
    std::set<std::string> outs = pattern_outputs(g, p);
    return {{"saved_bytes", saved_bytes(g, p)},
            {"feasible", feasible},
            {"requested", requested},
            {"requests", requests_json(reqs)},
            {"alloc", alloc_json(shared_planning(g, p, reqs))},
            {"score", sc.score_us},
            {"score_feasible", sc.feasible},
            {"complex", is_complex_pattern(g, p)},
            {"category", to_string(classify(g, p))},
            {"connected", pattern_is_connected(g, p)},
            {"outputs", std::vector<std::string>(outs.begin(), outs.end())}};
  }
  if (fn == "shared_planning") {  // emitter.cpp shared_planning on explicit requests
    FusionPattern p = pattern_arg(a.at("nodes"));
    std::vector<SharedRequest> reqs;
    for (const auto& r : a.at("requests"))
      reqs.push_back({r.at("op").get<std::string>(), r.at("bytes").get<int64_t>(),
                      SharedReason::kElemwiseStage});
    return alloc_json(shared_planning(g, p, reqs));
  }
  if (fn == "postdom") {  // emitter.cpp PostDominance
    FusionPattern p = pattern_arg(a.at("nodes"));
    PostDominance pd(g, p);
    ordered_json out = ordered_json::array();
    for (const auto& x : p.node_ids)
      for (const auto& y : p.node_ids)
        if (pd.dominates(x, y)) out.push_back({x, y});
    return out;
  }
  if (fn == "m_of_v") {  // cost_model.cpp m_of_v / bandwidth_at
    BandwidthModel bm = bm_arg(a);
    ordered_json out = ordered_json::array();
    for (const auto& v : a.at("v")) {
      int64_t x = v.get<int64_t>();
      out.push_back({m_of_v(bm, x), bm.bandwidth_at(x)});
    }
    return out;
  }
  if (fn == "score_execution") {  // cost_model.cpp score_execution_based
    FusionPattern p = pattern_arg(a.at("nodes"));
    std::optional<double> fused;
    if (!a.at("fused_us").is_null()) fused = a["fused_us"].get<double>();
    PatternScore s = score_execution_based(p, a.at("per_op_us").get<std::vector<double>>(), fused, cost_cfg(a));
    return {{"score", s.score_us}, {"feasible", s.feasible}};
  }
  if (fn == "solve") {  // ilp_solver.cpp solve
    IlpInstance inst;
    inst.num_vars = a.at("num_vars").get<int>();
    inst.scores = a.at("scores").get<std::vector<double>>();
    for (const auto& pr : a.at("pairs")) inst.pairs.push_back({pr[0].get<int>(), pr[1].get<int>()});
    if (a.contains("cycles"))
      for (const auto& c : a["cycles"]) inst.cycles.push_back({c.get<std::vector<int>>()});
    FusionPlan pl = solve(inst);
    return {{"selected", pl.selected}, {"total", pl.total_score}};
  }
  if (fn == "solve_cycle") {  // ilp_solver.cpp solve_with_cycle_elimination
    std::vector<FusionPattern> ps;
    int i = 0;
    for (const auto& ids : a.at("patterns")) ps.push_back(pattern_arg(ids, i++));
    FusionPlan pl = solve_with_cycle_elimination(g, ps, a.at("scores").get<std::vector<double>>());
    return {{"selected", pl.selected}, {"total", pl.total_score}};
  }
  if (fn == "apply_plan") {  // transform.cpp apply_plan
    std::vector<FusionPattern> ps;
    int i = 0;
    for (const auto& ids : a.at("patterns")) ps.push_back(pattern_arg(ids, i++));
    FusionPlan pl;
    pl.selected = a.at("selected").get<std::vector<int>>();
    Graph f = apply_plan(g, pl, ps);
    return {{"graph", ordered_json::parse(print_graph(f))},
            {"compression", compression_ratio(g, f)},
            {"edges_equal", dependence_edges(f) == dependence_edges(g)}};
  }
  if (fn == "plan") {  // pipeline.cpp run_plan
    PlanOptions o;
    o.strategy = strategy_arg(a);
    o.seed_cfg = seed_cfg(a);
    o.ms_cfg = ms_cfg(a);
    o.cost_cfg = cost_cfg(a);
    o.emit_cfg.shared_limit_bytes = o.cost_cfg.shared_limit_bytes;
    // Execution-based scores from measured kernel times (pipeline.cpp
    // CsvExecutionEvaluator, the CLI's --kernel-times CSV).
    std::optional<CsvExecutionEvaluator> ev;
    if (a.contains("kernel_times_csv")) ev = CsvExecutionEvaluator::from_csv_text(a["kernel_times_csv"].get<std::string>());
    PlanResult r = run_plan(g, bm_arg(a), o, ev ? &*ev : nullptr);
    return {{"plan", ordered_json::parse(plan_to_json(r))},
            {"fused", ordered_json::parse(print_graph(r.fused))},
            {"report_text", report_to_text(r.report)}};
  }
  if (fn == "codegen") {  // pipeline.cpp run_codegen (kernel sketches)
    CodegenOptions o;
    if (a.contains("shared_limit_bytes")) o.emit_cfg.shared_limit_bytes = a["shared_limit_bytes"].get<int64_t>();
    if (a.contains("template")) o.user_template = parse_template(a["template"].get<std::string>());
    CodegenResult r = run_codegen(g, bm_arg(a), o);
    ordered_json src = ordered_json::object();
    for (const auto& k : r.kernels) src[k.name] = k.source;
    return {{"manifest", ordered_json::parse(manifest_to_json(r))}, {"sources", src}};
  }
  if (fn == "templates") {  // template_ir.cpp generate_templates
    FusionPattern p = pattern_arg(a.at("nodes"));
    TemplateLimits lim;
    if (a.contains("max_templates")) lim.max_templates = a["max_templates"].get<int>();
    ordered_json out = ordered_json::array();
    for (const auto& t : generate_templates(g, p, lim)) out.push_back(print_template(t));
    return out;
  }
  if (fn == "template_roundtrip") return print_template(parse_template(a.at("text").get<std::string>()));
  throw std::runtime_error("unknown function: " + fn);
}

}  // namespace

extern "C" {

// Returns a malloc'd JSON string {"ok":true,"result":...} or
// {"ok":false,"error":"..."}; free with stitch_ref_free.
__attribute__((visibility("default"))) char* stitch_ref_call(const char* fn, const char* args_json) {
  ordered_json out;
  try {
    ordered_json a = ordered_json::parse(args_json);
    out = {{"ok", true}, {"result", dispatch(fn, a)}};
  } catch (const std::exception& e) {
    out = {{"ok", false}, {"error", e.what()}};
  }
  std::string s = out.dump();
  char* buf = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return buf;
}

__attribute__((visibility("default"))) void stitch_ref_free(char* p) { std::free(p); }

}  // extern "C"
