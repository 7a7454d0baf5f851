// Executes a fusion plan on the graph (paper §4.1 "the final fusion plan is
// used to transform the computation graph"): every selected pattern becomes
// one fused super-op whose body holds the induced subgraph behind parameter
// leaves and a terminal tuple. Mirrors reference proj/include/stitch/
// transform.hpp.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "ilp.hpp"
#include "ir.hpp"

namespace stitch {

enum class PatternCategory { kElemwise, kReduction, kGemm };
std::string to_string(PatternCategory c);

PatternCategory classify(const Graph& g, const FusionPattern& p);
PatternCategory classify_fused(const OpNode& fused);

Graph apply_plan(const Graph& g, const FusionPlan& plan, const std::vector<FusionPattern>& patterns);
Graph flatten(const Graph& g);
std::vector<std::pair<std::string, std::string>> dependence_edges(const Graph& g);
int kernel_op_count(const Graph& g);
double compression_ratio(const Graph& before, const Graph& after);

}  // namespace stitch
