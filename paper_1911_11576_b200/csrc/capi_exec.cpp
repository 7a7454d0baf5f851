// C ABI, execution half (declared in include/stitch_b200.h).
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "exec/runtime.hpp"
#include "capi_common.hpp"
#include "stitch_b200.h"

using namespace stitch;

struct stitch_executor {
  std::unique_ptr<exec::Executor> impl;
};

namespace {

#define g_exec_error capi_last_error()

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ParseError& e) {
    g_exec_error = e.what();
    return 1;
  } catch (const ValidationError& e) {
    g_exec_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_exec_error = e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

int stitch_executor_create(const char* fused_graph_json, const char* options_json, stitch_executor** out) {
  *out = nullptr;
  return guarded([&] {
    json::Value o = options_json && *options_json ? json::parse(options_json) : json::Value::object();
    exec::ExecOptions opts;
    if (o.has("device")) opts.device = static_cast<int>(o.at("device").as_int());
    if (o.has("cache_dir")) opts.cache_dir = o.at("cache_dir").as_string();
    if (o.has("use_graph")) opts.use_graph = o.at("use_graph").as_bool();
    if (o.has("compile_only")) opts.compile_only = o.at("compile_only").as_bool();
    exec::apply_codegen_options(opts.codegen, o);
    if (o.has("kernel_options")) opts.kernel_options = o.at("kernel_options");
    if (o.has("chunking")) opts.chunking = o.at("chunking").as_bool();
    if (o.has("chunk_l2_bytes")) opts.chunk_l2_bytes = o.at("chunk_l2_bytes").as_int();
    if (o.has("pdl")) opts.pdl = o.at("pdl").as_bool();
    if (o.has("pdl_cooperative")) opts.pdl_cooperative = o.at("pdl_cooperative").as_bool();
    if (o.has("concurrent_lanes")) opts.concurrent_lanes = static_cast<int>(o.at("concurrent_lanes").as_int());
    if (o.has("critical_priority")) opts.critical_priority = o.at("critical_priority").as_bool();
    if (o.has("big_lane_bytes")) opts.big_lane_bytes = o.at("big_lane_bytes").as_int();
    if (o.has("grid_fraction")) opts.grid_fraction = o.at("grid_fraction").as_real();
    if (o.has("fold_off_lane")) opts.fold_off_lane = o.at("fold_off_lane").as_bool();
    if (o.has("issue_order")) opts.issue_order = static_cast<int>(o.at("issue_order").as_int());
    if (o.has("pdl_true_deps_only")) opts.pdl_true_deps_only = o.at("pdl_true_deps_only").as_bool();
    if (o.has("pdl_low_priority")) opts.pdl_low_priority = o.at("pdl_low_priority").as_bool();
    if (o.has("tma_l2_promotion")) opts.tma_l2_promotion = static_cast<int>(o.at("tma_l2_promotion").as_int());
    if (o.has("fold_threads")) {
      opts.fold_threads = static_cast<int>(o.at("fold_threads").as_int());
      if (opts.fold_threads < 32 || opts.fold_threads > 1024 || opts.fold_threads % 32)
        throw GraphError("fold_threads must be a multiple of 32 in [32, 1024]");
    }
    if (o.has("fold_constants")) opts.fold_constants = o.at("fold_constants").as_bool();
    if (o.has("sink_broadcasts")) opts.sink_broadcasts = o.at("sink_broadcasts").as_bool();
    if (o.has("overlap_copies")) opts.overlap_copies = o.at("overlap_copies").as_bool();
    if (o.has("chunk_pipeline")) opts.chunk_pipeline = o.at("chunk_pipeline").as_bool();
    if (o.has("chunk_ring")) opts.chunk_ring = static_cast<int>(o.at("chunk_ring").as_int());
    if (o.has("chunk_fill")) opts.chunk_fill = o.at("chunk_fill").as_bool();
    if (o.has("max_chunks")) opts.max_chunks = static_cast<int>(o.at("max_chunks").as_int());
    Graph g = parse_graph(fused_graph_json);
    auto* ex = new stitch_executor;
    ex->impl = std::make_unique<exec::Executor>(g, opts);
    *out = ex;
  });
}

void stitch_executor_destroy(stitch_executor* ex) { delete ex; }

int stitch_executor_describe(const stitch_executor* ex, char** json_out) {
  return guarded([&] { *json_out = dup(ex->impl->describe().dump()); });
}

int stitch_executor_run(stitch_executor* ex, const void* const* inputs, void* const* outputs, void* stream) {
  return guarded([&] { ex->impl->run(inputs, outputs, stream); });
}

int stitch_executor_run_host(stitch_executor* ex, const void* const* host_inputs, void* const* host_outputs,
                             void* stream) {
  return guarded([&] { ex->impl->run_host(host_inputs, host_outputs, stream); });
}

int stitch_executor_trace(stitch_executor* ex, const void* const* inputs, void* const* outputs, void* stream,
                          char** json_out) {
  *json_out = nullptr;
  return guarded([&] { *json_out = dup(ex->impl->trace(inputs, outputs, stream).dump()); });
}

int stitch_executor_profile(stitch_executor* ex, const void* const* inputs, void* const* outputs, void* stream,
                            int iters, char** json_out) {
  return guarded([&] { *json_out = dup(ex->impl->profile(inputs, outputs, stream, iters).dump()); });
}

// Generated source of every kernel (debugging / golden tests): {"name": src}.
char* stitch_executor_sources(const stitch_executor* ex) {
  json::Value o = json::Value::object();
  for (const exec::KernelInst& k : ex->impl->kernels()) o.set(k.spec.name, exec::full_source(k.spec));
  return dup(o.dump());
}

}  // extern "C"
