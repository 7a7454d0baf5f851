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
    if (o.has("smem_limit_bytes")) opts.codegen.max_smem = static_cast<int>(o.at("smem_limit_bytes").as_int());
    if (o.has("allow_row")) opts.codegen.allow_row = o.at("allow_row").as_bool();
    if (o.has("num_sms")) opts.codegen.num_sms = static_cast<int>(o.at("num_sms").as_int());
    if (o.has("tc_pipeline")) opts.codegen.tc_pipeline = o.at("tc_pipeline").as_bool();
    if (o.has("tc_direct_loads")) opts.codegen.tc_direct_loads = o.at("tc_direct_loads").as_bool();
    if (o.has("tensor_cores")) opts.codegen.tensor_cores = o.at("tensor_cores").as_bool();
    if (o.has("pack_sequential")) opts.codegen.pack_sequential = o.at("pack_sequential").as_bool();
    if (o.has("wide_cross_threads")) opts.codegen.wide_cross_threads = static_cast<int>(o.at("wide_cross_threads").as_int());
    if (o.has("wide_cross_cta")) opts.codegen.wide_cross_cta = o.at("wide_cross_cta").as_bool();
    if (o.has("lazy_inputs")) opts.codegen.lazy_inputs = o.at("lazy_inputs").as_bool();
    if (o.has("colred")) opts.codegen.colred = o.at("colred").as_bool();
    if (o.has("row_prefetch_warp")) opts.codegen.row_prefetch_warp = o.at("row_prefetch_warp").as_bool();
    if (o.has("rcp_divide")) opts.codegen.rcp_divide = o.at("rcp_divide").as_bool();
    if (o.has("gws")) opts.codegen.gws = o.at("gws").as_bool();
    if (o.has("tma_early")) opts.codegen.tma_early = o.at("tma_early").as_bool();
    if (o.has("cross_smem")) opts.codegen.cross_smem = o.at("cross_smem").as_bool();
    if (o.has("cross_smem_min_regs")) opts.codegen.cross_smem_min_regs = static_cast<int>(o.at("cross_smem_min_regs").as_int());
    if (o.has("colred_fused")) opts.codegen.colred_fused = o.at("colred_fused").as_bool();
    if (o.has("colred_cp_async")) opts.codegen.colred_cp_async = o.at("colred_cp_async").as_bool();
    if (o.has("colred_cols")) opts.codegen.colred_cols = static_cast<int>(o.at("colred_cols").as_int());
    if (o.has("colred_ctas_per_sm")) opts.codegen.colred_ctas_per_sm = static_cast<int>(o.at("colred_ctas_per_sm").as_int());
    if (o.has("loop_fusion")) opts.codegen.loop_fusion = o.at("loop_fusion").as_bool();
    if (o.has("row_prefetch")) opts.codegen.row_prefetch = o.at("row_prefetch").as_bool();
    if (o.has("tma_double_buffer")) opts.codegen.tma_double_buffer = o.at("tma_double_buffer").as_bool();
    if (o.has("chunking")) opts.chunking = o.at("chunking").as_bool();
    if (o.has("chunk_l2_bytes")) opts.chunk_l2_bytes = o.at("chunk_l2_bytes").as_int();
    if (o.has("pdl")) opts.pdl = o.at("pdl").as_bool();
    if (o.has("fold_constants")) opts.fold_constants = o.at("fold_constants").as_bool();
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
