/*
 * stitch_b200.h -- C ABI of the B200-native FusionStitching executor.
 *
 * Drop-in boundary for the reference's pipeline API
 * (/root/reference/proj/include/stitch/pipeline.hpp). Plain pointers, sizes
 * and UTF-8 JSON strings only; no C++ or torch types cross this line. All
 * returned strings are malloc'd: release them with stitch_free(). Functions
 * returning int yield 0 on success, 1 on bad input (parse / validation /
 * infeasible), 2 on an internal invariant violation or a CUDA failure --
 * the reference CLI's exit-code convention (tools/stitch_main.cpp:201-208);
 * stitch_last_error() then describes the failure (thread-local).
 */
#ifndef STITCH_B200_H_
#define STITCH_B200_H_

#if defined(__GNUC__)
#define STITCH_API __attribute__((visibility("default")))
#else
#define STITCH_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- planning (host) -------------------------------------------------- */

/* Replaces stitch::run_plan + plan_to_json / print_graph / report_to_json
 * (reference pipeline.hpp:87-101, pipeline.cpp:43).
 * graph_json: the reference graph format (SPEC graph-ir External Interfaces).
 * options_json: {"strategy","phi_us","shared_limit_bytes","max_operands",
 *   "seed_min_bytes","exploration_budget","large_dot_flops","mode","seed",
 *   "bandwidth_csv","threads"} -- every key optional, reference defaults.
 * *result_json: {"plan": <plan.json>, "fused": <fused_graph.json>,
 *   "report_text": "...", "timings": {...}}. */
STITCH_API int stitch_plan_graph(const char* graph_json, const char* options_json, char** result_json);

/* Introspection used by the parity tests: runs one planner stage by name
 * (topo, contract, substitution, multi_step, exploratory, seeds,
 * generate_patterns, pattern_info, shared_planning, postdom, m_of_v,
 * score_execution, solve, solve_cycle, apply_plan, plan, validate, parse)
 * and returns {"ok":true,"result":...} or {"ok":false,"error":"..."}.
 * Mirrors the reference functions of the same names (graph.hpp,
 * pattern_gen.hpp, cost_model.hpp, emitter.hpp, ilp_solver.hpp). */
STITCH_API char* stitch_debug_call(const char* fn, const char* args_json);

/* ---- stitched execution (B200) ------------------------------------------ */

typedef struct stitch_executor stitch_executor;

/* Replaces stitch::run_codegen (reference pipeline.hpp:95, pipeline.cpp:99):
 * instead of kernel-sketch text, every fused op of `fused_graph_json`
 * becomes ONE compiled sm_100a kernel composed from the stitched device
 * templates, and every unfused kernel op one plain kernel. options_json:
 * {"device": int, "smem_limit_bytes": int, "cache_dir": str, "chunking": bool,
 *  "chunk_l2_bytes": int, "max_chunks": int,
 *  "use_graph": bool}. The executor owns an HBM arena for intermediates. */
STITCH_API int stitch_executor_create(const char* fused_graph_json, const char* options_json, stitch_executor** out);
STITCH_API void stitch_executor_destroy(stitch_executor* ex);

/* Inputs (graph parameters without a constant value, in node order), outputs
 * (graph outputs, flattened through tuples), per-kernel launch geometry,
 * composition scheme and algorithmic bytes, as JSON. */
STITCH_API int stitch_executor_describe(const stitch_executor* ex, char** json);

/* One pass on device memory: inputs[i] / outputs[j] are device pointers in
 * describe() order; `stream` is a cudaStream_t (NULL = legacy stream). */
STITCH_API int stitch_executor_run(stitch_executor* ex, const void* const* inputs, void* const* outputs, void* stream);

/* End-to-end pass on host memory (ideally pinned): copies inputs host to
 * device, runs, copies outputs back, synchronises `stream`. */
STITCH_API int stitch_executor_run_host(stitch_executor* ex, const void* const* host_inputs, void* const* host_outputs,
                             void* stream);

/* Measured kernel times (replaces the reference's KernelEvaluator /
 * ExecutionEvaluator stubs, emitter.hpp:155, cost_model.hpp:64): runs
 * `iters` passes with CUDA events around every launch and returns
 * {"kernels":[{"name","us"}...],"total_us":...}. */
STITCH_API int stitch_executor_profile(stitch_executor* ex, const void* const* inputs, void* const* outputs, void* stream,
                            int iters, char** json);

/* Timeline of one pass (executor created with {"trace": true}): runs once
 * through the normal launch path (CUDA graph, dataflow lanes) and returns
 * {"kernels":[{"name","start_us","end_us"}...],"span_us":...} from
 * %globaltimer stamps taken by every warp at kernel entry and exit. */
STITCH_API int stitch_executor_trace(stitch_executor* ex, const void* const* inputs, void* const* outputs, void* stream,
                          char** json);

/* Generated CUDA source of every kernel, {"<kernel name>": "<source>"}
 * (the inspectable counterpart of the reference's emitted <fused_op>.cu
 * files, pipeline.cpp:99 / stitch_main.cpp cmd_codegen). */
STITCH_API char* stitch_executor_sources(const stitch_executor* ex);

/* ---- misc ------------------------------------------------------------------ */
STITCH_API const char* stitch_last_error(void);
STITCH_API void stitch_free(char* p);

#ifdef __cplusplus
}
#endif

#endif /* STITCH_B200_H_ */
