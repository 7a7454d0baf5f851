// Stitched-kernel runtime: NVRTC compilation to sm_100a cubins (with an
// on-disk cache that build() pre-populates), an HBM arena for the values
// crossing kernel boundaries, and the launch scheduler that replays the
// fused graph's kernels in topological order -- directly or as one CUDA
// graph. Replaces the reference's text-file codegen output
// (proj/src/pipeline.cpp:99 run_codegen + tools/stitch_main.cpp cmd_codegen).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../host/ir.hpp"
#include "../host/json.hpp"
#include "codegen.hpp"

namespace stitch {
namespace exec {

struct ExecOptions {
  int device = 0;
  std::string cache_dir;   // "" = no disk cache
  bool use_graph = true;   // replay launches as a CUDA graph on non-null streams
  bool compile_only = false;  // generate + compile, no device work (build-time cache fill)
  // L2-resident chunking: consecutive row-chunkable kernels that hand
  // intermediates to each other run chunk by chunk (rows [c R/C, (c+1) R/C)
  // of every kernel), each intermediate held in a one-chunk buffer reused by
  // every chunk, so it stays in L2 and is overwritten before write-back.
  int64_t chunk_l2_bytes = 24ll << 20;  // target intermediate bytes per chunk (L2 is 126 MB)
  int max_chunks = 64;
  // Measured on B200: chunked launches lose to whole-tensor launches on the
  // bench configs (softmax 43 -> 51 us, encoder 145 -> 172 us: per-launch
  // ramp and tail dominate the L2 savings), so chunking is opt-in.
  bool chunking = false;
  bool chunk_fill = true;  // require enough rows per chunk to fill every SM (tests force small chunks)
  // Pipelined chunks: kernel j of a chunked segment runs on its own stream,
  // chunk c waiting only for kernel j-1's chunk c, so kernel j's chunk c
  // overlaps kernel j-1's chunk c+1 (tails filled); intermediates use a ring
  // of `chunk_ring` chunk slots.
  bool chunk_pipeline = true;
  // run_host: dataflow copy schedule (H2D in first-use order on one copy
  // stream, D2H of each output right after its producer on another)
  bool overlap_copies = true;
  // broadcasts of constants left unfused by the plan are folded into their
  // consumers as literals instead of being materialised by a kernel
  bool fold_constants = true;
  // Unfused broadcasts of small tensors (LayerNorm gamma/beta [H] ->
  // [T, H]) are not materialised: each consumer kernel reads the source
  // through the broadcast map instead (the broadcast moves into its body).
  bool sink_broadcasts = true;
  int64_t sink_max_bytes = 1 << 20;
  // programmatic dependent launch between consecutive (non-cooperative) kernels
  bool pdl = true;
  // PDL for grid-barrier kernels too: they get scheduled as the previous
  // kernel drains (every CTA of a PDL primary is resident before any
  // dependent CTA launches, so the barrier's co-residency still holds)
  bool pdl_cooperative = true;  // BERT step 1.739 -> 1.728 ms (dataflow), 1.989 -> 1.966 (serial)
  // Dataflow launch: kernels go out on up to `concurrent_lanes` streams
  // with event edges for their true dependencies only (producer -> consumer,
  // arena reuse, grid-barrier kernels one at a time), so independent fusion
  // groups (parameter-gradient column reductions beside the activation-
  // gradient chain) fill each other's tails. <= 1: one stream in launch order.
  // Not used for chunked schedules or per-kernel profiling.
  // measured (BERT step): serial 2.003 ms; before split folds 3 lanes 1.739,
  // 4: 1.771, 8: 1.762; final executor 4 lanes + fold_off_lane 1.518 vs
  // 3 lanes 1.553, 5: 1.544, 6: 1.545
  int concurrent_lanes = 4;
  // dataflow launch: kernels on the estimated critical path (longest chain
  // of algorithmic bytes + per-launch overhead) launch at the highest
  // stream priority, so freed SM slots go to them before side branches
  bool critical_priority = false;
  // > 0: kernels moving at least this many algorithmic bytes all go to lane
  // 0 (back to back, PDL-chained); smaller ones spread over the other lanes
  // and fill the big kernels' ramps and tails. 0: lane of the latest
  // predecessor, else a fresh / the longest-idle lane.
  int64_t big_lane_bytes = 0;  // measured worse (BERT 1.568 -> 1.610-1.648 ms)
  // dataflow launch: persistent grids capped at this fraction of the
  // resident CTA slots, so concurrent kernels co-reside instead of waiting
  // for each other's CTAs to retire (1 = a full resident wave)
  double grid_fraction = 1.0;
  // a fold kernel goes to another lane than its row kernel (waiting on its
  // event), so the row kernel's lane moves on without queueing behind it
  bool fold_off_lane = true;
  // dataflow issue order: 0 = the fused graph's topological order; 1 = ready
  // list, largest algorithmic bytes first; 2 = ready list alternating the
  // largest and the smallest ready kernel; 3 = two largest then one
  // smallest (folds as soon as ready in 1-3); 4 = as 2 with folds ranked by
  // their (zero) algorithmic bytes like any other kernel
  // measured (BERT step, 4 lanes): 0: 1.509-1.520 ms, 1: 1.555, 2: 1.489-1.491;
  // with the final defaults 2: 1.448, 3: 1.504, 4: 1.464
  int issue_order = 2;
  // dataflow launch: PDL only when the lane's previous kernel is a true
  // predecessor (else the early-launched CTAs would hold SM slots waiting on
  // an unrelated kernel)
  // measured (BERT step): 1.493 -> 1.445 ms
  bool pdl_true_deps_only = true;
  // threads per CTA of the fold kernels (split_cross): blockDim / 32 slices
  // of the partial rows per column block (the association follows it)
  // gws tensor maps: L2 promotion of the TMA tile reads (0 none, 1 64B,
  // 2 128B, 3 256B)
  int tma_l2_promotion = 3;
  int fold_threads = 256;
  // dataflow launch: kernels launched without PDL get the highest stream
  // priority, so CTA slots freed by a draining kernel go to runnable work
  // before the early-launched (waiting) CTAs of its PDL dependent
  bool pdl_low_priority = false;  // measured neutral (BERT 1.452 vs 1.453 ms)  // measured: 512 neutral, 1024 +1.7 % (BERT step)  // measured neutral-to-worse (1.775 vs 1.783 ms at 4 lanes): opt-in
  int chunk_ring = 2;
  CodegenOptions codegen;
  // per fused-op codegen overrides {op id: {option: value}} (the measured
  // per-group variant table, paper Alg. 3 KernelEvalUpdate)
  json::Value kernel_options = json::Value::object();
};

// Codegen options from an options JSON object (keys as in stitch_executor_create).
void apply_codegen_options(CodegenOptions& c, const json::Value& o);

const std::string& device_header_source();
std::string full_source(const KernelSpec& spec);
// NVRTC -> sm_100a cubin, through the disk cache when `cache_dir` is set.
std::string compile_cubin(const std::string& source, const std::string& cache_dir, bool* cache_hit = nullptr);

struct ValueBuf {
  std::string key;
  int64_t bytes = 0;
  enum Kind { kInput, kOutput, kArena } kind = kArena;
  int slot = -1;        // input / output position
  int64_t offset = 0;   // arena byte offset
  int first = -1, last = -1;  // producing / last consuming kernel
  int chunks = 1;             // > 1: chunk-local intermediate, arena holds `ring` chunk slots
  int ring = 1;
  int64_t chunk_bytes() const { return bytes / chunks; }
  int64_t arena_bytes() const { return chunk_bytes() * (chunks > 1 ? ring : 1); }
};

struct Segment {  // kernels [first, last] in launch order, run chunk by chunk when chunks > 1
  int first = 0, last = 0, chunks = 1;
};

struct alignas(64) TmapBytes {  // a CUtensorMap
  unsigned long long v[16];
};

struct KernelInst {
  KernelSpec spec;
  json::Value variant = json::Value::object();  // per-group codegen overrides applied
  // gws scheme: TMA tensor maps encoded for the input pointers of the last
  // launch, re-encoded when they change
  std::vector<TmapBytes> tmaps;
  std::vector<unsigned long long> tmap_ptrs;
  std::string op_id;                 // fused op or unfused op id in the fused graph
  std::vector<int> in_bufs, out_bufs;  // pointer arguments, in order
  // buffers this launch reads / writes (dependencies, lifetimes): = in_bufs /
  // out_bufs, except for a split row kernel and its fold (split_cross), which
  // share one argument list but write disjoint outputs
  std::vector<int> reads, writes;
  int fold_of = -1;                  // fold kernel: index of the row kernel whose partials it combines
  void* module = nullptr;            // CUmodule
  void* fn = nullptr;                // CUfunction
  int grid = 1;
  int block = 0;                     // launch block (spec.block, or the best warp count for flex kernels)
  int smem = 0;                      // dynamic shared memory at that block
  int64_t ws_off = 0;                // floats into the workspace pool
  int64_t sync_off = 0;              // u32 words into the sync pool
  bool cache_hit = false;
};

class Executor {
 public:
  Executor(const Graph& fused, const ExecOptions& opts);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  json::Value describe() const;
  void run(const void* const* inputs, void* const* outputs, void* stream);
  void run_host(const void* const* host_inputs, void* const* host_outputs, void* stream);
  json::Value profile(const void* const* inputs, void* const* outputs, void* stream, int iters);
  json::Value trace(const void* const* inputs, void* const* outputs, void* stream);

  const std::vector<KernelInst>& kernels() const { return kernels_; }
  const std::vector<std::string>& input_ids() const { return input_ids_; }
  const std::vector<std::string>& output_ids() const { return output_ids_; }

 private:
  void build_kernels();
  void plan_arena();
  void init_device();
  void plan_chunks();
  void plan_deps();
  bool ordered_before(int a, int b) const;
  void launch_all(const void* const* inputs, void* const* outputs, void* stream, std::vector<void*>* events);
  void launch_dag(const void* const* inputs, void* const* outputs, void* stream);
  void copy_aliased_outputs(const void* const* inputs, void* const* outputs, void* stream);
  void launch_one(int i, int c, int chunks, const void* const* inputs, void* const* outputs, void* stream);

  Graph g_;
  ExecOptions opts_;
  std::vector<ValueBuf> bufs_;
  std::map<std::string, int> buf_of_;
  std::vector<KernelInst> kernels_;
  std::vector<Segment> segments_;
  int launches_per_run_ = 0;
  int folded_kernels_ = 0;
  int sunk_kernels_ = 0;
  std::vector<void*> lanes_;        // CUstreams for pipelined chunk lanes
  std::vector<void*> lane_events_;  // CUevents: [segment-local kernel j][chunk c] done, plus fork/join
  // dataflow launch (ExecOptions::concurrent_lanes)
  bool dag_ = false;
  std::vector<std::vector<int>> preds_;  // kernel -> kernels it must follow
  std::vector<std::vector<uint64_t>> anc_;  // kernel -> ancestor bitset
  std::vector<bool> critical_;              // kernel on the estimated critical path
  std::vector<int> issue_;                  // dataflow issue order (a topological order)
  bool pdl_this_launch_ = true;             // launch_dag's per-launch PDL decision
  int high_priority_ = 0;                   // greatest stream priority of the context
  std::vector<int> writer_;                 // value buffer -> producing kernel
  std::vector<std::vector<int>> touch_;     // value buffer -> kernels reading / writing it
  std::vector<void*> dag_lanes_;         // CUstreams for lanes 1.. (lane 0 = the caller's stream)
  std::vector<void*> dag_events_;        // per kernel "done", plus the fork event
  void* copy_streams_[2] = {nullptr, nullptr};  // run_host: H2D and D2H copy streams
  std::vector<void*> in_events_, kernel_events_;
  void* start_event_ = nullptr;
  bool segments_ok_for_overlap() const;
  std::vector<std::string> input_ids_, output_ids_;
  std::vector<int64_t> input_bytes_, output_bytes_;
  std::vector<std::vector<int64_t>> input_dims_, output_dims_;
  std::vector<std::pair<int, int>> output_copies_;  // (output slot, source buffer) when an output aliases another value
  int64_t arena_bytes_ = 0, ws_floats_ = 0, sync_words_ = 0;
  uint64_t arena_ = 0, ws_ = 0, sync_ = 0;  // CUdeviceptr
  int sms_ = 148;
  bool device_ready_ = false;
  void* ctx_ = nullptr;  // retained primary context of opts_.device
  // CUDA-graph replay cache for the last pointer set
  void* graph_exec_ = nullptr;
  void* graph_stream_ = nullptr;
  std::vector<const void*> graph_ptrs_;
  std::vector<uint64_t> host_staging_;  // device buffers for run_host
  std::vector<std::string> cubins_tmp_;  // compiled images until modules load
};

}  // namespace exec
}  // namespace stitch
