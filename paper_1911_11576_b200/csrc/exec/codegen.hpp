// Stitched-kernel code generation: one fused op (its body graph) in, one
// sm_100a CUDA kernel out. This replaces the reference's template search +
// CUDA-C sketch emitter (proj/include/stitch/emitter.hpp) with kernels that
// actually run: the paper's composition mechanisms (§5.1) become
//
//   ROW scheme   the group's tensors share a leading "row" index space; a
//                warp (or a CTA) owns one row at a time and runs every fused
//                op for it with intermediates in registers (thread
//                composition), row reductions by shuffles (warp
//                composition) or through shared memory plus TMA-staged
//                operand tiles for gemm stages (block composition); column /
//                scalar reductions accumulate per thread across rows and
//                finish with a deterministic grid-wide combine;
//   FLAT scheme  elementwise groups without a row structure: vectorised
//                grid-stride loops;
//   SECTIONED    the general fallback: one grid-stride section per
//                materialised value, separated by a grid barrier;
//   packing      independent components of one group run on disjoint CTA
//                ranges of the same launch (§5.1(a)).
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "../host/ir.hpp"

namespace stitch {
namespace exec {

struct KernelSpec {
  std::string name;
  std::string source;  // generated kernel body; the device header is prepended at compile time
  std::string scheme;  // human-readable scheme summary, e.g. "row_warp(k=1,S=768)"
  std::set<std::string> composition;  // packing | thread | warp | block
  int block = 256;
  int max_grid = 1;          // useful CTAs; the runtime clamps cooperative grids to residency
  bool cooperative = false;  // needs co-residency (grid barrier)
  int smem_bytes = 0;        // dynamic shared memory per CTA
  int64_t workspace_floats = 0;
  int sync_words = 0;                // grid-barrier words
  std::vector<std::string> inputs;   // pointer arguments, in order
  std::vector<std::string> outputs;  // pointer arguments, in order
  int64_t algo_bytes = 0;            // each input read once + each output written once
  int64_t flops = 0;                 // 2*M*N*K summed over gemm stages
  // Row-chunkable: one ROW component with no cross-row reduction, so the
  // kernel can run any row range [row_lo, row_hi) (trailing kernel args) and
  // touches exactly that range's bytes of every rowed tensor.
  bool chunkable = false;
  // Warp-per-row kernels read blockDim at run time, so the runtime may launch
  // them with any warp count <= block; shared memory scales per warp.
  bool flex_block = false;
  int min_grid = 1;                  // ranged packing: at least one CTA per component
  int cluster = 0;                   // thread-block cluster size (1-D); grid = max_grid exactly
  // TMA tensor maps passed by value after the standard arguments (gws scheme):
  // input argument index, box rows, 0 = 128B swizzle (K-major A operand),
  // 1 = 128B swizzle of 32-byte atoms (MN-major B operand); [S][64][64] fp32
  struct TmaParam {
    int input = 0;
    int box_rows = 64;
    int swizzle = 0;
    int64_t samples = 0;
  };
  std::vector<TmaParam> tma;
  int smem_per_warp = 0;
  int64_t rows = 0;
  int rows_per_cta = 1;
  int row_threads = 32;  // threads per row of a single warp-row component (flex_block grids)
  int max_partials = 0;  // > 0: the workspace holds this many per-CTA partial rows (grid cap)
  // split_cross: the fixed-order combine of the per-CTA column partials runs
  // as a second kernel `fin_name` (same arguments; row_lo = the partial count,
  // i.e. this kernel's grid) -- no grid barrier, so this kernel is not
  // cooperative and its row outputs release their consumers before the
  // column reductions are folded. fin_outputs: the outputs it writes.
  std::string fin_name, fin_source;
  int fin_max_grid = 0;
  int fin_smem_bytes = 0;
  std::vector<std::string> fin_outputs;
};

struct CodegenOptions {
  int num_sms = 148;
  int max_smem = 232448 - 1024;  // per-CTA opt-in limit minus a static-smem margin
  bool allow_row = true;         // false forces SECTIONED (tests)
  // Measured on B200 (scripts/time_graph.py): the double buffer loses to
  // the occupancy it costs (GRU 139 -> 170 us at 1 CTA/SM), so it is
  // opt-in; row prefetching (only where the prefetched tiles take <= 32
  // registers) helps CTA rows (BERT row_cta groups ~5 % each, step 2419 ->
  // 2382 us) but costs warp rows occupancy (layernorm 18.4 -> 20.5 us), so
  // it is on for CTA rows only.
  bool row_prefetch = true;        // prefetch the next row's register tiles (CTA rows)
  bool row_prefetch_warp = false;  // ... and warp rows
  // Narrow rows (<= `narrow_row_max` elements, warp scheme, no column
  // reductions): a group of 4..16 lanes per row, so each lane keeps ~16
  // elements (4 x 128-bit loads per operand) in flight and a warp works on
  // several rows at once (softmax rows of 128 keys: 1 load per lane with a
  // whole warp per row).
  bool narrow_rows = true;
  // purely elementwise components (row-vector broadcasts only) as FLAT
  // grid-stride loops instead of ROW: balanced over the grid whatever the
  // row count (4096 rows on 1184 CTA slots leave a 14 % round-up tail)
  bool flat_elementwise = false;
  // cross-row (column) reductions of a row group folded by a separate
  // dependent kernel instead of after a grid barrier (KernelSpec::fin_*)
  bool split_cross = true;
  // > 0: a CTA of this many threads per row for row groups that would run a
  // warp per row (register-heavy multi-layer groups: more warps resident,
  // fewer values per thread); a per-group tuning candidate
  int cta_rows = 0;
  // > 0: threads per row of CTA-row groups (default 256 up to 4096 elements):
  // fewer elements per thread and more, smaller CTAs per SM -- a finer
  // round-up tail over 4096 rows; a per-group tuning candidate
  int cta_threads = 0;
  // Row-scheme inputs (body parameter ids) whose only reader is this kernel
  // and that are not graph outputs (arena intermediates): after a row is
  // consumed its 128-byte lines are invalidated in L2 (discard.global.L2),
  // so dirty lines the producer left there are never written back to HBM.
  // Filled per kernel by the executor when `l2_discard` is on.
  std::set<std::string> discard_inputs;
  bool l2_discard = true;
  // griddepcontrol.launch_dependents at kernel entry (a PDL dependent may be
  // scheduled as soon as every CTA of this kernel runs); false: implicit at
  // CTA exit
  bool pdl_early_trigger = true;
  // CTA rows: in-row reductions alternate two scratch buffers, one CTA
  // barrier per reduction instead of two
  bool pp_reduce = false;
  // gws tail: evict-first (st.global.cs) stores of the outputs
  bool gws_stream_stores = false;  // measured neutral-to-worse on BERT (1.454 -> 1.469 ms): opt-in  // measured worse (BERT 1.726 -> 1.773 ms): one 128-bit load per thread in flight
  int narrow_row_max = 256;
  bool loop_fusion = true;
  bool colred = true;
  bool colred_fused = true;
  bool rcp_divide = true;
  // timeline tracing: every warp's lane 0 folds %globaltimer at kernel entry
  // and exit into two u64 words just before the kernel's sync line
  // (Executor::trace; never on in timed runs)
  bool trace = false;  // c / x with c = +-2^k as the exact c * rcp.rn(x)
  // every elementwise divide / reciprocal as branch-free rcp.approx + Newton
  // (<= 1 ulp; __frcp_rn / IEEE division carry a slow-path call)
  bool nr_divide = false;
  // Row groups of [S][64][64] tiles with two batched dots on kernel inputs
  // (the GRU group): the warp-specialised tcgen05 scheme (device gws::run,
  // TMA producer / MMA issuer / split / tail warps). Off: the ROW scheme.
  bool gws = true;
  // A kernel that is one unfused dot / batched dot (operands from HBM): the
  // tiled fp32 GEMM scheme (device gemm::run). Off: SECTIONED / BLOCK loops.
  bool gemm = true;
  // __launch_bounds__ minimum CTAs per SM (register budget hint; 0: none)
  int min_ctas_per_sm = 0;
  // Groups ROW / COLRED / FLAT cannot take (dots + reductions over different
  // index spaces, paper Fig. 1) run as BLOCK composition -- one CTA per
  // leading index, shared memory at the planner's Alg. 4 alloc map -- instead
  // of grid-barrier SECTIONED when they share a leading index.
  bool block_compose = true;
  bool tma_early = false;  // CTA rows: next row's TMA tiles requested as soon as their last reader is done
  bool cross_smem = true;  // warp rows: many column-reduction partials in the warp's shared slab
  int cross_smem_min_regs = 16;  // ... when they would take more than this many registers per lane
  int colred_ctas_per_sm = 4;  // COLRED tiles per SM (one resident wave)
  // COLRED row chunks of a column block as one thread-block cluster of this
  // many CTAs, combined through distributed shared memory (cluster barrier
  // + DSMEM loads, fixed rank order) instead of global partials + fence +
  // arrival counter + last-CTA fold; 0: the global scheme
  int colred_cluster = 16;
  // COLRED also for groups whose other outputs are elementwise over the
  // reduce input's [R, C] (written from the same tiles). Off by default:
  // measured slower than CTA rows on BERT's [4096, 3072] GeLU-backward groups
  // (step 2.111 -> 2.433 ms); a per-group tuning candidate.
  bool colred_eout = false;  // BERT step 2.257 -> 2.195 ms (8: 2.205; 2: 2.473)
  int colred_cols = 32;        // COLRED column-block width: 32, 64 or 128 floats (32: BERT 2387 -> 2375 us)
  bool colred_cp_async = true;  // COLRED loads staged through cp.async (all of a pass in flight)  // COLRED also for reduces of an inline elementwise producer chain
  // many-input rows: load inputs per fused-loop step, not per row (measured
  // neutral on the BERT LayerNorm-backward groups: the column-reduction
  // partials, not the inputs, hold most of the registers)
  bool lazy_inputs = false;
  // Many column reductions in a wide warp-row group spill registers; CTA per
  // row avoids the spills but serialises 16 barriers per LayerNorm-backward
  // row: measured slower on B200 (BERT LN-backward groups 88 -> 123 us).
  bool wide_cross_cta = false;
  int wide_cross_threads = 0;     // CTA size for those rows (0: ~12 columns per thread)             // dedicated 2-D tiled scheme for lone column reductions
  // Packed independent components: disjoint CTA ranges (default; measured
  // faster on B200: encoder 96 vs 107 us, the streaming column reduction
  // overlaps the compute-heavier row group) or one after another on every CTA.
  bool pack_sequential = false;
  // Batched-GEMM stages of 64x64 row tiles on tcgen05 (3xTF32, TMEM
  // accumulator) instead of register-tiled FFMA.
  // Measured on B200 (GRU group): 207 us with staged operands (1 CTA/SM),
  // 291 us reading operands straight from global, vs 137 us for the
  // register-tiled FFMA stage -- the per-row split + commit latency is not
  // yet overlapped, so both are opt-in.
  bool tensor_cores = false;
  bool tc_direct_loads = false;
  bool tc_pipeline = true;        // with tensor_cores: next row's split + MMAs before this row's epilogue        // one loop per run of same-extent elementwise ops (scalars inside)
  bool tma_double_buffer = false; // double-buffer external TMA row tiles
};

// `constants` maps body-parameter ids whose value is a known scalar constant
// to that value; those become literals instead of pointer arguments.
KernelSpec generate_kernel(const Graph& body, const std::string& name, const std::map<std::string, double>& constants,
                           const CodegenOptions& opts = {});

}  // namespace exec
}  // namespace stitch
