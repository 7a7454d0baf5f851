// Stitched-kernel runtime (see runtime.hpp).
#include "runtime.hpp"

#include <nvrtc.h>

#include <algorithm>
#include <set>
#include <numeric>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <sys/stat.h>
#include <unistd.h>

#include "cuda_api.hpp"

namespace stitch {
namespace exec {

namespace {

#include "device_header.inc"  // defines kDeviceHeader (generated from device/stitch_device.cuh)

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

const char* kCompileOpts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-DSTITCH_NVRTC=1"};

std::string sanitize(const std::string& id) {
  std::string s;
  for (char c : id) s += (std::isalnum(static_cast<unsigned char>(c)) ? c : '_');
  if (s.empty() || std::isdigit(static_cast<unsigned char>(s[0]))) s = "k_" + s;
  return s;
}

std::mutex g_compile_mu;

}  // namespace

const std::string& device_header_source() {
  static const std::string h(kDeviceHeader);
  return h;
}

std::string full_source(const KernelSpec& spec) { return device_header_source() + "\n" + spec.source; }

std::string compile_cubin(const std::string& source, const std::string& cache_dir, bool* cache_hit) {
  std::string key = source;
  for (const char* o : kCompileOpts) key += std::string("\n//opt ") + o;
  char hex[32];
  std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(fnv1a(key)));
  const std::string path = cache_dir.empty() ? "" : cache_dir + "/" + hex + ".cubin";
  if (cache_hit) *cache_hit = false;
  if (!path.empty()) {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      std::stringstream buf;
      buf << in.rdbuf();
      if (cache_hit) *cache_hit = true;
      return buf.str();
    }
  }
  std::lock_guard<std::mutex> lock(g_compile_mu);
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, source.c_str(), "stitched.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw std::runtime_error("nvrtcCreateProgram failed");
  nvrtcResult rc = nvrtcCompileProgram(prog, static_cast<int>(sizeof(kCompileOpts) / sizeof(kCompileOpts[0])), kCompileOpts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string log(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &log[0]);
  if (rc != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    throw std::runtime_error(std::string("NVRTC compile failed: ") + nvrtcGetErrorString(rc) + "\n" + log);
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::string cubin(n, '\0');
  nvrtcGetCUBIN(prog, &cubin[0]);
  nvrtcDestroyProgram(&prog);
  if (!path.empty()) {
    mkdir(cache_dir.c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string(getpid());
    std::ofstream out(tmp, std::ios::binary);
    out.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
    out.close();
    std::rename(tmp.c_str(), path.c_str());
  }
  return cubin;
}

// ---------------------------------------------------------------------------

void apply_codegen_options(CodegenOptions& c, const json::Value& o) {
  if (o.has("smem_limit_bytes")) c.max_smem = static_cast<int>(o.at("smem_limit_bytes").as_int());
  if (o.has("allow_row")) c.allow_row = o.at("allow_row").as_bool();
  if (o.has("num_sms")) c.num_sms = static_cast<int>(o.at("num_sms").as_int());
  if (o.has("tc_pipeline")) c.tc_pipeline = o.at("tc_pipeline").as_bool();
  if (o.has("tc_direct_loads")) c.tc_direct_loads = o.at("tc_direct_loads").as_bool();
  if (o.has("tensor_cores")) c.tensor_cores = o.at("tensor_cores").as_bool();
  if (o.has("pack_sequential")) c.pack_sequential = o.at("pack_sequential").as_bool();
  if (o.has("wide_cross_threads")) c.wide_cross_threads = static_cast<int>(o.at("wide_cross_threads").as_int());
  if (o.has("wide_cross_cta")) c.wide_cross_cta = o.at("wide_cross_cta").as_bool();
  if (o.has("lazy_inputs")) c.lazy_inputs = o.at("lazy_inputs").as_bool();
  if (o.has("colred")) c.colred = o.at("colred").as_bool();
  if (o.has("row_prefetch_warp")) c.row_prefetch_warp = o.at("row_prefetch_warp").as_bool();
  if (o.has("narrow_rows")) c.narrow_rows = o.at("narrow_rows").as_bool();
  if (o.has("flat_elementwise")) c.flat_elementwise = o.at("flat_elementwise").as_bool();
  if (o.has("split_cross")) c.split_cross = o.at("split_cross").as_bool();
  if (o.has("cta_rows")) c.cta_rows = static_cast<int>(o.at("cta_rows").as_int());
  if (o.has("cta_threads")) c.cta_threads = static_cast<int>(o.at("cta_threads").as_int());
  if (o.has("l2_discard")) c.l2_discard = o.at("l2_discard").as_bool();
  if (o.has("pdl_early_trigger")) c.pdl_early_trigger = o.at("pdl_early_trigger").as_bool();
  if (o.has("pp_reduce")) c.pp_reduce = o.at("pp_reduce").as_bool();
  if (o.has("gws_stream_stores")) c.gws_stream_stores = o.at("gws_stream_stores").as_bool();
  if (o.has("narrow_row_max")) c.narrow_row_max = static_cast<int>(o.at("narrow_row_max").as_int());
  if (o.has("rcp_divide")) c.rcp_divide = o.at("rcp_divide").as_bool();
  if (o.has("trace")) c.trace = o.at("trace").as_bool();
  if (o.has("gws")) c.gws = o.at("gws").as_bool();
  if (o.has("gemm")) c.gemm = o.at("gemm").as_bool();
  if (o.has("nr_divide")) c.nr_divide = o.at("nr_divide").as_bool();
  if (o.has("min_ctas_per_sm")) c.min_ctas_per_sm = static_cast<int>(o.at("min_ctas_per_sm").as_int());
  if (o.has("block_compose")) c.block_compose = o.at("block_compose").as_bool();
  if (o.has("tma_early")) c.tma_early = o.at("tma_early").as_bool();
  if (o.has("cross_smem")) c.cross_smem = o.at("cross_smem").as_bool();
  if (o.has("cross_smem_min_regs")) c.cross_smem_min_regs = static_cast<int>(o.at("cross_smem_min_regs").as_int());
  if (o.has("colred_fused")) c.colred_fused = o.at("colred_fused").as_bool();
  if (o.has("colred_cp_async")) c.colred_cp_async = o.at("colred_cp_async").as_bool();
  if (o.has("colred_cols")) c.colred_cols = static_cast<int>(o.at("colred_cols").as_int());
  if (o.has("colred_ctas_per_sm")) c.colred_ctas_per_sm = static_cast<int>(o.at("colred_ctas_per_sm").as_int());
  if (o.has("colred_cluster")) c.colred_cluster = static_cast<int>(o.at("colred_cluster").as_int());
  if (o.has("colred_eout")) c.colred_eout = o.at("colred_eout").as_bool();
  if (o.has("loop_fusion")) c.loop_fusion = o.at("loop_fusion").as_bool();
  if (o.has("row_prefetch")) c.row_prefetch = o.at("row_prefetch").as_bool();
  if (o.has("tma_double_buffer")) c.tma_double_buffer = o.at("tma_double_buffer").as_bool();
}

Executor::Executor(const Graph& fused, const ExecOptions& opts) : g_(fused), opts_(opts) {
  for (const OpNode& n : g_.nodes)
    if (n.type == OpType::kParameter || (n.type == OpType::kConstant && !n.value)) {
      input_ids_.push_back(n.id);
      input_dims_.push_back(n.shape.dims);
      input_bytes_.push_back(n.shape.byte_count());
      if (n.shape.dtype != DType::f32()) throw GraphError("stitched executor: only f32 inputs are supported (" + n.id + ")");
    }
  for (const std::string& o : g_.outputs) {
    const OpNode& n = g_.at(o);
    if (n.type == OpType::kTuple)
      for (const std::string& e : n.operands) output_ids_.push_back(e);
    else
      output_ids_.push_back(o);
  }
  for (const std::string& o : output_ids_) {
    output_dims_.push_back(g_.at(o).shape.dims);
    output_bytes_.push_back(g_.at(o).shape.byte_count());
  }
  build_kernels();
  plan_chunks();
  plan_deps();
  plan_arena();
  if (!opts_.compile_only) init_device();
}

Executor::~Executor() {
  if (!ctx_) return;
  CudaApi& cu = CudaApi::get();
  {
  CtxScope scope(ctx_);
  if (graph_exec_) cu.cuGraphExecDestroy(static_cast<CUgraphExec>(graph_exec_));
  for (void* e : in_events_) cu.cuEventDestroy(static_cast<CUevent>(e));
  for (void* e : kernel_events_) cu.cuEventDestroy(static_cast<CUevent>(e));
  if (start_event_) cu.cuEventDestroy(static_cast<CUevent>(start_event_));
  for (void* st : copy_streams_)
    if (st) cu.cuStreamDestroy(static_cast<CUstream>(st));
  for (void* e : lane_events_) cu.cuEventDestroy(static_cast<CUevent>(e));
  for (void* st : lanes_) cu.cuStreamDestroy(static_cast<CUstream>(st));
  for (void* e : dag_events_) cu.cuEventDestroy(static_cast<CUevent>(e));
  for (void* st : dag_lanes_) cu.cuStreamDestroy(static_cast<CUstream>(st));
  for (KernelInst& k : kernels_)
    if (k.module) cu.cuModuleUnload(static_cast<CUmodule>(k.module));
  if (arena_) cu.cuMemFree(arena_);
  if (ws_) cu.cuMemFree(ws_);
  if (sync_) cu.cuMemFree(sync_);
  for (uint64_t p : host_staging_)
    if (p) cu.cuMemFree(p);
  }
  CUdevice dev;
  if (cu.cuDeviceGet(&dev, opts_.device) == CUDA_SUCCESS) cu.cuDevicePrimaryCtxRelease(dev);
}

void Executor::build_kernels() {
  // Buffer key of a value id in the fused graph.
  auto key_of = [&](const std::string& id) -> std::string {
    const OpNode& n = g_.at(id);
    if (n.type == OpType::kGetElement) return n.operands[0] + "#" + std::to_string(n.tuple_index);
    if (n.type == OpType::kFused) return id + "#0";
    return id;
  };
  std::map<std::string, int> input_slot;
  for (size_t i = 0; i < input_ids_.size(); ++i) input_slot[input_ids_[i]] = static_cast<int>(i);
  auto buffer = [&](const std::string& key, int64_t bytes) {
    auto it = buf_of_.find(key);
    if (it != buf_of_.end()) return it->second;
    ValueBuf b;
    b.key = key;
    b.bytes = bytes;
    auto s = input_slot.find(key);
    if (s != input_slot.end()) {
      b.kind = ValueBuf::kInput;
      b.slot = s->second;
    }
    bufs_.push_back(b);
    buf_of_[key] = static_cast<int>(bufs_.size()) - 1;
    return static_cast<int>(bufs_.size()) - 1;
  };

  // Uniform constants: value-carrying constants and (unfused) broadcasts of
  // them. Consumers read them as literals, so a broadcast-of-constant
  // kernel whose value is not a graph output is dead and never launched.
  std::map<std::string, double> uniform;
  std::set<std::string> graph_outs(output_ids_.begin(), output_ids_.end());
  const std::vector<std::string> topo = topological_sort(g_);
  for (const std::string& id : topo) {
    const OpNode& n = g_.at(id);
    if (n.type == OpType::kConstant && n.value) uniform[id] = *n.value;
    else if (opts_.fold_constants && n.type == OpType::kElementwise && n.elem_name == "broadcast" &&
             uniform.count(n.operands.at(0)))
      uniform[id] = uniform[n.operands[0]];
  }
  // Broadcast sinking: top-level (unfused) broadcasts of small tensors.
  std::map<std::string, std::string> sink_src;  // broadcast id -> its source
  if (opts_.sink_broadcasts)
    for (const std::string& id : topo) {
      const OpNode& n = g_.at(id);
      if (n.type != OpType::kElementwise || n.elem_name != "broadcast" || uniform.count(id)) continue;
      const OpNode& src = g_.at(n.operands.at(0));
      if (src.type == OpType::kTuple || src.type == OpType::kFused) continue;
      if (src.shape.byte_count() <= opts_.sink_max_bytes && src.shape.byte_count() * 4 <= n.shape.byte_count())
        sink_src[id] = n.operands[0];
    }
  std::map<std::string, std::string> names;
  struct Regen {  // what generated each kernel (L2-discard second pass)
    size_t ki;
    Graph body;
    std::string kname;
    std::map<std::string, double> consts;
    CodegenOptions co;
  };
  std::vector<Regen> regen;
  for (const std::string& id : topo) {
    const OpNode& n = g_.at(id);
    if (n.type != OpType::kFused && !is_fusible(n)) continue;
    if (n.type != OpType::kFused && uniform.count(id) && !graph_outs.count(id)) {
      ++folded_kernels_;
      continue;
    }
    if (sink_src.count(id) && !graph_outs.count(id)) {
      ++sunk_kernels_;  // every consumer kernel recomputes it from the source
      continue;
    }
    Graph body;
    std::vector<std::string> outer_inputs;
    std::vector<std::string> out_keys;
    if (n.type == OpType::kFused) {
      body = *n.body;
      int p = 0;
      for (const OpNode& bn : body.nodes)
        if (bn.type == OpType::kParameter) outer_inputs.push_back(n.operands.at(p++));
      const OpNode& tup = body.at(body.outputs.front());
      for (size_t i = 0; i < tup.operands.size(); ++i) out_keys.push_back(id + "#" + std::to_string(i));
    } else {
      // Unfused kernel op: a one-op body, so it runs through the same generator.
      for (const std::string& o : n.operands) {
        if (body.contains(o)) continue;
        OpNode prm;
        prm.id = o;
        prm.type = OpType::kParameter;
        prm.shape = g_.at(o).shape;
        body.add(prm);
        outer_inputs.push_back(o);
      }
      body.add(n);
      OpNode tup;
      tup.id = "__outputs";
      tup.type = OpType::kTuple;
      tup.operands = {n.id};
      tup.shape = n.shape;
      body.add(tup);
      body.outputs = {"__outputs"};
      out_keys.push_back(id);
    }
    // Sink broadcasts into this body: a parameter fed by a sunk broadcast
    // becomes that broadcast over a parameter of its (small) source.
    bool sinks = false;
    {
      int q = 0;
      for (const OpNode& bn : body.nodes)
        if (bn.type == OpType::kParameter) sinks = sinks || sink_src.count(outer_inputs.at(q++));
    }
    if (sinks) {
      Graph nb;
      std::vector<std::string> nouter;
      std::map<std::string, std::string> param_of;  // outer value -> body parameter id
      std::vector<std::pair<const OpNode*, std::string>> conv;  // body param node, source outer id
      int q = 0;
      for (const OpNode& bn : body.nodes) {
        if (bn.type != OpType::kParameter) continue;
        const std::string& outer = outer_inputs.at(q++);
        auto it = sink_src.find(outer);
        if (it != sink_src.end()) {
          conv.push_back({&bn, it->second});
        } else {
          nb.add(bn);
          nouter.push_back(outer);
          param_of[outer] = bn.id;
        }
      }
      for (auto& [bn, src] : conv) {
        if (param_of.count(src)) continue;
        OpNode prm;
        prm.id = src + "__sunk";
        while (body.contains(prm.id) || nb.contains(prm.id)) prm.id += "_";
        prm.type = OpType::kParameter;
        prm.shape = g_.at(src).shape;
        nb.add(prm);
        nouter.push_back(src);
        param_of[src] = prm.id;
      }
      for (auto& [bn, src] : conv) {
        OpNode b;
        b.id = bn->id;
        b.type = OpType::kElementwise;
        b.elem_name = "broadcast";
        b.operands = {param_of.at(src)};
        b.shape = bn->shape;
        nb.add(b);
      }
      for (const OpNode& bn : body.nodes)
        if (bn.type != OpType::kParameter) nb.add(bn);
      nb.outputs = body.outputs;
      body = std::move(nb);
      outer_inputs = std::move(nouter);
    }
    // Body parameter id -> outer value (positional for fused bodies).
    std::map<std::string, std::string> outer_of;
    std::map<std::string, double> consts;
    int p = 0;
    for (const OpNode& bn : body.nodes) {
      if (bn.type != OpType::kParameter) continue;
      const std::string& outer = outer_inputs.at(p++);
      outer_of[bn.id] = outer;
      auto u = uniform.find(outer);
      if (u != uniform.end()) consts[bn.id] = u->second;
    }
    std::string kname = sanitize(id);
    while (names.count(kname)) kname += "_";
    names[kname] = id;
    KernelInst k;
    k.op_id = id;
    // per-group codegen variant (Alg. 3 KernelEvalUpdate's measured choice)
    CodegenOptions co = opts_.codegen;
    if (opts_.kernel_options.is_object() && opts_.kernel_options.has(id)) {
      apply_codegen_options(co, opts_.kernel_options.at(id));
      k.variant = opts_.kernel_options.at(id);
    }
    k.spec = generate_kernel(body, kname, consts, co);
    if (co.l2_discard) regen.push_back({kernels_.size(), body, kname, consts, co});
    const OpNode& tup = body.at(body.outputs.front());
    for (const std::string& in : k.spec.inputs) {
      const std::string& outer = outer_of.at(in);
      k.in_bufs.push_back(buffer(key_of(outer), g_.at(outer).shape.byte_count()));
    }
    for (const std::string& o : k.spec.outputs) {
      auto pos = std::find(tup.operands.begin(), tup.operands.end(), o) - tup.operands.begin();
      k.out_bufs.push_back(buffer(out_keys.at(pos), body.at(o).shape.byte_count()));
    }
    k.reads = k.in_bufs;
    k.writes = k.out_bufs;
    if (!k.spec.fin_source.empty()) {
      // split_cross: the row kernel writes its row outputs, the fold kernel
      // (next in launch order) the column reductions from the partials
      KernelInst f;
      f.op_id = id;
      f.variant = k.variant;
      f.spec = k.spec;
      f.spec.name = k.spec.fin_name;
      f.spec.source = k.spec.fin_source;
      f.spec.fin_source.clear();
      f.spec.scheme = "fold(" + std::to_string(k.spec.fin_outputs.size()) + " column reductions of " + k.spec.name + ")";
      f.spec.composition = {"block"};
      f.spec.block = opts_.fold_threads;
      f.spec.max_grid = k.spec.fin_max_grid;
      f.spec.min_grid = 1;
      f.spec.cooperative = false;
      f.spec.smem_bytes = opts_.fold_threads * 4 + 16;
      f.spec.sync_words = 0;
      f.spec.chunkable = false;
      f.spec.flex_block = false;
      f.spec.cluster = 0;
      f.spec.tma.clear();
      f.spec.rows = 0;
      f.spec.algo_bytes = 0;  // partials only; the group's bytes are counted on the row kernel
      f.in_bufs = k.in_bufs;
      f.out_bufs = k.out_bufs;
      f.reads = k.in_bufs;
      std::set<std::string> folded(k.spec.fin_outputs.begin(), k.spec.fin_outputs.end());
      k.writes.clear();
      for (size_t j = 0; j < k.out_bufs.size(); ++j) {
        if (folded.count(k.spec.outputs[j]))
          f.writes.push_back(k.out_bufs[j]);
        else
          k.writes.push_back(k.out_bufs[j]);
      }
      f.reads.insert(f.reads.end(), k.writes.begin(), k.writes.end());  // kept alive (passed, not read)
      f.fold_of = static_cast<int>(kernels_.size());
      kernels_.push_back(std::move(k));
      kernels_.push_back(std::move(f));
      continue;
    }
    kernels_.push_back(std::move(k));
  }
  // L2 discard: an arena value (not a graph output) read by exactly one
  // kernel is dead once that kernel has consumed a row of it; regenerate
  // those consumers with the value in their discard set.
  if (!regen.empty()) {
    std::set<std::string> out_keys_all;
    for (const std::string& o : output_ids_) {
      const OpNode& n = g_.at(o);
      out_keys_all.insert(n.type == OpType::kGetElement ? n.operands[0] + "#" + std::to_string(n.tuple_index)
                          : n.type == OpType::kFused    ? o + "#0"
                                                        : o);
    }
    std::vector<int> readers(bufs_.size(), 0), produced(bufs_.size(), 0);
    for (const KernelInst& k : kernels_) {
      if (k.fold_of >= 0) continue;  // a fold passes the pointers but reads only its partials
      std::set<int> r(k.in_bufs.begin(), k.in_bufs.end());
      for (int b : r) ++readers[b];
      for (int b : k.writes) ++produced[b];
    }
    for (Regen& rg : regen) {
      KernelInst& k = kernels_[rg.ki];
      std::set<std::string> dead;
      for (size_t j = 0; j < k.in_bufs.size(); ++j) {
        const int b = k.in_bufs[j];
        if (bufs_[b].kind == ValueBuf::kArena && produced[b] == 1 && readers[b] == 1 && !out_keys_all.count(bufs_[b].key))
          dead.insert(k.spec.inputs[j]);
      }
      if (dead.empty()) continue;
      rg.co.discard_inputs = dead;
      KernelSpec spec = generate_kernel(rg.body, rg.kname, rg.consts, rg.co);
      if (spec.inputs != k.spec.inputs || spec.outputs != k.spec.outputs || spec.fin_name != k.spec.fin_name)
        throw InternalError("L2-discard regeneration changed kernel " + rg.kname + "'s arguments");
      k.spec = std::move(spec);
    }
  }
  // Lifetimes.
  for (size_t ki = 0; ki < kernels_.size(); ++ki) {
    for (int b : kernels_[ki].writes) {
      if (bufs_[b].first >= 0) throw InternalError("value produced twice: " + bufs_[b].key);
      bufs_[b].first = bufs_[b].last = static_cast<int>(ki);
    }
    for (int b : kernels_[ki].reads) {
      if (bufs_[b].kind == ValueBuf::kInput) continue;
      if (bufs_[b].first < 0) throw InternalError("value consumed before it is produced: " + bufs_[b].key);
      bufs_[b].last = std::max(bufs_[b].last, static_cast<int>(ki));
    }
  }
  // Graph outputs.
  for (size_t i = 0; i < output_ids_.size(); ++i) {
    const OpNode& n = g_.at(output_ids_[i]);
    std::string key = n.type == OpType::kGetElement ? n.operands[0] + "#" + std::to_string(n.tuple_index)
                      : n.type == OpType::kFused    ? output_ids_[i] + "#0"
                                                    : output_ids_[i];
    auto it = buf_of_.find(key);
    if (it == buf_of_.end() || bufs_[it->second].kind != ValueBuf::kArena) {
      if (it == buf_of_.end()) throw GraphError("stitched executor: output " + output_ids_[i] + " is not computed by any kernel");
      output_copies_.push_back({static_cast<int>(i), it->second});
      continue;
    }
    bufs_[it->second].kind = ValueBuf::kOutput;
    bufs_[it->second].slot = static_cast<int>(i);
  }
  // Compile (or fetch from the cache). STITCH_DUMP_DIR: also write every
  // generated kernel body there as <name>.cu (inspection / profiling aid).
  const char* dump = std::getenv("STITCH_DUMP_DIR");
  for (KernelInst& k : kernels_) {
    if (dump && *dump) {
      std::ofstream f(std::string(dump) + "/" + k.spec.name + ".cu");
      f << k.spec.source;
    }
    bool hit = false;
    std::string cubin = compile_cubin(full_source(k.spec), opts_.cache_dir, &hit);
    k.cache_hit = hit;
    k.module = nullptr;
    k.spec.source.shrink_to_fit();
    cubins_tmp_.push_back(std::move(cubin));
  }
}

void Executor::plan_chunks() {
  segments_.clear();
  const int nk = static_cast<int>(kernels_.size());
  int i = 0;
  while (i < nk) {
    Segment seg;
    seg.first = i;
    int j = i;
    if (opts_.chunking && kernels_[i].spec.chunkable)
      while (j + 1 < nk && kernels_[j + 1].spec.chunkable) ++j;
    seg.last = j;
    i = j + 1;
    // Intermediates produced and fully consumed inside the segment.
    std::vector<int> local;
    int64_t inter = 0;
    for (size_t b = 0; b < bufs_.size(); ++b) {
      const ValueBuf& x = bufs_[b];
      if (x.kind == ValueBuf::kArena && x.first >= seg.first && x.last <= seg.last && x.last > x.first) {
        local.push_back(static_cast<int>(b));
        inter += x.bytes;
      }
    }
    if (seg.last > seg.first && !local.empty()) {
      // Smallest power-of-two chunk count that brings the per-chunk
      // intermediates under the L2 budget, dividing every kernel's rows and
      // every local buffer, with enough rows per chunk to fill the GPU.
      int best = 1;
      for (int C = 2; C <= opts_.max_chunks; C *= 2) {
        bool ok = true;
        for (int k = seg.first; k <= seg.last && ok; ++k) {
          const KernelSpec& sp = kernels_[k].spec;
          ok = sp.rows % C == 0 && (!opts_.chunk_fill || sp.rows / C >= static_cast<int64_t>(sms_) * 2 * sp.rows_per_cta);
        }
        for (int b : local) ok = ok && bufs_[b].bytes % (static_cast<int64_t>(C) * 256) == 0;
        if (!ok) break;
        best = C;
        if (inter / C <= opts_.chunk_l2_bytes) break;
      }
      seg.chunks = best;
      if (best > 1) {
        for (int b : local) {
          bufs_[b].chunks = best;
          bufs_[b].ring = opts_.chunk_pipeline ? std::min(best, std::max(1, opts_.chunk_ring)) : 1;
        }
        // A chunked segment runs all of its kernels once per chunk, so any
        // buffer it touches is live across the whole segment (not just its
        // own kernel-index interval): widen lifetimes before plan_arena so
        // no chunk ring is placed on top of a value a later chunk still
        // writes or reads.
        for (int k = seg.first; k <= seg.last; ++k) {
          for (const std::vector<int>* v : {&kernels_[k].reads, &kernels_[k].writes})
            for (int b : *v) {
              bufs_[b].first = std::min(bufs_[b].first, seg.first);
              bufs_[b].last = std::max(bufs_[b].last, seg.last);
            }
        }
      }
    }
    segments_.push_back(seg);
  }
  launches_per_run_ = 0;
  for (const Segment& sg : segments_) launches_per_run_ += (sg.last - sg.first + 1) * sg.chunks;
}

void Executor::plan_arena() {
  std::vector<int> order;
  for (size_t b = 0; b < bufs_.size(); ++b)
    if (bufs_[b].kind == ValueBuf::kArena) order.push_back(static_cast<int>(b));
  std::sort(order.begin(), order.end(), [&](int a, int b) { return bufs_[a].arena_bytes() > bufs_[b].arena_bytes(); });
  std::vector<int> placed;
  const int64_t align = 256;
  for (int b : order) {
    ValueBuf& x = bufs_[b];
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (int p : placed) {
      const ValueBuf& y = bufs_[p];
      const bool live = dag_ ? !(ordered_before(b, p) || ordered_before(p, b)) : (y.first <= x.last && x.first <= y.last);
      if (live) busy.push_back({y.offset, y.offset + y.arena_bytes()});
    }
    std::sort(busy.begin(), busy.end());
    int64_t off = 0;
    for (auto [lo, hi] : busy) {
      if (off + x.arena_bytes() <= lo) break;
      off = std::max(off, (hi + align - 1) / align * align);
    }
    x.offset = off;
    arena_bytes_ = std::max(arena_bytes_, off + x.arena_bytes());
    placed.push_back(b);
  }
  for (KernelInst& k : kernels_) {
    k.ws_off = 0;  // serial schedule: one shared workspace
    ws_floats_ = std::max(ws_floats_, k.spec.workspace_floats);
    if (opts_.codegen.trace) sync_words_ = (sync_words_ + 1) / 2 * 2 + 4;  // two u64 trace words before the line
    k.sync_off = sync_words_;
    sync_words_ += std::max(2, k.spec.sync_words) + 30;  // one 128-byte line per kernel
  }
  if (!dag_) return;
  // Workspace: kernels that may run concurrently (neither an ancestor of the
  // other) get disjoint ranges; an ancestor's range is free again.
  const int nk = static_cast<int>(kernels_.size());
  ws_floats_ = 0;
  for (int k = 0; k < nk; ++k) {
    const int64_t need = (kernels_[k].spec.workspace_floats + 63) / 64 * 64;
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (int j = 0; j < k; ++j)
      if (!(anc_[k][j / 64] >> (j % 64) & 1) && kernels_[j].spec.workspace_floats > 0)
        busy.push_back({kernels_[j].ws_off, kernels_[j].ws_off + kernels_[j].spec.workspace_floats});
    std::sort(busy.begin(), busy.end());
    int64_t off = 0;
    for (auto [lo, hi] : busy) {
      if (off + need <= lo) break;
      off = std::max(off, (hi + 63) / 64 * 64);
    }
    kernels_[k].ws_off = need > 0 ? off : 0;
    if (kernels_[k].fold_of >= 0) {  // reads the partials its row kernel (the previous index) left there
      kernels_[k].ws_off = kernels_[kernels_[k].fold_of].ws_off;
      continue;
    }
    ws_floats_ = std::max(ws_floats_, off + need);
  }
  // invariant: values sharing arena bytes are ordered by true dependencies
  for (size_t a = 0; a < bufs_.size(); ++a)
    for (size_t b = a + 1; b < bufs_.size(); ++b) {
      const ValueBuf &x = bufs_[a], &y = bufs_[b];
      if (x.kind != ValueBuf::kArena || y.kind != ValueBuf::kArena) continue;
      if (x.offset >= y.offset + y.arena_bytes() || y.offset >= x.offset + x.arena_bytes()) continue;
      if (!ordered_before(static_cast<int>(a), static_cast<int>(b)) && !ordered_before(static_cast<int>(b), static_cast<int>(a)))
        throw InternalError("dataflow arena: " + x.key + " and " + y.key + " share memory but may run concurrently");
    }
}

void Executor::plan_deps() {
  // Dataflow launch order (ExecOptions::concurrent_lanes): true dependencies
  // only. Arena placement (plan_arena) then lets two values share memory
  // only when every kernel touching one is an ancestor of the other's
  // producer, so memory reuse adds no edge.
  const int nk = static_cast<int>(kernels_.size());
  dag_ = opts_.concurrent_lanes > 1 && nk > 1;
  for (const Segment& sg : segments_) dag_ = dag_ && sg.chunks == 1;
  preds_.assign(nk, {});
  writer_.assign(bufs_.size(), -1);
  touch_.assign(bufs_.size(), {});
  for (int k = 0; k < nk; ++k) {
    for (int b : kernels_[k].writes) {
      writer_[b] = k;
      touch_[b].push_back(k);
    }
    for (int b : kernels_[k].reads) touch_[b].push_back(k);
  }
  if (!dag_) return;
  int last_coop = -1;
  for (int k = 0; k < nk; ++k) {
    std::set<int> p;
    for (int b : kernels_[k].reads)  // read after write
      if (writer_[b] >= 0 && writer_[b] != k) p.insert(writer_[b]);
    if (kernels_[k].fold_of >= 0) p.insert(kernels_[k].fold_of);  // partials in the workspace
    // grid-barrier kernels spin until every CTA is resident: never two in
    // flight (every other kernel in flight runs to completion unconditionally,
    // and PDL dependents launch only once all of their primary's CTAs run)
    if (kernels_[k].spec.cooperative) {
      if (last_coop >= 0) p.insert(last_coop);
      last_coop = k;
    }
    preds_[k].assign(p.begin(), p.end());
  }
  // critical path estimate: algorithmic bytes at 6 TB/s + 2 us per launch
  std::vector<double> cost(nk), top(nk, 0.0), bot(nk, 0.0);
  for (int k = 0; k < nk; ++k) cost[k] = static_cast<double>(kernels_[k].spec.algo_bytes) / 6e6 + 2.0;
  for (int k = 0; k < nk; ++k)
    for (int q : preds_[k]) top[k] = std::max(top[k], top[q] + cost[q]);
  for (int k = nk - 1; k >= 0; --k) {
    bot[k] += cost[k];
    for (int q : preds_[k]) bot[q] = std::max(bot[q], bot[k]);
  }
  double span = 0;
  for (int k = 0; k < nk; ++k) span = std::max(span, top[k] + bot[k]);
  critical_.assign(nk, false);
  for (int k = 0; k < nk; ++k) critical_[k] = top[k] + bot[k] >= 0.97 * span;
  // issue order
  issue_.clear();
  {
    std::vector<int> indeg(nk, 0);
    std::vector<std::vector<int>> succ(nk);
    for (int k = 0; k < nk; ++k)
      for (int q : preds_[k]) {
        ++indeg[k];
        succ[q].push_back(k);
      }
    std::vector<int> ready;
    for (int k = 0; k < nk; ++k)
      if (!indeg[k]) ready.push_back(k);
    bool big = true;
    int phase = 0;  // issue_order 3: two largest, then one smallest
    while (!ready.empty()) {
      size_t pick = 0;
      if (opts_.issue_order == 0) {
        pick = std::min_element(ready.begin(), ready.end()) - ready.begin();
      } else {
        auto key = [&](int k) {
          return kernels_[k].fold_of >= 0 && opts_.issue_order != 4 ? INT64_MAX : kernels_[k].spec.algo_bytes;
        };
        bool fold = false;
        for (size_t r = 0; r < ready.size() && !fold && opts_.issue_order != 4; ++r)
          if (kernels_[ready[r]].fold_of >= 0) pick = r, fold = true;
        if (!fold)
          for (size_t r = 1; r < ready.size(); ++r) {
            const bool big_now = opts_.issue_order == 1 || (opts_.issue_order == 3 ? (phase % 3) != 2 : big);
            const bool better = big_now ? key(ready[r]) > key(ready[pick]) : key(ready[r]) < key(ready[pick]);
            if (better || (key(ready[r]) == key(ready[pick]) && ready[r] < ready[pick])) pick = r;
          }
        if (!fold) {
          big = !big;
          ++phase;
        }
      }
      const int k = ready[pick];
      ready.erase(ready.begin() + static_cast<long>(pick));
      issue_.push_back(k);
      for (int q : succ[k])
        if (--indeg[q] == 0) ready.push_back(q);
    }
    if (static_cast<int>(issue_.size()) != nk) throw InternalError("dataflow: dependency cycle");
  }
  const size_t words = (static_cast<size_t>(nk) + 63) / 64;
  anc_.assign(nk, std::vector<uint64_t>(words, 0));
  for (int k = 0; k < nk; ++k)
    for (int q : preds_[k]) {
      for (size_t w = 0; w < words; ++w) anc_[k][w] |= anc_[q][w];
      anc_[k][q / 64] |= 1ull << (q % 64);
    }
}

bool Executor::ordered_before(int a, int b) const {
  // every kernel touching value a finishes before value b's producer starts
  const int w = writer_[b];
  if (w < 0) return false;
  for (int t : touch_[a])
    if (!(anc_[w][t / 64] >> (t % 64) & 1)) return false;
  return true;
}

void Executor::init_device() {
  CudaApi& cu = CudaApi::get();
  cu_check(cu.cuInit(0), "cuInit");
  CUdevice dev;
  cu_check(cu.cuDeviceGet(&dev, opts_.device), "cuDeviceGet");
  // Always the primary context of opts_.device (the one torch / the CUDA
  // runtime use for that device), made current around every call, whatever
  // context the calling thread has current.
  CUcontext ctx = nullptr;
  cu_check(cu.cuDevicePrimaryCtxRetain(&ctx, dev), "cuDevicePrimaryCtxRetain");
  ctx_ = ctx;
  CtxScope scope(ctx_);
  cu_check(cu.cuDeviceGetAttribute(&sms_, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev), "sm count");
  int major = 0, minor = 0;
  cu.cuDeviceGetAttribute(&major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, dev);
  cu.cuDeviceGetAttribute(&minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, dev);
  if (major != 10 || minor != 0)
    throw std::runtime_error("stitched executor kernels are built for sm_100a; device is sm_" + std::to_string(major) +
                             std::to_string(minor));
  CUdeviceptr p = 0;
  cu_check(cu.cuMemAlloc(&p, std::max<int64_t>(arena_bytes_, 256)), "arena alloc");
  arena_ = p;
  cu_check(cu.cuMemAlloc(&p, std::max<int64_t>(ws_floats_ * 4, 256)), "workspace alloc");
  ws_ = p;
  cu_check(cu.cuMemAlloc(&p, std::max<int64_t>(sync_words_ * 4, 256)), "sync alloc");
  sync_ = p;
  cu_check(cu.cuMemsetD8Async(sync_, 0, std::max<int64_t>(sync_words_ * 4, 256), nullptr), "sync memset");
  cu_check(cu.cuStreamSynchronize(nullptr), "sync");
  for (size_t i = 0; i < kernels_.size(); ++i) {
    KernelInst& k = kernels_[i];
    CUmodule mod;
    cu_check(cu.cuModuleLoadData(&mod, cubins_tmp_[i].data()), "cuModuleLoadData");
    CUfunction fn;
    cu_check(cu.cuModuleGetFunction(&fn, mod, k.spec.name.c_str()), "cuModuleGetFunction");
    k.module = mod;
    k.fn = fn;
    if (k.spec.smem_bytes > 48 * 1024)
      cu_check(cu.cuFuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, k.spec.smem_bytes),
               "smem attribute");
    k.block = k.spec.block;
    k.smem = k.spec.smem_bytes;
    int occ = 0;
    cu_check(cu.cuOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, k.block, k.smem), "occupancy");
    if (k.spec.flex_block) {
      // Register-limited warp-row kernels: the warp count per CTA that keeps
      // the most warps resident (finer CTAs fill the register file better).
      int best_warps = occ * k.block / 32;
      for (int b = k.spec.block - 32; b >= 64; b -= 32) {
        const int smem = k.spec.smem_per_warp * (b / 32);
        int o = 0;
        cu_check(cu.cuOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, b, smem), "occupancy");
        if (o * b / 32 > best_warps) {
          best_warps = o * b / 32;
          k.block = b;
          k.smem = smem;
          occ = o;
        }
      }
    }
    if (occ < 1) throw std::runtime_error("kernel " + k.spec.name + " cannot be resident (block/smem too large)");
    const int64_t resident = static_cast<int64_t>(occ) * sms_;
    int64_t useful = std::max(1, k.spec.max_grid);
    if (k.spec.flex_block && k.spec.rows > 0) {
      const int64_t rpc = k.block / k.spec.row_threads;
      useful = (k.spec.rows + rpc - 1) / rpc;
    }
    if (k.spec.flex_block && k.spec.rows == 0) useful = static_cast<int64_t>(k.spec.max_grid) * k.spec.block / k.block;
    useful = std::max<int64_t>(useful, k.spec.min_grid);
    int64_t cap = resident;
    if (dag_ && opts_.grid_fraction < 1.0 && !k.spec.cooperative)
      cap = std::max<int64_t>(sms_, static_cast<int64_t>(static_cast<double>(resident) * opts_.grid_fraction));
    k.grid = static_cast<int>(std::min<int64_t>(useful, cap));
    if (k.grid < k.spec.min_grid)
      throw std::runtime_error("kernel " + k.spec.name + ": packed components need " + std::to_string(k.spec.min_grid) +
                               " resident CTAs");
    if (k.spec.cooperative) k.grid = static_cast<int>(std::min<int64_t>(k.grid, static_cast<int64_t>(sms_) * 32));
    if (k.spec.max_partials > 0 && k.spec.cluster == 0 && !k.spec.chunkable)
      k.grid = std::min(k.grid, k.spec.max_partials);  // one workspace partial row per CTA
    if (k.spec.cluster > 0) {
      // cluster kernels map CTAs to work statically: exactly max_grid CTAs
      // (a multiple of the cluster size), clusters scheduled in waves
      k.grid = k.spec.max_grid;
      if (k.grid % k.spec.cluster != 0) throw InternalError("cluster kernel grid is not a multiple of its cluster");
      if (k.spec.cluster > 8)
        cu_check(cu.cuFuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_NON_PORTABLE_CLUSTER_SIZE_ALLOWED, 1), "cluster attribute");
    }
  }
  cubins_tmp_.clear();
  int lanes = 0, nev = 0;
  for (const Segment& sg : segments_)
    if (sg.chunks > 1 && sg.last > sg.first) {
      lanes = std::max(lanes, sg.last - sg.first + 1);
      nev += 1 + (sg.last - sg.first + 1) * sg.chunks;
    }
  for (int j = 0; j < lanes; ++j) {
    CUstream st;
    cu_check(cu.cuStreamCreate(&st, CU_STREAM_NON_BLOCKING), "lane stream");
    lanes_.push_back(st);
  }
  for (int e = 0; e < nev; ++e) {
    CUevent x;
    cu_check(cu.cuEventCreate(&x, CU_EVENT_DISABLE_TIMING), "lane event");
    lane_events_.push_back(x);
  }
  if (dag_) {
    int least = 0, greatest = 0;
    cu_check(cu.cuCtxGetStreamPriorityRange(&least, &greatest), "stream priority range");
    high_priority_ = greatest;
    for (int j = 1; j < opts_.concurrent_lanes; ++j) {
      CUstream st;
      cu_check(cu.cuStreamCreate(&st, CU_STREAM_NON_BLOCKING), "dag lane stream");
      dag_lanes_.push_back(st);
    }
    for (size_t e = 0; e <= kernels_.size(); ++e) {
      CUevent x;
      cu_check(cu.cuEventCreate(&x, CU_EVENT_DISABLE_TIMING), "dag event");
      dag_events_.push_back(x);
    }
  }
  device_ready_ = true;
}

void Executor::launch_one(int i, int c, int chunks, const void* const* inputs, void* const* outputs, void* stream) {
  CudaApi& cu = CudaApi::get();
  // Address of buffer b as seen by chunk c: a chunk-local buffer holds
  // `ring` chunk slots and kernels index rows absolutely, so chunk c's slot
  // base is shifted back by c chunks.
  auto addr = [&](int b) -> CUdeviceptr {
    const ValueBuf& x = bufs_[b];
    if (x.kind == ValueBuf::kInput) return reinterpret_cast<CUdeviceptr>(inputs[x.slot]);
    if (x.kind == ValueBuf::kOutput) return reinterpret_cast<CUdeviceptr>(outputs[x.slot]);
    if (x.chunks <= 1) return arena_ + x.offset;
    const CUdeviceptr cb = static_cast<CUdeviceptr>(x.chunk_bytes());
    return arena_ + x.offset + static_cast<CUdeviceptr>(c % x.ring) * cb - static_cast<CUdeviceptr>(c) * cb;
  };
  KernelInst& k = kernels_[i];
  const size_t nargs = k.in_bufs.size() + k.out_bufs.size() + 2;
  std::vector<CUdeviceptr> vals(nargs);
  long long rng[2];
  std::vector<void*> args(nargs + 2);
  int na = 0;
  for (int b : k.in_bufs) vals[na++] = addr(b);
  for (int b : k.out_bufs) vals[na++] = addr(b);
  vals[na++] = ws_ + k.ws_off * 4;
  vals[na++] = sync_ + k.sync_off * 4;
  for (int a = 0; a < na; ++a) args[a] = &vals[a];
  int grid = k.grid;
  rng[0] = rng[1] = 0;
  if (k.spec.chunkable) {
    const int64_t rows = k.spec.rows / chunks;
    rng[0] = static_cast<long long>(rows * c);
    rng[1] = static_cast<long long>(rows * (c + 1));
    if (chunks > 1) {
      const int rpc = k.spec.flex_block ? k.block / k.spec.row_threads : k.spec.rows_per_cta;
      const int64_t need = (rows + rpc - 1) / rpc;
      grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid, need)));
    }
  }
  if (k.fold_of >= 0) rng[0] = kernels_[k.fold_of].grid;  // partial count
  args[na] = &rng[0];
  args[na + 1] = &rng[1];
  // gws scheme: tensor maps of the operand tiles, by value after row_lo/row_hi
  if (!k.spec.tma.empty()) {
    k.tmaps.resize(k.spec.tma.size());
    k.tmap_ptrs.resize(k.spec.tma.size(), 0);
    for (size_t t = 0; t < k.spec.tma.size(); ++t) {
      const KernelSpec::TmaParam& tp = k.spec.tma[t];
      const CUdeviceptr ptr = vals[tp.input];
      if (k.tmap_ptrs[t] != ptr) {
        cuuint64_t dims[3] = {64, 64, static_cast<cuuint64_t>(tp.samples)};
        cuuint64_t strides[2] = {256, 16384};
        cuuint32_t box[3] = {32, static_cast<cuuint32_t>(tp.box_rows), 1};
        cuuint32_t es[3] = {1, 1, 1};
        cu_check(cu.cuTensorMapEncodeTiled(reinterpret_cast<CUtensorMap*>(k.tmaps[t].v), CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                           3, reinterpret_cast<void*>(ptr), dims, strides, box, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           tp.swizzle ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                                           opts_.tma_l2_promotion == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                           : opts_.tma_l2_promotion == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                           : opts_.tma_l2_promotion == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                                         : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
                 "cuTensorMapEncodeTiled");
        k.tmap_ptrs[t] = ptr;
      }
      args.push_back(k.tmaps[t].v);
    }
  }
  CUlaunchConfig cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.gridDimX = grid;
  cfg.gridDimY = cfg.gridDimZ = 1;
  cfg.blockDimX = k.block;
  cfg.blockDimY = cfg.blockDimZ = 1;
  cfg.sharedMemBytes = k.smem;
  cfg.hStream = static_cast<CUstream>(stream);
  CUlaunchAttribute attr[4];
  unsigned na_attr = 0;
  const bool pdl_launch = opts_.pdl && pdl_this_launch_ && (!k.spec.cooperative || opts_.pdl_cooperative);
  if (dag_ && high_priority_ != 0 &&
      ((opts_.critical_priority && critical_[i]) || (opts_.pdl_low_priority && !pdl_launch))) {
    attr[na_attr].id = CU_LAUNCH_ATTRIBUTE_PRIORITY;
    attr[na_attr++].value.priority = high_priority_;
  }
  if (k.spec.cooperative) {
    attr[na_attr].id = CU_LAUNCH_ATTRIBUTE_COOPERATIVE;
    attr[na_attr++].value.cooperative = 1;
  }
  if (pdl_launch) {
    // overlap this launch with the previous kernel's tail (the kernel waits
    // in griddepcontrol.wait before reading anything)
    attr[na_attr].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[na_attr++].value.programmaticStreamSerializationAllowed = 1;
  }
  if (k.spec.cluster > 0) {
    attr[na_attr].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
    attr[na_attr].value.clusterDim.x = static_cast<unsigned>(k.spec.cluster);
    attr[na_attr].value.clusterDim.y = 1;
    attr[na_attr++].value.clusterDim.z = 1;
  }
  if (na_attr) {
    cfg.attrs = attr;
    cfg.numAttrs = na_attr;
  }
  cu_check(cu.cuLaunchKernelEx(&cfg, static_cast<CUfunction>(k.fn), args.data(), nullptr), k.spec.name.c_str());
}

void Executor::launch_dag(const void* const* inputs, void* const* outputs, void* stream) {
  // Kernels in launch (topological) order; each goes on the lane whose last
  // kernel is its latest predecessor, else on a fresh lane, else on the lane
  // idle longest, and waits on the done-events of its other predecessors'
  // lanes (only the latest predecessor per lane).
  CudaApi& cu = CudaApi::get();
  const int nk = static_cast<int>(kernels_.size());
  const int nl = static_cast<int>(dag_lanes_.size()) + 1;
  auto lane_stream = [&](int l) { return static_cast<CUstream>(l == 0 ? stream : dag_lanes_[l - 1]); };
  auto ev = [&](int k) { return static_cast<CUevent>(dag_events_[k]); };
  CUevent fork = static_cast<CUevent>(dag_events_[nk]);
  cu_check(cu.cuEventRecord(fork, lane_stream(0)), "dag fork");
  std::vector<int> tail(nl, -1), lane_of(nk, -1), pos(nk, -1);
  std::vector<bool> used(nl, false);
  used[0] = true;
  for (int it = 0; it < nk; ++it) {
    const int k = issue_[it];
    pos[k] = it;
    // latest-issued predecessor first (pk.back())
    std::vector<int> pk = preds_[k];
    std::sort(pk.begin(), pk.end(), [&](int a, int b) { return pos[a] < pos[b]; });
    auto older = [&](int l, int m) { return (tail[l] < 0 ? -1 : pos[tail[l]]) < (tail[m] < 0 ? -1 : pos[tail[m]]); };
    int lane = -1;
    if (opts_.fold_off_lane && kernels_[k].fold_of >= 0 && nl > 1) {
      const int own = lane_of[kernels_[k].fold_of];
      for (int l = 0; l < nl && lane < 0; ++l)
        if (l != own && !used[l]) lane = l;
      if (lane < 0) {
        lane = own == 0 ? 1 : 0;
        for (int l = 0; l < nl; ++l)
          if (l != own && older(l, lane)) lane = l;
      }
    }
    if (lane < 0 && opts_.big_lane_bytes > 0 && nl > 1) {
      if (kernels_[k].spec.algo_bytes >= opts_.big_lane_bytes) {
        lane = 0;
      } else {
        for (int l = 1; l < nl && lane < 0; ++l)
          if (!pk.empty() && tail[l] == pk.back()) lane = l;
        for (int l = 1; l < nl && lane < 0; ++l)
          if (!used[l]) lane = l;
        if (lane < 0) {
          lane = 1;
          for (int l = 2; l < nl; ++l)
            if (older(l, lane)) lane = l;
        }
      }
    }
    for (int l = 0; l < nl && lane < 0; ++l)
      if (!pk.empty() && tail[l] == pk.back()) lane = l;
    if (lane < 0 && tail[0] < 0) lane = 0;
    for (int l = 1; l < nl && lane < 0; ++l)
      if (!used[l]) lane = l;
    if (lane < 0) {
      lane = 0;
      for (int l = 1; l < nl; ++l)
        if (older(l, lane)) lane = l;
    }
    CUstream st = lane_stream(lane);
    if (!used[lane]) {
      cu_check(cu.cuStreamWaitEvent(st, fork, 0), "dag fork wait");
      used[lane] = true;
    }
    std::vector<int> latest(nl, -1);
    for (int p : pk)
      if (latest[lane_of[p]] < 0 || pos[p] > pos[latest[lane_of[p]]]) latest[lane_of[p]] = p;
    for (int l = 0; l < nl; ++l)
      if (l != lane && latest[l] >= 0) cu_check(cu.cuStreamWaitEvent(st, ev(latest[l]), 0), "dag wait");
    pdl_this_launch_ = !opts_.pdl_true_deps_only || tail[lane] < 0 ||
                       std::find(pk.begin(), pk.end(), tail[lane]) != pk.end();
    launch_one(k, 0, 1, inputs, outputs, st);
    pdl_this_launch_ = true;
    cu_check(cu.cuEventRecord(ev(k), st), "dag done");
    tail[lane] = k;
    lane_of[k] = lane;
  }
  for (int l = 1; l < nl; ++l)
    if (used[l] && tail[l] >= 0) cu_check(cu.cuStreamWaitEvent(lane_stream(0), ev(tail[l]), 0), "dag join");
}

void Executor::launch_all(const void* const* inputs, void* const* outputs, void* stream, std::vector<void*>* events) {
  CudaApi& cu = CudaApi::get();
  CUstream s0 = static_cast<CUstream>(stream);
  if (dag_ && !events) {
    launch_dag(inputs, outputs, stream);
    copy_aliased_outputs(inputs, outputs, stream);
    return;
  }
  int launch = 0;
  size_t ev = 0;  // next lane event
  auto next_event = [&]() { return static_cast<CUevent>(lane_events_.at(ev++)); };
  for (const Segment& sg : segments_) {
    const int m = sg.last - sg.first + 1;
    const bool pipelined = !events && sg.chunks > 1 && m > 1 && opts_.chunk_pipeline;
    if (!pipelined) {
      for (int c = 0; c < sg.chunks; ++c)
        for (int i = sg.first; i <= sg.last; ++i, ++launch) {
          if (events) cu_check(cu.cuEventRecord(static_cast<CUevent>((*events)[2 * launch]), s0), "event");
          launch_one(i, c, sg.chunks, inputs, outputs, stream);
          if (events) cu_check(cu.cuEventRecord(static_cast<CUevent>((*events)[2 * launch + 1]), s0), "event");
        }
      continue;
    }
    // Fork: every lane starts after what s0 has queued so far.
    CUevent fork = next_event();
    cu_check(cu.cuEventRecord(fork, s0), "fork");
    for (int j = 0; j < m; ++j) cu_check(cu.cuStreamWaitEvent(static_cast<CUstream>(lanes_.at(j)), fork, 0), "fork wait");
    std::vector<CUevent> done(static_cast<size_t>(m) * sg.chunks);
    int ring = 1 << 30;
    for (const ValueBuf& b : bufs_)
      if (b.chunks > 1 && b.first >= sg.first && b.last <= sg.last) ring = std::min(ring, b.ring);
    for (int c = 0; c < sg.chunks; ++c)
      for (int j = 0; j < m; ++j, ++launch) {
        CUstream lane = static_cast<CUstream>(lanes_[j]);
        if (j > 0) cu_check(cu.cuStreamWaitEvent(lane, done[(j - 1) * sg.chunks + c], 0), "producer wait");
        // ring slot reuse: chunk c - ring must have left the whole chain
        if (j == 0 && c >= ring) cu_check(cu.cuStreamWaitEvent(lane, done[(m - 1) * sg.chunks + c - ring], 0), "ring wait");
        launch_one(sg.first + j, c, sg.chunks, inputs, outputs, lane);
        CUevent e = next_event();
        cu_check(cu.cuEventRecord(e, lane), "done");
        done[j * sg.chunks + c] = e;
      }
    // Join: s0 continues after every lane's last chunk.
    for (int j = 0; j < m; ++j) cu_check(cu.cuStreamWaitEvent(s0, done[j * sg.chunks + sg.chunks - 1], 0), "join");
  }
  copy_aliased_outputs(inputs, outputs, stream);
}

void Executor::copy_aliased_outputs(const void* const* inputs, void* const* outputs, void* stream) {
  CudaApi& cu = CudaApi::get();
  CUstream s0 = static_cast<CUstream>(stream);
  for (auto [slot, b] : output_copies_) {
    const ValueBuf& x = bufs_[b];
    CUdeviceptr src = x.kind == ValueBuf::kInput ? reinterpret_cast<CUdeviceptr>(inputs[x.slot])
                      : x.kind == ValueBuf::kOutput ? reinterpret_cast<CUdeviceptr>(outputs[x.slot])
                                                    : arena_ + x.offset;
    cu_check(cu.cuMemcpyDtoDAsync(reinterpret_cast<CUdeviceptr>(outputs[slot]), src, output_bytes_[slot], s0),
             "output copy");
  }
}

void Executor::run(const void* const* inputs, void* const* outputs, void* stream) {
  if (!device_ready_) throw std::runtime_error("executor was created compile-only");
  CudaApi& cu = CudaApi::get();
  CtxScope scope(ctx_);
  if (!opts_.use_graph || stream == nullptr) {
    launch_all(inputs, outputs, stream, nullptr);
    return;
  }
  std::vector<const void*> ptrs(inputs, inputs + input_ids_.size());
  ptrs.insert(ptrs.end(), outputs, outputs + output_ids_.size());
  if (!graph_exec_ || graph_stream_ != stream || ptrs != graph_ptrs_) {
    if (graph_exec_) cu.cuGraphExecDestroy(static_cast<CUgraphExec>(graph_exec_));
    graph_exec_ = nullptr;
    cu_check(cu.cuStreamBeginCapture(static_cast<CUstream>(stream), CU_STREAM_CAPTURE_MODE_THREAD_LOCAL), "begin capture");
    try {
      launch_all(inputs, outputs, stream, nullptr);
    } catch (...) {
      CUgraph g = nullptr;
      cu.cuStreamEndCapture(static_cast<CUstream>(stream), &g);
      if (g) cu.cuGraphDestroy(g);
      throw;
    }
    CUgraph graph = nullptr;
    cu_check(cu.cuStreamEndCapture(static_cast<CUstream>(stream), &graph), "end capture");
    CUgraphExec exec = nullptr;
    cu_check(cu.cuGraphInstantiate(&exec, graph, 0), "graph instantiate");
    cu.cuGraphDestroy(graph);
    graph_exec_ = exec;
    graph_stream_ = stream;
    graph_ptrs_ = ptrs;
  }
  cu_check(cu.cuGraphLaunch(static_cast<CUgraphExec>(graph_exec_), static_cast<CUstream>(stream)), "graph launch");
}

void Executor::run_host(const void* const* host_inputs, void* const* host_outputs, void* stream) {
  if (!device_ready_) throw std::runtime_error("executor was created compile-only");
  CudaApi& cu = CudaApi::get();
  CtxScope scope(ctx_);
  const size_t ni = input_ids_.size(), no = output_ids_.size();
  if (host_staging_.empty()) {
    host_staging_.resize(ni + no, 0);
    for (size_t i = 0; i < ni + no; ++i) {
      CUdeviceptr p;
      cu_check(cu.cuMemAlloc(&p, std::max<int64_t>(i < ni ? input_bytes_[i] : output_bytes_[i - ni], 256)), "staging");
      host_staging_[i] = p;
    }
  }
  CUstream s = static_cast<CUstream>(stream);
  std::vector<const void*> din(ni);
  std::vector<void*> dout(no);
  for (size_t i = 0; i < ni; ++i) din[i] = reinterpret_cast<const void*>(host_staging_[i]);
  for (size_t i = 0; i < no; ++i) dout[i] = reinterpret_cast<void*>(host_staging_[ni + i]);
  if (!opts_.overlap_copies || !segments_ok_for_overlap()) {
    for (size_t i = 0; i < ni; ++i) cu_check(cu.cuMemcpyHtoDAsync(host_staging_[i], host_inputs[i], input_bytes_[i], s), "H2D");
    run(din.data(), dout.data(), stream);
    for (size_t i = 0; i < no; ++i)
      cu_check(cu.cuMemcpyDtoHAsync(host_outputs[i], host_staging_[ni + i], output_bytes_[i], s), "D2H");
    cu_check(cu.cuStreamSynchronize(s), "stream sync");
    return;
  }
  // Dataflow copy schedule: inputs go up on a copy stream in order of first
  // use, each kernel waits only for its own inputs, and every output goes
  // down on a second copy stream as soon as its producing kernel is done --
  // host->device and device->host transfers overlap each other (full-duplex
  // link) and the kernels.
  if (!copy_streams_[0]) {
    for (int j = 0; j < 2; ++j) {
      CUstream st;
      cu_check(cu.cuStreamCreate(&st, CU_STREAM_NON_BLOCKING), "copy stream");
      copy_streams_[j] = st;
    }
    in_events_.resize(ni);
    for (void*& e : in_events_) {
      CUevent x;
      cu_check(cu.cuEventCreate(&x, CU_EVENT_DISABLE_TIMING), "event");
      e = x;
    }
    kernel_events_.resize(kernels_.size());
    for (void*& e : kernel_events_) {
      CUevent x;
      cu_check(cu.cuEventCreate(&x, CU_EVENT_DISABLE_TIMING), "event");
      e = x;
    }
    CUevent x;
    cu_check(cu.cuEventCreate(&x, CU_EVENT_DISABLE_TIMING), "event");
    start_event_ = x;
  }
  CUstream up = static_cast<CUstream>(copy_streams_[0]), down = static_cast<CUstream>(copy_streams_[1]);
  cu_check(cu.cuEventRecord(static_cast<CUevent>(start_event_), s), "start");
  cu_check(cu.cuStreamWaitEvent(up, static_cast<CUevent>(start_event_), 0), "up wait");
  cu_check(cu.cuStreamWaitEvent(down, static_cast<CUevent>(start_event_), 0), "down wait");
  // first consumer of every input buffer
  std::vector<int> first_use(ni, static_cast<int>(kernels_.size()));
  for (size_t k = 0; k < kernels_.size(); ++k)
    for (int b : kernels_[k].in_bufs)
      if (bufs_[b].kind == ValueBuf::kInput) first_use[bufs_[b].slot] = std::min<int>(first_use[bufs_[b].slot], static_cast<int>(k));
  std::vector<int> order(ni);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return first_use[a] < first_use[b]; });
  for (int i : order) {
    cu_check(cu.cuMemcpyHtoDAsync(host_staging_[i], host_inputs[i], input_bytes_[i], up), "H2D");
    cu_check(cu.cuEventRecord(static_cast<CUevent>(in_events_[i]), up), "in event");
  }
  // output slot -> producing kernel
  std::vector<int> producer(no, -1);
  for (size_t k = 0; k < kernels_.size(); ++k)
    for (int b : kernels_[k].writes)
      if (bufs_[b].kind == ValueBuf::kOutput) producer[bufs_[b].slot] = static_cast<int>(k);
  std::vector<std::vector<int>> outs_of(kernels_.size());
  for (size_t o = 0; o < no; ++o)
    if (producer[o] >= 0) outs_of[producer[o]].push_back(static_cast<int>(o));
  for (size_t k = 0; k < kernels_.size(); ++k) {
    for (int b : kernels_[k].in_bufs)
      if (bufs_[b].kind == ValueBuf::kInput)
        cu_check(cu.cuStreamWaitEvent(s, static_cast<CUevent>(in_events_[bufs_[b].slot]), 0), "input wait");
    launch_one(static_cast<int>(k), 0, 1, din.data(), dout.data(), stream);
    if (outs_of[k].empty()) continue;
    cu_check(cu.cuEventRecord(static_cast<CUevent>(kernel_events_[k]), s), "kernel event");
    cu_check(cu.cuStreamWaitEvent(down, static_cast<CUevent>(kernel_events_[k]), 0), "output wait");
    for (int o : outs_of[k])
      cu_check(cu.cuMemcpyDtoHAsync(host_outputs[o], host_staging_[ni + o], output_bytes_[o], down), "D2H");
  }
  // outputs that alias inputs / other values: copied after everything
  for (auto [slot, b] : output_copies_) {
    (void)b;
    producer[slot] = -2;
  }
  bool tail = false;
  for (size_t o = 0; o < no; ++o) tail = tail || producer[o] < 0;
  if (tail) {
    // any output not produced by a kernel directly (aliases): device copy on s, then down
    for (auto [slot, b] : output_copies_) {
      const ValueBuf& x = bufs_[b];
      CUdeviceptr src = x.kind == ValueBuf::kInput ? host_staging_[x.slot]
                        : x.kind == ValueBuf::kOutput ? host_staging_[ni + x.slot]
                                                      : arena_ + x.offset;
      if (x.kind == ValueBuf::kInput)
        cu_check(cu.cuStreamWaitEvent(s, static_cast<CUevent>(in_events_[x.slot]), 0), "input wait");
      cu_check(cu.cuMemcpyDtoDAsync(host_staging_[ni + slot], src, output_bytes_[slot], s), "output copy");
    }
    CUevent e = static_cast<CUevent>(start_event_);
    cu_check(cu.cuEventRecord(e, s), "tail event");
    cu_check(cu.cuStreamWaitEvent(down, e, 0), "tail wait");
    for (size_t o = 0; o < no; ++o)
      if (producer[o] < 0) cu_check(cu.cuMemcpyDtoHAsync(host_outputs[o], host_staging_[ni + o], output_bytes_[o], down), "D2H");
  }
  cu_check(cu.cuStreamSynchronize(down), "down sync");
  cu_check(cu.cuStreamSynchronize(s), "stream sync");
  cu_check(cu.cuStreamSynchronize(up), "up sync");
}

bool Executor::segments_ok_for_overlap() const {
  // the per-kernel dataflow schedule launches every kernel whole (chunked
  // schedules keep the plain path)
  for (const Segment& sg : segments_)
    if (sg.chunks > 1) return false;
  return true;
}

json::Value Executor::trace(const void* const* inputs, void* const* outputs, void* stream) {
  if (!opts_.codegen.trace) throw std::runtime_error("trace needs an executor created with trace=true");
  CudaApi& cu = CudaApi::get();
  CtxScope scope(ctx_);
  CUstream s = static_cast<CUstream>(stream);
  const int64_t bytes = std::max<int64_t>(sync_words_ * 4, 256);
  cu_check(cu.cuStreamSynchronize(s), "sync");
  cu_check(cu.cuMemsetD8Async(sync_, 0, bytes, s), "trace reset");
  run(inputs, outputs, stream);
  cu_check(cu.cuStreamSynchronize(s), "sync");
  std::vector<uint32_t> host(static_cast<size_t>(bytes / 4));
  cu_check(cu.cuMemcpyDtoHAsync(host.data(), sync_, bytes, s), "trace read");
  cu_check(cu.cuStreamSynchronize(s), "sync");
  auto u64 = [&](int64_t w) { return static_cast<uint64_t>(host[w]) | static_cast<uint64_t>(host[w + 1]) << 32; };
  uint64_t t0 = ~0ull, t1 = 0;
  std::vector<std::pair<uint64_t, uint64_t>> se(kernels_.size());
  for (size_t i = 0; i < kernels_.size(); ++i) {
    se[i] = {~u64(kernels_[i].sync_off - 4), u64(kernels_[i].sync_off - 2)};
    t0 = std::min(t0, se[i].first);
    t1 = std::max(t1, se[i].second);
  }
  json::Value out = json::Value::object();
  json::Value ks = json::Value::array();
  for (size_t i = 0; i < kernels_.size(); ++i) {
    json::Value k = json::Value::object();
    k.set("name", kernels_[i].spec.name);
    k.set("start_us", static_cast<double>(se[i].first - t0) / 1e3);
    k.set("end_us", static_cast<double>(se[i].second - t0) / 1e3);
    k.set("algo_bytes", kernels_[i].spec.algo_bytes);
    ks.push(k);
  }
  out.set("kernels", ks);
  out.set("span_us", static_cast<double>(t1 - t0) / 1e3);
  return out;
}

json::Value Executor::profile(const void* const* inputs, void* const* outputs, void* stream, int iters) {
  if (!device_ready_) throw std::runtime_error("executor was created compile-only");
  CudaApi& cu = CudaApi::get();
  CtxScope scope(ctx_);
  std::vector<void*> ev(2 * launches_per_run_);
  for (void*& e : ev) {
    CUevent x;
    cu_check(cu.cuEventCreate(&x, CU_EVENT_DEFAULT), "event create");
    e = x;
  }
  std::vector<double> acc(kernels_.size(), 0.0);
  std::vector<int> kernel_of;
  for (const Segment& sg : segments_)
    for (int c = 0; c < sg.chunks; ++c)
      for (int i = sg.first; i <= sg.last; ++i) kernel_of.push_back(i);
  for (int it = 0; it < std::max(1, iters); ++it) {
    launch_all(inputs, outputs, stream, &ev);
    cu_check(cu.cuStreamSynchronize(static_cast<CUstream>(stream)), "sync");
    for (int l = 0; l < launches_per_run_; ++l) {
      float ms = 0.f;
      cu_check(cu.cuEventElapsedTime(&ms, static_cast<CUevent>(ev[2 * l]), static_cast<CUevent>(ev[2 * l + 1])), "elapsed");
      acc[kernel_of[l]] += ms;
    }
  }
  for (void* e : ev) cu.cuEventDestroy(static_cast<CUevent>(e));
  json::Value out = json::Value::object();
  json::Value ks = json::Value::array();
  double total = 0;
  for (size_t i = 0; i < kernels_.size(); ++i) {
    json::Value k = json::Value::object();
    k.set("name", kernels_[i].spec.name);
    k.set("op", kernels_[i].op_id);
    double us = acc[i] * 1000.0 / std::max(1, iters);
    k.set("us", us);
    k.set("algo_bytes", kernels_[i].spec.algo_bytes);
    k.set("gbps", us > 0 ? static_cast<double>(kernels_[i].spec.algo_bytes) / (us * 1e3) : 0.0);
    total += us;
    ks.push(k);
  }
  out.set("kernels", ks);
  out.set("total_us", total);
  out.set("launches", launches_per_run_);
  return out;
}

json::Value Executor::describe() const {
  json::Value j = json::Value::object();
  auto tensors = [](const std::vector<std::string>& ids, const std::vector<std::vector<int64_t>>& dims,
                    const std::vector<int64_t>& bytes) {
    json::Value a = json::Value::array();
    for (size_t i = 0; i < ids.size(); ++i) {
      json::Value t = json::Value::object();
      t.set("id", ids[i]);
      t.set("dims", json::Value::array_of(dims[i]));
      t.set("dtype", "f32");
      t.set("bytes", bytes[i]);
      a.push(t);
    }
    return a;
  };
  j.set("inputs", tensors(input_ids_, input_dims_, input_bytes_));
  j.set("outputs", tensors(output_ids_, output_dims_, output_bytes_));
  json::Value ks = json::Value::array();
  int64_t algo = 0;
  for (const KernelInst& k : kernels_) {
    json::Value e = json::Value::object();
    e.set("name", k.spec.name);
    e.set("op", k.op_id);
    e.set("scheme", k.spec.scheme);
    e.set("variant", k.variant);
    json::Value comp = json::Value::array();
    for (const std::string& c : k.spec.composition) comp.push(c);
    e.set("composition", comp);
    e.set("grid", k.grid);
    e.set("block", k.block ? k.block : k.spec.block);
    e.set("smem_bytes", k.block ? k.smem : k.spec.smem_bytes);
    e.set("cooperative", k.spec.cooperative);
    e.set("algo_bytes", k.spec.algo_bytes);
    e.set("flops", k.spec.flops);
    e.set("chunkable", k.spec.chunkable);
    e.set("rows", k.spec.rows);
    e.set("inputs", json::Value::array_of(k.spec.inputs));
    e.set("outputs", json::Value::array_of(k.spec.outputs));
    e.set("cache_hit", k.cache_hit);
    if (k.fold_of >= 0) e.set("fold_of", kernels_[k.fold_of].spec.name);
    if (dag_) {
      const size_t ki = static_cast<size_t>(&k - kernels_.data());
      json::Value after = json::Value::array();
      for (int q : preds_[ki]) after.push(kernels_[q].spec.name);
      e.set("after", after);
      e.set("issue_pos", static_cast<int64_t>(std::find(issue_.begin(), issue_.end(), static_cast<int>(ki)) - issue_.begin()));
    }
    algo += k.spec.algo_bytes;
    ks.push(e);
  }
  j.set("kernels", ks);
  json::Value sched = json::Value::array();
  for (const Segment& sg : segments_) {
    json::Value e = json::Value::object();
    json::Value names = json::Value::array();
    for (int i = sg.first; i <= sg.last; ++i) names.push(kernels_[i].spec.name);
    e.set("kernels", names);
    e.set("chunks", sg.chunks);
    sched.push(e);
  }
  j.set("schedule", sched);
  j.set("launches", launches_per_run_);
  int64_t edges = 0;
  for (const std::vector<int>& p : preds_) edges += static_cast<int64_t>(p.size());
  j.set("launch_order", dag_ ? "dataflow" : "serial");
  j.set("concurrent_lanes", dag_ ? opts_.concurrent_lanes : 1);
  j.set("dependency_edges", edges);
  int ncrit = 0;
  for (bool c : critical_) ncrit += c;
  j.set("critical_kernels", dag_ ? ncrit : 0);
  j.set("folded_constant_kernels", folded_kernels_);
  j.set("sunk_broadcast_kernels", sunk_kernels_);
  j.set("algo_bytes", algo);
  j.set("arena_bytes", arena_bytes_);
  j.set("workspace_bytes", ws_floats_ * 4);
  return j;
}

}  // namespace exec
}  // namespace stitch
