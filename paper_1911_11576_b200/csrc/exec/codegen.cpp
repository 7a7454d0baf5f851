// Stitched-kernel generator (see codegen.hpp for the scheme overview).
//
// Value semantics follow the reference emitter's per-op C expressions
// (proj/src/emitter.cpp:883-915) and broadcast indexing (graph.cpp:158):
// out[c] = in[c[map[0]], ..., c[map[r-1]]] with map the right-most greedy
// subsequence match. Reductions: sum (reference) or max (extension).
#include "codegen.hpp"

#include "../host/cost.hpp"

#include <algorithm>
#include <cstring>
#include <functional>
#include <numeric>
#include <sstream>

namespace stitch {
namespace exec {

namespace {

std::string flit(double v) {
  float f = static_cast<float>(v);
  uint32_t bits;
  std::memcpy(&bits, &f, 4);
  char buf[64];
  std::snprintf(buf, sizeof buf, "__int_as_float(0x%08x)", bits);
  return buf;
}

int64_t prod(const std::vector<int64_t>& d, size_t from = 0, size_t to = std::string::npos) {
  int64_t p = 1;
  for (size_t i = from; i < std::min(to, d.size()); ++i) p *= d[i];
  return p;
}

std::string join(const std::vector<std::string>& xs, const char* sep) {
  std::string s;
  for (size_t i = 0; i < xs.size(); ++i) s += (i ? sep : "") + xs[i];
  return s;
}

// Row-major linear index of `coords` in `dims`, as a C expression.
std::string linear(const std::vector<std::string>& coords, const std::vector<int64_t>& dims) {
  if (coords.empty()) return "0";
  std::string e = "(long long)(" + coords[0] + ")";
  for (size_t i = 1; i < coords.size(); ++i) e = "(" + e + " * " + std::to_string(dims[i]) + "LL + (" + coords[i] + "))";
  return e;
}

// Coordinates of linear index `lin` (a C expression) in `dims`.
std::vector<std::string> decode(const std::string& lin, const std::vector<int64_t>& dims) {
  std::vector<std::string> c(dims.size());
  int64_t stride = 1;
  for (size_t i = dims.size(); i-- > 0;) {
    std::string e = stride == 1 ? "(" + lin + ")" : "((" + lin + ") / " + std::to_string(stride) + "LL)";
    c[i] = i == 0 ? e : "(" + e + " % " + std::to_string(dims[i]) + "LL)";
    stride *= dims[i];
  }
  return c;
}

enum class Cls { kNone, kRowed, kFree, kCross, kPost };

struct Val {
  std::string id;
  const OpNode* node = nullptr;
  bool external = false;
  bool constant = false;
  double cval = 0.0;
  bool member = false;
  bool output = false;
  std::vector<int64_t> dims;
  std::vector<int> operands;   // value indices
  std::vector<int> consumers;  // member value indices (dups removed)
};

struct Layout {  // per-thread ownership of an inner tile of S elements
  int64_t S = 1;
  int vec = 1, iters = 1;
  bool guard = false;
  int elems() const { return vec * iters; }
};

struct Component {
  std::vector<int> members;  // topo order
  std::vector<int> outputs;
  std::string scheme;        // row | flat | sectioned
  int64_t weight = 1;
  // ROW
  int k = 0;
  std::vector<int64_t> P;
  int64_t R = 0;
  int NT = 32;
  bool cta = false;
  std::vector<Cls> cls;
  std::vector<char> staged;
  std::vector<int64_t> smem_off;  // floats within the row-group slab
  std::map<int, int64_t> cross_off;  // cross_smem: per-warp column accumulators within the slab
  int64_t slab_floats = 0;
  bool tma = false;
  bool dbuf = false;          // external TMA tiles double-buffered (prefetch the next row)
  bool prefetch = false;      // register-loaded row inputs prefetched one row ahead
  std::vector<char> cheap;    // rowed broadcasts of constants / free tensors: recomputed at each use, never stored
  std::vector<char> lazy;     // rowed inputs loaded per fused-loop step (float4) instead of preloaded per row
  // COLRED: a lone column reduction of an external [R][C] tensor
  int64_t cr_R = 0, cr_C = 0, cr_ncb = 0, cr_nch = 0, cr_rpc = 0;
  int cr_sync = 0, cr_m = -1, cr_w = 128;
  int cr_cluster = 0;         // COLRED: row chunks of a column block form a cluster of this many CTAs
  std::vector<int> cr_eouts;  // COLRED: elementwise outputs written from the same tiles
  bool tc = false;            // gemm stages on tcgen05 (3xTF32): smem scratch + TMEM accumulator
  int tc_k = 0;               // largest K among the tensor-core gemm stages
  std::vector<char> tc_dot;   // value -> gemm stage runs on tcgen05
  std::vector<int> tc_direct;  // tcgen05 stages with unstaged external operands
  bool tcp = false;            // pipelined tcgen05 schedule (next row's MMAs overlap this row's epilogue)
  std::vector<int> tc_list;    // tcgen05 gemm members in order
  std::vector<char> tc_raw;    // TMA-staged operand tiles only the tcgen05 split reads
  int64_t ext_floats = 0;     // floats of one copy of the external staged tiles
  std::vector<int> cross, post, free_out;
  int64_t max_grid = 1;
};

class Builder {
 public:
  Builder(const Graph& body, const std::string& name, const std::map<std::string, double>& constants,
          const CodegenOptions& opts)
      : body_(body), name_(name), consts_(constants), opts_(opts) {}

  KernelSpec build();

 private:
  bool build_gws();  // the warp-specialised tcgen05 scheme, when the group fits it
  bool build_gemm();  // one unfused dot: the tiled fp32 GEMM scheme
  bool nr_div_ = false;  // elementwise divides as branch-free rcp + Newton (gws tails)
  // ---- analysis ----
  void collect();
  std::vector<Component> components();
  bool plan_row(Component& c);
  bool plan_colred(Component& c);
  void emit_colred(Component& c, const std::string& lo, const std::string& n);
  int colred_sync_ = 2;  // next free sync word (0..1: grid barrier)
  bool all_elementwise(const Component& c) const;
  Layout layout(int64_t S, int NT) const;
  bool identity_broadcast(int in, int out, int k) const;

  // ---- emission helpers ----
  void ln(const std::string& s) { out_ << std::string(indent_ * 2, ' ') << s << "\n"; }
  void open(const std::string& s) { ln(s + " {"); ++indent_; }
  void close(const std::string& tail = "") { --indent_; ln("}" + tail); }
  std::string fresh(const char* stem) { return std::string(stem) + std::to_string(tmp_++); }
  std::string in_ptr(int v) const { return "in" + std::to_string(v); }
  std::string out_ptr(int v) const { return "out" + std::to_string(v); }
  std::string elem_expr(const OpNode& op, const std::vector<std::string>& a) const;
  std::vector<std::string> map_broadcast(int in, int out, const std::vector<std::string>& coords) const;

  // Inline expression machinery (FLAT / SECTIONED / FREE values).
  std::string at(int v, const std::vector<std::string>& coords);
  std::vector<std::map<std::string, std::string>> memo_;
  std::map<int, std::string> materialized_;  // value -> buffer pointer expression (SECTIONED / post)
  std::function<std::string(int, const std::vector<std::string>&)> row_hook_;

  void emit_flat(const Component& c, const std::string& lo, const std::string& n);
  void emit_row(Component& c, const std::string& lo, const std::string& n, const std::string& cta_rank);
  void emit_row_finalize(std::vector<Component*>& comps, bool split);
  void emit_sectioned(const std::vector<int>& members);
  // BLOCK: heterogeneous groups over a common leading index G (paper Fig. 1:
  // dots + reductions + elementwise over different inner index spaces), one
  // CTA per leading index, sections separated by __syncthreads, staged values
  // in shared memory at the planner's Alg. 4 alloc map. Returns the shared
  // bytes, or -1 when the group does not fit the scheme.
  int64_t plan_block(int64_t* G);
  void emit_block(const std::vector<int>& members, int64_t G);
  std::string emit_heavy(int m, const std::vector<std::string>& oc);  // reduce / dot value at coords (loops)
  bool inline_heavy_ = false;  // at() may recompute reductions and dots inline (BLOCK)
  std::map<int, std::pair<int64_t, int64_t>> block_smem_;  // value -> (byte offset, bytes) per leading index
  std::map<int, int> block_reuse_;  // value -> value whose shared block it reuses (planner's reused_from)
  std::string block_alloc_note_;

  bool reg_input(const Component& c, int v) const;
  bool tc_direct(const Component& c, int m) const;
  bool free_vector_access(const Component& c, int o, int v) const;
  void emit_row_scalar(const Component& c, int m);
  void emit_row_load(int v, const std::string& dst, const std::string& row, const Layout& L, int NT);

  // ROW emission state
  std::string row_access(const Component& c, int o, int v, const std::string& it, const std::string& u,
                         const Layout& L);
  std::map<int, std::string> reg_;  // value -> register array name (per row body)
  std::map<int, std::string> loop_scalar_;  // value -> scalar of the current fused elementwise loop
  std::map<int, std::string> freevec_;      // free external -> float[4] of the current `it` (fused loop)
  std::map<int, std::string> rowvec_;       // lazy rowed input -> float[4] of the current `it` (fused loop)
  std::map<int, std::string> scalar_;

  const Graph& body_;
  std::string name_;
  const std::map<std::string, double>& consts_;
  CodegenOptions opts_;

  std::vector<Val> vals_;
  std::map<std::string, int> idx_;
  std::vector<int> topo_members_;
  std::vector<int> outputs_;
  std::vector<int> inputs_;  // pointer inputs

  std::ostringstream out_;
  int indent_ = 0;
  int tmp_ = 0;
  KernelSpec spec_;
  int64_t ws_floats_ = 0;
  bool uses_barrier_ = false;
  std::map<int, int64_t> ws_off_;  // value -> workspace offset (floats)
  std::map<int, std::string> cross_parts_;  // cross value -> nparts expression
  std::string fin_body_;  // split_cross: body of the column-reduction fold kernel
  size_t n_comps_ = 1;    // components of the kernel being emitted
  bool chunked_ = false;  // the single ROW component runs rows [row_lo, row_hi) (launch-time chunking)
};

// ---------------------------------------------------------------------------
// analysis
// ---------------------------------------------------------------------------

void Builder::collect() {
  const std::vector<std::string> topo = topological_sort(body_);
  vals_.resize(body_.nodes.size());
  for (size_t i = 0; i < body_.nodes.size(); ++i) {
    const OpNode& n = body_.nodes[i];
    Val& v = vals_[i];
    v.id = n.id;
    v.node = &n;
    v.dims = n.shape.dims;
    idx_[n.id] = static_cast<int>(i);
    if (n.type == OpType::kParameter || n.type == OpType::kConstant) {
      auto c = consts_.find(n.id);
      if (c != consts_.end()) {
        v.constant = true;
        v.cval = c->second;
      } else if (n.type == OpType::kConstant && n.value) {
        v.constant = true;
        v.cval = *n.value;
      } else {
        v.external = true;
      }
    } else if (is_fusible(n)) {
      v.member = true;
      if (n.shape.dtype != DType::f32())
        throw GraphError("stitched executor: only f32 tensors are supported (" + n.id + ")");
    }
  }
  for (size_t i = 0; i < body_.nodes.size(); ++i)
    for (const std::string& o : body_.nodes[i].operands) vals_[i].operands.push_back(idx_.at(o));
  for (const std::string& id : topo) {
    int i = idx_.at(id);
    if (!vals_[i].member) continue;
    topo_members_.push_back(i);
    for (int o : vals_[i].operands)
      if (std::find(vals_[o].consumers.begin(), vals_[o].consumers.end(), i) == vals_[o].consumers.end())
        vals_[o].consumers.push_back(i);
  }
  for (const OpNode& n : body_.nodes)
    if (n.type == OpType::kTuple)
      for (const std::string& o : n.operands) {
        int i = idx_.at(o);
        if (!vals_[i].member) throw GraphError("stitched executor: fused output " + o + " is not computed in the group");
        if (!vals_[i].output) outputs_.push_back(i);
        vals_[i].output = true;
      }
  if (outputs_.empty()) throw GraphError("stitched executor: fused body has no outputs");
  for (int i = 0; i < static_cast<int>(vals_.size()); ++i)
    if (vals_[i].external) {
      bool used = !vals_[i].consumers.empty();
      if (used) inputs_.push_back(i);
      if (vals_[i].node->shape.dtype != DType::f32())
        throw GraphError("stitched executor: only f32 tensors are supported (" + vals_[i].id + ")");
    }
}

std::vector<Component> Builder::components() {
  std::vector<int> parent(vals_.size());
  std::iota(parent.begin(), parent.end(), 0);
  std::function<int(int)> find = [&](int x) { return parent[x] == x ? x : parent[x] = find(parent[x]); };
  for (int m : topo_members_)
    for (int o : vals_[m].operands)
      if (vals_[o].member) parent[find(m)] = find(o);
  std::map<int, int> comp_of_root;
  std::vector<Component> comps;
  for (int m : topo_members_) {
    int r = find(m);
    auto it = comp_of_root.find(r);
    if (it == comp_of_root.end()) {
      it = comp_of_root.emplace(r, static_cast<int>(comps.size())).first;
      comps.emplace_back();
    }
    comps[it->second].members.push_back(m);
    if (vals_[m].output) comps[it->second].outputs.push_back(m);
  }
  for (Component& c : comps) {
    int64_t w = 0;
    std::set<int> ins;
    for (int m : c.members)
      for (int o : vals_[m].operands)
        if (vals_[o].external) ins.insert(o);
    for (int i : ins) w += vals_[i].node->shape.byte_count();
    for (int o : c.outputs) w += vals_[o].node->shape.byte_count();
    c.weight = std::max<int64_t>(w, 1);
  }
  return comps;
}

bool Builder::all_elementwise(const Component& c) const {
  for (int m : c.members)
    if (vals_[m].node->type != OpType::kElementwise) return false;
  return true;
}

Layout Builder::layout(int64_t S, int NT) const {
  Layout L;
  L.S = S;
  L.vec = S % 4 == 0 ? 4 : S % 2 == 0 ? 2 : 1;
  if (S < NT * L.vec && S % NT == 0) L.vec = static_cast<int>(S / NT);  // spread small tiles over the group
  if (L.vec < 1) L.vec = 1;
  const int64_t per = static_cast<int64_t>(NT) * L.vec;
  L.iters = static_cast<int>((S + per - 1) / per);
  L.guard = S % per != 0;
  return L;
}

std::vector<std::string> Builder::map_broadcast(int in, int out, const std::vector<std::string>& coords) const {
  const Shape& is = vals_[in].node->shape;
  const Shape& os = vals_[out].node->shape;
  std::vector<int> m = broadcast_dim_map(is, os);
  std::vector<std::string> c;
  for (int d : m) c.push_back(coords[d]);
  return c;
}

bool Builder::identity_broadcast(int in, int out, int k) const {
  // Broadcast whose input, seen from the row tile, is indexed exactly like
  // the output tile (same inner dims, inner map is the identity).
  const auto& id = vals_[in].dims;
  const auto& od = vals_[out].dims;
  std::vector<int> m = broadcast_dim_map(vals_[in].node->shape, vals_[out].node->shape);
  if (id.size() < static_cast<size_t>(k)) return false;
  if (std::vector<int64_t>(id.begin() + k, id.end()) != std::vector<int64_t>(od.begin() + k, od.end())) return false;
  for (size_t i = 0; i < m.size(); ++i)
    if (m[i] != static_cast<int>(i)) return false;
  return true;
}

// COLRED scheme: out[C] = sum/max over R rows of f(in...)[R][C], where f is
// the component's elementwise producer chain evaluated inline (LayerNorm
// dgamma = sum(dy * xhat), a bias gradient = sum(dy)); reduce_dims a leading
// prefix, the reduce the component's only output. 2-D tiles (128-column
// block x row chunk) over one wave of CTAs, float4 streaming loads of the
// same-shape inputs coalesced along the row, a fixed warp-order CTA sum,
// per-chunk partials in the workspace, and the last CTA of a column block
// (atomic arrival counter) combining the chunks in chunk order:
// deterministic, no grid barrier, no cooperative launch.
// COLRED shared layout (floats): warp partials + flag, then the cp.async
// stage of kColredStageSlots float4 per thread (256 threads)
constexpr int kColredStageOff = 8 * 128 + 16;
constexpr int kColredStageSlots = 8;

bool Builder::plan_colred(Component& c) {
  if (!opts_.colred) return false;
  int m = -1;
  for (int x : c.members) {
    const OpNode& xo = *vals_[x].node;
    if (xo.type == OpType::kReduce) {
      if (m >= 0) return false;
      m = x;
    } else if (xo.type != OpType::kElementwise) {
      return false;
    }
  }
  if (m < 0 || !vals_[m].output) return false;
  // elementwise outputs over the reduce input's index space (e.g. the GeLU
  // backward dx beside its bias gradient) are written from the same tiles
  c.cr_eouts.clear();
  for (int x : c.members)
    if (x != m && vals_[x].output) {
      if (!opts_.colred_eout || vals_[x].dims != vals_[vals_[m].operands[0]].dims) return false;
      c.cr_eouts.push_back(x);
    }
  if (c.members.size() > 1 && !opts_.colred_fused) return false;
  const OpNode& op = *vals_[m].node;
  const int in = vals_[m].operands[0];
  if (!vals_[in].external && !vals_[in].member) return false;
  const auto& d = vals_[in].dims;
  const int j = static_cast<int>(op.reduce_dims.size());
  if (j < 1 || j >= static_cast<int>(d.size())) return false;
  for (int i = 0; i < j; ++i)
    if (op.reduce_dims[i] != i) return false;
  c.cr_m = m;
  c.cr_R = prod(d, 0, j);
  c.cr_C = prod(d, j);
  if (c.cr_C % 4 != 0 || c.cr_R < 1) return false;
  // W-column blocks (colred_cols: 32, 64 or 128): a warp load covers
  // 128 / W * 4 rows x W floats; the last CTA of a block folds W columns
  const int W = opts_.colred_cols == 32 || opts_.colred_cols == 64 ? opts_.colred_cols : 128;  // default 32
  c.cr_w = W;
  c.cr_ncb = (c.cr_C + W - 1) / W;
  // one wave of colred_ctas_per_sm CTAs of 8 warps per SM
  int64_t nch = std::max<int64_t>(1, (static_cast<int64_t>(opts_.num_sms) * opts_.colred_ctas_per_sm) / c.cr_ncb);
  // at least one full pass of the CTA's row groups per chunk
  const int64_t pass = 8 * (128 / W);
  nch = std::min<int64_t>(nch, std::max<int64_t>(1, c.cr_R / pass));
  // cluster combine: exactly colred_cluster chunks per column block (one
  // cluster each), when every chunk keeps at least one full pass
  const int K = opts_.colred_cluster;
  c.cr_cluster = 0;
  if ((K == 2 || K == 4 || K == 8 || K == 16) && c.cr_R >= static_cast<int64_t>(K) * pass) {
    c.cr_cluster = K;
    nch = K;
  }
  // chunks of whole passes: every pass but the matrix's last is unpredicated
  c.cr_rpc = ((c.cr_R + nch - 1) / nch + pass - 1) / pass * pass;
  c.cr_nch = (c.cr_R + c.cr_rpc - 1) / c.cr_rpc;
  // a cluster always has K chunks (trailing ones may be empty: their
  // partial is the reduction's identity)
  if (c.cr_cluster) c.cr_nch = c.cr_cluster;
  c.cr_sync = colred_sync_;
  colred_sync_ += static_cast<int>(c.cr_ncb);
  c.scheme = "colred";
  c.max_grid = c.cr_ncb * c.cr_nch;
  return true;
}

void Builder::emit_colred(Component& c, const std::string& lo, const std::string& n) {
  const int m = c.cr_m;
  const OpNode& op = *vals_[m].node;
  const int in = vals_[m].operands[0];
  const std::string Op = op.elem_name == "max" ? "stitch_dev::MaxOp" : "stitch_dev::SumOp";
  const std::string C = std::to_string(c.cr_C) + "LL", NCB = std::to_string(c.cr_ncb), NCH = std::to_string(c.cr_nch);
  const int W = c.cr_w, LPR = W / 4, G = 32 / LPR;  // lanes per row, rows per warp load
  const std::string Ws = std::to_string(W);
  const std::string parts = "(ws + " + std::to_string(ws_off_[m]) + "LL)";
  int64_t iters = std::min<int64_t>(8, c.cr_rpc / (8 * G));  // loads per thread per pass (8-warp CTA)
  const std::string Gs = std::to_string(G);
  open("");
  ln("// colred: " + vals_[m].id + "[" + std::to_string(c.cr_C) + "] over " + std::to_string(c.cr_R) + " rows; " + NCB +
     " column blocks of " + Ws + " x " + NCH + " row chunks of " + std::to_string(c.cr_rpc));
  ln("const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;");
  ln("const int sub = lane / " + std::to_string(LPR) + ", cl = lane % " + std::to_string(LPR) + ";");
  ln("int* last = reinterpret_cast<int*>(smem + " + std::to_string(kColredStageOff - 8) + ");  // past every partial row");
  open("for (long long tile = (long long)blockIdx.x - " + lo + "; tile < " + NCB + "LL * " + NCH + "LL; tile += " + n + ")");
  if (c.cr_cluster)  // the K row chunks of a column block are one cluster (consecutive CTAs)
    ln("const int cb = (int)(tile / " + std::to_string(c.cr_cluster) + "), ch = (int)(tile % " + std::to_string(c.cr_cluster) + ");");
  else
    ln("const int cb = (int)(tile % " + NCB + "), ch = (int)(tile / " + NCB + ");");
  ln("const long long col = (long long)cb * " + Ws + " + cl * 4;");
  ln("const long long r0 = (long long)ch * " + std::to_string(c.cr_rpc) + "LL;");
  ln("const long long r1 = r0 + " + std::to_string(c.cr_rpc) + "LL < " + std::to_string(c.cr_R) + "LL ? r0 + " +
     std::to_string(c.cr_rpc) + "LL : " + std::to_string(c.cr_R) + "LL;");
  ln("float a0 = " + Op + "::init(), a1 = a0, a2 = a0, a3 = a0;");
  // f(...) at (r, col + u): same-shape external inputs as one float4 each,
  // then the producer chain inline (broadcast vectors through L1)
  const auto& d = vals_[in].dims;
  const int j = static_cast<int>(op.reduce_dims.size());
  std::vector<int64_t> rd(d.begin(), d.begin() + j), cd(d.begin() + j, d.end());
  std::set<int> ins, seen;
  std::function<void(int)> walk = [&](int v) {
    if (!seen.insert(v).second) return;
    if (vals_[v].external && vals_[v].dims == d) ins.insert(v);
    if (vals_[v].member && vals_[v].node->type == OpType::kElementwise && vals_[v].node->elem_name != "broadcast")
      for (int o : vals_[v].operands) walk(o);
  };
  walk(in);
  for (int eo : c.cr_eouts) walk(eo);
  if (opts_.colred_cp_async)
    iters = std::max<int64_t>(1, std::min<int64_t>(iters, kColredStageSlots / std::max<int64_t>(1, static_cast<int64_t>(ins.size()))));
  const std::string IT = std::to_string(iters);
  // staging: with colred_cp_async every load of a pass goes through
  // cp.async into this thread's shared slots (ptxas otherwise keeps only
  // ~2 rows of float4 loads in flight per thread)
  const bool cpa = opts_.colred_cp_async;
  const int nin = static_cast<int>(ins.size());
  auto body = [&](bool guarded) {
    std::map<int, std::string> qname;
    int vi = 0;
    std::map<int, int> slot;
    for (int v : ins) {
      slot[v] = vi++;
      qname[v] = fresh("q");
      if (!cpa) ln("float4 " + qname[v] + "[" + IT + "];");
    }
    ln("#pragma unroll");
    open("for (int i = 0; i < " + IT + "; ++i)");
    ln("const long long r = rb + (i * nw + warp) * " + Gs + " + sub;");
    for (int v : ins) {
      const std::string src = in_ptr(v) + " + " + (guarded ? "(r < r1 ? r : r0)" : "r") + " * " + C + " + col";
      if (cpa)
        ln("stitch_dev::cp_async16(cstage + (i * " + std::to_string(nin) + " + " + std::to_string(slot[v]) + ") * blockDim.x, " + src +
           ", " + (guarded ? "r < r1" : "true") + ");");
      else
        ln(qname[v] + "[i] = " + (guarded ? "r < r1 ? " : "") + "stitch_dev::ld4_stream(" + src + ")" +
           (guarded ? " : make_float4(0.f, 0.f, 0.f, 0.f)" : "") + ";");
    }
    close();
    if (cpa) ln("stitch_dev::cp_async_wait_all();");
    ln("#pragma unroll");
    open("for (int i = 0; i < " + IT + "; ++i)");
    ln("const long long r = rb + (i * nw + warp) * " + Gs + " + sub;");
    if (guarded) open("if (r < r1)");
    for (int v : ins)
      if (cpa) ln("const float4 " + qname[v] + " = cstage[(i * " + std::to_string(nin) + " + " + std::to_string(slot[v]) + ") * blockDim.x];");
    memo_.emplace_back();
    std::vector<std::string> rc = decode("r", rd);
    auto coords = [&](int u) {
      std::vector<std::string> cc = rc;
      std::vector<std::string> k2 = decode(u ? "(col + " + std::to_string(u) + ")" : std::string("col"), cd);
      cc.insert(cc.end(), k2.begin(), k2.end());
      return cc;
    };
    const char* lanes[4] = {".x", ".y", ".z", ".w"};
    for (int v : ins)
      for (int u = 0; u < 4; ++u)
        memo_.back()[std::to_string(v) + "@" + join(coords(u), ",")] = qname[v] + (cpa ? "" : "[i]") + lanes[u];
    std::vector<std::string> xv;
    for (int u = 0; u < 4; ++u) xv.push_back(at(in, coords(u)));
    for (int eo : c.cr_eouts) {
      std::vector<std::string> ev;
      for (int u = 0; u < 4; ++u) ev.push_back(at(eo, coords(u)));
      ln("stitch_dev::st4(" + out_ptr(eo) + " + r * " + C + " + col, " + ev[0] + ", " + ev[1] + ", " + ev[2] + ", " + ev[3] + ");");
    }
    memo_.pop_back();
    ln("a0 = " + Op + "::apply(a0, " + xv[0] + "); a1 = " + Op + "::apply(a1, " + xv[1] + "); a2 = " + Op + "::apply(a2, " +
       xv[2] + "); a3 = " + Op + "::apply(a3, " + xv[3] + ");");
    if (guarded) close();
    close();
  };
  if (cpa) ln("float4* cstage = reinterpret_cast<float4*>(smem + " + std::to_string(kColredStageOff) + ") + threadIdx.x;");
  open("if (col < " + C + ")");
  open("for (long long rb = r0; rb < r1; rb += " + IT + " * nw * " + Gs + ")");
  // full passes without predicates (predicate registers would otherwise
  // serialise the loads), the ragged last pass guarded
  open("if (rb + " + IT + " * nw * " + Gs + " <= r1)");
  body(false);
  close();
  open("else");
  body(true);
  close();
  close();
  close();
  // the warp's row groups, then the CTA's warps in warp order
  for (int x = LPR; x < 32; x *= 2)
    for (int u = 0; u < 4; ++u) {
      const std::string a = "a" + std::to_string(u);
      ln(a + " = " + Op + "::apply(" + a + ", __shfl_xor_sync(0xffffffffu, " + a + ", " + std::to_string(x) + "));");
    }
  ln("if (sub == 0) { smem[warp * " + Ws + " + cl * 4 + 0] = a0; smem[warp * " + Ws + " + cl * 4 + 1] = a1; smem[warp * " + Ws +
     " + cl * 4 + 2] = a2; smem[warp * " + Ws + " + cl * 4 + 3] = a3; }");
  ln("__syncthreads();");
  open("for (int i = threadIdx.x; i < " + Ws + "; i += blockDim.x)");
  open("if ((long long)cb * " + Ws + " + i < " + C + ")");
  ln("float a = " + Op + "::init();");
  ln("for (int w = 0; w < nw; ++w) a = " + Op + "::apply(a, smem[w * " + Ws + " + i]);");
  if (c.cr_cluster) {
    // this chunk's partial row stays in shared memory (the staging area,
    // free now); rank 0 folds the cluster's K partials in rank order
    // through DSMEM after a cluster barrier
    const std::string K = std::to_string(c.cr_cluster);
    ln("smem[" + std::to_string(kColredStageOff) + " + i] = a;");
    close();
    close();
    ln("stitch_dev::cluster_sync();");
    open("if (ch == 0)");
    open("for (int i = threadIdx.x; i < " + Ws + "; i += blockDim.x)");
    open("if ((long long)cb * " + Ws + " + i < " + C + ")");
    ln("float v = " + Op + "::init();");
    ln("#pragma unroll");
    ln("for (unsigned r = 0; r < " + K + "u; ++r) v = " + Op + "::apply(v, stitch_dev::dsmem_ld(smem + " +
       std::to_string(kColredStageOff) + " + i, r));");
    ln(out_ptr(m) + "[(long long)cb * " + Ws + " + i] = v;");
    close();
    close();
    close();
    ln("stitch_dev::cluster_sync();  // every remote read of this CTA's partial is done");
    close();
    close();
    return;
  }
  ln(parts + "[(long long)ch * " + C + " + (long long)cb * " + Ws + " + i] = a;");
  close();
  close();
  ln("__threadfence();");
  ln("__syncthreads();");
  ln("if (threadIdx.x == 0) *last = atomicAdd(gsync + " + std::to_string(c.cr_sync) + " + cb, 1u) == " + NCH + "u - 1u;");
  ln("__syncthreads();");
  open("if (*last)");
  ln("__threadfence();");
  if (cpa) {
    // float4 column groups x strided chunk slices; each round puts
    // kColredStageSlots partial rows per thread in flight through cp.async,
    // chunks fold in ascending order per slice, slices join in slice order
    const std::string S = std::to_string(kColredStageSlots), LG = std::to_string(LPR);
    ln("const int slices = blockDim.x / " + LG + ", sl = threadIdx.x / " + LG + ", cg = threadIdx.x % " + LG + ";");
    ln("const long long fcol = (long long)cb * " + Ws + " + cg * 4;");
    ln("float f0 = " + Op + "::init(), f1 = f0, f2 = f0, f3 = f0;");
    open("for (int k0 = sl; k0 < " + NCH + "; k0 += slices * " + S + ")");
    ln("#pragma unroll");
    open("for (int i = 0; i < " + S + "; ++i)");
    ln("const int k = k0 + i * slices;");
    ln("const bool ok = k < " + NCH + " && fcol < " + C + ";");
    ln("stitch_dev::cp_async16(cstage + i * blockDim.x, " + parts + " + (ok ? (long long)k * " + C + " + fcol : 0LL), ok);");
    close();
    ln("stitch_dev::cp_async_wait_all();");
    ln("#pragma unroll");
    open("for (int i = 0; i < " + S + "; ++i)");
    open("if (k0 + i * slices < " + NCH + ")");
    ln("const float4 p = cstage[i * blockDim.x];");
    ln("f0 = " + Op + "::apply(f0, p.x); f1 = " + Op + "::apply(f1, p.y); f2 = " + Op + "::apply(f2, p.z); f3 = " + Op + "::apply(f3, p.w);");
    close();
    close();
    close();
    ln("smem[sl * " + Ws + " + cg * 4 + 0] = f0; smem[sl * " + Ws + " + cg * 4 + 1] = f1; smem[sl * " + Ws + " + cg * 4 + 2] = f2; smem[sl * " +
       Ws + " + cg * 4 + 3] = f3;");
    ln("__syncthreads();");
    open("for (int i = threadIdx.x; i < " + Ws + "; i += blockDim.x)");
    open("if ((long long)cb * " + Ws + " + i < " + C + ")");
    ln("float v = smem[i];");
    ln("for (int j = 1; j < slices; ++j) v = " + Op + "::apply(v, smem[j * " + Ws + " + i]);");
    ln(out_ptr(m) + "[(long long)cb * " + Ws + " + i] = v;");
    close();
    close();
  } else {
    // every slice of W threads folds a strided set of the chunks (4
    // interleaved chains, fixed order), then slice partials join in slice order
    ln("const int slices = blockDim.x / " + Ws + ", sl = threadIdx.x / " + Ws + ", cc = threadIdx.x % " + Ws + ";");
    ln("float a = " + Op + "::init();");
    open("if ((long long)cb * " + Ws + " + cc < " + C + ")");
    ln("float q[4];");
    ln("#pragma unroll");
    ln("for (int u = 0; u < 4; ++u) q[u] = " + Op + "::init();");
    ln("int k = sl;");
    open("for (; k + 3 * slices < " + NCH + "; k += 4 * slices)");
    ln("#pragma unroll");
    ln("for (int u = 0; u < 4; ++u) q[u] = " + Op + "::apply(q[u], __ldcg(" + parts + " + (long long)(k + u * slices) * " + C +
       " + (long long)cb * " + Ws + " + cc));");
    close();
    ln("for (; k < " + NCH + "; k += slices) q[0] = " + Op + "::apply(q[0], __ldcg(" + parts + " + (long long)k * " + C +
       " + (long long)cb * " + Ws + " + cc));");
    ln("a = " + Op + "::apply(" + Op + "::apply(q[0], q[1]), " + Op + "::apply(q[2], q[3]));");
    close();
    ln("smem[threadIdx.x] = a;");
    ln("__syncthreads();");
    open("if (sl == 0 && (long long)cb * " + Ws + " + cc < " + C + ")");
    ln("float v = smem[cc];");
    ln("for (int j = 1; j < slices; ++j) v = " + Op + "::apply(v, smem[j * " + Ws + " + cc]);");
    ln(out_ptr(m) + "[(long long)cb * " + Ws + " + cc] = v;");
    close();

  }
  ln("if (threadIdx.x == 0) atomicExch(gsync + " + std::to_string(c.cr_sync) + " + cb, 0u);");
  close();
  ln("__syncthreads();");
  close();
  close();
}

bool Builder::plan_row(Component& c) {
  if (!opts_.allow_row) return false;
  // Anchor: the largest tensor the component touches.
  int anchor = -1;
  auto better = [&](int a) {
    if (anchor < 0) return true;
    int64_t ea = prod(vals_[a].dims), eb = prod(vals_[anchor].dims);
    return ea > eb || (ea == eb && vals_[a].dims.size() > vals_[anchor].dims.size());
  };
  for (int m : c.members) {
    if (better(m)) anchor = m;
    for (int o : vals_[m].operands)
      if (!vals_[o].constant && better(o)) anchor = o;
  }
  const std::vector<int64_t>& A = vals_[anchor].dims;
  if (A.size() < 2) return false;

  const int N = static_cast<int>(vals_.size());
  int chosen_k = -1;
  std::vector<Cls> best_cls;
  for (int k = static_cast<int>(A.size()) - 1; k >= 1; --k) {
    std::vector<int64_t> P(A.begin(), A.begin() + k);
    auto rowed = [&](int v) {
      const auto& d = vals_[v].dims;
      return d.size() >= static_cast<size_t>(k) && std::equal(P.begin(), P.end(), d.begin());
    };
    std::vector<Cls> cls(N, Cls::kNone);
    bool ok = true;
    for (int v = 0; v < N; ++v)
      if (vals_[v].external || vals_[v].constant) cls[v] = rowed(v) ? Cls::kRowed : Cls::kFree;
    for (int m : c.members) {
      const OpNode& op = *vals_[m].node;
      const auto& ops = vals_[m].operands;
      auto is_post_src = [&](int o) { return cls[o] == Cls::kCross || cls[o] == Cls::kPost; };
      bool any_post = std::any_of(ops.begin(), ops.end(), is_post_src);
      if (op.type == OpType::kElementwise) {
        if (any_post) {
          for (int o : ops)
            if (cls[o] == Cls::kRowed) ok = false;
          cls[m] = Cls::kPost;
          continue;
        }
        if (op.elem_name == "broadcast") {
          int in = ops[0];
          if (rowed(m)) {
            if (cls[in] == Cls::kRowed) {
              std::vector<int> mp = broadcast_dim_map(vals_[in].node->shape, op.shape);
              for (int i = 0; i < k; ++i) ok = ok && mp[i] == i;
            } else {
              std::vector<int> mp = broadcast_dim_map(vals_[in].node->shape, op.shape);
              for (int d : mp) ok = ok && d >= k;
            }
            cls[m] = Cls::kRowed;
          } else {
            if (cls[in] == Cls::kRowed) ok = false;
            cls[m] = Cls::kFree;
          }
        } else {
          Cls want = rowed(m) ? Cls::kRowed : Cls::kFree;
          for (int o : ops)
            if (!vals_[o].constant && cls[o] != want) ok = false;
          cls[m] = want;
        }
      } else if (op.type == OpType::kReduce) {
        int in = ops[0];
        if (cls[in] != Cls::kRowed) {
          ok = false;
          break;
        }
        int nrow = 0;
        for (int d : op.reduce_dims) nrow += d < k;
        const int rank_in = static_cast<int>(vals_[in].dims.size());
        if (nrow == 0) {
          cls[m] = Cls::kRowed;
        } else if (nrow == k && (static_cast<int>(op.reduce_dims.size()) == k ||
                                 static_cast<int>(op.reduce_dims.size()) == rank_in)) {
          cls[m] = Cls::kCross;
        } else {
          ok = false;
        }
      } else if (op.type == OpType::kBatchedDot) {
        int r = static_cast<int>(op.shape.dims.size());
        ok = ok && k <= r - 2 && cls[ops[0]] == Cls::kRowed && cls[ops[1]] == Cls::kRowed;
        cls[m] = Cls::kRowed;
      } else if (op.type == OpType::kDot) {
        auto cd = effective_contract_dims(body_, op);
        ok = ok && cls[ops[0]] == Cls::kRowed && cd[0] >= k && cls[ops[1]] == Cls::kFree &&
             vals_[ops[1]].external;
        cls[m] = Cls::kRowed;
      } else {
        ok = false;
      }
      if (!ok) break;
      // A rowed op may not consume post-phase values.
      if (cls[m] == Cls::kRowed && any_post) ok = false;
      if (!ok) break;
    }
    if (!ok) continue;
    // Free members must be pure elementwise over free / constant inputs.
    for (int m : c.members)
      if (cls[m] == Cls::kFree && vals_[m].node->type != OpType::kElementwise) ok = false;
    if (!ok) continue;
    const int64_t inner = prod(A, k);
    if (chosen_k < 0) {
      chosen_k = k;
      best_cls = cls;
    }
    if (inner >= 128) {
      chosen_k = k;
      best_cls = cls;
      break;
    }
  }
  if (chosen_k < 0) return false;
  const int k = chosen_k;
  c.k = k;
  c.P.assign(A.begin(), A.begin() + k);
  c.R = prod(c.P);
  c.cls = best_cls;
  c.staged.assign(N, 0);

  bool has_dot = false;
  int64_t max_inner = 1;
  for (int m : c.members) {
    const OpNode& op = *vals_[m].node;
    if (c.cls[m] == Cls::kRowed) max_inner = std::max(max_inner, prod(vals_[m].dims, k));
    for (int o : vals_[m].operands)
      if (c.cls[o] == Cls::kRowed && !vals_[o].constant) max_inner = std::max(max_inner, prod(vals_[o].dims, k));
    if (op.type == OpType::kBatchedDot || op.type == OpType::kDot) {
      has_dot = true;
      const int a = vals_[m].operands[0], b = vals_[m].operands[1];
      if (tc_direct(c, m)) {
        // tcgen05 stage reading its external operands straight from global
        // memory into the split tiles: nothing to stage
        c.tc_direct.push_back(m);
        continue;
      }
      c.staged[a] = 1;
      if (op.type == OpType::kBatchedDot) c.staged[b] = 1;
    }
    if (op.type == OpType::kReduce && c.cls[m] == Cls::kRowed) {
      int in = vals_[m].operands[0];
      int n_inner = static_cast<int>(vals_[in].dims.size()) - k;
      if (static_cast<int>(op.reduce_dims.size()) != n_inner) c.staged[in] = 1;  // partial in-row reduce
    }
    if (op.type == OpType::kElementwise && op.elem_name == "broadcast" && c.cls[m] == Cls::kRowed) {
      int in = vals_[m].operands[0];
      if (c.cls[in] == Cls::kRowed && prod(vals_[in].dims, k) > 1 && !identity_broadcast(in, m, k) &&
          !vals_[in].external)
        c.staged[in] = 1;
    }
    if (c.cls[m] == Cls::kCross) c.cross.push_back(m);
    if (c.cls[m] == Cls::kPost) c.post.push_back(m);
    if (c.cls[m] == Cls::kFree && vals_[m].output) c.free_out.push_back(m);
  }
  bool any_staged = std::any_of(c.staged.begin(), c.staged.end(), [](char s) { return s != 0; });
  c.cta = has_dot || any_staged || max_inner > 1024;
  // Register pressure of a warp-per-row group: every cross-row (column)
  // reduction keeps max_inner/32 partial sums per lane for the whole row
  // loop. Wide multi-gradient groups (LayerNorm backward with dgamma / dbeta
  // / bias gradients: 7 x 24 registers) spill badly, so they go CTA-per-row
  // where each thread owns max_inner/NT columns.
  bool wide_cross = false;
  if (!c.cta && opts_.wide_cross_cta) {
    int n_cross = 0;
    for (int m : c.members) n_cross += c.cls[m] == Cls::kCross;
    wide_cross = n_cross * ((max_inner + 31) / 32) > 48;
    c.cta = wide_cross;
  }
  const bool forced_cta = !c.cta && opts_.cta_rows > 0 && max_inner >= opts_.cta_rows;
  if (forced_cta) c.cta = true;
  if (c.cta) {
    int nt = 256;
    if (max_inner > 4096) nt = 512;
    if (max_inner > 8192) nt = 1024;
    if (forced_cta) nt = opts_.cta_rows;
    if (!forced_cta && opts_.cta_threads > 0 && max_inner >= opts_.cta_threads) nt = opts_.cta_threads;
    // wide multi-gradient rows: a small CTA (2 warps for 768 columns) per
    // row -- ~12 columns per thread, cheap 64-thread barriers, many rows
    // in flight per SM
    if (wide_cross) {
      nt = static_cast<int>(std::min<int64_t>(256, std::max<int64_t>(64, (max_inner / 12 + 31) / 32 * 32)));
      while (nt > 64 && max_inner % (nt * 4) != 0 && max_inner % nt != 0) nt -= 32;
      if (opts_.wide_cross_threads > 0) nt = opts_.wide_cross_threads;
    }
    c.NT = nt;
  } else {
    c.NT = 32;
    if (opts_.narrow_rows && c.cross.empty() && c.post.empty() && c.free_out.empty() && max_inner <= opts_.narrow_row_max) {
      // ~16 elements per lane, 4..32 lanes per row
      int nt = 4;
      while (nt < 32 && static_cast<int64_t>(nt) * 16 < max_inner) nt *= 2;
      c.NT = nt;
    }
  }
  if (max_inner > static_cast<int64_t>(c.NT) * 64) return false;  // too large for registers
  // shared-memory slab per row group
  // Tensor-core gemm stages: batched dots whose per-row product is one
  // 64x64 output from staged row-major operands (A [64][K], B [K][64]).
  c.tc_dot.assign(N, 0);
  if (c.cta && c.NT == 256 && opts_.tensor_cores)
    for (int m : c.tc_direct) {
      auto cd = effective_contract_dims(body_, *vals_[m].node);
      c.tc_dot[m] = 1;
      c.tc = true;
      c.tc_k = std::max<int>(c.tc_k, static_cast<int>(vals_[vals_[m].operands[0]].dims[cd[0]]));
    }
  if (c.cta && c.NT == 256 && opts_.tensor_cores)
    for (int m : c.members) {
      const OpNode& op = *vals_[m].node;
      if (op.type != OpType::kBatchedDot || c.cls[m] != Cls::kRowed) continue;
      const int a = vals_[m].operands[0], b = vals_[m].operands[1];
      std::vector<int64_t> od(vals_[m].dims.begin() + k, vals_[m].dims.end());
      auto cd = effective_contract_dims(body_, op);
      const int64_t K = vals_[a].dims[cd[0]];
      if (od.size() == 2 && od[0] == 64 && od[1] == 64 && K % 32 == 0 && K <= 256 && c.staged[a] && c.staged[b] &&
          prod(vals_[a].dims, k) == 64 * K && prod(vals_[b].dims, k) == K * 64) {
        c.tc_dot[m] = 1;
        c.tc = true;
        c.tc_k = std::max<int>(c.tc_k, static_cast<int>(K));
      }
    }
  // Pipelined tcgen05 schedule: every staged tile is an external operand of
  // a tcgen05 stage (so the raw TMA buffer is free once the split ran) and
  // at most two stages per row (2 rows x 2 accumulators x 64 TMEM columns).
  c.tc_raw.assign(N, 0);
  if (c.tc && opts_.tc_pipeline) {
    bool ok = true;
    for (int m : c.members)
      if (c.tc_dot[m]) c.tc_list.push_back(m);
    for (int v = 0; v < N && ok; ++v) {
      if (!c.staged[v]) continue;
      bool tc_operand = false;
      for (int m : c.tc_list)
        tc_operand = tc_operand || vals_[m].operands[0] == v || vals_[m].operands[1] == v;
      ok = vals_[v].external && tc_operand;
    }
    ok = ok && !c.tc_list.empty() && c.tc_list.size() <= 2 && c.tc_direct.empty();
    if (ok) {
      c.tcp = true;
      for (int v = 0; v < N; ++v)
        if (c.staged[v]) c.tc_raw[v] = 1;
    } else {
      c.tc_list.clear();
    }
  }
  // Slab layout: computed staged values first, then the external (TMA)
  // tiles; with double buffering a second copy of the external tiles
  // follows so the next row's loads overlap this row's compute.
  int64_t off = 0;
  c.smem_off.assign(N, -1);
  for (int pass = 0; pass < 2; ++pass)
    for (int v = 0; v < N; ++v)
      if (c.staged[v] && vals_[v].external == (pass == 1)) {
        c.smem_off[v] = off;
        const int64_t f = (prod(vals_[v].dims, k) + 3) / 4 * 4;
        off += f;
        if (pass == 1) c.ext_floats += f;
      }
  // Register relief for warp rows with many column reductions (BERT
  // LayerNorm-backward groups carry 5-9 [768] parameter gradients, 24
  // registers each per lane): with cross_smem the per-warp column partials
  // live in the warp's slab instead of registers when 8 warps still fit.
  c.cross_off.clear();
  if (opts_.cross_smem && !c.cta) {
    int64_t regs = 0, extra = 0;
    for (int x : c.cross) {
      const int in = vals_[x].operands[0];
      if (vals_[x].node->reduce_dims.size() == vals_[in].dims.size()) continue;  // scalar: one register
      const int64_t S = prod(vals_[in].dims, k);
      regs += layout(S, 32).elems();
      extra += (S + 3) / 4 * 4;
    }
    if (regs > opts_.cross_smem_min_regs && (off + extra + 32) * 4 * 8 <= opts_.max_smem)
      for (int x : c.cross) {
        const int in = vals_[x].operands[0];
        if (vals_[x].node->reduce_dims.size() == vals_[in].dims.size()) continue;
        c.cross_off[x] = off;
        off += (prod(vals_[in].dims, k) + 3) / 4 * 4;
      }
  }
  c.slab_floats = off;
  if (c.cta) {
    bool tma_ok = true;
    for (int v = 0; v < N; ++v)
      if (c.staged[v] && vals_[v].external) tma_ok = tma_ok && prod(vals_[v].dims, k) % 4 == 0;
    c.tma = tma_ok && std::any_of(inputs_.begin(), inputs_.end(), [&](int v) { return c.staged[v] != 0; });
    const int64_t tc_bytes = c.tc ? (c.tcp ? static_cast<int64_t>(c.tc_list.size()) : 1) * 4LL * 64 * c.tc_k * 4 + 64 * 68 * 4 + 1024 : 0;
    if (opts_.tma_double_buffer && c.tma && (c.slab_floats + c.ext_floats + 32 + 8) * 4 + tc_bytes <= opts_.max_smem) {
      c.dbuf = true;
      c.slab_floats += c.ext_floats;
    }
  }
  const int64_t tc_sets = c.tcp ? static_cast<int64_t>(c.tc_list.size()) : 1;
  const int64_t slab_bytes = (c.slab_floats + 32) * 4 + (c.tc ? tc_sets * 4 * 64 * c.tc_k * 4 + 64 * 68 * 4 + 1024 : 0);
  if (c.cta ? slab_bytes > opts_.max_smem : slab_bytes * 8 > opts_.max_smem) return false;
  c.scheme = "row";
  c.max_grid = c.cta ? c.R : (c.R + 7) / 8;
  // Broadcasts of constants or free (row-independent) tensors read only at
  // the identity element by elementwise consumers are recomputed at each use
  // (a literal or an L1-resident gather) instead of occupying registers.
  c.cheap.assign(N, 0);
  for (int m : c.members) {
    const OpNode& op = *vals_[m].node;
    if (c.cls[m] != Cls::kRowed || op.type != OpType::kElementwise || op.elem_name != "broadcast") continue;
    const int in = vals_[m].operands[0];
    // (also broadcasts of row scalars -- rstd, mean: the scalar is in a
    // register already, so the [row] -> [row, C] broadcast costs nothing)
    if (!(vals_[in].constant || c.cls[in] == Cls::kFree || (c.cls[in] == Cls::kRowed && prod(vals_[in].dims, k) == 1)))
      continue;
    if (vals_[m].output || c.staged[m] || prod(vals_[m].dims, k) == 1) continue;
    bool ok = true;
    for (int cns : vals_[m].consumers) {
      if (std::find(c.members.begin(), c.members.end(), cns) == c.members.end()) continue;
      const OpNode& co = *vals_[cns].node;
      ok = ok && c.cls[cns] == Cls::kRowed && co.type == OpType::kElementwise &&
           prod(vals_[cns].dims, k) == prod(vals_[m].dims, k) &&
           (co.elem_name != "broadcast" || identity_broadcast(m, cns, k));
    }
    if (ok && opts_.loop_fusion) c.cheap[m] = 1;
  }
  // Register relief for many-input rows (LayerNorm backward reads ~15 row
  // tensors): beyond 64 preloaded elements per thread, inputs that only
  // elementwise ops read at their own element are loaded inside each fused
  // loop step (one 128-bit load per 4 elements) instead of for the whole row.
  c.lazy.assign(N, 0);
  {
    int64_t pre = 0;
    std::vector<int> cand;
    for (int v : inputs_)
      if (c.cls[v] == Cls::kRowed && !c.staged[v] && prod(vals_[v].dims, k) > 1 && reg_input(c, v)) {
        pre += layout(prod(vals_[v].dims, k), c.NT).elems();
        bool only_ew = true;
        for (int cns : vals_[v].consumers) {
          if (std::find(c.members.begin(), c.members.end(), cns) == c.members.end()) continue;
          const OpNode& co = *vals_[cns].node;
          only_ew = only_ew && co.type == OpType::kElementwise && c.cls[cns] == Cls::kRowed &&
                    (co.elem_name != "broadcast" || identity_broadcast(v, cns, k)) &&
                    prod(vals_[cns].dims, k) == prod(vals_[v].dims, k);
        }
        if (only_ew) cand.push_back(v);
      }
    if (opts_.lazy_inputs && opts_.loop_fusion && pre > 64 && layout(prod(vals_[cand.empty() ? 0 : cand[0]].dims, k), c.NT).vec == 4)
      for (int v : cand) c.lazy[v] = 1;
  }
  // Prefetch the next row's register tiles when the extra registers fit.
  int64_t pf_regs = 0;
  for (int v : inputs_)
    if (c.cls[v] == Cls::kRowed && !c.staged[v] && prod(vals_[v].dims, k) > 1 && reg_input(c, v))
      pf_regs += layout(prod(vals_[v].dims, k), c.NT).elems();
  c.prefetch = opts_.row_prefetch && pf_regs > 0 && pf_regs <= 32 && (c.cta || opts_.row_prefetch_warp);
  return true;
}

// ---------------------------------------------------------------------------
// expressions
// ---------------------------------------------------------------------------

std::string Builder::elem_expr(const OpNode& op, const std::vector<std::string>& a) const {
  const std::string& f = op.elem_name;
  if (f == "add") return "(" + a[0] + " + " + a[1] + ")";
  if (f == "subtract") return "(" + a[0] + " - " + a[1] + ")";
  if (f == "multiply") return "(" + a[0] + " * " + a[1] + ")";
  if (f == "divide") {
    // c / x with c = +-2^k: c * rcp.rn(x) is exactly rn(c / x) (scaling by
    // a power of two commutes with rounding) at a fraction of div.rn's cost
    unsigned bits = 0;
    if (opts_.rcp_divide && std::sscanf(a[0].c_str(), "__int_as_float(0x%x)", &bits) == 1 && a[0].size() == 26 && (bits & 0x7fffffu) == 0 &&
        ((bits >> 23) & 0xffu) > 0 && ((bits >> 23) & 0xffu) < 0xffu)
      return "(" + a[0] + (nr_div_ ? " * stitch_dev::rcp_nr(" : " * __frcp_rn(") + a[1] + "))";
    if (nr_div_) return "stitch_dev::div_nr(" + a[0] + ", " + a[1] + ")";
    return "(" + a[0] + " / " + a[1] + ")";
  }
  if (f == "maximum") return "fmaxf(" + a[0] + ", " + a[1] + ")";
  if (f == "minimum") return "fminf(" + a[0] + ", " + a[1] + ")";
  if (f == "log") return "logf(" + a[0] + ")";
  if (f == "exp") return "expf(" + a[0] + ")";
  if (f == "negate") return "(-" + a[0] + ")";
  if (f == "rsqrt") return "rsqrtf(" + a[0] + ")";
  if (f == "compare") return "stitch_dev::op_compare(" + a[0] + ", " + a[1] + ")";
  if (f == "select") return "stitch_dev::op_select(" + a[0] + ", " + a[1] + ", " + a[2] + ")";
  if (f == "broadcast") return a[0];
  throw GraphError("stitched executor: unknown elementwise op " + f);
}

std::string Builder::at(int v, const std::vector<std::string>& coords) {
  const Val& x = vals_[v];
  if (x.constant) return flit(x.cval);
  const std::string key = std::to_string(v) + "@" + join(coords, ",");
  for (auto it = memo_.rbegin(); it != memo_.rend(); ++it) {
    auto f = it->find(key);
    if (f != it->end()) return f->second;
  }
  std::string expr;
  auto m = materialized_.find(v);
  if (row_hook_) {
    std::string h = row_hook_(v, coords);
    if (!h.empty()) return h;
  }
  if (m != materialized_.end()) {
    expr = "__ldcg(" + m->second + " + " + linear(coords, x.dims) + ")";
  } else if (x.external) {
    expr = "__ldg(" + in_ptr(v) + " + " + linear(coords, x.dims) + ")";
  } else if (x.member && x.node->type == OpType::kElementwise) {
    std::vector<std::string> args;
    if (x.node->elem_name == "broadcast") {
      args.push_back(at(x.operands[0], map_broadcast(x.operands[0], v, coords)));
      // a broadcast literal stays a literal (constant folding downstream,
      // e.g. c / x with c = 2^k as c * rcp(x))
      if (args[0].rfind("__int_as_float(0x", 0) == 0 && args[0].size() == 26) return args[0];
    } else {
      for (int o : x.operands) args.push_back(at(o, coords));
    }
    expr = elem_expr(*x.node, args);
  } else if (inline_heavy_ && x.member &&
             (x.node->type == OpType::kReduce || x.node->type == OpType::kDot || x.node->type == OpType::kBatchedDot)) {
    return emit_heavy(v, coords);
  } else {
    throw InternalError("stitched executor: value " + x.id + " needed inline but not materialised");
  }
  std::string t = fresh("t");
  ln("const float " + t + " = " + expr + ";  // " + x.id);
  memo_.back()[key] = t;
  return t;
}

// ---------------------------------------------------------------------------
// FLAT: vectorised grid-stride loops, one per output shape
// ---------------------------------------------------------------------------

void Builder::emit_flat(const Component& c, const std::string& lo, const std::string& n) {
  std::map<std::vector<int64_t>, std::vector<int>> by_shape;
  for (int o : c.outputs) by_shape[vals_[o].dims].push_back(o);
  for (auto& [dims, outs] : by_shape) {
    const int64_t total = prod(dims);
    const int64_t last = dims.empty() ? 1 : dims.back();
    const int vec = (last % 4 == 0) ? 4 : 1;
    const int64_t chunks = total / vec;
    open("");
    ln("// flat section over [" + [&] {
      std::string s;
      for (size_t i = 0; i < dims.size(); ++i) s += (i ? "," : "") + std::to_string(dims[i]);
      return s;
    }() + "]");
    open("for (long long e = (long long)(blockIdx.x - " + lo + ") * blockDim.x + threadIdx.x; e < " +
         std::to_string(chunks) + "LL; e += (long long)(" + n + ") * blockDim.x)");
    memo_.emplace_back();
    ln("const long long base = e * " + std::to_string(vec) + "LL;");
    std::vector<std::string> bc = decode("base", dims);
    std::map<int, std::vector<std::string>> results;
    // Identity loads of same-shaped inputs as one 128-bit load.
    if (vec == 4) {
      std::set<int> ins, seen;
      std::function<void(int)> walk = [&](int v) {
        if (!seen.insert(v).second) return;
        if (vals_[v].external && vals_[v].dims == dims) ins.insert(v);
        if (vals_[v].member && !(vals_[v].node->elem_name == "broadcast"))
          for (int o : vals_[v].operands) walk(o);
      };
      for (int o : outs) walk(o);
      for (int v : ins) {
        std::string t = fresh("q");
        ln("const float4 " + t + " = stitch_dev::ld4_stream(" + in_ptr(v) + " + base);");
        const char* lane[4] = {".x", ".y", ".z", ".w"};
        for (int u = 0; u < 4; ++u) {
          std::vector<std::string> cu = bc;
          if (!cu.empty() && u) cu.back() = "(" + bc.back() + " + " + std::to_string(u) + ")";
          memo_.back()[std::to_string(v) + "@" + join(cu, ",")] = t + lane[u];
        }
      }
    }
    for (int u = 0; u < vec; ++u) {
      std::vector<std::string> cu = bc;
      if (!cu.empty() && u) cu.back() = "(" + bc.back() + " + " + std::to_string(u) + ")";
      for (int o : outs) results[o].push_back(at(o, cu));
    }
    for (int o : outs) {
      if (vec == 4)
        ln("stitch_dev::st4(" + out_ptr(o) + " + base, " + join(results[o], ", ") + ");");
      else
        ln(out_ptr(o) + "[base] = " + results[o][0] + ";");
    }
    memo_.pop_back();
    close();
    close();
  }
}

// ---------------------------------------------------------------------------
// ROW
// ---------------------------------------------------------------------------

// Expression for operand `o` of rowed value `v` at v's owned element (it, u).
std::string Builder::row_access(const Component& c, int o, int v, const std::string& it, const std::string& u,
                                const Layout& L) {
  const Val& x = vals_[o];
  if (x.constant) return flit(x.cval);
  const int k = c.k;
  const std::string e = "(" + it + ") * " + std::to_string(L.vec) + " + (" + u + ")";
  const std::string lin = "((" + it + ") * " + std::to_string(c.NT) + " + t) * " + std::to_string(L.vec) + " + (" + u + ")";
  if (c.cls[o] == Cls::kRowed && !c.cheap.empty() && c.cheap[o])
    return row_access(c, vals_[o].operands[0], o, it, u, L);
  if (c.cls[o] == Cls::kRowed) {
    const int64_t So = prod(x.dims, k);
    if (So == 1) {
      auto s = scalar_.find(o);
      if (s != scalar_.end()) return s->second;
      if (x.external) return "__ldg(" + in_ptr(o) + " + row)";
    }
    const bool ident = (vals_[v].node->type == OpType::kElementwise &&
                        (vals_[v].node->elem_name != "broadcast" || identity_broadcast(o, v, k)));
    if (ident) {
      auto ls = loop_scalar_.find(o);
      if (ls != loop_scalar_.end()) return ls->second;
      auto rv = rowvec_.find(o);
      if (rv != rowvec_.end()) return rv->second + "[" + u + "]";
      auto r = reg_.find(o);
      if (r != reg_.end()) return r->second + "[" + e + "]";
      if (c.staged[o] && !(c.tcp && c.tc_raw[o])) return "sm" + std::to_string(o) + "[" + lin + "]";
      if (x.external) return "__ldg(" + in_ptr(o) + " + row * " + std::to_string(So) + "LL + " + lin + ")";
    }
    // Gather through the broadcast map within the row.
    std::vector<int64_t> vin(vals_[v].dims.begin() + k, vals_[v].dims.end());
    std::vector<std::string> vc = decode(lin, vin);
    std::vector<std::string> full;
    for (int i = 0; i < k; ++i) full.push_back("0");
    full.insert(full.end(), vc.begin(), vc.end());
    std::vector<std::string> oc = map_broadcast(o, v, full);
    std::vector<std::string> oin(oc.begin() + k, oc.end());
    std::vector<int64_t> odims(x.dims.begin() + k, x.dims.end());
    const std::string olin = linear(oin, odims);
    if (c.staged[o]) return "sm" + std::to_string(o) + "[" + olin + "]";
    if (x.external) return "__ldg(" + in_ptr(o) + " + row * " + std::to_string(So) + "LL + " + olin + ")";
    throw InternalError("stitched executor: rowed value " + x.id + " gathered without staging");
  }
  // free operand: inline expression at the mapped coordinates
  std::vector<int64_t> vin(vals_[v].dims.begin() + k, vals_[v].dims.end());
  std::vector<std::string> vc = decode(lin, vin);
  std::vector<std::string> full;
  for (int i = 0; i < k; ++i) full.push_back("0");
  full.insert(full.end(), vc.begin(), vc.end());
  std::vector<std::string> oc = (vals_[v].node->elem_name == "broadcast") ? map_broadcast(o, v, full) : full;
  // Same-shape free input read at the identity element: vector-friendly index
  // (a float4 loaded once per `it` by the fused loop when available).
  if (free_vector_access(c, o, v)) {
    auto fv = freevec_.find(o);
    if (fv != freevec_.end()) return fv->second + "[" + u + "]";
    return "__ldg(" + in_ptr(o) + " + " + lin + ")";
  }
  return at(o, oc);
}

// Row-scalar elementwise op (one value per row, S == 1): every thread of the
// row group holds it.
void Builder::emit_row_scalar(const Component& c, int m) {
  const OpNode& op = *vals_[m].node;
  std::vector<std::string> args;
  for (int o : vals_[m].operands) {
    if (vals_[o].constant) {
      args.push_back(flit(vals_[o].cval));
    } else if (c.cls[o] == Cls::kRowed) {
      auto s = scalar_.find(o);
      args.push_back(s != scalar_.end() ? s->second : "__ldg(" + in_ptr(o) + " + row)");
    } else {
      std::vector<std::string> zero(vals_[o].dims.size(), "0");
      args.push_back(at(o, zero));
    }
  }
  std::string s = fresh("s");
  ln("const float " + s + " = " + elem_expr(op, args) + ";  // " + vals_[m].id);
  scalar_[m] = s;
}

// v reads free external o at v's own in-row element (o's dims are v's inner
// dims and the access is the identity): a row-invariant vector like a bias.
bool Builder::free_vector_access(const Component& c, int o, int v) const {
  const Val& x = vals_[o];
  if (!x.external || c.cls[o] != Cls::kFree || vals_[v].node->type != OpType::kElementwise) return false;
  std::vector<int64_t> vin(vals_[v].dims.begin() + c.k, vals_[v].dims.end());
  if (x.dims != vin) return false;
  if (vals_[v].node->elem_name != "broadcast") return true;
  std::vector<int> mp = broadcast_dim_map(x.node->shape, vals_[v].node->shape);
  for (size_t i = 0; i < mp.size(); ++i)
    if (mp[i] != static_cast<int>(i) + c.k) return false;
  return true;
}

// Batched dot eligible for the tcgen05 stage with both operands external
// rowed inputs (64 x K and K x 64 per row, K % 32 == 0).
bool Builder::tc_direct(const Component& c, int m) const {
  if (!opts_.tensor_cores || !opts_.tc_direct_loads) return false;
  const OpNode& op = *vals_[m].node;
  if (op.type != OpType::kBatchedDot) return false;
  const int a = vals_[m].operands[0], b = vals_[m].operands[1];
  if (!vals_[a].external || !vals_[b].external) return false;
  std::vector<int64_t> od(vals_[m].dims.begin() + c.k, vals_[m].dims.end());
  auto cd = effective_contract_dims(body_, op);
  const int64_t K = vals_[a].dims[cd[0]];
  return od.size() == 2 && od[0] == 64 && od[1] == 64 && K % 32 == 0 && K <= 256 && prod(vals_[a].dims, c.k) == 64 * K &&
         prod(vals_[b].dims, c.k) == K * 64;
}

// A rowed external input some member reads at the identity element (so it is
// loaded once per row into registers).
bool Builder::reg_input(const Component& c, int v) const {
  for (int m : vals_[v].consumers) {
    if (std::find(c.members.begin(), c.members.end(), m) == c.members.end()) continue;
    const OpNode& op = *vals_[m].node;
    if (op.type == OpType::kReduce) return true;
    if (op.type == OpType::kElementwise && (op.elem_name != "broadcast" || identity_broadcast(v, m, c.k))) return true;
  }
  return false;
}

// Loads this thread's elements of row `row` of input v into register array
// `dst` (128-bit streaming loads when the row extent allows).
void Builder::emit_row_load(int v, const std::string& dst, const std::string& row, const Layout& L, int NT) {
  const int64_t S = L.S;
  ln("#pragma unroll");
  open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
  ln("const int lin = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + ";");
  if (L.guard) open("if (lin < " + std::to_string(S) + ")");
  const std::string src = in_ptr(v) + " + (" + row + ") * " + std::to_string(S) + "LL + lin";
  if (L.vec == 4) {
    ln("const float4 q = stitch_dev::ld4_stream(" + src + ");");
    ln(dst + "[it * 4 + 0] = q.x; " + dst + "[it * 4 + 1] = q.y; " + dst + "[it * 4 + 2] = q.z; " + dst + "[it * 4 + 3] = q.w;");
  } else {
    for (int u = 0; u < L.vec; ++u)
      ln(dst + "[it * " + std::to_string(L.vec) + " + " + std::to_string(u) + "] = __ldg(" + src + " + " + std::to_string(u) + ");");
  }
  if (L.guard) {
    close();
    ln("else { for (int u = 0; u < " + std::to_string(L.vec) + "; ++u) " + dst + "[it * " + std::to_string(L.vec) + " + u] = 0.0f; }");
  }
  close();
}

void Builder::emit_row(Component& c, const std::string& lo, const std::string& n, const std::string& cta_rank) {
  const int k = c.k;
  const int NT = c.NT;
  (void)cta_rank;
  open("");
  ln("// row scheme: k=" + std::to_string(k) + " rows=" + std::to_string(c.R) + " threads/row=" + std::to_string(NT));
  const std::string rlo = chunked_ ? "row_lo" : "0LL";
  const std::string rhi = chunked_ ? "row_hi" : std::to_string(c.R) + "LL";
  if (c.cta) {
    ln("const int t = threadIdx.x;");
    if (c.tc) {
      // tcgen05 region at the 1024-aligned start of dynamic smem: hi/lo
      // operand tiles (swizzled), the D tile, then the slab
      const int64_t scratch_b = 4LL * 64 * c.tc_k * 4;
      const int64_t sets = c.tcp ? static_cast<int64_t>(c.tc_list.size()) : 1;
      ln("unsigned char* tcs = reinterpret_cast<unsigned char*>(smem);  // " + std::to_string(sets) + " split set(s)");
      ln("float* tcD = smem + " + std::to_string(sets * scratch_b / 4) + ";  // one padded 64x64 D tile, reused by each stage");
      ln("float* slab = smem + " + std::to_string(sets * scratch_b / 4 + 64 * 68) + ";");
    } else {
      ln("float* slab = smem;");
    }
    ln("const long long g0 = blockIdx.x - " + lo + ", gstride = " + n + ";");
  } else {
    ln("const int t = threadIdx.x & " + std::to_string(NT - 1) + ";");
    ln("const int wib = threadIdx.x / " + std::to_string(NT) + ", wpb = blockDim.x / " + std::to_string(NT) + ";");
    ln("float* slab = smem + wib * " + std::to_string(c.slab_floats + 32) + ";");
    ln("const long long g0 = (long long)(blockIdx.x - " + lo + ") * wpb + wib, gstride = (long long)(" + n + ") * wpb;");
  }
  ln("float* red = slab + " + std::to_string(c.slab_floats) + ";");
  ln("(void)red;");
  const bool pp = c.cta && NT > 32 && opts_.pp_reduce;
  if (pp) ln("int rpp = 0;  // in-row reductions alternate red[0..31] / red[64..95]");
  for (int v = 0; v < static_cast<int>(vals_.size()); ++v)
    if (c.staged[v] && !(c.dbuf && vals_[v].external))
      ln("float* sm" + std::to_string(v) + " = slab + " + std::to_string(c.smem_off[v]) + ";  // " + vals_[v].id);

  // Free outputs (not depending on rows): grid-stride over their elements.
  for (int f : c.free_out) {
    open("for (long long i = (long long)(blockIdx.x - " + lo + ") * blockDim.x + threadIdx.x; i < " +
         std::to_string(prod(vals_[f].dims)) + "LL; i += (long long)(" + n + ") * blockDim.x)");
    memo_.emplace_back();
    ln(out_ptr(f) + "[i] = " + at(f, decode("i", vals_[f].dims)) + ";");
    memo_.pop_back();
    close();
  }

  // Cross-row partial accumulators.
  std::map<int, Layout> cross_layout;
  for (int x : c.cross) {
    const OpNode& op = *vals_[x].node;
    int in = vals_[x].operands[0];
    Layout L = layout(prod(vals_[in].dims, k), NT);
    cross_layout[x] = L;
    bool scalar = static_cast<int>(op.reduce_dims.size()) == static_cast<int>(vals_[in].dims.size());
    const std::string Op = op.elem_name == "max" ? "stitch_dev::MaxOp" : "stitch_dev::SumOp";
    if (scalar)
      ln("float p" + std::to_string(x) + " = " + Op + "::init();  // " + vals_[x].id);
    else if (c.cross_off.count(x)) {
      ln("float* p" + std::to_string(x) + " = slab + " + std::to_string(c.cross_off[x]) + ";  // " + vals_[x].id + " (warp partials in shared memory)");
      ln("#pragma unroll");
      open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
      ln("#pragma unroll");
      open("for (int u = 0; u < " + std::to_string(L.vec) + "; ++u)");
      ln("const int lin = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + " + u;");
      ln((L.guard ? "if (lin < " + std::to_string(L.S) + ") " : std::string()) + "p" + std::to_string(x) + "[lin] = " + Op + "::init();");
      close();
      close();
    } else {
      ln("float p" + std::to_string(x) + "[" + std::to_string(L.elems()) + "];  // " + vals_[x].id);
      ln("#pragma unroll");
      ln("for (int e = 0; e < " + std::to_string(L.elems()) + "; ++e) p" + std::to_string(x) + "[e] = " + Op + "::init();");
    }
  }

  if (c.tc) {
    ln("stitch_dev::u64* tcbar = reinterpret_cast<stitch_dev::u64*>(red + 36);  // after the TMA barriers at red + 32");
    ln("unsigned* tcslot = reinterpret_cast<unsigned*>(red + 38);");
    ln("if (t == 0) stitch_dev::mbar_init(tcbar, 1);");
    const int cols = c.tcp ? (c.tc_list.size() > 1 ? 256 : 128) : 64;
    ln("const unsigned tmem = stitch_dev::tc::alloc(tcslot, " + std::to_string(cols) +
       ");  // 64 fp32 columns per 64x64 accumulator" + (c.tcp ? " (x2 rows in flight)" : ""));
    ln("unsigned tcphase = 0;");
  }
  // External tiles of one row: total bytes and the bulk copies into buffer `b`.
  int64_t tma_bytes = 0;
  for (int v : inputs_)
    if (c.staged[v]) tma_bytes += prod(vals_[v].dims, k) * 4;
  auto issue_tma = [&](const std::string& r, const std::string& b) {
    ln("stitch_dev::mbar_expect_tx(bar + " + b + ", " + std::to_string(tma_bytes) + "u);");
    for (int v : inputs_)
      if (c.staged[v]) {
        const int64_t S = prod(vals_[v].dims, k);
        ln("stitch_dev::bulk_g2s(slab + " + std::to_string(c.smem_off[v]) + " + " + b + " * " + std::to_string(c.ext_floats) +
           ", " + in_ptr(v) + " + (" + r + ") * " + std::to_string(S) + "LL, " + std::to_string(S * 4) + "u, bar + " + b + ");");
      }
  };
  // tma_early: a staged input's tile for the next row is requested as soon
  // as this row's last reader of it is done (one CTA barrier per release
  // point), so the next row's loads overlap this row's remaining stages.
  const bool early_tma = opts_.tma_early && c.cta && c.tma && !c.dbuf && !c.tcp;
  std::map<size_t, std::vector<int>> release_at;  // member index -> inputs whose last reader it is
  if (early_tma) {
    const size_t kEnd = c.members.size();
    std::map<int, size_t> last;
    for (int v : inputs_)
      if (c.staged[v]) last[v] = 0;
    std::function<void(int, size_t)> reads = [&](int o, size_t j) {
      if (last.count(o)) last[o] = std::max(last[o], j);
      if (c.cls[o] == Cls::kRowed && !c.cheap.empty() && c.cheap[o] && vals_[o].member)
        for (int q : vals_[o].operands) reads(q, j);
    };
    for (size_t j = 0; j < c.members.size(); ++j) {
      const int m = c.members[j];
      const bool after_loop = c.cls[m] == Cls::kCross || c.cls[m] == Cls::kPost;
      for (int o : vals_[m].operands) reads(o, after_loop ? kEnd : j);
    }
    for (auto& [v, j] : last) release_at[j].push_back(v);
  }
  auto issue_some = [&](const std::vector<int>& vs, bool with_expect) {
    if (with_expect) ln("stitch_dev::mbar_expect_tx(bar, " + std::to_string(tma_bytes) + "u);");
    for (int v : vs) {
      const int64_t S = prod(vals_[v].dims, k);
      ln("stitch_dev::bulk_g2s(slab + " + std::to_string(c.smem_off[v]) + ", " + in_ptr(v) + " + (row + gstride) * " +
         std::to_string(S) + "LL, " + std::to_string(S * 4) + "u, bar);  // next row's " + vals_[v].id);
    }
  };
  bool early_expect_done = false;
  auto release_upto = [&](size_t idx) {
    while (!release_at.empty() && release_at.begin()->first <= idx && release_at.begin()->first < c.members.size()) {
      ln("__syncthreads();  // every reader of these tiles is done with this row");
      open("if (t == 0 && row + gstride < " + rhi + ")");
      issue_some(release_at.begin()->second, !early_expect_done);
      close();
      early_expect_done = true;
      release_at.erase(release_at.begin());
    }
  };
  if (c.tma) {
    // TMA barriers right after the reduction scratch `red` (relative to the
    // slab, which the tcgen05 region may displace)
    ln("stitch_dev::u64* bar = reinterpret_cast<stitch_dev::u64*>(red + 32);");
    ln(c.dbuf ? "if (t == 0) { stitch_dev::mbar_init(bar, 1); stitch_dev::mbar_init(bar + 1, 1); }"
              : "if (t == 0) stitch_dev::mbar_init(bar, 1);");
    ln("__syncthreads();");
    ln("unsigned phase = 0;");
    if (early_tma) {
      // this CTA's first row; later rows are issued from inside the loop
      open("if (t == 0 && " + rlo + " + g0 < " + rhi + ")");
      issue_tma(rlo + " + g0", "0");
      close();
    }
    if (c.dbuf) {
      ln("int buf = 0;");
      open("if (t == 0 && " + rlo + " + g0 < " + rhi + ")");
      issue_tma(rlo + " + g0", "0");
      close();
    }
  }
  // tcp: row r+1's split and MMAs are issued before row r's epilogue, into
  // the other TMEM buffer; row r+2's tiles stream in meanwhile
  const int ntc = static_cast<int>(c.tc_list.size());
  auto tcp_split_issue = [&](const std::string& buf_expr) {
    for (int j = 0; j < ntc; ++j) {
      const int m = c.tc_list[j];
      const int a = vals_[m].operands[0], b = vals_[m].operands[1];
      ln("stitch_dev::tc::split_operands<" + std::to_string(c.tc_k) + ">(slab + " + std::to_string(c.smem_off[a]) +
         ", slab + " + std::to_string(c.smem_off[b]) + ", tcs + " + std::to_string(j * 4LL * 64 * c.tc_k * 4) + ");");
    }
    ln("stitch_dev::tc::publish_operands();  // also: every thread is done with the raw tiles");
  };
  auto tcp_issue = [&](const std::string& buf_expr) {
    open("if (t == 0)");
    for (int j = 0; j < ntc; ++j)
      ln("stitch_dev::tc::issue_tf32x3<" + std::to_string(c.tc_k) + ">(tcs + " + std::to_string(j * 4LL * 64 * c.tc_k * 4) +
         ", tmem + ((" + buf_expr + ") * " + std::to_string(ntc) + " + " + std::to_string(j) + ") * 64);");
    ln("stitch_dev::tc::commit(tcbar);");
    close();
  };
  if (c.tcp) {
    ln("int tb = 0;");
    open("if (" + rlo + " + g0 < " + rhi + ")");
    open("if (t == 0)");
    issue_tma(rlo + " + g0", "0");
    close();
    ln("stitch_dev::mbar_wait(bar, phase);");
    ln("phase ^= 1u;");
    tcp_split_issue("0");
    open("if (t == 0 && " + rlo + " + g0 + gstride < " + rhi + ")");
    issue_tma(rlo + " + g0 + gstride", "0");
    close();
    tcp_issue("0");
    close();
  }
  if (c.prefetch) {
    for (int v : inputs_)
      if (c.cls[v] == Cls::kRowed && !c.staged[v] && prod(vals_[v].dims, k) > 1 && reg_input(c, v)) {
        const Layout L = layout(prod(vals_[v].dims, k), NT);
        ln("float pf" + std::to_string(v) + "[" + std::to_string(L.elems()) + "];  // next row of " + vals_[v].id);
      }
    open("if (" + rlo + " + g0 < " + rhi + ")");
    for (int v : inputs_)
      if (c.cls[v] == Cls::kRowed && !c.staged[v] && prod(vals_[v].dims, k) > 1 && reg_input(c, v))
        emit_row_load(v, "pf" + std::to_string(v), rlo + " + g0", layout(prod(vals_[v].dims, k), NT), NT);
    close();
  }
  open("for (long long row = " + rlo + " + g0; row < " + rhi + "; row += gstride" + (c.dbuf ? ", buf ^= 1" : "") + ")");
  reg_.clear();
  scalar_.clear();
  memo_.emplace_back();
  const std::string sync = c.cta ? "__syncthreads();" : "__syncwarp();";

  // Stage external operand tiles (TMA bulk copies in CTA mode).
  bool any_ext_staged = false;
  for (int v : inputs_)
    if (c.staged[v]) any_ext_staged = true;
  if (c.tcp) {
    any_ext_staged = false;  // the tcgen05 pipeline owns the raw tiles
    ln("stitch_dev::mbar_wait(tcbar, tcphase);  // this row's MMAs are done");
    ln("tcphase ^= 1u;");
    ln("stitch_dev::tc::fence_after();");
    open("if (row + gstride < " + rhi + ")");
    ln("stitch_dev::mbar_wait(bar, phase);  // next row's tiles landed");
    ln("phase ^= 1u;");
    tcp_split_issue("tb ^ 1");
    open("if (t == 0 && row + 2 * gstride < " + rhi + ")");
    issue_tma("row + 2 * gstride", "0");
    close();
    tcp_issue("tb ^ 1");
    close();
  }
  if (any_ext_staged) {
    if (c.dbuf) {
      // prefetch the next row into the other buffer (its readers finished at
      // the previous iteration's trailing barrier), then wait for this one
      open("if (t == 0 && row + gstride < " + rhi + ")");
      issue_tma("row + gstride", "(buf ^ 1)");
      close();
      ln("stitch_dev::mbar_wait(bar + buf, (phase >> buf) & 1u);");
      ln("phase ^= 1u << buf;");
      for (int v : inputs_)
        if (c.staged[v])
          ln("float* sm" + std::to_string(v) + " = slab + " + std::to_string(c.smem_off[v]) + " + buf * " +
             std::to_string(c.ext_floats) + ";  // " + vals_[v].id);
    } else if (c.tma) {
      if (!early_tma) {
        open("if (t == 0)");
        issue_tma("row", "0");
        close();
      }
      ln("stitch_dev::mbar_wait(bar, phase);");
      ln("phase ^= 1u;");
    } else {
      for (int v : inputs_)
        if (c.staged[v]) {
          const int64_t S = prod(vals_[v].dims, k);
          ln("for (int i = t; i < " + std::to_string(S) + "; i += " + std::to_string(NT) + ") sm" + std::to_string(v) +
             "[i] = __ldg(" + in_ptr(v) + " + row * " + std::to_string(S) + "LL + i);");
        }
      ln(sync);
    }
  }

  // Register loads of rowed inputs read at identity by elementwise ops.
  // With prefetching (row_pf), the next row's tiles are already in flight in
  // pf<v> while this row computes: the loop renames pf -> r and re-issues.
  for (int v : inputs_) {
    if (c.cls[v] != Cls::kRowed || (c.staged[v] && !(c.tcp && c.tc_raw[v]))) continue;
    const int64_t S = prod(vals_[v].dims, k);
    if (S == 1) {
      std::string s = fresh("s");
      ln("const float " + s + " = __ldg(" + in_ptr(v) + " + row);  // " + vals_[v].id);
      scalar_[v] = s;
      continue;
    }
    if (!reg_input(c, v)) continue;
    if (!c.lazy.empty() && c.lazy[v]) continue;  // loaded inside the fused loops
    const Layout L = layout(S, NT);
    const std::string r = "r" + std::to_string(v);
    ln("float " + r + "[" + std::to_string(L.elems()) + "];  // " + vals_[v].id);
    if (c.prefetch) {
      ln("#pragma unroll");
      ln("for (int e = 0; e < " + std::to_string(L.elems()) + "; ++e) " + r + "[e] = pf" + std::to_string(v) + "[e];");
    } else {
      emit_row_load(v, r, "row", L, NT);
    }
    reg_[v] = r;
  }
  if (c.prefetch) {
    open("if (row + gstride < " + rhi + ")");
    for (int v : inputs_)
      if (c.cls[v] == Cls::kRowed && !c.staged[v] && prod(vals_[v].dims, k) > 1 && reg_input(c, v))
        emit_row_load(v, "pf" + std::to_string(v), "row + gstride", layout(prod(vals_[v].dims, k), NT), NT);
    close();
  }

  auto emit_elementwise_loop = [&](int m, const Layout& L, const std::function<std::string(const std::string&, const std::string&)>& body_fn) {
    std::string r = "r" + std::to_string(m);
    ln("float " + r + "[" + std::to_string(L.elems()) + "];  // " + vals_[m].id);
    ln("#pragma unroll");
    open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
    ln("#pragma unroll");
    open("for (int u = 0; u < " + std::to_string(L.vec) + "; ++u)");
    memo_.emplace_back();
    if (L.guard) {
      ln("const int lin_g = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + " + u;");
      open("if (lin_g < " + std::to_string(L.S) + ")");
    }
    ln(r + "[it * " + std::to_string(L.vec) + " + u] = " + body_fn("it", "u") + ";");
    if (L.guard) {
      close();
      ln("else " + r + "[it * " + std::to_string(L.vec) + " + u] = 0.0f;");
    }
    memo_.pop_back();
    close();
    close();
    reg_[m] = r;
  };

  auto stage_value = [&](int m, const Layout& L, int64_t S) {
    ln(sync);  // previous readers of this slab region are done
    ln("#pragma unroll");
    open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
    ln("#pragma unroll");
    open("for (int u = 0; u < " + std::to_string(L.vec) + "; ++u)");
    ln("const int lin = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + " + u;");
    std::string val = S == 1 ? scalar_[m] : reg_[m] + "[it * " + std::to_string(L.vec) + " + u]";
    ln((L.guard ? "if (lin < " + std::to_string(S) + ") " : std::string()) + "sm" + std::to_string(m) + "[lin] = " + val + ";");
    close();
    close();
    ln(sync);
  };
  auto in_comp = [&](int x) { return std::find(c.members.begin(), c.members.end(), x) != c.members.end(); };

  for (size_t mi = 0; mi < c.members.size(); ++mi) {
    if (early_tma && mi > 0) release_upto(mi - 1);
    const int m = c.members[mi];
    if (c.cls[m] != Cls::kRowed) continue;
    const OpNode& op = *vals_[m].node;
    const int64_t S = prod(vals_[m].dims, k);
    const Layout L = layout(S, NT);
    if (op.type == OpType::kElementwise && S > 1 && opts_.loop_fusion) {
      // Aggressive loop fusion (paper §5.1: "merge as many elementwise ops
      // as possible into a single loop structure"): the run of consecutive
      // rowed elementwise ops over the same row extent becomes one loop
      // over this thread's elements; values used only inside the run live
      // in scalars, only escaping values get register arrays.
      std::vector<int> grp, hoisted;
      std::set<int> in_grp;
      size_t mj = mi;
      for (; mj < c.members.size(); ++mj) {
        const int x = c.members[mj];
        if (c.cls[x] != Cls::kRowed) {
          bool reads_grp = false;
          for (int o : vals_[x].operands) reads_grp = reads_grp || in_grp.count(o);
          if (reads_grp) break;  // e.g. a cross-row reduce of a run value: keep order simple
          continue;
        }
        const OpNode& xo = *vals_[x].node;
        if (c.cheap[x]) continue;  // recomputed at its uses
        if (xo.type == OpType::kElementwise && prod(vals_[x].dims, k) == 1) {
          bool reads_grp = false;
          for (int o : vals_[x].operands) reads_grp = reads_grp || in_grp.count(o);
          if (reads_grp) break;
          hoisted.push_back(x);  // row scalar, independent of the run: emitted before the loop
          continue;
        }
        if (xo.type != OpType::kElementwise || prod(vals_[x].dims, k) != S) break;
        bool ok = true;
        for (int o : vals_[x].operands)
          if (in_grp.count(o) && xo.elem_name == "broadcast" && !identity_broadcast(o, x, k)) ok = false;
        if (!ok) break;
        grp.push_back(x);
        in_grp.insert(x);
      }
      for (int x : hoisted) emit_row_scalar(c, x);
      std::set<int> escapes;
      for (int g : grp) {
        bool esc = vals_[g].output || c.staged[g];
        for (int cns : vals_[g].consumers)
          if (in_comp(cns) && !in_grp.count(cns)) esc = true;
        if (esc) escapes.insert(g);
      }
      for (int g : grp)
        if (escapes.count(g)) ln("float r" + std::to_string(g) + "[" + std::to_string(L.elems()) + "];  // " + vals_[g].id);
      ln("#pragma unroll");
      open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
      if (L.vec == 4) {
        // row-invariant vectors (bias, gamma, mask, ...) this run reads at
        // its own element: one 128-bit L1-cached load per `it`
        std::set<int> fvs;
        std::function<void(int, int)> scan = [&](int g, int depth) {
          for (int o : vals_[g].operands) {
            if (free_vector_access(c, o, g)) fvs.insert(o);
            if (depth < 4 && c.cls[o] == Cls::kRowed && !c.cheap.empty() && c.cheap[o]) scan(o, depth + 1);
          }
        };
        for (int g : grp) scan(g, 0);
        for (int o : fvs) {
          const std::string f = "fv" + std::to_string(o);
          ln("float " + f + "[4];");
          open("");
          ln("const int lin4 = (it * " + std::to_string(NT) + " + t) * 4;");
          if (L.guard) open("if (lin4 < " + std::to_string(L.S) + ")");
          ln("const float4 q = stitch_dev::ld4(" + in_ptr(o) + " + lin4);");
          ln(f + "[0] = q.x; " + f + "[1] = q.y; " + f + "[2] = q.z; " + f + "[3] = q.w;");
          if (L.guard) {
            close();
            ln("else { " + f + "[0] = " + f + "[1] = " + f + "[2] = " + f + "[3] = 0.0f; }");
          }
          close();
          freevec_[o] = f;
        }
        // lazily loaded row inputs this run reads at its own element
        std::set<int> lz;
        for (int g : grp)
          for (int o : vals_[g].operands)
            if (!c.lazy.empty() && c.lazy[o] && !reg_.count(o)) lz.insert(o);
        for (int o : lz) {
          const std::string f = "rv" + std::to_string(o);
          const int64_t So = prod(vals_[o].dims, k);
          ln("float " + f + "[4];");
          open("");
          ln("const int lin4 = (it * " + std::to_string(NT) + " + t) * 4;");
          if (L.guard) open("if (lin4 < " + std::to_string(So) + ")");
          ln("const float4 q = stitch_dev::ld4(" + in_ptr(o) + " + row * " + std::to_string(So) + "LL + lin4);");
          ln(f + "[0] = q.x; " + f + "[1] = q.y; " + f + "[2] = q.z; " + f + "[3] = q.w;");
          if (L.guard) {
            close();
            ln("else { " + f + "[0] = " + f + "[1] = " + f + "[2] = " + f + "[3] = 0.0f; }");
          }
          close();
          rowvec_[o] = f;
        }
      }
      ln("#pragma unroll");
      open("for (int u = 0; u < " + std::to_string(L.vec) + "; ++u)");
      memo_.emplace_back();
      if (L.guard) {
        ln("const int lin_g = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + " + u;");
        open("if (lin_g < " + std::to_string(L.S) + ")");
      }
      for (int g : grp) {
        std::vector<std::string> args;
        for (int o : vals_[g].operands) args.push_back(row_access(c, o, g, "it", "u", L));
        const std::string v = "v" + std::to_string(g);
        ln("const float " + v + " = " + elem_expr(*vals_[g].node, args) + ";  // " + vals_[g].id);
        loop_scalar_[g] = v;
        if (escapes.count(g)) ln("r" + std::to_string(g) + "[it * " + std::to_string(L.vec) + " + u] = " + v + ";");
      }
      if (L.guard) {
        close();
        open("else");
        for (int g : grp)
          if (escapes.count(g)) ln("r" + std::to_string(g) + "[it * " + std::to_string(L.vec) + " + u] = 0.0f;");
        close();
      }
      memo_.pop_back();
      close();
      close();
      freevec_.clear();
      rowvec_.clear();
      for (int g : grp) {
        loop_scalar_.erase(g);
        if (escapes.count(g)) reg_[g] = "r" + std::to_string(g);
      }
      for (int g : grp)
        if (c.staged[g]) stage_value(g, L, S);
      // continue after the last fused / hoisted member (skipped non-rowed and
      // cheap members emit nothing here)
      size_t last = mi;
      for (size_t q = mi; q < c.members.size(); ++q)
        if (in_grp.count(c.members[q]) ||
            std::find(hoisted.begin(), hoisted.end(), c.members[q]) != hoisted.end())
          last = q;
      mi = last;
      continue;
    }
    if (!c.cheap.empty() && c.cheap[m]) continue;
    if (op.type == OpType::kElementwise) {
      if (S == 1) {
        emit_row_scalar(c, m);
      } else {
        emit_elementwise_loop(m, L, [&](const std::string& it, const std::string& u) {
          std::vector<std::string> args;
          for (int o : vals_[m].operands) args.push_back(row_access(c, o, m, it, u, L));
          return elem_expr(op, args);
        });
      }
    } else if (op.type == OpType::kReduce) {
      const int in = vals_[m].operands[0];
      const std::string Op = op.elem_name == "max" ? "stitch_dev::MaxOp" : "stitch_dev::SumOp";
      const int64_t Sin = prod(vals_[in].dims, k);
      const Layout Li = layout(Sin, NT);
      if (S == 1 && Sin == 1) {
        // a reduce over a single element per row is the element itself
        int src = in;
        while (c.cls[src] == Cls::kRowed && !c.cheap.empty() && c.cheap[src]) src = vals_[src].operands[0];
        std::string x;
        auto sc = scalar_.find(src);
        auto r = reg_.find(src);
        if (vals_[src].constant) x = flit(vals_[src].cval);
        else if (sc != scalar_.end()) x = sc->second;
        else if (r != reg_.end()) x = r->second + "[0]";
        else if (c.staged[src]) x = "sm" + std::to_string(src) + "[0]";
        else if (c.cls[src] == Cls::kRowed && vals_[src].external) x = "__ldg(" + in_ptr(src) + " + row)";
        else if (c.cls[src] != Cls::kRowed) x = at(src, std::vector<std::string>(vals_[src].dims.size(), "0"));
        else throw InternalError("row reduce input not in registers: " + vals_[in].id);
        std::string s = fresh("s");
        ln("const float " + s + " = " + x + ";  // " + vals_[m].id + " (one element)");
        scalar_[m] = s;
      } else if (S == 1) {
        std::string acc = fresh("a");
        ln("float " + acc + " = " + Op + "::init();");
        ln("#pragma unroll");
        open("for (int it = 0; it < " + std::to_string(Li.iters) + "; ++it)");
        ln("#pragma unroll");
        open("for (int u = 0; u < " + std::to_string(Li.vec) + "; ++u)");
        if (Li.guard) open("if ((it * " + std::to_string(NT) + " + t) * " + std::to_string(Li.vec) + " + u < " + std::to_string(Sin) + ")");
        std::string x;
        auto r = reg_.find(in);
        if (r != reg_.end()) x = r->second + "[it * " + std::to_string(Li.vec) + " + u]";
        else if (c.staged[in]) x = "sm" + std::to_string(in) + "[(it * " + std::to_string(NT) + " + t) * " + std::to_string(Li.vec) + " + u]";
        else throw InternalError("row reduce input not in registers: " + vals_[in].id);
        ln(acc + " = " + Op + "::apply(" + acc + ", " + x + ");");
        if (Li.guard) close();
        close();
        close();
        std::string s = fresh("s");
        if (c.cta && NT > 32 && opts_.pp_reduce) {
          ln("const float " + s + " = stitch_dev::row_allreduce_pp<" + std::to_string(NT) + ", " + Op + ">(" + acc + ", red + 64 * rpp);  // " + vals_[m].id);
          ln("rpp ^= 1;");
        } else {
          ln("const float " + s + " = stitch_dev::row_allreduce<" + std::to_string(NT) + ", " + Op + ">(" + acc + ", red);  // " + vals_[m].id);
        }
        scalar_[m] = s;
      } else {
        // partial in-row reduce from the staged input tile
        std::vector<int64_t> ind(vals_[in].dims.begin() + k, vals_[in].dims.end());
        emit_elementwise_loop(m, L, [&](const std::string& it, const std::string& u) {
          std::string lin = "((" + it + ") * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + " + (" + u + ")";
          std::vector<int64_t> od(vals_[m].dims.begin() + k, vals_[m].dims.end());
          std::vector<std::string> oc = decode(lin, od);
          std::string acc = fresh("a");
          ln("float " + acc + " = " + Op + "::init();");
          std::vector<std::string> ic;
          size_t kept = 0;
          int loops = 0;
          for (size_t d = 0; d < ind.size(); ++d) {
            int gd = static_cast<int>(d) + k;
            if (std::find(op.reduce_dims.begin(), op.reduce_dims.end(), gd) != op.reduce_dims.end()) {
              std::string lv = fresh("q");
              open("for (int " + lv + " = 0; " + lv + " < " + std::to_string(ind[d]) + "; ++" + lv + ")");
              ++loops;
              ic.push_back(lv);
            } else {
              ic.push_back(oc[kept++]);
            }
          }
          ln(acc + " = " + Op + "::apply(" + acc + ", sm" + std::to_string(in) + "[" + linear(ic, ind) + "]);");
          for (int i = 0; i < loops; ++i) close();
          return acc;
        });
      }
    } else if (op.type == OpType::kBatchedDot || op.type == OpType::kDot) {
      const int a = vals_[m].operands[0], b = vals_[m].operands[1];
      auto cd = effective_contract_dims(body_, op);
      const int64_t K = vals_[a].dims[cd[0]];
      std::vector<int64_t> od(vals_[m].dims.begin() + k, vals_[m].dims.end());
      std::vector<int64_t> ad(vals_[a].dims.begin() + k, vals_[a].dims.end());
      std::vector<int64_t> bd = op.type == OpType::kBatchedDot
                                    ? std::vector<int64_t>(vals_[b].dims.begin() + k, vals_[b].dims.end())
                                    : vals_[b].dims;
      const int64_t Nn = od.back();
      const bool fast = op.type == OpType::kBatchedDot && L.vec == 4 && Nn % 4 == 0 && !L.guard;
      // Register tile: the L.iters row chunks a thread owns share its
      // column quad, so each k step loads one B quad and one A quad per
      // owned row (k-vectorised) and issues 16 FMAs per B quad.
      const bool tiled = fast && od.size() == 2 && (static_cast<int64_t>(NT) * 4) % Nn == 0 && K % 4 == 0 &&
                         c.staged[a] && c.staged[b];
      std::string r = "r" + std::to_string(m);
      ln("float " + r + "[" + std::to_string(L.elems()) + "];  // " + vals_[m].id + " (gemm stage)");
      if (c.tcp && c.tc_dot[m]) {
        const int j = static_cast<int>(std::find(c.tc_list.begin(), c.tc_list.end(), m) - c.tc_list.begin());
        ln("stitch_dev::tc::accum_to_smem(tmem + (tb * " + std::to_string(ntc) + " + " + std::to_string(j) + ") * 64, tcD);");
        ln("#pragma unroll");
        open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
        ln("const int e4 = (it * " + std::to_string(NT) + " + t) * 4;");
        ln("const float4 q = *reinterpret_cast<const float4*>(tcD + (e4 >> 6) * stitch_dev::tc::kDStride + (e4 & 63));");
        ln(r + "[it * 4 + 0] = q.x; " + r + "[it * 4 + 1] = q.y; " + r + "[it * 4 + 2] = q.z; " + r + "[it * 4 + 3] = q.w;");
        close();
      } else if (!c.tc_dot.empty() && c.tc_dot[m]) {
        // 5th-gen tensor cores: 3xTF32 tcgen05.mma into TMEM, D back through
        // shared memory into this thread's elements of the row tile
        if (std::find(c.tc_direct.begin(), c.tc_direct.end(), m) != c.tc_direct.end())
          ln("stitch_dev::tc::gemm_64x64_tf32x3<" + std::to_string(K) + ", true>(" + in_ptr(a) + " + row * " +
             std::to_string(64 * K) + "LL, " + in_ptr(b) + " + row * " + std::to_string(64 * K) + "LL, tcD, tcs, tmem, tcbar, tcphase);");
        else
          ln("stitch_dev::tc::gemm_64x64_tf32x3<" + std::to_string(K) + ">(sm" + std::to_string(a) + ", sm" + std::to_string(b) +
             ", tcD, tcs, tmem, tcbar, tcphase);");
        ln("#pragma unroll");
        open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
        ln("const int e4 = (it * " + std::to_string(NT) + " + t) * 4;");
        ln("const float4 q = *reinterpret_cast<const float4*>(tcD + (e4 >> 6) * stitch_dev::tc::kDStride + (e4 & 63));");
        ln(r + "[it * 4 + 0] = q.x; " + r + "[it * 4 + 1] = q.y; " + r + "[it * 4 + 2] = q.z; " + r + "[it * 4 + 3] = q.w;");
        close();
      } else if (tiled) {
        const int64_t RS = static_cast<int64_t>(NT) * 4 / Nn;  // rows between a thread's row chunks
        const int I = L.iters;
        open("");
        ln("const int n0 = (4 * t) % " + std::to_string(Nn) + ", m0 = (4 * t) / " + std::to_string(Nn) + ";");
        ln("const float* A = sm" + std::to_string(a) + " + m0 * " + std::to_string(K) + ";");
        ln("const float* B = sm" + std::to_string(b) + " + n0;");
        ln("float acc[" + std::to_string(I * 4) + "];");
        ln("#pragma unroll");
        ln("for (int e = 0; e < " + std::to_string(I * 4) + "; ++e) acc[e] = 0.f;");
        ln("#pragma unroll 2");
        open("for (int kk = 0; kk < " + std::to_string(K) + "; kk += 4)");
        ln("float4 av[" + std::to_string(I) + "];");
        ln("#pragma unroll");
        ln("for (int i = 0; i < " + std::to_string(I) + "; ++i) av[i] = *reinterpret_cast<const float4*>(A + i * " +
           std::to_string(RS * K) + " + kk);");
        for (int j = 0; j < 4; ++j) {
          const char* comp = j == 0 ? "x" : j == 1 ? "y" : j == 2 ? "z" : "w";
          ln("{ const float4 bv = *reinterpret_cast<const float4*>(B + (kk + " + std::to_string(j) + ") * " + std::to_string(Nn) + ");");
          ln("#pragma unroll");
          ln("  for (int i = 0; i < " + std::to_string(I) + "; ++i) { const float s = av[i]." + comp +
             "; acc[i * 4 + 0] = fmaf(s, bv.x, acc[i * 4 + 0]); acc[i * 4 + 1] = fmaf(s, bv.y, acc[i * 4 + 1]); "
             "acc[i * 4 + 2] = fmaf(s, bv.z, acc[i * 4 + 2]); acc[i * 4 + 3] = fmaf(s, bv.w, acc[i * 4 + 3]); } }");
        }
        close();
        ln("#pragma unroll");
        ln("for (int e = 0; e < " + std::to_string(I * 4) + "; ++e) " + r + "[e] = acc[e];");
        close();
      } else if (fast) {
        // Output element chunk (.., m, n0..n0+3) per (it): A scalar x B float4.
        const int rb = static_cast<int>(od.size());
        ln("#pragma unroll");
        open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
        ln("const int lin = (it * " + std::to_string(NT) + " + t) * 4;");
        std::vector<std::string> oc = decode("lin", od);
        ln("const int n0 = (int)" + oc[rb - 1] + ";");
        ln("const int mm = (int)" + oc[rb - 2] + ";");
        std::string bb = "0";
        {
          std::vector<int64_t> bdims(od.begin(), od.end() - 2);
          std::vector<std::string> bcs(oc.begin(), oc.end() - 2);
          bb = linear(bcs, bdims);
        }
        ln("const long long bb = " + bb + ";");
        ln("float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;");
        const int64_t M = od[rb - 2];
        ln("const float* A = sm" + std::to_string(a) + " + bb * " + std::to_string(M * K) + "LL + (long long)mm * " + std::to_string(K) + ";");
        ln("const float* B = sm" + std::to_string(b) + " + bb * " + std::to_string(K * Nn) + "LL + n0;");
        ln("#pragma unroll 8");
        open("for (int kk = 0; kk < " + std::to_string(K) + "; ++kk)");
        ln("const float av = A[kk];");
        ln("const float4 bv = *reinterpret_cast<const float4*>(B + kk * " + std::to_string(Nn) + ");");
        ln("c0 = fmaf(av, bv.x, c0); c1 = fmaf(av, bv.y, c1); c2 = fmaf(av, bv.z, c2); c3 = fmaf(av, bv.w, c3);");
        close();
        ln(r + "[it * 4 + 0] = c0; " + r + "[it * 4 + 1] = c1; " + r + "[it * 4 + 2] = c2; " + r + "[it * 4 + 3] = c3;");
        close();
      } else {
        ln("#pragma unroll");
        open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
        ln("#pragma unroll");
        open("for (int u = 0; u < " + std::to_string(L.vec) + "; ++u)");
        ln("const int lin = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + " + u;");
        ln("float acc = 0.f;");
        if (L.guard) open("if (lin < " + std::to_string(L.S) + ")");
        std::vector<std::string> oc = decode("lin", od);
        std::vector<std::string> ac, bc;
        if (op.type == OpType::kBatchedDot) {
          const int rb = static_cast<int>(od.size());
          for (int d = 0; d < rb - 2; ++d) {
            ac.push_back(oc[d]);
            bc.push_back(oc[d]);
          }
          ac.push_back(oc[rb - 2]);
          ac.push_back("kk");
          bc.push_back("kk");
          bc.push_back(oc[rb - 1]);
        } else {
          int pos = 0;
          for (int d = k; d < static_cast<int>(vals_[a].dims.size()); ++d) ac.push_back(d == cd[0] ? "kk" : oc[pos++]);
          for (int d = 0; d < static_cast<int>(vals_[b].dims.size()); ++d) bc.push_back(d == cd[1] ? "kk" : oc[pos++]);
        }
        open("for (int kk = 0; kk < " + std::to_string(K) + "; ++kk)");
        std::string bval = op.type == OpType::kBatchedDot ? "sm" + std::to_string(b) + "[" + linear(bc, bd) + "]"
                                                            : "__ldg(" + in_ptr(b) + " + " + linear(bc, bd) + ")";
        ln("acc = fmaf(sm" + std::to_string(a) + "[" + linear(ac, ad) + "], " + bval + ", acc);");
        close();
        if (L.guard) close();
        ln(r + "[it * " + std::to_string(L.vec) + " + u] = acc;");
        close();
        close();
      }
      reg_[m] = r;
      int64_t mnk = prod(vals_[m].dims) * K;
      spec_.flops += 2 * mnk;
    }
    // Stage computed values that later ops gather from.
    if (c.staged[m]) stage_value(m, L, S);
  }

  // Cross-row accumulation.
  for (int x : c.cross) {
    const OpNode& op = *vals_[x].node;
    const int in = vals_[x].operands[0];
    const Layout& L = cross_layout[x];
    const std::string Op = op.elem_name == "max" ? "stitch_dev::MaxOp" : "stitch_dev::SumOp";
    bool scalar = static_cast<int>(op.reduce_dims.size()) == static_cast<int>(vals_[in].dims.size());
    std::string src;
    auto r = reg_.find(in);
    ln("#pragma unroll");
    open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
    ln("#pragma unroll");
    open("for (int u = 0; u < " + std::to_string(L.vec) + "; ++u)");
    ln("const int lin = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + " + u;");
    if (r != reg_.end()) src = r->second + "[it * " + std::to_string(L.vec) + " + u]";
    else if (c.staged[in]) src = "sm" + std::to_string(in) + "[lin]";
    else if (scalar_.count(in)) src = scalar_[in];
    else throw InternalError("cross-row reduce input unavailable: " + vals_[in].id);
    std::string tgt = scalar ? "p" + std::to_string(x)
                             : "p" + std::to_string(x) + (c.cross_off.count(x) ? "[lin]" : "[it * " + std::to_string(L.vec) + " + u]");
    ln((L.guard ? "if (lin < " + std::to_string(L.S) + ") " : std::string()) + tgt + " = " + Op + "::apply(" + tgt + ", " + src + ");");
    close();
    close();
  }

  // Row outputs.
  for (int o : c.outputs) {
    if (c.cls[o] != Cls::kRowed) continue;
    const int64_t S = prod(vals_[o].dims, k);
    if (S == 1) {
      // a reduction's row scalar, or element 0 of a one-element row tile
      // (e.g. a [1, K] . [K, 1] dot)
      auto sc = scalar_.find(o);
      const std::string v = sc != scalar_.end() && !sc->second.empty() ? sc->second : reg_[o] + "[0]";
      ln("if (t == 0) " + out_ptr(o) + "[row] = " + v + ";");
      continue;
    }
    const Layout L = layout(S, NT);
    const std::string r = reg_[o];
    ln("#pragma unroll");
    open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
    ln("const int lin = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + ";");
    if (L.guard) open("if (lin < " + std::to_string(S) + ")");
    const std::string dst = out_ptr(o) + " + row * " + std::to_string(S) + "LL + lin";
    if (L.vec == 4)
      ln("stitch_dev::st4(" + dst + ", " + r + "[it * 4], " + r + "[it * 4 + 1], " + r + "[it * 4 + 2], " + r + "[it * 4 + 3]);");
    else
      for (int u = 0; u < L.vec; ++u) ln("(" + dst + ")[" + std::to_string(u) + "] = " + r + "[it * " + std::to_string(L.vec) + " + " + std::to_string(u) + "];");
    if (L.guard) close();
    close();
  }
  memo_.pop_back();
  if (c.tcp) ln("tb ^= 1;");
  if (c.cta && (any_ext_staged || std::any_of(c.staged.begin(), c.staged.end(), [](char s) { return s; }))) ln("__syncthreads();");
  if (early_tma) {
    std::vector<int> rest;
    for (auto& [j, vs] : release_at) rest.insert(rest.end(), vs.begin(), vs.end());
    if (!rest.empty() || !early_expect_done) {
      open("if (t == 0 && row + gstride < " + rhi + ")");
      issue_some(rest, !early_expect_done);
      close();
    }
    release_at.clear();
  }
  {
    // dead intermediates: drop this row's lines from L2 without write-back
    std::vector<int> dead;
    for (int v : inputs_)
      if (n_comps_ == 1 && opts_.discard_inputs.count(vals_[v].id) && c.cls[v] == Cls::kRowed && prod(vals_[v].dims, k) * 4 % 128 == 0)
        dead.push_back(v);
    if (!dead.empty()) {
      if (c.cta)
        ln("__syncthreads();  // every thread is done with this row's inputs");
      else if (NT == 32)
        ln("__syncwarp();  // every lane is done with this row's inputs");
      else
        ln("__syncwarp(((1u << " + std::to_string(NT) + ") - 1u) << ((threadIdx.x & 31) & ~" + std::to_string(NT - 1) +
           "));  // the row group is done with this row's inputs");
      for (int v : dead) {
        const int64_t So = prod(vals_[v].dims, k);
        ln("for (int l = t; l < " + std::to_string(So * 4 / 128) + "; l += " + std::to_string(NT) + ") stitch_dev::discard_l2(" +
           in_ptr(v) + " + row * " + std::to_string(So) + "LL + l * 32);  // " + vals_[v].id + " (dead after this kernel)");
      }
    }
  }
  close();  // row loop
  if (c.tc) ln("stitch_dev::tc::dealloc(tmem, " + std::string(c.tcp ? (c.tc_list.size() > 1 ? "256" : "128") : "64") + ");");

  // Write this CTA's cross-row partials: combine the CTA's row groups first.
  for (int x : c.cross) {
    const OpNode& op = *vals_[x].node;
    const int in = vals_[x].operands[0];
    const Layout& L = cross_layout[x];
    const std::string Op = op.elem_name == "max" ? "stitch_dev::MaxOp" : "stitch_dev::SumOp";
    bool scalar = static_cast<int>(op.reduce_dims.size()) == static_cast<int>(vals_[in].dims.size());
    const int64_t So = scalar ? 1 : L.S;
    const std::string parts = "(ws + " + std::to_string(ws_off_[x]) + "LL)";
    const std::string rank = "(long long)(blockIdx.x - " + lo + ")";
    if (scalar) {
      if (c.cta) {
        ln("{ const float v = stitch_dev::row_allreduce<" + std::to_string(NT) + ", " + Op + ">(p" + std::to_string(x) + ", red);");
        ln("  if (threadIdx.x == 0) " + parts + "[" + rank + "] = v; }");
      } else {
        ln("{ float v = stitch_dev::warp_allreduce<" + Op + ">(p" + std::to_string(x) + ");");
        ln("  __syncthreads(); if (t == 0) smem[wib] = v; __syncthreads();");
        ln("  if (threadIdx.x == 0) { float a = " + Op + "::init(); for (int w = 0; w < wpb; ++w) a = " + Op + "::apply(a, smem[w]); " + parts + "[" + rank + "] = a; }");
        ln("  __syncthreads(); }");
      }
    } else if (c.cta) {
      ln("#pragma unroll");
      open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
      ln("#pragma unroll");
      open("for (int u = 0; u < " + std::to_string(L.vec) + "; ++u)");
      ln("const int lin = (it * " + std::to_string(NT) + " + t) * " + std::to_string(L.vec) + " + u;");
      ln((L.guard ? "if (lin < " + std::to_string(So) + ") " : std::string()) + parts + "[" + rank + " * " + std::to_string(So) + "LL + lin] = p" + std::to_string(x) + "[it * " + std::to_string(L.vec) + " + u];");
      close();
      close();
    } else if (c.cross_off.count(x)) {
      // the warps' partial rows already sit in their slabs: fixed-order CTA sum
      ln("__syncthreads();");
      open("for (int i = threadIdx.x; i < " + std::to_string(So) + "; i += blockDim.x)");
      ln("float a = " + Op + "::init();");
      ln("for (int w = 0; w < wpb; ++w) a = " + Op + "::apply(a, smem[w * " + std::to_string(c.slab_floats + 32) + " + " +
         std::to_string(c.cross_off[x]) + " + i]);");
      ln(parts + "[" + rank + " * " + std::to_string(So) + "LL + i] = a;");
      close();
      ln("__syncthreads();");
    } else {
      // warps -> shared partial rows -> fixed-order CTA sum
      ln("__syncthreads();");
      ln("#pragma unroll");
      open("for (int it = 0; it < " + std::to_string(L.iters) + "; ++it)");
      ln("#pragma unroll");
      open("for (int u = 0; u < " + std::to_string(L.vec) + "; ++u)");
      ln("const int lin = (it * 32 + t) * " + std::to_string(L.vec) + " + u;");
      ln((L.guard ? "if (lin < " + std::to_string(So) + ") " : std::string()) + "smem[wib * " + std::to_string(So) + " + lin] = p" + std::to_string(x) + "[it * " + std::to_string(L.vec) + " + u];");
      close();
      close();
      ln("__syncthreads();");
      open("for (int i = threadIdx.x; i < " + std::to_string(So) + "; i += blockDim.x)");
      ln("float a = " + Op + "::init();");
      ln("for (int w = 0; w < wpb; ++w) a = " + Op + "::apply(a, smem[w * " + std::to_string(So) + " + i]);");
      ln(parts + "[" + rank + " * " + std::to_string(So) + "LL + i] = a;");
      close();
      ln("__syncthreads();");
    }
  }
  close();
}

void Builder::emit_row_finalize(std::vector<Component*>& comps, bool split) {
  bool any = false;
  for (Component* c : comps) any = any || !c->cross.empty();
  if (!any) return;
  if (split) {
    ln("// partials of every CTA of the row kernel are complete (this kernel");
    ln("// runs after it); row_lo = their count");
  } else {
    uses_barrier_ = true;
    ln("stitch_dev::grid_barrier(gsync);");
  }
  ln("// deterministic combine of the per-CTA partials: every (output, column");
  ln("// block) item of every cross output in ONE grid-stride loop, so all CTAs");
  ln("// work at once (not one output after another on So / 32 CTAs)");
  struct Item {
    int x;
    int64_t So;
    int CW;
    int64_t first, count;
  };
  std::vector<Item> items;
  int64_t total = 0;
  for (Component* c : comps)
    for (int x : c->cross) {
      const OpNode& op = *vals_[x].node;
      const int in = vals_[x].operands[0];
      bool scalar = static_cast<int>(op.reduce_dims.size()) == static_cast<int>(vals_[in].dims.size());
      const int64_t So = scalar ? 1 : prod(vals_[in].dims, c->k);
      const int CW = So >= 32 ? 32 : 1;
      const int64_t cnt = (So + CW - 1) / CW;
      items.push_back({x, So, CW, total, cnt});
      total += cnt;
    }
  open("for (long long item = blockIdx.x; item < " + std::to_string(total) + "LL; item += gridDim.x)");
  for (size_t j = 0; j < items.size(); ++j) {
    const Item& it = items[j];
    const int x = it.x;
    const OpNode& op = *vals_[x].node;
    const int64_t So = it.So;
    const int CW = it.CW;
    const std::string Op = op.elem_name == "max" ? "stitch_dev::MaxOp" : "stitch_dev::SumOp";
    // Parallel fixed-order combine: a CTA owns a block of CW columns, its
    // threads split the partial rows (slice s of S), then slice 0 joins
    // the S slice sums in order through shared memory.
    open(std::string(j ? "else " : "") + "if (item < " + std::to_string(it.first + it.count) + "LL)");
    ln("const long long cb = item - " + std::to_string(it.first) + "LL;");
    ln("const int CW = " + std::to_string(CW) + ", S = blockDim.x / CW;");
    ln("const int c = threadIdx.x % CW, s = threadIdx.x / CW;");
    ln("const long long i = cb * CW + c;");
    ln("float a = " + Op + "::init();");
    ln("if (i < " + std::to_string(So) + "LL) a = stitch_dev::combine_strided<" + Op + ">(ws + " +
       std::to_string(ws_off_[x]) + "LL, " + cross_parts_[x] + ", " + std::to_string(So) + "LL, i, s, S);");
    ln("__syncthreads();");
    ln("smem[s * CW + c] = a;");
    ln("__syncthreads();");
    if (CW == 1) {
      // scalar: warp 0 folds the slices (lane l: slices l, l+32, ...) and
      // finishes with a fixed xor-shuffle tree
      open("if (threadIdx.x < 32)");
      ln("float v = " + Op + "::init();");
      ln("for (int j = threadIdx.x; j < S; j += 32) v = " + Op + "::apply(v, smem[j]);");
      ln("v = stitch_dev::warp_allreduce<" + Op + ">(v);");
      open("if (threadIdx.x == 0)");
    } else {
      open("if (s == 0 && i < " + std::to_string(So) + "LL)");
      ln("float v = " + Op + "::init();");
      ln("for (int j = 0; j < S; ++j) v = " + Op + "::apply(v, smem[j * CW + c]);");
    }
    if (vals_[x].output) ln(out_ptr(x) + "[i] = v;");
    if (materialized_.count(x) && !vals_[x].output) ln(materialized_[x] + "[i] = v;");
    close();
    if (CW == 1) close();
    close();
  }
  close();
  bool any_post = false;
  for (Component* c : comps) any_post = any_post || !c->post.empty();
  if (!any_post) return;
  if (split) throw InternalError("split cross finalize with post-reduction ops");
  ln("stitch_dev::grid_barrier(gsync);");
  for (Component* c : comps)
    for (int p : c->post) {
      if (!vals_[p].output) continue;
      open("for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < " + std::to_string(prod(vals_[p].dims)) + "LL; i += (long long)gridDim.x * blockDim.x)");
      memo_.emplace_back();
      ln(out_ptr(p) + "[i] = " + at(p, decode("i", vals_[p].dims)) + ";");
      memo_.pop_back();
      close();
    }
}

// ---------------------------------------------------------------------------
// SECTIONED
// ---------------------------------------------------------------------------

void Builder::emit_sectioned(const std::vector<int>& members) {
  std::vector<int> mat;
  for (int m : members) {
    const Val& v = vals_[m];
    bool need = v.output || v.node->type != OpType::kElementwise;
    for (int c : v.consumers)
      need = need || vals_[c].node->type == OpType::kDot || vals_[c].node->type == OpType::kBatchedDot;
    if (need) mat.push_back(m);
  }
  for (int m : mat)
    if (!vals_[m].output) {
      ws_off_[m] = ws_floats_;
      ws_floats_ += (prod(vals_[m].dims) + 63) / 64 * 64;
    }
  for (size_t s = 0; s < mat.size(); ++s) {
    const int m = mat[s];
    const Val& v = vals_[m];
    const OpNode& op = *v.node;
    const std::string dst = v.output ? out_ptr(m) : "(ws + " + std::to_string(ws_off_[m]) + "LL)";
    if (s > 0) {
      uses_barrier_ = true;
      ln("stitch_dev::grid_barrier(gsync);");
    }
    ln("// section: " + v.id);
    open("for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < " + std::to_string(prod(v.dims)) + "LL; i += (long long)gridDim.x * blockDim.x)");
    memo_.emplace_back();
    std::vector<std::string> oc = decode("i", v.dims);
    if (op.type == OpType::kElementwise) {
      ln(dst + "[i] = " + at(m, oc) + ";");
    } else if (op.type == OpType::kReduce) {
      const int in = v.operands[0];
      const auto& ind = vals_[in].dims;
      const std::string Op = op.elem_name == "max" ? "stitch_dev::MaxOp" : "stitch_dev::SumOp";
      ln("float acc = " + Op + "::init();");
      std::vector<std::string> ic;
      size_t kept = 0;
      int loops = 0;
      for (size_t d = 0; d < ind.size(); ++d) {
        if (std::find(op.reduce_dims.begin(), op.reduce_dims.end(), static_cast<int>(d)) != op.reduce_dims.end()) {
          std::string lv = fresh("q");
          open("for (long long " + lv + " = 0; " + lv + " < " + std::to_string(ind[d]) + "LL; ++" + lv + ")");
          memo_.emplace_back();
          ++loops;
          ic.push_back(lv);
        } else {
          ic.push_back(oc[kept++]);
        }
      }
      ln("acc = " + Op + "::apply(acc, " + at(in, ic) + ");");
      for (int l = 0; l < loops; ++l) {
        memo_.pop_back();
        close();
      }
      ln(dst + "[i] = acc;");
    } else if (op.type == OpType::kDot || op.type == OpType::kBatchedDot) {
      const int a = v.operands[0], b = v.operands[1];
      auto cd = effective_contract_dims(body_, op);
      const int64_t K = vals_[a].dims[cd[0]];
      std::vector<std::string> ac, bc;
      if (op.type == OpType::kBatchedDot) {
        const int r = static_cast<int>(v.dims.size());
        for (int d = 0; d < r - 2; ++d) {
          ac.push_back(oc[d]);
          bc.push_back(oc[d]);
        }
        ac.push_back(oc[r - 2]);
        ac.push_back("kk");
        bc.push_back("kk");
        bc.push_back(oc[r - 1]);
      } else {
        int pos = 0;
        for (int d = 0; d < static_cast<int>(vals_[a].dims.size()); ++d) ac.push_back(d == cd[0] ? "kk" : oc[pos++]);
        for (int d = 0; d < static_cast<int>(vals_[b].dims.size()); ++d) bc.push_back(d == cd[1] ? "kk" : oc[pos++]);
      }
      ln("float acc = 0.f;");
      open("for (long long kk = 0; kk < " + std::to_string(K) + "LL; ++kk)");
      memo_.emplace_back();
      ln("acc = fmaf(" + at(a, ac) + ", " + at(b, bc) + ", acc);");
      memo_.pop_back();
      close();
      ln(dst + "[i] = acc;");
      spec_.flops += 2 * prod(v.dims) * K;
    }
    memo_.pop_back();
    close();
    materialized_[m] = v.output ? out_ptr(m) : "(ws + " + std::to_string(ws_off_[m]) + "LL)";
  }
}


// ---------------------------------------------------------------------------
// BLOCK: block composition of heterogeneous groups (paper Fig. 1)
// ---------------------------------------------------------------------------

int64_t Builder::plan_block(int64_t* G) {
  if (topo_members_.empty() || !opts_.allow_row) return -1;
  const int64_t g0 = vals_[topo_members_.front()].dims.empty() ? -1 : vals_[topo_members_.front()].dims[0];
  if (g0 < 1) return -1;
  auto member = [&](int v) { return vals_[v].member; };
  for (int m : topo_members_) {
    const Val& v = vals_[m];
    const OpNode& op = *v.node;
    if (v.dims.empty() || v.dims[0] != g0) return -1;
    if (op.type == OpType::kElementwise) {
      if (op.elem_name == "broadcast") {
        const int in = v.operands[0];
        if (vals_[in].constant || vals_[in].dims.empty()) continue;
        std::vector<int> mp = broadcast_dim_map(vals_[in].node->shape, op.shape);
        const bool batched = vals_[in].dims[0] == g0 && !mp.empty() && mp[0] == 0;
        if (member(in) && !batched) return -1;  // a computed value's leading index moves
      } else {
        for (int o : v.operands)
          if (!vals_[o].constant && vals_[o].dims != v.dims && member(o)) return -1;
      }
    } else if (op.type == OpType::kReduce) {
      if (std::find(op.reduce_dims.begin(), op.reduce_dims.end(), 0) != op.reduce_dims.end()) return -1;
    } else if (op.type == OpType::kBatchedDot) {
      if (v.dims.size() < 3) return -1;
    } else if (op.type == OpType::kDot) {
      auto cd = effective_contract_dims(body_, op);
      if (cd[0] == 0 || member(v.operands[1])) return -1;
    } else {
      return -1;
    }
  }
  // Shared memory: the planner's Alg. 4 alloc map for this group (requests
  // and post-dominance reuse, cost.cpp shared_planning), per leading index.
  FusionPattern pat;
  for (int m : topo_members_) pat.node_ids.insert(vals_[m].id);
  AllocMap am = shared_planning(body_, pat, canonical_shared_requests(body_, pat));
  std::map<std::string, int> idx;
  for (int m : topo_members_) idx[vals_[m].id] = m;
  int64_t total = 0;
  block_smem_.clear();
  block_reuse_.clear();
  for (const AllocEntry& e : am.entries) {
    auto it = idx.find(e.op_id);
    if (it == idx.end()) continue;  // "<op>__tree" scratch: reductions here run per element
    const int m = it->second;
    const int64_t bytes = (prod(vals_[m].dims, 1) * 4 + 15) / 16 * 16;
    if (e.reused_from && idx.count(*e.reused_from) && block_smem_.count(idx[*e.reused_from]) &&
        block_smem_[idx[*e.reused_from]].second >= bytes) {
      block_smem_[m] = {block_smem_[idx[*e.reused_from]].first, bytes};
      block_reuse_[m] = idx[*e.reused_from];
    } else {
      block_smem_[m] = {total, bytes};
      total += bytes;
    }
  }
  if (total > opts_.max_smem) return -1;
  std::ostringstream note;
  note << "planner alloc total " << am.total << " B, requested " << am.requested() << " B";
  block_alloc_note_ = note.str();
  *G = g0;
  return total;
}


std::string Builder::emit_heavy(int m, const std::vector<std::string>& oc) {
  const Val& v = vals_[m];
  const OpNode& op = *v.node;
  const std::string acc = fresh("acc");
  if (op.type == OpType::kReduce) {
    const int in = v.operands[0];
    const auto& ind = vals_[in].dims;
    const std::string Op = op.elem_name == "max" ? "stitch_dev::MaxOp" : "stitch_dev::SumOp";
    ln("float " + acc + " = " + Op + "::init();  // " + v.id);
    std::vector<std::string> ic;
    size_t kept = 0;
    int loops = 0;
    for (size_t d = 0; d < ind.size(); ++d) {
      if (std::find(op.reduce_dims.begin(), op.reduce_dims.end(), static_cast<int>(d)) != op.reduce_dims.end()) {
        std::string lv = fresh("q");
        open("for (long long " + lv + " = 0; " + lv + " < " + std::to_string(ind[d]) + "LL; ++" + lv + ")");
        memo_.emplace_back();
        ++loops;
        ic.push_back(lv);
      } else {
        ic.push_back(oc[kept++]);
      }
    }
    ln(acc + " = " + Op + "::apply(" + acc + ", " + at(in, ic) + ");");
    for (int l = 0; l < loops; ++l) {
      memo_.pop_back();
      close();
    }
    return acc;
  }
  const int a = v.operands[0], b = v.operands[1];
  auto cd = effective_contract_dims(body_, op);
  const int64_t K = vals_[a].dims[cd[0]];
  std::vector<std::string> ac, bc;
  const std::string kk = fresh("k");
  if (op.type == OpType::kBatchedDot) {
    const int r = static_cast<int>(v.dims.size());
    for (int d = 0; d < r - 2; ++d) {
      ac.push_back(oc[d]);
      bc.push_back(oc[d]);
    }
    ac.push_back(oc[r - 2]);
    ac.push_back(kk);
    bc.push_back(kk);
    bc.push_back(oc[r - 1]);
  } else {
    int pos = 0;
    for (int d = 0; d < static_cast<int>(vals_[a].dims.size()); ++d) ac.push_back(d == cd[0] ? kk : oc[pos++]);
    for (int d = 0; d < static_cast<int>(vals_[b].dims.size()); ++d) bc.push_back(d == cd[1] ? kk : oc[pos++]);
  }
  ln("float " + acc + " = 0.f;  // " + v.id);
  open("for (long long " + kk + " = 0; " + kk + " < " + std::to_string(K) + "LL; ++" + kk + ")");
  memo_.emplace_back();
  ln(acc + " = fmaf(" + at(a, ac) + ", " + at(b, bc) + ", " + acc + ");");
  memo_.pop_back();
  close();
  return acc;
}

void Builder::emit_block(const std::vector<int>& members, int64_t G) {
  // materialised values: outputs, reductions, dots, dot operands, and the
  // planner's shared-memory values; everything else is recomputed inline
  // (a reduction or dot with a single elementwise consumer over its own index
  // space is computed inline in that consumer's section, as the reference's
  // sketches do -- e.g. fig1's dot_2 inside divide)
  std::vector<int> mat;
  for (int m : members) {
    const Val& v = vals_[m];
    bool need = v.output || block_smem_.count(m);
    if (v.node->type != OpType::kElementwise) {
      int in_group = 0;
      bool simple = true;
      for (int c : v.consumers) {
        if (!vals_[c].member) continue;
        ++in_group;
        simple = simple && vals_[c].node->type == OpType::kElementwise && vals_[c].node->elem_name != "broadcast" &&
                 vals_[c].dims == v.dims;
      }
      need = need || in_group != 1 || !simple;
    }
    for (int c : v.consumers)
      need = need || vals_[c].node->type == OpType::kDot || vals_[c].node->type == OpType::kBatchedDot;
    if (need) mat.push_back(m);
  }
  inline_heavy_ = true;
  // per-CTA workspace for materialised values neither in shared memory nor outputs
  int64_t wsb = 0;
  std::map<int, int64_t> wso;
  for (int m : mat)
    if (!vals_[m].output && !block_smem_.count(m)) {
      wso[m] = wsb;
      wsb += (prod(vals_[m].dims, 1) + 63) / 64 * 64;
    }
  const int64_t ws_base = ws_floats_;
  ws_floats_ += wsb * static_cast<int64_t>(opts_.num_sms) * 8;  // one slice per resident CTA (grid <= 8 x SMs)
  ln("// block composition: one CTA per leading index g < " + std::to_string(G) + "; " + block_alloc_note_);
  for (auto& [m, ob] : block_smem_)
    ln("float* sh" + std::to_string(m) + " = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(smem) + " +
       std::to_string(ob.first) + ");  // " + vals_[m].id + (block_reuse_.count(m) ? " (reuses " + vals_[block_reuse_[m]].id + ")" : ""));
  ln("float* wsb = ws + " + std::to_string(ws_base) + "LL + (long long)blockIdx.x * " + std::to_string(wsb) + "LL;");
  ln("(void)wsb;");
  std::set<int> done;
  row_hook_ = [&](int v, const std::vector<std::string>& coords) -> std::string {
    if (!done.count(v)) return "";
    std::vector<std::string> inner(coords.begin() + 1, coords.end());
    std::vector<int64_t> idims(vals_[v].dims.begin() + 1, vals_[v].dims.end());
    const std::string lin = idims.empty() ? std::string("0") : linear(inner, idims);
    if (block_smem_.count(v)) return "sh" + std::to_string(v) + "[" + lin + "]";
    if (wso.count(v)) return "wsb[" + std::to_string(wso[v]) + "LL + " + lin + "]";
    return "__ldcg(" + out_ptr(v) + " + " + linear(coords, vals_[v].dims) + ")";
  };
  open("for (long long g = blockIdx.x; g < " + std::to_string(G) + "LL; g += gridDim.x)");
  for (size_t s = 0; s < mat.size(); ++s) {
    const int m = mat[s];
    const Val& v = vals_[m];
    const OpNode& op = *v.node;
    const int64_t inner = prod(v.dims, 1);
    std::vector<int64_t> idims(v.dims.begin() + 1, v.dims.end());
    // A value that reuses another's shared block is computed into registers
    // first, then written after a barrier (its section may still read the
    // block it overwrites); one register slot per element of the thread.
    const bool two_phase = block_reuse_.count(m) > 0;
    const int64_t per_thread = (inner + 255) / 256;
    ln("// section " + std::to_string(s) + ": " + v.id + (block_smem_.count(m) ? " -> shared" : v.output ? " -> output" : " -> workspace"));
    if (two_phase) ln("float st" + std::to_string(m) + "[" + std::to_string(per_thread) + "];");
    open("for (long long i = threadIdx.x, slot = 0; i < " + std::to_string(inner) + "LL; i += blockDim.x, ++slot)");
    ln("(void)slot;");
    memo_.emplace_back();
    std::vector<std::string> oc = {"g"};
    for (const std::string& c : decode("i", idims)) oc.push_back(c);
    if (idims.empty()) oc.resize(1);
    std::string val;
    if (op.type == OpType::kElementwise) {
      val = at(m, oc);
    } else {
      val = emit_heavy(m, oc);
    }
    if (two_phase) {
      ln("st" + std::to_string(m) + "[slot] = " + val + ";");
    } else {
      if (block_smem_.count(m)) ln("sh" + std::to_string(m) + "[i] = " + val + ";");
      else if (wso.count(m)) ln("wsb[" + std::to_string(wso[m]) + "LL + i] = " + val + ";");
      if (v.output) ln(out_ptr(m) + "[g * " + std::to_string(inner) + "LL + i] = " + val + ";");
    }
    memo_.pop_back();
    close();
    if (two_phase) {
      ln("__syncthreads();  // every reader of the block " + vals_[m].id + " reuses is done");
      open("for (long long i = threadIdx.x, slot = 0; i < " + std::to_string(inner) + "LL; i += blockDim.x, ++slot)");
      ln("sh" + std::to_string(m) + "[i] = st" + std::to_string(m) + "[slot];");
      if (v.output) ln(out_ptr(m) + "[g * " + std::to_string(inner) + "LL + i] = st" + std::to_string(m) + "[slot];");
      close();
    }
    ln("__syncthreads();");
    done.insert(m);
  }
  close();
  row_hook_ = nullptr;
  inline_heavy_ = false;
}

// ---------------------------------------------------------------------------
// driver
// ---------------------------------------------------------------------------


// ---------------------------------------------------------------------------
// GWS: warp-specialised tcgen05 batched-GEMM stage + generated tail
// (device template stitch_dev::gws::run). Eligible fused groups: exactly two
// batched dots over [S][64][64] whose four operands are kernel inputs of
// that shape, every other member elementwise over [S][64][64] (broadcasts of
// constants or inputs included), every output [S][64][64].
// ---------------------------------------------------------------------------

namespace {
constexpr int kGwsThreads = 32 * (2 + 8 + 4 * 2);  // stitch_dev::gws::kThreads (STITCH_GWS_EPQ = 2)
constexpr int kGwsElems = 16;                      // stitch_dev::gws::kElems
constexpr int kGwsSmem = 3 * 65536 + 32768 + 8 * (2 * 3 + 9) + 16 + 1024;  // stitch_dev::gws::Smem::kAlloc
}  // namespace

bool Builder::build_gws() {
  if (!opts_.gws || !opts_.allow_row) return false;
  std::vector<int> dots;
  int64_t S = -1;
  auto tile = [&](int v) {
    const auto& d = vals_[v].dims;
    return d.size() == 3 && d[1] == 64 && d[2] == 64 && (S < 0 || d[0] == S);
  };
  for (int m : topo_members_) {
    const OpNode& op = *vals_[m].node;
    if (op.type == OpType::kBatchedDot) {
      if (S < 0 && vals_[m].dims.size() == 3) S = vals_[m].dims[0];
      if (!tile(m)) return false;
      const auto& cd = op.contract_dims;
      if (!(cd[0] < 0 || (cd[0] == 2 && cd[1] == 1))) return false;
      for (int o : vals_[m].operands)
        if (!vals_[o].external || !tile(o)) return false;
      dots.push_back(m);
    }
  }
  if (dots.size() != 2 || S < 1 || S > (1LL << 31) - 1) return false;
  for (int m : topo_members_) {
    const OpNode& op = *vals_[m].node;
    if (op.type == OpType::kBatchedDot) continue;
    if (op.type != OpType::kElementwise || !tile(m)) return false;
  }
  for (int o : outputs_)
    if (!tile(o)) return false;
  const int A0 = vals_[dots[0]].operands[0], B0 = vals_[dots[0]].operands[1];
  const int A1 = vals_[dots[1]].operands[0], B1 = vals_[dots[1]].operands[1];
  if (A0 == A1) return false;  // the stacked A' needs two tiles

  // values the tail reads: dot results, staged A tiles, other full-tile
  // inputs (prefetched one sample ahead), anything else through at()
  std::set<int> tail_ext;  // full-tile external inputs read by the tail
  int staged = 0;
  for (int m : topo_members_) {
    if (vals_[m].node->type == OpType::kBatchedDot) continue;
    const bool bc = vals_[m].node->elem_name == "broadcast";
    for (int o : vals_[m].operands) {
      if (!vals_[o].external || bc || !tile(o)) continue;
      if (o == A0) staged |= 1;
      else if (o == A1) staged |= 2;
      else tail_ext.insert(o);
    }
  }
  std::map<int, std::string> argname;
  for (int v : inputs_) argname[v] = in_ptr(v);

  // ---- the tail functor
  std::ostringstream& o = out_;
  indent_ = 0;
  ln("struct Tail {");
  ++indent_;
  for (int v : inputs_) ln("const float* __restrict__ " + in_ptr(v) + ";");
  for (int v : outputs_) ln("float* __restrict__ " + out_ptr(v) + ";");
  open("struct Regs");
  for (int v : tail_ext) ln("float r" + std::to_string(v) + "[" + std::to_string(kGwsElems) + "];");
  if (tail_ext.empty()) ln("int unused;");
  close(";");
  open("__device__ __forceinline__ void load(long long s, int q, int lane, int e, Regs& rg) const");
  if (!tail_ext.empty()) {
    ln("#pragma unroll");
    open("for (int i = 0; i < " + std::to_string(kGwsElems) + "; i += 2)");
    ln("const long long off = (s * 64 + stitch_dev::gws::elem_row(q, lane, i)) * 64 + stitch_dev::gws::elem_col(e, lane, i);");
    for (int v : tail_ext) {
      ln("{ const float2 t = __ldg(reinterpret_cast<const float2*>(" + in_ptr(v) + " + off)); rg.r" + std::to_string(v) +
         "[i] = t.x; rg.r" + std::to_string(v) + "[i + 1] = t.y; }");
    }
    close();
  } else {
    ln("(void)s; (void)q; (void)lane; (void)e; (void)rg;");
  }
  close();
  open("__device__ __forceinline__ void operator()(long long s, int q, int lane, int e, const float* d0, const float* d1, "
       "const float* a0, const float* a1, const Regs& rg) const");
  ln("(void)a0; (void)a1; (void)rg;");
  ln("#pragma unroll");
  open("for (int i = 0; i < " + std::to_string(kGwsElems) + "; i += 2)");
  ln("const int row = stitch_dev::gws::elem_row(q, lane, i), col = stitch_dev::gws::elem_col(e, lane, i);");
  ln("const long long off = (s * 64 + row) * 64 + col;");
  for (int v : outputs_) ln("float o" + std::to_string(v) + "[2];");
  ln("#pragma unroll");
  open("for (int x = 0; x < 2; ++x)");
  ln("const int ii = i + x, cc = col + x;");
  ln("(void)ii; (void)cc;");
  nr_div_ = true;
  row_hook_ = [&](int v, const std::vector<std::string>& coords) -> std::string {
    (void)coords;
    if (v == dots[0]) return "d0[ii]";
    if (v == dots[1]) return "d1[ii]";
    if (v == A0 && (staged & 1)) return "a0[ii]";
    if (v == A1 && (staged & 2)) return "a1[ii]";
    if (tail_ext.count(v)) return "rg.r" + std::to_string(v) + "[ii]";
    return "";
  };
  memo_.emplace_back();
  for (int v : outputs_) {
    std::string e = at(v, {"s", "row", "cc"});
    ln("o" + std::to_string(v) + "[x] = " + e + ";");
  }
  memo_.pop_back();
  row_hook_ = nullptr;
  nr_div_ = opts_.nr_divide;
  close();
  for (int v : outputs_) {
    const std::string val = "make_float2(o" + std::to_string(v) + "[0], o" + std::to_string(v) + "[1])";
    if (opts_.gws_stream_stores)
      ln("__stcs(reinterpret_cast<float2*>(" + out_ptr(v) + " + off), " + val + ");  // evict-first");
    else
      ln("*reinterpret_cast<float2*>(" + out_ptr(v) + " + off) = " + val + ";");
  }
  close();
  close();
  --indent_;
  ln("};");
  std::string tail_src = o.str();
  out_.str("");

  // ---- signature: standard pointers, then the four tensor maps by value
  std::vector<std::string> params;
  auto input_index = [&](int v) {
    return static_cast<int>(std::find(inputs_.begin(), inputs_.end(), v) - inputs_.begin());
  };
  for (int v : inputs_) {
    params.push_back("const float* __restrict__ " + in_ptr(v));
    spec_.inputs.push_back(vals_[v].id);
    spec_.algo_bytes += vals_[v].node->shape.byte_count();
  }
  for (int v : outputs_) {
    params.push_back("float* __restrict__ " + out_ptr(v));
    spec_.outputs.push_back(vals_[v].id);
    spec_.algo_bytes += vals_[v].node->shape.byte_count();
  }
  params.push_back("float* __restrict__ ws");
  params.push_back("unsigned int* __restrict__ gsync");
  params.push_back("const long long row_lo");
  params.push_back("const long long row_hi");
  const int ops[4] = {A0, A1, B0, B1};
  for (int k = 0; k < 4; ++k) {
    params.push_back("const __grid_constant__ stitch_dev::gws::TmaDesc tm" + std::to_string(k));
    KernelSpec::TmaParam tp;
    tp.input = input_index(ops[k]);
    tp.box_rows = k < 2 ? 16 : 64;
    tp.swizzle = k < 2 ? 0 : 1;
    tp.samples = S;
    spec_.tma.push_back(tp);
  }
  std::ostringstream head;
  head << "// stitched kernel for fused op '" << name_ << "': " << topo_members_.size()
       << " ops, scheme gws (warp-specialised tcgen05 3xTF32 batched-GEMM stage, " << S << " samples of 64x64)\n";
  for (int m : topo_members_) {
    head << "//   " << vals_[m].id << " = " << to_string(vals_[m].node->type);
    if (!vals_[m].node->elem_name.empty()) head << ":" << vals_[m].node->elem_name;
    head << "(";
    for (size_t i = 0; i < vals_[m].operands.size(); ++i) head << (i ? ", " : "") << vals_[vals_[m].operands[i]].id;
    head << ")\n";
  }
  head << tail_src;
  head << "static_assert(stitch_dev::gws::kThreads == " << kGwsThreads << " && stitch_dev::gws::kElems == " << kGwsElems
       << " && stitch_dev::gws::Smem::kAlloc == " << kGwsSmem << ", \"codegen / device gws constants\");\n";
  head << "extern \"C\" __global__ void __launch_bounds__(" << kGwsThreads << ", 1) " << name_ << "(" << join(params, ", ")
       << ") {\n";
  head << "  extern __shared__ __align__(1024) unsigned char smem[];\n";
  head << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  if (opts_.pdl_early_trigger) head << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  if (opts_.trace) head << "  stitch_dev::TraceScope stitch_trace_(gsync);\n";
  head << "  (void)ws; (void)gsync; (void)row_lo; (void)row_hi;\n";
  head << "  const Tail tail{";
  {
    std::vector<std::string> init;
    for (int v : inputs_) init.push_back(in_ptr(v));
    for (int v : outputs_) init.push_back(out_ptr(v));
    head << join(init, ", ");
  }
  head << "};\n";
  head << "  stitch_dev::gws::run<" << staged << ">(&tm0, &tm1, &tm2, &tm3, 0, " << S << "LL, smem, tail);\n";
  head << "}\n";
  spec_.source = head.str();
  spec_.scheme = "gws(S=" + std::to_string(S) + ",tcgen05)";
  spec_.composition = {"thread", "block", "tensor"};
  spec_.block = kGwsThreads;
  spec_.smem_bytes = kGwsSmem;
  spec_.max_grid = static_cast<int>(std::min<int64_t>(S, 1 << 20));
  spec_.flops = 2LL * 2 * 64 * 64 * 64 * S;
  spec_.workspace_floats = 0;
  spec_.sync_words = 0;
  return true;
}

bool Builder::build_gemm() {
  if (!opts_.gemm || topo_members_.size() != 1) return false;
  const int m = topo_members_[0];
  const Val& v = vals_[m];
  const OpNode& op = *v.node;
  if (op.type != OpType::kDot && op.type != OpType::kBatchedDot) return false;
  if (!v.output || outputs_.size() != 1 || outputs_[0] != m) return false;
  const int a = v.operands[0], b = v.operands[1];
  if (a == b || !vals_[a].external || !vals_[b].external) return false;
  const auto& ad = vals_[a].dims;
  const auto& bd = vals_[b].dims;
  int64_t M, N, K, batch = 1, sam, sak, sab = 0, sbk, sbn, sbb = 0;
  if (op.type == OpType::kDot) {
    if (ad.size() != 2 || bd.size() != 2) return false;
    auto cd = effective_contract_dims(body_, op);
    K = ad[cd[0]];
    M = ad[1 - cd[0]];
    N = bd[1 - cd[1]];
    if (bd[cd[1]] != K) return false;
    sam = cd[0] == 1 ? K : 1;
    sak = cd[0] == 1 ? 1 : M;
    sbk = cd[1] == 0 ? N : 1;
    sbn = cd[1] == 0 ? 1 : K;
  } else {
    const auto cd = effective_contract_dims(body_, op);
    const size_t r = v.dims.size();
    if (r < 3 || ad.size() != r || bd.size() != r) return false;
    if (!(cd[0] == static_cast<int>(r) - 1 && cd[1] == static_cast<int>(r) - 2)) return false;
    for (size_t d = 0; d + 2 < r; ++d) {
      if (ad[d] != v.dims[d] || bd[d] != v.dims[d]) return false;
      batch *= v.dims[d];
    }
    M = ad[r - 2];
    K = ad[r - 1];
    N = bd[r - 1];
    if (bd[r - 2] != K) return false;
    sam = K, sak = 1, sab = M * K, sbk = N, sbn = 1, sbb = K * N;
  }
  if (v.dims.size() < 2 || v.dims[v.dims.size() - 2] != M || v.dims.back() != N || M < 1 || N < 1 || K < 1)
    return false;
  // small matrices waste most of a 128 x 128 tile: the row scheme is faster
  // there (4096 batched 64^3 dots: 64 vs 125 us, scripts/gemm_perf.py)
  if (M * N < 128 * 64) return false;
  const int64_t tiles = batch * ((M + 127) / 128) * ((N + 127) / 128);
  auto L = [](int64_t x) { return std::to_string(x) + "LL"; };
  std::vector<std::string> params;
  for (int x : inputs_) {
    params.push_back("const float* __restrict__ " + in_ptr(x));
    spec_.inputs.push_back(vals_[x].id);
    spec_.algo_bytes += vals_[x].node->shape.byte_count();
  }
  params.push_back("float* __restrict__ " + out_ptr(m));
  spec_.outputs.push_back(v.id);
  spec_.algo_bytes += v.node->shape.byte_count();
  params.push_back("float* __restrict__ ws");
  params.push_back("unsigned int* __restrict__ gsync");
  params.push_back("const long long row_lo");
  params.push_back("const long long row_hi");
  std::ostringstream h;
  h << "// kernel for op '" << name_ << "': " << v.id << " = " << to_string(op.type) << "(" << vals_[a].id << ", "
    << vals_[b].id << "), scheme gemm (tiled fp32, " << batch << " x [" << M << " x " << K << "] . [" << K << " x "
    << N << "])\n";
  h << "extern \"C\" __global__ void __launch_bounds__(256) " << name_ << "(" << join(params, ", ") << ") {\n";
  h << "  extern __shared__ __align__(128) float smem[];\n";
  h << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  if (opts_.pdl_early_trigger) h << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  if (opts_.trace) h << "  stitch_dev::TraceScope stitch_trace_(gsync);\n";
  h << "  (void)ws; (void)gsync; (void)row_lo; (void)row_hi;\n";
  h << "  stitch_dev::gemm::run<" << L(M) << ", " << L(N) << ", " << L(K) << ", " << L(batch) << ", " << L(sam) << ", "
    << L(sak) << ", " << L(sab) << ", " << L(sbk) << ", " << L(sbn) << ", " << L(sbb) << ">(" << in_ptr(a) << ", "
    << in_ptr(b) << ", " << out_ptr(m) << ", smem);\n";
  h << "}\n";
  spec_.source = h.str();
  spec_.scheme = "gemm(" + std::to_string(batch) + "x" + std::to_string(M) + "x" + std::to_string(N) + "x" +
                 std::to_string(K) + ")";
  spec_.composition = {"thread", "block"};
  spec_.block = 256;
  spec_.smem_bytes = 2 * 8 * (128 + 128) * 4;
  spec_.max_grid = static_cast<int>(std::min<int64_t>(tiles, 1 << 20));
  spec_.flops = 2 * batch * M * N * K;
  spec_.workspace_floats = 0;
  spec_.sync_words = 0;
  return true;
}

KernelSpec Builder::build() {
  collect();
  spec_.name = name_;
  nr_div_ = opts_.nr_divide;
  if (build_gws()) return spec_;
  if (build_gemm()) return spec_;
  std::vector<Component> comps = components();
  bool sectioned = false;
  for (Component& c : comps) {
    // COLRED only for a kernel's sole component: packed beside a row group,
    // the streaming cross-row scheme overlaps better (encoder 96 vs 133 us)
    if (comps.size() == 1 && plan_colred(c)) continue;
    if (!(opts_.flat_elementwise && all_elementwise(c)) && plan_row(c)) continue;
    if (all_elementwise(c)) {
      c.scheme = "flat";
      int64_t total = 0;
      for (int o : c.outputs) total = std::max(total, prod(vals_[o].dims));
      c.max_grid = std::max<int64_t>(1, (total / 4 + 255) / 256);
      continue;
    }
    c.scheme = "sectioned";
    sectioned = true;
  }

  // Block size: the widest CTA-mode row component, else 256.
  // (A kernel made only of CTA-row components may use a narrower CTA, e.g.
  // 192 threads x 4 columns for 768-wide LayerNorm-backward rows; COLRED
  // needs >= 128 threads; everything else adapts to blockDim.)
  int block = 0;
  bool all_cta = true;
  for (const Component& c : comps) {
    if (c.scheme == "row" && c.cta) block = std::max(block, c.NT);
    else all_cta = false;
    if (c.scheme == "colred") block = std::max(block, 256);
  }
  if (!all_cta || block == 0) block = std::max(block, 256);
  for (Component& c : comps)
    if (c.scheme == "row" && c.cta) {
      if (c.NT != block && c.tc) block = std::max(block, 256);
      c.NT = block;
    }

  std::ostringstream head;
  std::string body_src;
  int64_t smem_floats = 0;
  int64_t block_G = 0, block_smem = -1;
  if (sectioned && opts_.block_compose) block_smem = plan_block(&block_G);
  if (sectioned && block_smem >= 0) {
    spec_.scheme = "block(G=" + std::to_string(block_G) + ",smem=" + std::to_string(block_smem) + ")";
    spec_.composition = {"thread", "block"};
    memo_.emplace_back();
    indent_ = 1;
    emit_block(topo_members_, block_G);
    memo_.pop_back();
    body_src = out_.str();
    block = 256;
    spec_.max_grid = static_cast<int>(std::min<int64_t>(block_G, static_cast<int64_t>(opts_.num_sms) * 8));
    smem_floats = (block_smem + 3) / 4;
  } else if (sectioned) {
    spec_.scheme = "sectioned";
    spec_.cooperative = true;
    spec_.composition = {"block"};
    memo_.emplace_back();
    indent_ = 1;
    emit_sectioned(topo_members_);
    memo_.pop_back();
    body_src = out_.str();
    int64_t maxe = 1;
    for (int m : topo_members_) maxe = std::max(maxe, prod(vals_[m].dims));
    spec_.max_grid = static_cast<int>(std::min<int64_t>((maxe + block - 1) / block, opts_.num_sms * 8));
  } else {
    // Workspace for cross-row partials: one row of partials per CTA.
    // (resident CTAs: <= 2048 threads and <= 32 CTAs per SM; warp-row
    // kernels may be launched with blocks down to 64 threads)
    bool flex_rows = true;
    for (const Component& c : comps) flex_rows = flex_rows && ((c.scheme == "row" && !c.cta) || c.scheme == "flat");
    const int min_block = flex_rows ? 64 : block;
    const int64_t max_ctas = static_cast<int64_t>(opts_.num_sms) * std::min(32, 2048 / std::max(32, min_block));
    spec_.max_partials = static_cast<int>(max_ctas);
    bool coop = false;
    for (Component& c : comps)
      for (int x : c.cross) {
        coop = true;
        const OpNode& op = *vals_[x].node;
        const int in = vals_[x].operands[0];
        bool scalar = static_cast<int>(op.reduce_dims.size()) == static_cast<int>(vals_[in].dims.size());
        const int64_t So = scalar ? 1 : prod(vals_[in].dims, c.k);
        ws_off_[x] = ws_floats_;
        ws_floats_ += max_ctas * ((So + 63) / 64 * 64);
        if (!c.post.empty()) {
          // post-reduction ops read the finished reduce after the second
          // grid barrier: from its output buffer, or a workspace row
          if (vals_[x].output) {
            materialized_[x] = out_ptr(x);
          } else {
            int64_t off = ws_floats_;
            ws_floats_ += (So + 63) / 64 * 64;
            materialized_[x] = "(ws + " + std::to_string(off) + "LL)";
          }
        }
      }
    for (Component& c : comps)
      if (c.scheme == "colred") {
        const int x = c.cr_m;
        ws_off_[x] = ws_floats_;
        ws_floats_ += c.cr_nch * ((c.cr_C + 63) / 64 * 64);
      }
    spec_.cooperative = coop;
    // CTA ranges per component, proportional to weight.
    int64_t total_w = 0;
    for (const Component& c : comps) total_w += c.weight;
    std::vector<std::string> lo(comps.size()), n(comps.size());
    indent_ = 1;
    if (comps.size() > 1 && opts_.pack_sequential) {
      // Kernel packing by composition: every CTA runs every component over
      // its share of that component's rows, one after the other, so the
      // load balances by construction (no idle CTA ranges at the barrier).
      ln("// kernel packing: " + std::to_string(comps.size()) + " independent components, each over the whole grid");
      for (size_t i = 0; i < comps.size(); ++i) {
        lo[i] = "0";
        n[i] = "gridDim.x";
      }
      spec_.composition.insert("packing");
    } else if (comps.size() > 1) {
      int64_t cum = 0;
      ln("// kernel packing: " + std::to_string(comps.size()) + " independent components on disjoint CTA ranges");
      std::vector<std::string> bounds;
      for (size_t i = 0; i <= comps.size(); ++i) {
        // b_i = max(i, floor(G * cum_i / W)), clipped so every component keeps a CTA
        std::string b = "cb" + std::to_string(i);
        if (i == 0) ln("const int cb0 = 0;");
        else if (i == comps.size()) ln("const int " + b + " = gridDim.x;");
        else
          ln("const int " + b + " = max(cb" + std::to_string(i - 1) + " + 1, min((int)gridDim.x - " + std::to_string(comps.size() - i) +
             ", (int)(((long long)gridDim.x * " + std::to_string(cum) + "LL) / " + std::to_string(total_w) + "LL)));");
        if (i < comps.size()) cum += comps[i].weight;
      }
      for (size_t i = 0; i < comps.size(); ++i) {
        lo[i] = "cb" + std::to_string(i);
        n[i] = "(cb" + std::to_string(i + 1) + " - cb" + std::to_string(i) + ")";
      }
      spec_.composition.insert("packing");
    } else {
      lo[0] = "0";
      n[0] = "gridDim.x";
    }
    std::vector<Component*> rowc;
    std::string scheme;
    n_comps_ = comps.size();
    chunked_ = comps.size() == 1 && comps[0].scheme == "row" && comps[0].cross.empty() && comps[0].post.empty() &&
               comps[0].free_out.empty();
    if (comps.size() == 1 && comps[0].scheme == "row") spec_.rows = comps[0].R;
    if (comps.size() > 1)
      for (const Component& c : comps)
        if (c.scheme == "row") spec_.rows = std::max(spec_.rows, c.R);
    if (chunked_) {
      spec_.chunkable = true;
      spec_.rows_per_cta = comps[0].cta ? 1 : block / comps[0].NT;
    }
    for (size_t i = 0; i < comps.size(); ++i) {
      Component& c = comps[i];
      for (int x : c.cross) cross_parts_[x] = "(int)" + n[i];
      const bool ranged = comps.size() > 1 && !opts_.pack_sequential;
      if (ranged) open("if ((int)blockIdx.x >= " + lo[i] + " && (int)blockIdx.x < cb" + std::to_string(i + 1) + ")");
      memo_.emplace_back();
      if (c.scheme == "row") {
        emit_row(c, lo[i], n[i], "");
        rowc.push_back(&c);
        smem_floats = std::max<int64_t>(smem_floats, c.cta ? c.slab_floats + 32 + 8 + (opts_.pp_reduce ? 64 : 0) +
                                                                 (c.tc ? (c.tcp ? static_cast<int64_t>(c.tc_list.size()) : 1) *
                                                                                 int64_t{4} * 64 * c.tc_k + 64 * 68
                                                                       : 0)
                                                          : (c.slab_floats + 32) * (block / c.NT));
        if (c.tc) spec_.composition.insert("tensor");
        if (!c.cta)
          for (int x : c.cross) {
            const int in = vals_[x].operands[0];
            smem_floats = std::max(smem_floats, (block / 32) * prod(vals_[in].dims, c.k));
          }
        spec_.composition.insert("thread");
        bool has_red = false, has_block = c.cta;
        for (int m : c.members) has_red = has_red || vals_[m].node->type == OpType::kReduce;
        if (has_red && !c.cta) spec_.composition.insert("warp");
        if (has_block) spec_.composition.insert("block");
        std::ostringstream s;
        s << (c.cta ? "row_cta" : "row_warp") << "(k=" << c.k << ",rows=" << c.R << ",nt=" << c.NT
          << (c.tma ? (c.dbuf ? ",tma2" : ",tma") : "") << (c.tc ? ",tcgen05" : "") << (c.cross.empty() ? "" : ",cross") << ")";
        scheme += (scheme.empty() ? "" : "+") + s.str();
        spec_.max_grid = std::max<int>(spec_.max_grid, static_cast<int>(std::min<int64_t>(c.max_grid, 1 << 20)));
      } else if (c.scheme == "colred") {
        emit_colred(c, lo[i], n[i]);
        spec_.composition.insert("block");
        smem_floats = std::max<int64_t>(smem_floats, opts_.colred_cp_async ? kColredStageOff + 256 * 4 * kColredStageSlots : kColredStageOff);
        if (c.cr_cluster) smem_floats = std::max<int64_t>(smem_floats, kColredStageOff + c.cr_w);  // the cluster partial row
        std::ostringstream cs;
        cs << "colred(" << c.cr_ncb << "x" << c.cr_nch << ",w" << c.cr_w << (c.cr_cluster ? ",cluster" : "") << ")";
        if (c.cr_cluster) spec_.cluster = c.cr_cluster;
        scheme += (scheme.empty() ? "" : "+") + cs.str();
        spec_.max_grid = std::max<int>(spec_.max_grid, static_cast<int>(std::min<int64_t>(c.max_grid, 1 << 20)));
      } else {
        emit_flat(c, lo[i], n[i]);
        spec_.composition.insert("thread");
        scheme += (scheme.empty() ? "" : "+") + std::string("flat");
        spec_.max_grid = std::max<int>(spec_.max_grid, static_cast<int>(std::min<int64_t>(c.max_grid, 1 << 20)));
      }
      memo_.pop_back();
      if (ranged) close();
    }
    bool split = opts_.split_cross && comps.size() == 1 && comps[0].scheme == "row" && !comps[0].cross.empty() &&
                 comps[0].post.empty();
    if (split)
      for (int x : comps[0].cross) split = split && vals_[x].output;
    if (split) {
      // the fold goes to its own kernel (KernelSpec::fin_*), emitted into a
      // separate buffer; the partial count arrives as row_lo
      for (int x : comps[0].cross) cross_parts_[x] = "(int)row_lo";
      std::ostringstream fin;
      std::swap(out_, fin);
      const int saved_indent = indent_;
      indent_ = 1;
      memo_.emplace_back();
      open("");
      emit_row_finalize(rowc, true);
      close();
      memo_.pop_back();
      indent_ = saved_indent;
      std::swap(out_, fin);
      fin_body_ = fin.str();
      for (int x : comps[0].cross) spec_.fin_outputs.push_back(vals_[x].id);
      spec_.fin_smem_bytes = 256 * 4 + 16;
      int64_t items = 0;
      for (int x : comps[0].cross) {
        const int in = vals_[x].operands[0];
        const bool scalar = static_cast<int>(vals_[x].node->reduce_dims.size()) == static_cast<int>(vals_[in].dims.size());
        const int64_t So = scalar ? 1 : prod(vals_[in].dims, comps[0].k);
        items += (So + (So >= 32 ? 31 : 0)) / (So >= 32 ? 32 : 1);
      }
      spec_.fin_max_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(items, 1 << 20)));
      spec_.cooperative = false;  // no grid barrier left in the row kernel
    } else {
      for (Component* c : rowc)
        if (!c->cross.empty()) smem_floats = std::max<int64_t>(smem_floats, block);
      memo_.emplace_back();
      emit_row_finalize(rowc, false);
      memo_.pop_back();
    }
    spec_.max_grid = std::max<int>(spec_.max_grid, static_cast<int>(comps.size()));
    if (comps.size() > 1 && !opts_.pack_sequential) spec_.min_grid = static_cast<int>(comps.size());
    spec_.scheme = scheme;
    body_src = out_.str();
  }

  // Signature.
  std::vector<std::string> params;
  for (int v : inputs_) {
    params.push_back("const float* __restrict__ " + in_ptr(v));
    spec_.inputs.push_back(vals_[v].id);
    spec_.algo_bytes += vals_[v].node->shape.byte_count();
  }
  for (int o : outputs_) {
    params.push_back("float* __restrict__ " + out_ptr(o));
    spec_.outputs.push_back(vals_[o].id);
    spec_.algo_bytes += vals_[o].node->shape.byte_count();
  }
  params.push_back("float* __restrict__ ws");
  params.push_back("unsigned int* __restrict__ gsync");
  params.push_back("const long long row_lo");
  params.push_back("const long long row_hi");
  head << "// stitched kernel for fused op '" << name_ << "': " << topo_members_.size() << " ops, scheme "
       << spec_.scheme << "\n";
  for (int m : topo_members_) {
    head << "//   " << vals_[m].id << " = " << to_string(vals_[m].node->type);
    if (!vals_[m].node->elem_name.empty()) head << ":" << vals_[m].node->elem_name;
    head << "(";
    for (size_t i = 0; i < vals_[m].operands.size(); ++i) head << (i ? ", " : "") << vals_[vals_[m].operands[i]].id;
    head << ")\n";
  }
  head << "extern \"C\" __global__ void __launch_bounds__(" << block
       << (opts_.min_ctas_per_sm > 0 ? ", " + std::to_string(opts_.min_ctas_per_sm) : std::string()) << ") " << name_ << "("
       << join(params, ", ") << ") {\n";
  head << "  extern __shared__ __align__(128) float smem[];\n";
  // Programmatic dependent launch: this grid may be scheduled while the
  // previous kernel drains; wait for it (and its memory) before touching any
  // global data, and let the next kernel get scheduled right away (our grids
  // are one resident wave, so its CTAs only take slots this one leaves free).
  head << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
  if (opts_.pdl_early_trigger) head << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
  if (opts_.trace) head << "  stitch_dev::TraceScope stitch_trace_(gsync);\n";
  head << "  (void)ws; (void)gsync; (void)smem; (void)row_lo; (void)row_hi;\n";
  spec_.source = head.str() + body_src + "}\n";
  if (!fin_body_.empty()) {
    spec_.fin_name = name_ + "_fold";
    std::ostringstream fh;
    fh << "// column-reduction fold of fused op '" << name_ << "': fixed-order combine of the per-CTA partials "
       << name_ << " wrote to the workspace\n";
    fh << "extern \"C\" __global__ void __launch_bounds__(1024) " << spec_.fin_name << "(" << join(params, ", ") << ") {\n";
    fh << "  extern __shared__ __align__(128) float smem[];\n";
    fh << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
    if (opts_.pdl_early_trigger) fh << "  asm volatile(\"griddepcontrol.launch_dependents;\");\n";
    if (opts_.trace) fh << "  stitch_dev::TraceScope stitch_trace_(gsync);\n";
    fh << "  (void)ws; (void)gsync; (void)smem; (void)row_lo; (void)row_hi;\n";
    spec_.fin_source = fh.str() + fin_body_ + "}\n";
  }
  spec_.block = block;
  spec_.smem_bytes = static_cast<int>(smem_floats * 4 + (smem_floats ? 16 : 0));
  bool all_warp = !sectioned;
  for (const Component& c : comps) all_warp = all_warp && ((c.scheme == "row" && !c.cta) || c.scheme == "flat");
  // (colred components assume blockDim >= 128 and size smem for 8 warps)
  if (all_warp) {
    // every shared-memory term of a warp-row kernel is per warp
    spec_.flex_block = true;
    spec_.row_threads = comps.size() == 1 && comps[0].scheme == "row" ? comps[0].NT : 32;
    spec_.smem_per_warp = static_cast<int>((smem_floats * 4 + (block / 32) - 1) / (block / 32));
  }
  spec_.workspace_floats = ws_floats_;
  spec_.sync_words = std::max((spec_.cooperative || uses_barrier_) ? 2 : 0, colred_sync_ > 2 ? colred_sync_ : 0);
  if (uses_barrier_) spec_.cooperative = true;
  if (spec_.max_grid < 1) spec_.max_grid = 1;
  if (spec_.cluster > 0 && spec_.max_grid % spec_.cluster != 0)
    throw InternalError("stitched executor: cluster kernel " + name_ + " grid is not a multiple of its cluster");
  return spec_;
}

}  // namespace

KernelSpec generate_kernel(const Graph& body, const std::string& name, const std::map<std::string, double>& constants,
                           const CodegenOptions& opts) {
  Builder b(body, name, constants, opts);
  return b.build();
}

}  // namespace exec
}  // namespace stitch
