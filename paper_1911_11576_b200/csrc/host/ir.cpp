// Graph IR implementation. Semantics follow the reference's graph module
// (proj/src/graph.cpp): validation rules and their order, the lexicographic
// Kahn sort (graph.cpp:515), the contraction DFS whose witness feeds cycle
// elimination (graph.cpp:574) -- the witness must match node-for-node, so the
// vertex and adjacency orders below are the reference's.
#include "ir.hpp"

#include <algorithm>
#include <fstream>
#include <functional>
#include <queue>
#include <sstream>

namespace stitch {

std::string to_string(DType dt) {
  switch (dt.kind) {
    case DTypeKind::kF16: return "f16";
    case DTypeKind::kI32: return "i32";
    default: return "f32";
  }
}

DType dtype_from_string(const std::string& s) {
  if (s == "f32") return DType::f32();
  if (s == "f16") return DType::f16();
  if (s == "i32") return DType::i32();
  throw ParseError("unknown dtype: " + s);
}

int64_t Shape::element_count() const {
  int64_t n = 1;
  for (int64_t d : dims) n *= d;
  return n;
}

namespace {

struct KindName {
  OpType t;
  const char* name;
};
constexpr KindName kKinds[] = {
    {OpType::kParameter, "parameter"}, {OpType::kConstant, "constant"},
    {OpType::kElementwise, "elementwise"}, {OpType::kReduce, "reduce"},
    {OpType::kDot, "dot"}, {OpType::kBatchedDot, "batched_dot"},
    {OpType::kTuple, "tuple"}, {OpType::kGetElement, "get_element"},
    {OpType::kFused, "fused"},
};

OpType op_type_from(const std::string& s) {
  for (const auto& k : kKinds)
    if (s == k.name) return k.t;
  throw ParseError("unknown op kind: " + s);
}

// Arity by elementwise function (reference graph.cpp:82-94).
int elementwise_arity(const std::string& f) {
  static const std::set<std::string> unary = {"log", "exp", "negate", "rsqrt", "broadcast"};
  static const std::set<std::string> binary = {"add", "subtract", "multiply", "divide",
                                               "maximum", "minimum", "compare"};
  if (unary.count(f)) return 1;
  if (binary.count(f)) return 2;
  if (f == "select") return 3;
  return -1;
}

}  // namespace

std::string to_string(OpType t) {
  for (const auto& k : kKinds)
    if (k.t == t) return k.name;
  return "parameter";
}

std::string to_string(ReduceKind k) {
  return k == ReduceKind::kRow ? "row" : k == ReduceKind::kColumn ? "column" : "scalar";
}

const OpNode* Graph::find(const std::string& id) const {
  auto it = index_.find(id);
  return it == index_.end() ? nullptr : &nodes[it->second];
}

int Graph::index_of(const std::string& id) const {
  auto it = index_.find(id);
  return it == index_.end() ? -1 : it->second;
}

const OpNode& Graph::at(const std::string& id) const {
  const OpNode* n = find(id);
  if (!n) throw GraphError("no such node: " + id);
  return *n;
}

void Graph::add(OpNode node) {
  if (index_.count(node.id)) throw GraphError("duplicate node id: " + node.id);
  index_.emplace(node.id, static_cast<int>(nodes.size()));
  nodes.push_back(std::move(node));
}

bool is_fusible(const OpNode& op) {
  return op.type == OpType::kElementwise || op.type == OpType::kReduce ||
         op.type == OpType::kDot || op.type == OpType::kBatchedDot;
}

bool is_kernel_op(const OpNode& op) { return is_fusible(op) || op.type == OpType::kFused; }

ReduceKind reduce_kind(const Graph& g, const OpNode& op) {
  const int rank = g.at(op.operands.at(0)).shape.rank();
  const int k = static_cast<int>(op.reduce_dims.size());
  if (k == rank) return ReduceKind::kScalar;
  for (int i = 0; i < k; ++i)
    if (op.reduce_dims[i] != rank - k + i) return ReduceKind::kColumn;
  return ReduceKind::kRow;
}

std::array<int, 2> effective_contract_dims(const Graph& g, const OpNode& op) {
  if (op.contract_dims[0] >= 0) return op.contract_dims;
  const Shape& lhs = g.at(op.operands.at(0)).shape;
  const Shape& rhs = g.at(op.operands.at(1)).shape;
  if (op.type == OpType::kBatchedDot) return {lhs.rank() - 1, lhs.rank() - 2};
  return {lhs.rank() - 1, std::max(0, rhs.rank() - 2)};
}

int64_t dot_flops(const Graph& g, const OpNode& op) {
  // Reference graph.cpp:141 reads contract_dims[0] as stored.
  const Shape& lhs = g.at(op.operands.at(0)).shape;
  return 2 * op.shape.element_count() * lhs.dims.at(op.contract_dims[0]);
}

std::vector<int> broadcast_dim_map(const Shape& in, const Shape& out) {
  std::vector<int> map(in.rank(), -1);
  int o = out.rank() - 1;
  for (int i = in.rank() - 1; i >= 0; --i) {
    while (o >= 0 && out.dims[o] != in.dims[i]) --o;
    if (o < 0) return {};
    map[i] = o--;
  }
  return map;
}

// ---------------------------------------------------------------------------
// JSON <-> Graph
// ---------------------------------------------------------------------------

namespace {

Shape shape_from(const json::Value& j) {
  if (!j.has("dims") || !j.at("dims").is_array()) throw ParseError("shape requires a dims array");
  Shape s;
  for (const auto& d : j.at("dims").items()) s.dims.push_back(d.as_int());
  s.dtype = dtype_from_string(j.has("dtype") ? j.at("dtype").as_string() : "f32");
  return s;
}

json::Value shape_to(const Shape& s) {
  json::Value j = json::Value::object();
  j.set("dims", json::Value::array_of(s.dims));
  j.set("dtype", to_string(s.dtype));
  return j;
}

OpNode node_from(const json::Value& j) {
  OpNode n;
  if (!j.has("id")) throw ParseError("node missing id");
  n.id = j.at("id").as_string();
  if (!j.has("kind")) throw ParseError("node " + n.id + " missing kind");
  n.type = op_type_from(j.at("kind").as_string());
  if (j.has("name")) n.elem_name = j.at("name").as_string();
  if (j.has("operands"))
    for (const auto& o : j.at("operands").items()) n.operands.push_back(o.as_string());
  if (!j.has("shape")) throw ParseError("node " + n.id + " missing shape");
  n.shape = shape_from(j.at("shape"));
  if (j.has("reduce_dims"))
    for (const auto& d : j.at("reduce_dims").items()) n.reduce_dims.push_back(static_cast<int>(d.as_int()));
  if (j.has("contract_dims")) {
    const auto& cd = j.at("contract_dims");
    if (!cd.is_array() || cd.size() != 2)
      throw ParseError("node " + n.id + ": contract_dims must be [lhs,rhs]");
    n.contract_dims = {static_cast<int>(cd[0].as_int()), static_cast<int>(cd[1].as_int())};
  }
  if (j.has("index")) n.tuple_index = static_cast<int>(j.at("index").as_int());
  if (j.has("category")) n.fused_category = j.at("category").as_string();
  if (j.has("value") && j.at("value").is_number()) n.value = j.at("value").as_real();
  if (j.has("body")) n.body = std::make_shared<const Graph>(graph_from_json(j.at("body")));
  return n;
}

json::Value node_to(const OpNode& n) {
  json::Value j = json::Value::object();
  j.set("id", n.id);
  j.set("kind", to_string(n.type));
  if (!n.elem_name.empty()) j.set("name", n.elem_name);
  if (!n.operands.empty()) j.set("operands", json::Value::array_of(n.operands));
  j.set("shape", shape_to(n.shape));
  if (!n.reduce_dims.empty()) j.set("reduce_dims", json::Value::array_of(n.reduce_dims));
  if (n.contract_dims[0] >= 0) {
    json::Value cd = json::Value::array();
    cd.push(n.contract_dims[0]);
    cd.push(n.contract_dims[1]);
    j.set("contract_dims", cd);
  }
  if (n.tuple_index >= 0) j.set("index", n.tuple_index);
  if (!n.fused_category.empty()) j.set("category", n.fused_category);
  if (n.value) j.set("value", *n.value);
  if (n.body) j.set("body", graph_to_json(*n.body));
  return j;
}

}  // namespace

Graph graph_from_json(const json::Value& j) {
  if (!j.has("nodes") || !j.at("nodes").is_array()) throw ParseError("graph requires a nodes array");
  Graph g;
  for (const auto& nj : j.at("nodes").items()) {
    OpNode n = node_from(nj);
    if (g.contains(n.id)) throw ParseError("duplicate node id: " + n.id);
    g.add(std::move(n));
  }
  if (j.has("outputs"))
    for (const auto& o : j.at("outputs").items()) g.outputs.push_back(o.as_string());
  return g;
}

json::Value graph_to_json(const Graph& g) {
  json::Value j = json::Value::object();
  json::Value nodes = json::Value::array();
  for (const OpNode& n : g.nodes) nodes.push(node_to(n));
  j.set("nodes", nodes);
  j.set("outputs", json::Value::array_of(g.outputs));
  return j;
}

Graph parse_graph(const std::string& text) {
  json::Value j;
  try {
    j = json::parse(text);
  } catch (const json::Error& e) {
    throw ParseError(e.what());
  }
  Graph g;
  try {
    g = graph_from_json(j);
  } catch (const json::Error& e) {
    throw ParseError(e.what());
  }
  std::vector<Diagnostic> errors;
  for (const Diagnostic& d : validate(g))
    if (!d.warning) errors.push_back(d);
  if (!errors.empty()) throw ValidationError(format_diagnostics(errors));
  return g;
}

Graph load_graph(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open graph file: " + path);
  std::stringstream buf;
  buf << in.rdbuf();
  return parse_graph(buf.str());
}

std::string print_graph(const Graph& g) { return graph_to_json(g).dump(2) + "\n"; }

std::string format_diagnostics(const std::vector<Diagnostic>& diags) {
  std::string out;
  for (const Diagnostic& d : diags)
    out += std::string(d.warning ? "warning" : "error") + " [" + d.rule + "] " + d.node_id + ": " +
           d.message + "\n";
  return out;
}

// ---------------------------------------------------------------------------
// validation (reference graph.cpp:246-470)
// ---------------------------------------------------------------------------

namespace {

void shape_rules(const Graph& g, const OpNode& n, std::vector<Diagnostic>& out) {
  auto bad = [&](const std::string& m) { out.push_back({n.id, "shape", m, false}); };
  auto opnd = [&](size_t i) -> const Shape& { return g.at(n.operands[i]).shape; };
  switch (n.type) {
    case OpType::kElementwise: {
      if (n.elem_name == "broadcast") {
        const Shape& in = opnd(0);
        if (in.rank() > 0 && broadcast_dim_map(in, n.shape).empty())
          bad("broadcast input dims are not a subsequence of output dims");
        if (in.dtype != n.shape.dtype) bad("broadcast dtype mismatch");
        return;
      }
      for (size_t i = 0; i < n.operands.size(); ++i) {
        const Shape& s = opnd(i);
        if (s.dims != n.shape.dims) bad("operand " + n.operands[i] + " dims differ from output dims");
        bool free_dtype = n.elem_name == "compare" || (n.elem_name == "select" && i == 0);
        if (!free_dtype && s.dtype != n.shape.dtype)
          bad("operand " + n.operands[i] + " dtype differs from output");
      }
      return;
    }
    case OpType::kReduce: {
      const Shape& in = opnd(0);
      if (n.reduce_dims.empty()) return bad("reduce requires a nonempty reduce_dims list");
      for (size_t i = 0; i < n.reduce_dims.size(); ++i) {
        int d = n.reduce_dims[i];
        if (d < 0 || d >= in.rank()) return bad("reduce dim out of range");
        if (i > 0 && d <= n.reduce_dims[i - 1]) return bad("reduce_dims must be strictly increasing");
      }
      std::vector<int64_t> kept;
      for (int d = 0; d < in.rank(); ++d)
        if (std::find(n.reduce_dims.begin(), n.reduce_dims.end(), d) == n.reduce_dims.end())
          kept.push_back(in.dims[d]);
      if (kept != n.shape.dims) bad("output dims inconsistent with reduce_dims");
      if (in.dtype != n.shape.dtype) bad("reduce dtype mismatch");
      return;
    }
    case OpType::kDot: {
      const Shape& a = opnd(0);
      const Shape& b = opnd(1);
      std::array<int, 2> cd = n.contract_dims[0] >= 0
                                  ? n.contract_dims
                                  : std::array<int, 2>{a.rank() - 1, std::max(0, b.rank() - 2)};
      if (cd[0] >= a.rank() || cd[1] >= b.rank()) return bad("contract dim out of range");
      if (a.dims[cd[0]] != b.dims[cd[1]]) return bad("contracted extents differ");
      std::vector<int64_t> expect;
      for (int d = 0; d < a.rank(); ++d)
        if (d != cd[0]) expect.push_back(a.dims[d]);
      for (int d = 0; d < b.rank(); ++d)
        if (d != cd[1]) expect.push_back(b.dims[d]);
      if (expect != n.shape.dims) bad("output dims inconsistent with dot");
      return;
    }
    case OpType::kBatchedDot: {
      const Shape& a = opnd(0);
      const Shape& b = opnd(1);
      if (a.rank() != b.rank() || a.rank() < 3) return bad("batched_dot operands must share rank >= 3");
      const int r = a.rank();
      std::array<int, 2> cd = n.contract_dims[0] >= 0 ? n.contract_dims : std::array<int, 2>{r - 1, r - 2};
      if (cd[0] != r - 1 || cd[1] != r - 2) return bad("batched_dot contraction must be [rank-1, rank-2]");
      for (int d = 0; d < r - 2; ++d)
        if (a.dims[d] != b.dims[d]) bad("batch dims differ");
      if (a.dims[r - 1] != b.dims[r - 2]) return bad("contracted extents differ");
      std::vector<int64_t> expect(a.dims.begin(), a.dims.end() - 1);
      expect.push_back(b.dims[r - 1]);
      if (expect != n.shape.dims) bad("output dims inconsistent with batched_dot");
      return;
    }
    case OpType::kGetElement: {
      const OpNode& src = g.at(n.operands[0]);
      if (src.type == OpType::kTuple) {
        if (n.tuple_index < 0 || n.tuple_index >= static_cast<int>(src.operands.size()))
          bad("get_element index out of range");
      } else if (src.type == OpType::kFused) {
        if (!src.body) return;
        const OpNode* tup = nullptr;
        for (const auto& bn : src.body->nodes)
          if (bn.type == OpType::kTuple) tup = &bn;
        if (!tup || n.tuple_index < 0 || n.tuple_index >= static_cast<int>(tup->operands.size()))
          bad("get_element index out of range for fused body");
        else if (src.body->at(tup->operands[n.tuple_index]).shape != n.shape)
          bad("get_element shape differs from fused body element");
      } else {
        bad("get_element operand must be a tuple or fused op");
      }
      return;
    }
    case OpType::kFused: {
      if (!n.body) return bad("fused op requires a body graph");
      int params = 0;
      for (const auto& bn : n.body->nodes) params += bn.type == OpType::kParameter;
      if (params != static_cast<int>(n.operands.size()))
        bad("fused operand count differs from body parameter count");
      for (const Diagnostic& d : validate(*n.body))
        if (!d.warning) out.push_back({n.id, "fused-body", d.node_id + ": " + d.message, false});
      return;
    }
    default:
      return;
  }
}

}  // namespace

std::vector<Diagnostic> validate(const Graph& g) {
  std::vector<Diagnostic> out;
  for (const OpNode& n : g.nodes) {
    for (int64_t d : n.shape.dims)
      if (d < 1) out.push_back({n.id, "shape", "dims must be positive", false});
    int arity = -1;
    switch (n.type) {
      case OpType::kParameter:
      case OpType::kConstant: arity = 0; break;
      case OpType::kElementwise:
        arity = elementwise_arity(n.elem_name);
        if (arity < 0) {
          out.push_back({n.id, "kind", "unknown elementwise name: " + n.elem_name, false});
          continue;
        }
        break;
      case OpType::kReduce:
      case OpType::kGetElement: arity = 1; break;
      case OpType::kDot:
      case OpType::kBatchedDot: arity = 2; break;
      case OpType::kTuple:
      case OpType::kFused:
        if (n.operands.empty()) {
          out.push_back({n.id, "arity", "requires at least one operand", false});
          continue;
        }
        break;
    }
    if (arity >= 0 && static_cast<int>(n.operands.size()) != arity) {
      out.push_back({n.id, "arity",
                     "expected " + std::to_string(arity) + " operands, got " + std::to_string(n.operands.size()),
                     false});
      continue;
    }
    bool resolved = true;
    for (const std::string& o : n.operands)
      if (!g.contains(o)) {
        out.push_back({n.id, "operand", "unresolved operand id: " + o, false});
        resolved = false;
      }
    if (resolved) shape_rules(g, n, out);
  }
  for (const std::string& o : g.outputs)
    if (!g.contains(o)) out.push_back({o, "output", "unresolved output id", false});
  bool structural = std::none_of(out.begin(), out.end(), [](const Diagnostic& d) {
    return d.rule == "operand" || d.rule == "output";
  });
  if (!structural) return out;
  try {
    topological_sort(g);
  } catch (const CycleError& e) {
    out.push_back({"", "cycle", e.what(), false});
  }
  if (!g.outputs.empty()) {
    std::set<std::string> live = live_nodes(g);
    for (const OpNode& n : g.nodes)
      if (!live.count(n.id)) out.push_back({n.id, "dead", "unreachable from graph outputs", true});
  }
  return out;
}

std::vector<std::string> topological_sort(const Graph& g) {
  const int n = static_cast<int>(g.nodes.size());
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<int>> succ(n);
  for (int i = 0; i < n; ++i)
    for (const std::string& o : g.nodes[i].operands) {
      int s = g.index_of(o);
      if (s < 0) throw GraphError("unresolved operand: " + o);
      succ[s].push_back(i);
      ++indeg[i];
    }
  // Ready set ordered by id (byte-wise), as the reference's min-heap.
  auto later = [&](int a, int b) { return g.nodes[a].id > g.nodes[b].id; };
  std::priority_queue<int, std::vector<int>, decltype(later)> ready(later);
  for (int i = 0; i < n; ++i)
    if (indeg[i] == 0) ready.push(i);
  std::vector<std::string> order;
  order.reserve(n);
  while (!ready.empty()) {
    int v = ready.top();
    ready.pop();
    order.push_back(g.nodes[v].id);
    for (int s : succ[v])
      if (--indeg[s] == 0) ready.push(s);
  }
  if (static_cast<int>(order.size()) != n) {
    std::string msg = "cycle detected involving:";
    for (int i = 0; i < n; ++i)
      if (indeg[i] > 0) msg += " " + g.nodes[i].id;
    throw CycleError(msg);
  }
  return order;
}

std::unordered_map<std::string, std::vector<std::string>> consumer_map(const Graph& g) {
  std::unordered_map<std::string, std::vector<std::string>> c;
  for (const OpNode& n : g.nodes)
    for (const std::string& o : n.operands) c[o].push_back(n.id);
  return c;
}

std::set<std::string> live_nodes(const Graph& g) {
  std::set<std::string> live;
  if (g.outputs.empty()) {
    for (const OpNode& n : g.nodes) live.insert(n.id);
    return live;
  }
  std::vector<std::string> stack(g.outputs.begin(), g.outputs.end());
  while (!stack.empty()) {
    std::string id = std::move(stack.back());
    stack.pop_back();
    const OpNode* n = g.find(id);
    if (!n || !live.insert(id).second) continue;
    for (const std::string& o : n->operands) stack.push_back(o);
  }
  return live;
}

// ---------------------------------------------------------------------------
// contraction (reference graph.cpp:574-702)
// ---------------------------------------------------------------------------

ContractResult contract_plan(const Graph& g, const std::vector<FusionPattern>& plan) {
  const int n = static_cast<int>(g.nodes.size());
  std::vector<int> owner(n, -1);
  for (size_t i = 0; i < plan.size(); ++i)
    for (const std::string& id : plan[i].node_ids) {
      int v = g.index_of(id);
      if (v < 0) throw GraphError("pattern references unknown node: " + id);
      if (owner[v] >= 0) throw GraphError("patterns overlap on node " + id);
      owner[v] = static_cast<int>(i);
    }

  // Vertex numbering: plain nodes keep their index; each distinct pattern
  // label "__pattern_<id>" gets one super vertex n + k (patterns sharing a
  // pattern_id share a vertex, as the reference keys vertices by label).
  std::vector<std::string> super_label;
  std::vector<int> pvert(plan.size());
  for (size_t i = 0; i < plan.size(); ++i) {
    std::string l = "__pattern_" + std::to_string(plan[i].pattern_id >= 0 ? plan[i].pattern_id
                                                                           : static_cast<int>(i));
    auto it = std::find(super_label.begin(), super_label.end(), l);
    pvert[i] = n + static_cast<int>(it - super_label.begin());
    if (it == super_label.end()) super_label.push_back(l);
  }
  auto vtx = [&](int node) {
    const int o = owner[node];
    return o < 0 ? node : pvert.at(static_cast<size_t>(o));
  };
  auto label = [&](int v) { return v < n ? g.nodes[v].id : super_label[v - n]; };
  const int nv = n + static_cast<int>(super_label.size());
  std::vector<int> order;  // vertices by first appearance in node order
  std::vector<char> seen(nv, 0);
  for (int i = 0; i < n; ++i) {
    int v = vtx(i);
    if (!seen[v]) {
      seen[v] = 1;
      order.push_back(v);
    }
  }
  std::vector<std::vector<int>> adj(nv);
  for (int i = 0; i < n; ++i) {
    int dst = vtx(i);
    for (const std::string& o : g.nodes[i].operands) {
      int src = vtx(g.index_of(o));
      if (src != dst) adj[src].push_back(dst);
    }
  }

  // Iterative DFS keeping the gray path; the first back edge yields the witness.
  std::vector<char> color(nv, 0);
  std::vector<int> path;
  std::vector<std::pair<int, size_t>> stack;
  std::optional<std::vector<int>> cycle;
  for (int root : order) {
    if (color[root]) continue;
    color[root] = 1;
    path.push_back(root);
    stack.push_back({root, 0});
    while (!stack.empty() && !cycle) {
      auto& [v, next_edge] = stack.back();
      if (next_edge < adj[v].size()) {
        int w = adj[v][next_edge++];
        if (color[w] == 1) {
          cycle = std::vector<int>(std::find(path.begin(), path.end(), w), path.end());
        } else if (color[w] == 0) {
          color[w] = 1;
          path.push_back(w);
          stack.push_back({w, 0});
        }
      } else {
        color[v] = 2;
        path.pop_back();
        stack.pop_back();
      }
    }
    if (cycle) break;
  }

  ContractResult result;
  if (cycle) {
    CycleWitness w;
    for (int v : *cycle) {
      std::string l = label(v);
      if (l.rfind("__pattern_", 0) == 0)
        w.pattern_ids.push_back(std::stoi(l.substr(10)));
      else
        w.node_ids.push_back(l);
    }
    result.cycle = std::move(w);
    return result;
  }

  Graph out;
  std::fill(seen.begin(), seen.end(), 0);
  for (int i = 0; i < n; ++i) {
    int v = vtx(i);
    if (seen[v]) continue;
    seen[v] = 1;
    if (v == i) {
      OpNode copy = g.nodes[i];
      std::vector<std::string> ops;
      for (const std::string& o : copy.operands) {
        std::string r = label(vtx(g.index_of(o)));
        if (std::find(ops.begin(), ops.end(), r) == ops.end()) ops.push_back(r);
      }
      copy.operands = std::move(ops);
      out.add(std::move(copy));
    } else {
      const int pi = owner[i];
      OpNode super;
      super.id = label(v);
      super.type = OpType::kFused;
      for (int m = 0; m < n; ++m) {
        if (owner[m] != pi) continue;
        for (const std::string& o : g.nodes[m].operands) {
          int ov = vtx(g.index_of(o));
          if (ov == v) continue;
          std::string r = label(ov);
          if (std::find(super.operands.begin(), super.operands.end(), r) == super.operands.end())
            super.operands.push_back(r);
        }
      }
      super.shape = g.nodes[i].shape;
      out.add(std::move(super));
    }
  }
  for (const std::string& o : g.outputs) out.outputs.push_back(label(vtx(g.index_of(o))));
  result.graph = std::move(out);
  return result;
}

bool pattern_is_connected(const Graph& g, const FusionPattern& p) {
  if (p.node_ids.empty()) return false;
  auto consumers = consumer_map(g);
  std::set<std::string> seen;
  std::vector<std::string> stack{*p.node_ids.begin()};
  while (!stack.empty()) {
    std::string id = stack.back();
    stack.pop_back();
    if (!seen.insert(id).second) continue;
    for (const std::string& o : g.at(id).operands)
      if (p.node_ids.count(o) && !seen.count(o)) stack.push_back(o);
    for (const std::string& c : consumers[id])
      if (p.node_ids.count(c) && !seen.count(c)) stack.push_back(c);
  }
  return seen.size() == p.node_ids.size();
}

// ---------------------------------------------------------------------------
// GraphIndex
// ---------------------------------------------------------------------------

GraphIndex::GraphIndex(const Graph& graph) : g(graph), n(static_cast<int>(graph.nodes.size())) {
  node_of.resize(n);
  for (int i = 0; i < n; ++i) node_of[i] = i;
  std::sort(node_of.begin(), node_of.end(), [&](int a, int b) { return g.nodes[a].id < g.nodes[b].id; });
  rank_of.resize(n);
  for (int r = 0; r < n; ++r) rank_of[node_of[r]] = r;
  operands.resize(n);
  consumers.resize(n);
  for (int i = 0; i < n; ++i)
    for (const std::string& o : g.nodes[i].operands) {
      int s = g.index_of(o);
      if (s < 0) throw GraphError("unresolved operand: " + o);
      operands[i].push_back(s);
      consumers[s].push_back(i);
    }
  topo.reserve(n);
  for (const std::string& id : topological_sort(g)) topo.push_back(g.index_of(id));
  topo_pos.resize(n);
  for (int i = 0; i < n; ++i) topo_pos[topo[i]] = i;
  live.assign(n, 0);
  fusible.assign(n, 0);
  is_output.assign(n, 0);
  for (const std::string& id : live_nodes(g)) live[g.index_of(id)] = 1;
  for (int i = 0; i < n; ++i) fusible[i] = is_fusible(g.nodes[i]);
  for (const std::string& o : g.outputs) {
    int v = g.index_of(o);
    if (v >= 0) is_output[v] = 1;
  }
}

std::vector<int> GraphIndex::ranks_of(const std::set<std::string>& ids) const {
  std::vector<int> r;
  r.reserve(ids.size());
  for (const std::string& id : ids) r.push_back(rank_of[g.index_of(id)]);
  return r;  // already sorted: set order == rank order
}

std::set<std::string> GraphIndex::ids_of(const std::vector<int>& ranks) const {
  std::set<std::string> s;
  for (int r : ranks) s.insert(s.end(), g.nodes[node_of[r]].id);
  return s;
}

}  // namespace stitch
