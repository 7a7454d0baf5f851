"""Synthetic computation graphs for the benchmark configurations.

Each builder returns a graph in the reference's JSON graph format
(SPEC "graph-ir" External Interfaces; parsed by reference
proj/src/graph.cpp:node_from_json) using only op kinds and elementwise names
the reference validates (graph.cpp:82-94), so the reference planner can plan
every workload and the fusion groups can be compared bit for bit.

Two extensions ride along as extra JSON keys that the reference parser
ignores (graph.cpp:178-205 reads only known keys):
  * constants carry a scalar "value" (the reference has no constant data);
  * a reduce may carry "name": "max" (the reference's emitter only sums,
    emitter.cpp "var += val"; planning treats every reduce identically, so
    plans are unaffected).

The batch (leading) dimension is the shard axis: `batch` is the per-GPU
shard, and every config is data-parallel over it with no exchange.
"""

import math


class GraphBuilder:
    def __init__(self):
        self.nodes = []
        self.ids = set()

    def _add(self, node):
        if node["id"] in self.ids:
            raise ValueError("duplicate id " + node["id"])
        self.ids.add(node["id"])
        self.nodes.append(node)
        return node["id"]

    @staticmethod
    def _shape(dims, dtype="f32"):
        return {"dims": list(dims), "dtype": dtype}

    def param(self, id, dims, dtype="f32"):
        return self._add({"id": id, "kind": "parameter", "shape": self._shape(dims, dtype)})

    def const(self, id, value, dims=()):
        return self._add({"id": id, "kind": "constant", "shape": self._shape(dims),
                          "value": float(value)})

    def ew(self, id, name, operands, dims):
        return self._add({"id": id, "kind": "elementwise", "name": name,
                          "operands": list(operands), "shape": self._shape(dims)})

    def bcast(self, id, src, dims):
        return self.ew(id, "broadcast", [src], dims)

    def reduce(self, id, src, reduce_dims, dims, kind="sum"):
        node = {"id": id, "kind": "reduce", "operands": [src],
                "reduce_dims": list(reduce_dims), "shape": self._shape(dims)}
        if kind != "sum":
            node["name"] = kind
        return self._add(node)

    def bdot(self, id, a, b, dims):
        r = len(dims)
        return self._add({"id": id, "kind": "batched_dot", "operands": [a, b],
                          "contract_dims": [r - 1, r - 2], "shape": self._shape(dims)})

    def dot(self, id, a, b, dims, contract=(1, 0)):
        return self._add({"id": id, "kind": "dot", "operands": [a, b],
                          "contract_dims": list(contract), "shape": self._shape(dims)})

    def graph(self, outputs):
        return {"nodes": self.nodes, "outputs": list(outputs)}


# ---------------------------------------------------------------------------
# building blocks
# ---------------------------------------------------------------------------

def _layernorm(g, x, lead, C, pre, gamma, beta, eps=1e-5):
    """Row LayerNorm over the last dim of x[lead..., C]; returns y id.
    mean/var as sum * (1/C) so the graph stays within the reference op set."""
    full = list(lead) + [C]
    rdim = [len(lead)]
    inv = g.bcast(pre + "inv_b", g.const(pre + "inv_n", 1.0 / C), lead)
    epsb = g.bcast(pre + "eps_b", g.const(pre + "eps", eps), lead)
    s = g.reduce(pre + "sum", x, rdim, lead)
    mean = g.ew(pre + "mean", "multiply", [s, inv], lead)
    mb = g.bcast(pre + "mean_b", mean, full)
    xc = g.ew(pre + "xc", "subtract", [x, mb], full)
    sq = g.ew(pre + "sq", "multiply", [xc, xc], full)
    vs = g.reduce(pre + "var_sum", sq, rdim, lead)
    var = g.ew(pre + "var", "multiply", [vs, inv], lead)
    ve = g.ew(pre + "var_eps", "add", [var, epsb], lead)
    rs = g.ew(pre + "rstd", "rsqrt", [ve], lead)
    rb = g.bcast(pre + "rstd_b", rs, full)
    xn = g.ew(pre + "xn", "multiply", [xc, rb], full)
    gb = g.bcast(pre + "gamma_b", gamma, full)
    y1 = g.ew(pre + "scaled", "multiply", [xn, gb], full)
    bb = g.bcast(pre + "beta_b", beta, full)
    return g.ew(pre + "y", "add", [y1, bb], full)


def _gelu(g, x, dims, pre):
    """tanh-GeLU written with exp: x * sigmoid(2*sqrt(2/pi)*(x + 0.044715 x^3))."""
    k = g.bcast(pre + "k_b", g.const(pre + "k", 2.0 * math.sqrt(2.0 / math.pi)), dims)
    a = g.bcast(pre + "a_b", g.const(pre + "a", 0.044715), dims)
    one = g.bcast(pre + "one_b", g.const(pre + "one", 1.0), dims)
    x2 = g.ew(pre + "x2", "multiply", [x, x], dims)
    x3 = g.ew(pre + "x3", "multiply", [x2, x], dims)
    ax3 = g.ew(pre + "ax3", "multiply", [a, x3], dims)
    inner = g.ew(pre + "inner", "add", [x, ax3], dims)
    z = g.ew(pre + "z", "multiply", [k, inner], dims)
    nz = g.ew(pre + "nz", "negate", [z], dims)
    ez = g.ew(pre + "ez", "exp", [nz], dims)
    den = g.ew(pre + "den", "add", [one, ez], dims)
    return g.ew(pre + "gelu", "divide", [x, den], dims)


def _softmax_rows(g, x, lead, C, pre):
    """Numerically stable softmax over the last dim (row max + row sum)."""
    full = list(lead) + [C]
    rdim = [len(lead)]
    mx = g.reduce(pre + "rmax", x, rdim, lead, kind="max")
    mb = g.bcast(pre + "rmax_b", mx, full)
    sh = g.ew(pre + "shift", "subtract", [x, mb], full)
    e = g.ew(pre + "e", "exp", [sh], full)
    s = g.reduce(pre + "rsum", e, rdim, lead)
    sb = g.bcast(pre + "rsum_b", s, full)
    return g.ew(pre + "prob", "divide", [e, sb], full)


# ---------------------------------------------------------------------------
# the BASELINE.json configs
# ---------------------------------------------------------------------------

def layernorm(rows=16384, cols=768):
    """configs[0]: LayerNorm subgraph, fp32 [rows x cols]."""
    g = GraphBuilder()
    x = g.param("x", [rows, cols])
    gamma = g.param("gamma", [cols])
    beta = g.param("beta", [cols])
    y = _layernorm(g, x, [rows], cols, "", gamma, beta)
    return g.graph([y])


def softmax(heads=64, seq=512):
    """configs[1]: masked scaled softmax over [heads x seq x seq] attention
    scores, stored as rows [heads*seq, seq] with an additive key mask [seq].

    Why 2-D: the IR's broadcast has no explicit dimension list; it maps input
    dims onto output dims right-most-greedily (reference graph.cpp:146
    broadcast_dim_map). A row statistic [heads, seq] broadcast back to
    [heads, seq, seq] would land on dims (0, 2) -- a column broadcast -- because
    both trailing extents are 512. Flattening (head, query) into one row axis
    keeps every broadcast unambiguous and the arithmetic identical."""
    g = GraphBuilder()
    rows = heads * seq
    full = [rows, seq]
    x = g.param("x", full)
    mask = g.param("mask", [seq])
    sc = g.bcast("scale_b", g.const("scale", 1.0 / math.sqrt(64.0)), full)
    xs = g.ew("xs", "multiply", [x, sc], full)
    mb = g.bcast("mask_b", mask, full)
    xm = g.ew("xm", "add", [xs, mb], full)
    y = _softmax_rows(g, xm, [rows], seq, "")
    return g.graph([y])


def encoder(batch=64, seq=512, hidden=1024):
    """configs[2]: bias + GeLU + residual + LayerNorm on [batch, seq, hidden],
    plus the column-reduction bias gradient of an incoming dy."""
    g = GraphBuilder()
    full = [batch, seq, hidden]
    h = g.param("h", full)
    bias = g.param("bias", [hidden])
    res = g.param("res", full)
    gamma = g.param("gamma", [hidden])
    beta = g.param("beta", [hidden])
    dy = g.param("dy", full)
    bb = g.bcast("bias_b", bias, full)
    hb = g.ew("hb", "add", [h, bb], full)
    ge = _gelu(g, hb, full, "")
    r = g.ew("resid", "add", [ge, res], full)
    y = _layernorm(g, r, [batch, seq], hidden, "ln_", gamma, beta)
    db = g.reduce("dbias", dy, [0, 1], [hidden])
    return g.graph([y, db])


def gru(batch=4096, n=64):
    """configs[3]: attention-GRU style cell with per-sample 64x64 batched GEMMs
    feeding sigmoid / tanh gates (written with exp / divide).
        pre = h @ W + x @ U          (two fine-grained batched GEMMs)
        z   = sigmoid(pre);  c = tanh(pre) = 2*sigmoid(2 pre) - 1
        h'  = z * h + (1 - z) * c
    """
    g = GraphBuilder()
    full = [batch, n, n]
    h = g.param("h", full)
    W = g.param("W", full)
    x = g.param("x", full)
    U = g.param("U", full)
    one = g.bcast("one_b", g.const("one", 1.0), full)
    two = g.bcast("two_b", g.const("two", 2.0), full)
    hw = g.bdot("hw", h, W, full)
    xu = g.bdot("xu", x, U, full)
    pre = g.ew("pre", "add", [hw, xu], full)
    npre = g.ew("npre", "negate", [pre], full)
    e = g.ew("e", "exp", [npre], full)
    d = g.ew("d", "add", [one, e], full)
    z = g.ew("z", "divide", [one, d], full)
    p2 = g.ew("p2", "multiply", [two, pre], full)
    np2 = g.ew("np2", "negate", [p2], full)
    e2 = g.ew("e2", "exp", [np2], full)
    d2 = g.ew("d2", "add", [one, e2], full)
    s2 = g.ew("s2", "divide", [two, d2], full)
    c = g.ew("c", "subtract", [s2, one], full)
    zh = g.ew("zh", "multiply", [z, h], full)
    omz = g.ew("omz", "subtract", [one, z], full)
    oc = g.ew("oc", "multiply", [omz, c], full)
    hn = g.ew("hn", "add", [zh, oc], full)
    return g.graph([hn])


CONFIGS = {
    "layernorm": layernorm,
    "softmax": softmax,
    "encoder": encoder,
    "gru": gru,
}
