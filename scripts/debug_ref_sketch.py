"""Runs one reference-sketch variant on the GPU and reports, per graph
output, the worst err/tol against the oracle and where it sits."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import executor as orc  # noqa: E402
from oracle import ref_sketches as S  # noqa: E402
from oracle import tolerance  # noqa: E402

name, variant = sys.argv[1], sys.argv[2]
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 0.25
e = {x["name"]: x for x in json.load(open("tests/golden/ref_sketches.json"))}[name]
ins = orc.random_inputs(e["graph"], seed=5, scale=scale)
got = S.run(e["graph"], e["variants"][variant], ins, torch)
vals = orc.evaluate(e["graph"], ins)
ref, bound = tolerance.reference_with_bound(e["graph"], ins)
bnd = dict(zip(orc.graph_outputs(e["graph"]), bound))
for oid in sorted(got):
    r = np.asarray(vals[oid], dtype=np.float64)
    g = got[oid].reshape(r.shape)
    b = bnd.get(oid)
    if b is None:
        b = np.zeros_like(r)
    ok, worst = tolerance.check(g, r, b)
    rel = np.abs(g - r) / np.maximum(np.abs(r), 1e-6)
    bad = np.argwhere(rel > 1e-3)
    print("%-24s shape=%s ok=%s worst=%.3g maxrel=%.3g nbad=%d first_bad=%s" % (
        oid, list(r.shape), ok, worst, float(np.nanmax(rel)), len(bad), bad[:4].tolist()))
    if len(bad) and r.ndim == 2:
        rows = sorted(set(int(x[0]) for x in bad))
        print("   bad rows:", rows[:20], "...", len(rows))
        i = tuple(bad[0])
        print("   got", g[i], "ref", r[i])
