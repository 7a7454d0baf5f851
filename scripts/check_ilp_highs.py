"""Independent check of the planner's selection on a whole-graph instance
with an off-the-shelf MIP solver (scipy's HiGHS; a development check, not a
product dependency).

    STITCH_ILP_DUMP=/tmp/bert python -c "...rt.plan(W.bert(), ...)"   # writes /tmp/bert.0.txt
    python scripts/check_ilp_highs.py /tmp/bert.0.txt selected.json [out.json]
    (selected.json: the solver's own indices, e.g. from scripts/probes/ilp_driver.cpp)

1. max s.x over node-disjoint selections (plus the cycle constraints) -- the
   optimum must equal the canonical total of the planner's selection;
   solved per independent component (patterns sharing no node and no cycle
   constraint), the whole-graph MIP does not finish in 20 minutes;
2. whether HiGHS picks the same set per component (uniqueness of the
   optimum is what the planner's own search proves: it enumerates every
   selection within the rounding window of it).
"""
import json
import sys
import time

import numpy as np
import scipy.sparse as sp
from scipy.optimize import Bounds, LinearConstraint, milp


def load(path):
    L = open(path).read().split("\n")
    n, nn, npairs, ncyc, _ = map(int, L[0].split())
    s = np.array([float.fromhex(x) for x in L[1:1 + n]])
    sets = [list(map(int, l.split()))[1:] for l in L[1 + n:1 + 2 * n]] if nn else [[] for _ in range(n)]
    off = 1 + (2 * n if nn else n)
    pairs = [tuple(map(int, l.split())) for l in L[off:off + npairs]]
    cycles = [list(map(int, l.split()))[1:] for l in L[off + npairs:off + npairs + ncyc]]
    return n, nn, s, sets, pairs, cycles


def components(n, s, sets, pairs, cycles):
    par = list(range(n))

    def f(x):
        while par[x] != x:
            par[x] = par[par[x]]
            x = par[x]
        return x
    owner = {}
    for v in range(n):
        for x in sets[v]:
            if x in owner:
                par[f(v)] = f(owner[x])
            else:
                owner[x] = v
    for u, v in pairs:
        par[f(u)] = f(v)
    for c in cycles:
        for v in c[1:]:
            par[f(v)] = f(c[0])
    comps = {}
    for v in range(n):
        if s[v] > 0:
            comps.setdefault(f(v), []).append(v)
    return list(comps.values())


def solve_component(vs, s, sets, pairs, cycles, time_limit):
    col = {v: j for j, v in enumerate(vs)}
    nodes = sorted({x for v in vs for x in sets[v]})
    row = {x: i for i, x in enumerate(nodes)}
    r, c = [], []
    for j, v in enumerate(vs):
        for x in sets[v]:
            r.append(row[x])
            c.append(j)
    A = [sp.csr_matrix((np.ones(len(r)), (r, c)), shape=(max(len(nodes), 1), len(vs)))]
    ub = [np.ones(max(len(nodes), 1))]
    for u, v in pairs:
        if u in col and v in col:
            A.append(sp.csr_matrix(([1.0, 1.0], ([0, 0], [col[u], col[v]])), shape=(1, len(vs))))
            ub.append(np.ones(1))
    for cy in cycles:
        if cy and cy[0] in col:
            idx = [col[v] for v in cy if v in col]
            A.append(sp.csr_matrix((np.ones(len(idx)), ([0] * len(idx), idx)), shape=(1, len(vs))))
            ub.append(np.array([len(cy) - 1.0]))
    res = milp(-s[vs], constraints=LinearConstraint(sp.vstack(A), -np.inf, np.concatenate(ub)),
               integrality=np.ones(len(vs)), bounds=Bounds(0, 1),
               options={"mip_rel_gap": 0.0, "presolve": True, "time_limit": time_limit})
    return -res.fun, sorted(vs[j] for j in range(len(vs)) if res.x[j] > 0.5), res.message


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    path, selp = args[:2]
    n, nn, s, sets, pairs, cycles = load(path)
    sel = set(json.load(open(selp)))
    comps = components(n, s, sets, pairs, cycles)
    t = time.time()
    rows, worst = [], 0.0
    for vs in sorted(comps, key=len, reverse=True):
        best, hx, msg = solve_component(vs, s, sets, pairs, cycles, 1200)
        mine = sorted(v for v in vs if v in sel)
        tot = float(np.sum(s[mine])) if mine else 0.0
        worst = max(worst, abs(best - tot))
        rows.append({"vars": len(vs), "highs_optimum": best, "planner": tot, "same_set": hx == mine,
                     "status": msg})
    res = {"instance": path, "vars": n, "positive_vars": int(np.sum(s > 0)), "nodes": nn, "cycles": len(cycles),
           "components": len(comps), "max_abs_diff": worst,
           "all_same_set": all(r["same_set"] for r in rows),
           "highs_total": float(sum(r["highs_optimum"] for r in rows)),
           "planner_total": float(sum(r["planner"] for r in rows)), "seconds": round(time.time() - t, 1),
           "largest_components": rows[:6]}
    print(json.dumps(res, indent=1))
    if len(args) > 2:
        json.dump(res, open(args[2], "w"), indent=1)


if __name__ == "__main__":
    main()
