"""Multi-rank data-parallel path on CPU (gloo, world_size 2): each rank runs
its own batch shard (workloads.shard_range / shard_layout, the split
bench.py uses), with no exchange on the data path. Checks that the shards
reassemble into the full-batch result (row outputs concatenate, per-shard
column reductions sum to the full reduction), that every rank's shard graph
plans identically (same fusion groups on every GPU), and the bench's
max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import executor as orc
from paper_1911_11576_b200 import runtime as rt
from paper_1911_11576_b200 import workloads as W

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, name, kw, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        batch, rows = W.shard_layout(name, **kw)
        full = W.CONFIGS[name](**kw)
        rng = np.random.default_rng(5)
        nodes = {n["id"]: n for n in full["nodes"]}
        ins = {i: rng.standard_normal(nodes[i]["shape"]["dims"]).astype(np.float32) for i in orc.graph_inputs(full)}
        lo, hi = W.shard_range(batch, WORLD, rank)
        bk = W.BATCH_KW[name]
        shard = W.CONFIGS[name](**dict(kw, **{bk: hi - lo}))
        sin = {i: (v[lo * rows[i]:hi * rows[i]] if i in rows else v) for i, v in ins.items()}
        outs = orc.run(shard, sin)
        # plan of the shard graph: fusion groups must be the same on every rank
        plan = rt.plan(shard, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
        groups = sorted(sorted(b["id"] for b in n["body"]["nodes"] if b["kind"] not in ("parameter", "tuple"))
                        for n in plan["nodes"] if n["kind"] == "fused")
        gathered = [None] * WORLD
        dist.all_gather_object(gathered, (lo, hi, [o.tolist() for o in outs], groups))
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py: max over ranks
        if rank == 0:
            ref = orc.run(full, ins)
            names = orc.graph_outputs(full)
            ok = True
            for k, o in enumerate(names):
                parts = [np.asarray(g[2][k], dtype=np.float32) for g in gathered]
                got = np.concatenate(parts, 0) if o in rows else np.sum(parts, 0)
                ok = ok and np.allclose(got, ref[k], rtol=1e-5, atol=1e-4)
            # equal shard sizes (bench.py's weak scaling) plan identically on every rank
            ok = ok and all(g[3] == gathered[0][3] for g in gathered if g[1] - g[0] == gathered[0][1] - gathered[0][0])
            ok = ok and [g[:2] for g in gathered] == [W.shard_range(batch, WORLD, r) for r in range(WORLD)]
            q.put((ok, float(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,kw", [
    ("layernorm", dict(rows=37, cols=96)),
    ("softmax", dict(heads=4, seq=32)),  # heads != 1: rows == seq would make the row broadcast ambiguous
    ("encoder", dict(batch=3, seq=8, hidden=64)),
    ("gru", dict(batch=5, n=16)),
])
def test_two_rank_shards_reassemble(name, kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, name, kw, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    ok, tmax = q.get(timeout=5)
    assert ok
    assert tmax == float(WORLD)


def test_shard_range_balanced():
    for b in (1, 5, 64, 4096):
        for w in (1, 2, 3, 8):
            rs = [W.shard_range(b, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == b
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


def _bench(*args, env=None):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + list(args), capture_output=True,
                       text=True, timeout=600, env=e, cwd=root)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r.returncode, (json.loads(lines[-1]) if lines else None), r.stderr


def test_bench_gpus_2_spawns_ranks():
    """`bench.py --gpus 2` with no torchrun environment re-launches itself
    with two ranks; rank 0 prints one line with n_gpus 2, identical plans on
    both ranks and the max-over-ranks step time (rank 1 sleeps 2 ms/step)."""
    rc, line, err = _bench("--gpus", "2", "--dry-run", "--configs", "layernorm,gru", "--steps", "4", "--warmup", "1")
    assert rc == 0, err[-2000:]
    assert line["n_gpus"] == 2 and line["dry_run"] and line["value"] is None
    assert set(line["plan_digests"]) == {"layernorm", "gru"}
    assert line["ms_per_step"] >= 2.0


def test_bench_rejects_world_size_mismatch():
    rc, line, err = _bench("--gpus", "4", "--dry-run", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert rc != 0 and line is None and "WORLD_SIZE=2" in err
