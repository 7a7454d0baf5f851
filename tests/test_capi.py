"""The C-ABI drop-in boundary (include/stitch_b200.h): the library loads
without a GPU, exports every declared symbol, follows the reference CLI's
error-code convention, and the executor's compile-only path works on CPU."""
import ctypes
import os
import re

import pytest

from paper_1911_11576_b200 import runtime as rt
from paper_1911_11576_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "stitch_b200.h")).read()
    return re.findall(r"STITCH_API\s+[\w\s\*]+?\b(stitch_\w+)\s*\(", src)


def test_header_symbols_exported():
    names = declared()
    assert len(names) >= 10
    lib = ctypes.CDLL(rt.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n


def test_only_declared_symbols_exported():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", rt.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert {s for s in exported if s.startswith("stitch_")} == set(declared())


def test_error_codes():
    with pytest.raises(rt.StitchError) as e:
        rt.plan("[1, 2")
    assert e.value.code == 1
    with pytest.raises(rt.StitchError) as e:
        rt.Executor('{"nodes": [], "outputs": ["nope"]}', compile_only=True)
    assert e.value.code in (1, 2)


def test_executor_compile_only_describe():
    g = W.layernorm(rows=64, cols=768)
    fused = rt.plan(g, shared_limit_bytes=W.B200_SHARED_LIMIT)["fused"]
    ex = rt.Executor(fused, compile_only=True)
    d = ex.info
    assert sorted(t["id"] for t in d["inputs"]) == ["beta", "gamma", "x"]
    assert [t["dims"] for t in d["outputs"]] == [[64, 768]]
    assert len(d["kernels"]) == 1
    k = d["kernels"][0]
    assert k["algo_bytes"] == (64 * 768 * 2 + 768 * 2) * 4
    src = ex.sources()[k["name"]]
    assert "extern \"C\" __global__" in src and "row_allreduce" in src
    with pytest.raises(rt.StitchError):
        ex.run([0, 0, 0], [0])  # compile-only executors refuse device work
