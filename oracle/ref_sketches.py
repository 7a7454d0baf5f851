"""Test infrastructure (oracle) -- runs the REFERENCE's own emitted kernels.

NOT part of the product: only tests/ import this module.

The reference plans fusion and emits one CUDA-C kernel sketch per fused op
(proj/src/pipeline.cpp:112 run_codegen -> emitter.cpp:1367
generate_best_kernel -> :1329 emit_kernel; signature assembled at
emitter.cpp:1253-1290: inputs as `const T* __restrict__ <id>` in fused-op
operand order, then outputs as `T* __restrict__ <id>`, launch
<<<cta_num, cta_size>>> with static shared memory only). It never runs them
(SPEC fusion-transform Non-goals). This module does: the sketches committed
in tests/golden/ref_sketches.json (scripts/make_ref_sketches.py, generated
from oracle/_ref) are compiled UNMODIFIED with nvcc for sm_100a, loaded with
the CUDA driver API and launched in the fused graph's order on buffers named
by the reference's own ids. Their outputs are the reference's numerics for
the graph; tests/test_ref_sketches.py checks oracle/executor.py (and our
executor) against them.
"""
import ctypes
import hashlib
import os
import re
import subprocess
import tempfile

import numpy as np

_SIG = re.compile(r'extern "C" __global__ void (\w+)\((.*?)\) \{', re.S)
_ARG = re.compile(r'(const )?(float|int)\* __restrict__ (\w+)')


def sanitize(i):
    """emitter.cpp:50 sanitize (C identifier for a node id)."""
    out = "".join(c if (c.isalnum() or c == "_") else "_" for c in i)
    if not out or out[0].isdigit():
        out = "v_" + out
    return out


def signature(source):
    """(kernel name, [(arg name, is_output)]) parsed from a sketch."""
    m = _SIG.search(source)
    if m is None:
        raise ValueError("no kernel signature in sketch")
    args = [(a.group(3), a.group(1) is None) for a in _ARG.finditer(m.group(2))]
    return m.group(1), args


def launch_order_ok(graph, kernels):
    """True when every sketch's inputs are graph inputs or outputs of an
    earlier sketch (the manifest follows the fused graph's node order)."""
    names = {sanitize(n["id"]) for n in graph["nodes"] if n["kind"] in ("parameter", "constant")}
    for k in kernels:
        _, args = signature(k["source"])
        for a, out in args:
            if not out and a not in names:
                return False
        names.update(a for a, out in args if out)
    return True


def compile_cubin(kernels, cache_dir=None):
    """nvcc -cubin for sm_100a of all sketches of one variant (one module)."""
    src = "".join(k["source"] + "\n" for k in kernels)
    h = hashlib.sha1(src.encode()).hexdigest()[:16]
    d = cache_dir or os.path.join(tempfile.gettempdir(), "stitch_ref_sketches")
    os.makedirs(d, exist_ok=True)
    cu, cubin = os.path.join(d, h + ".cu"), os.path.join(d, h + ".cubin")
    if not os.path.exists(cubin):
        with open(cu, "w") as f:
            f.write(src)
        nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
        subprocess.run([nvcc, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-o", cubin + ".tmp", cu], check=True, capture_output=True)
        os.replace(cubin + ".tmp", cubin)
    with open(cubin, "rb") as f:
        return f.read()


def _ck(res):
    if int(res[0]) != 0:
        raise RuntimeError("CUDA driver error %s" % res[0])
    return res[1] if len(res) > 1 else None


def run(graph, kernels, inputs, torch):
    """Runs the reference sketches of one variant on cuda:0. `inputs` maps
    parameter ids (constants take their "value") to fp32 arrays. Returns
    {id: np.float32 array} for every value the sketches wrote."""
    from cuda.bindings import driver as cu

    nodes = {sanitize(n["id"]): n for n in graph["nodes"]}
    torch.cuda.init()
    bufs = {}
    for n in graph["nodes"]:
        if n["kind"] == "parameter" or (n["kind"] == "constant" and "value" not in n):
            bufs[sanitize(n["id"])] = torch.from_numpy(
                np.ascontiguousarray(inputs[n["id"]], dtype=np.float32)).cuda()
        elif n["kind"] == "constant":
            bufs[sanitize(n["id"])] = torch.full(n["shape"]["dims"] or [1], n["value"],
                                                 dtype=torch.float32, device="cuda")
    mod = _ck(cu.cuModuleLoadData(compile_cubin(kernels)))
    stream = torch.cuda.current_stream().cuda_stream
    written = []
    for k in kernels:
        name, args = signature(k["source"])
        fn = _ck(cu.cuModuleGetFunction(mod, name.encode()))
        ptrs = []
        for a, out in args:
            if out:
                bufs[a] = torch.full(nodes[a]["shape"]["dims"] or [1], float("nan"),
                                     dtype=torch.float32, device="cuda")
                written.append(a)
            ptrs.append(bufs[a].data_ptr())
        _ck(cu.cuLaunchKernel(fn, int(k["cta_num"]), 1, 1, int(k["cta_size"]), 1, 1, 0, cu.CUstream(stream),
                              (tuple(ptrs), tuple(ctypes.c_void_p for _ in ptrs)), 0))
    torch.cuda.synchronize()
    out = {}
    for a in written:
        out[nodes[a]["id"]] = bufs[a].cpu().numpy().reshape(nodes[a]["shape"]["dims"])
    _ck(cu.cuModuleUnload(mod))
    return out
