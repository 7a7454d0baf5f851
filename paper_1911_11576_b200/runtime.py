"""Python binding of the C ABI in include/stitch_b200.h (ctypes).

The product path is native: planning runs in libstitch_b200.so's C++ host
code, execution in sm_100a kernels it generates and launches. This module
only marshals JSON strings and pointers; it never computes anything itself
and raises if the library is missing.
"""

import ctypes
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstitch_b200.so")
CACHE_DIR = os.path.join(_HERE, "_kcache")
_lib = None


class StitchError(RuntimeError):
    """Error reported through stitch_last_error(); `code` is the C ABI
    return value (1 = bad input, 2 = internal / CUDA failure)."""

    def __init__(self, msg, code=1):
        super().__init__(msg)
        self.code = code


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise StitchError("libstitch_b200.so is not built; run __graft_entry__.build()", 2)
        L = ctypes.CDLL(LIB_PATH)
        vp, cp = ctypes.c_void_p, ctypes.c_char_p
        L.stitch_plan_graph.argtypes = [cp, cp, ctypes.POINTER(vp)]
        L.stitch_plan_graph.restype = ctypes.c_int
        L.stitch_debug_call.argtypes = [cp, cp]
        L.stitch_debug_call.restype = vp
        L.stitch_executor_create.argtypes = [cp, cp, ctypes.POINTER(vp)]
        L.stitch_executor_create.restype = ctypes.c_int
        L.stitch_executor_destroy.argtypes = [vp]
        L.stitch_executor_describe.argtypes = [vp, ctypes.POINTER(vp)]
        L.stitch_executor_describe.restype = ctypes.c_int
        L.stitch_executor_run.argtypes = [vp, vp, vp, vp]
        L.stitch_executor_run.restype = ctypes.c_int
        L.stitch_executor_run_host.argtypes = [vp, vp, vp, vp]
        L.stitch_executor_run_host.restype = ctypes.c_int
        L.stitch_executor_profile.argtypes = [vp, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
        L.stitch_executor_profile.restype = ctypes.c_int
        L.stitch_executor_trace.argtypes = [vp, vp, vp, vp, ctypes.POINTER(vp)]
        L.stitch_executor_trace.restype = ctypes.c_int
        L.stitch_executor_sources.argtypes = [vp]
        L.stitch_executor_sources.restype = vp
        L.stitch_last_error.restype = cp
        L.stitch_free.argtypes = [vp]
        _lib = L
    return _lib


def _take_string(ptr):
    try:
        return ctypes.string_at(ptr).decode()
    finally:
        lib().stitch_free(ptr)


def _check(rc):
    if rc != 0:
        raise StitchError(lib().stitch_last_error().decode(), rc)


def debug_call(fn, **args):
    """Runs one planner stage by name (stitch_debug_call)."""
    out = json.loads(_take_string(lib().stitch_debug_call(fn.encode(), json.dumps(args).encode())))
    if not out["ok"]:
        raise StitchError(out["error"])
    return out["result"]


def plan(graph, **options):
    """stitch_plan_graph: {"plan", "fused", "report_text", "timings"}."""
    res = ctypes.c_void_p()
    g = graph if isinstance(graph, str) else json.dumps(graph)
    _check(lib().stitch_plan_graph(g.encode(), json.dumps(options).encode(), ctypes.byref(res)))
    return json.loads(_take_string(res))


def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def _data_ptr(x):
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):  # torch tensor
        return x.data_ptr()
    if hasattr(x, "ctypes"):  # numpy array
        return x.ctypes.data
    raise TypeError("expected a pointer, torch tensor or numpy array")


class Executor:
    """One compiled sm_100a kernel per fused op of `fused_graph` (and one per
    unfused kernel op), launched in topological order over an HBM arena.
    Mirrors the reference's run_codegen(fused) -> kernels, but runnable."""

    def __init__(self, fused_graph, device=0, cache_dir=CACHE_DIR, use_graph=True, compile_only=False, **extra):
        opts = dict(device=device, cache_dir=cache_dir or "", use_graph=use_graph, compile_only=compile_only)
        opts.update(extra)
        h = ctypes.c_void_p()
        g = fused_graph if isinstance(fused_graph, str) else json.dumps(fused_graph)
        _check(lib().stitch_executor_create(g.encode(), json.dumps(opts).encode(), ctypes.byref(h)))
        self._h = h
        res = ctypes.c_void_p()
        _check(lib().stitch_executor_describe(self._h, ctypes.byref(res)))
        self.info = json.loads(_take_string(res))

    def close(self):
        if getattr(self, "_h", None):
            lib().stitch_executor_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def input_ids(self):
        return [t["id"] for t in self.info["inputs"]]

    @property
    def output_ids(self):
        return [t["id"] for t in self.info["outputs"]]

    def sources(self):
        return json.loads(_take_string(lib().stitch_executor_sources(self._h)))

    def run(self, inputs, outputs, stream=0):
        """Device pointers (or CUDA torch tensors) in describe() order."""
        ins = _ptr_array([_data_ptr(x) for x in inputs])
        outs = _ptr_array([_data_ptr(x) for x in outputs])
        _check(lib().stitch_executor_run(self._h, ins, outs, ctypes.c_void_p(stream)))

    def run_host(self, inputs, outputs, stream=0):
        """Host buffers (numpy / pinned torch CPU tensors); copies included."""
        ins = _ptr_array([_data_ptr(x) for x in inputs])
        outs = _ptr_array([_data_ptr(x) for x in outputs])
        _check(lib().stitch_executor_run_host(self._h, ins, outs, ctypes.c_void_p(stream)))

    def trace(self, inputs, outputs, stream=0):
        """Per-kernel [start, end] (us) of one pass; needs trace=True."""
        ins = _ptr_array([_data_ptr(x) for x in inputs])
        outs = _ptr_array([_data_ptr(x) for x in outputs])
        res = ctypes.c_void_p()
        _check(lib().stitch_executor_trace(self._h, ins, outs, ctypes.c_void_p(stream), ctypes.byref(res)))
        return json.loads(_take_string(res))

    def profile(self, inputs, outputs, stream=0, iters=10):
        ins = _ptr_array([_data_ptr(x) for x in inputs])
        outs = _ptr_array([_data_ptr(x) for x in outputs])
        res = ctypes.c_void_p()
        _check(lib().stitch_executor_profile(self._h, ins, outs, ctypes.c_void_p(stream), iters, ctypes.byref(res)))
        return json.loads(_take_string(res))
