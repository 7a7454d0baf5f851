"""Test infrastructure (oracle) -- loader for the compiled reference planner.

oracle/_ref/libstitch_ref.so is built by oracle/Makefile from the unmodified
sources under /root/reference/proj/src plus oracle/ref_driver.cpp. Only
tests/ and the golden-fixture generator import this module; the product never
does.
"""
import ctypes
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libstitch_ref.so")
_lib = None


def available():
    return os.path.exists(LIB_PATH)


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(LIB_PATH)
        lib.stitch_ref_call.restype = ctypes.c_void_p
        lib.stitch_ref_call.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
        lib.stitch_ref_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


def call(fn, **args):
    """Runs reference function `fn` (see ref_driver.cpp) and returns its JSON
    result; raises RuntimeError carrying the reference's error text."""
    lib = _load()
    ptr = lib.stitch_ref_call(fn.encode(), json.dumps(args).encode())
    try:
        out = json.loads(ctypes.string_at(ptr).decode())
    finally:
        lib.stitch_ref_free(ptr)
    if not out["ok"]:
        raise RuntimeError(out["error"])
    return out["result"]
