"""B200-native FusionStitching (arXiv 1911.11576): fusion planning on the
host (C++), one stitched sm_100a kernel per fusion group on the device.

    from paper_1911_11576_b200 import runtime, workloads
    res = runtime.plan(workloads.layernorm(), shared_limit_bytes=232448)
    ex = runtime.Executor(res["fused"])
"""
from . import runtime, workloads  # noqa: F401

__all__ = ["runtime", "workloads"]
