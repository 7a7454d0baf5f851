"""GEMM scheme vs the loop schemes it replaces, for unfused dots (CUDA events
via stitch_executor_profile, L2 flushed, median of 9). Writes JSON."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402

CASES = [("dot", (512, 512), (512, 512), (512, 512)), ("dot", (2048, 2048), (2048, 2048), (2048, 2048)),
         ("dot", (4096, 768), (768, 3072), (4096, 3072)), ("batched_dot", (4096, 64, 64), (4096, 64, 64), (4096, 64, 64))]


def graph(kind, ad, bd, od):
    return {"nodes": [{"id": "a", "kind": "parameter", "shape": {"dims": list(ad), "dtype": "f32"}},
                      {"id": "b", "kind": "parameter", "shape": {"dims": list(bd), "dtype": "f32"}},
                      {"id": "c", "kind": kind, "operands": ["a", "b"], "shape": {"dims": list(od), "dtype": "f32"}}],
            "outputs": ["c"]}


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = []
    for kind, ad, bd, od in CASES:
        g = graph(kind, ad, bd, od)
        a = torch.randn(ad, device="cuda")
        b = torch.randn(bd, device="cuda")
        c = torch.empty(od, device="cuda")
        flops = 2.0 * np.prod(od) * ad[-1]
        row = {"case": "%s %s x %s" % (kind, ad, bd), "gflop": flops / 1e9}
        for tag, opts in (("gemm", {}), ("loops", {"gemm": False})):
            ex = rt.Executor(g, **opts)
            s = torch.cuda.current_stream().cuda_stream
            ex.run([a, b], [c], stream=s)
            us = []
            for _ in range(9):
                flush.zero_()
                us.append(ex.profile([a, b], [c], stream=s, iters=1)["kernels"][0]["us"])
            t = float(np.median(us))
            row[tag] = {"scheme": ex.info["kernels"][0]["scheme"], "us": round(t, 2),
                        "tflops": round(flops / t / 1e6, 2)}
            ex.close()
        ref = torch.matmul(a.double(), b.double()).float() if kind == "dot" else torch.bmm(a.double(), b.double()).float()
        ex = rt.Executor(g)
        ex.run([a, b], [c], stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        row["max_rel_err_vs_fp64"] = float(((c - ref).abs() / (ref.abs() + 1e-3)).max())
        ex.close()
        print(json.dumps(row), flush=True)
        out.append(row)
    json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gemm_perf.json", "w"), indent=1)


if __name__ == "__main__":
    main()
