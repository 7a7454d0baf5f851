"""Runs the bench BERT plan once with per-kernel option overrides (the
command ncu wraps to profile one group's variant; never a timing source).
    python scripts/run_bert_variant.py '{"fusion_5": {"wide_cross_cta": true}}'"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1911_11576_b200 import runtime as rt  # noqa: E402
from paper_1911_11576_b200 import tuning  # noqa: E402

over = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
kopt = dict(tuning.kernel_variants("bert"))
kopt.update(over)
torch.cuda.set_device(0)
fused = tuning.config_plan("bert")[0]["fused"]
ex = rt.Executor(fused, use_graph=False, kernel_options=kopt)
ins = [torch.randn(t["dims"], device="cuda") for t in ex.info["inputs"]]
outs = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
ex.run(ins, outs, stream=torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print({k["name"]: (k["scheme"], k["block"], k["grid"], k["smem_bytes"]) for k in ex.info["kernels"] if k["name"] in over})
