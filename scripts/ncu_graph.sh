#!/bin/bash
# ncu --set full of the stitched kernels of fused-graph JSON files (one
# executor each, plain launches). Usage: scripts/ncu_graph.sh out_name g1.json [g2.json ...]
out=$1; shift
mkdir -p gpurun_out
cat > /tmp/run_graphs.py <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
from paper_1911_11576_b200 import runtime as rt
torch.cuda.set_device(0)
for p in sys.argv[1:]:
    ex = rt.Executor(json.load(open(p)), use_graph=False)
    ins = [torch.randn(t["dims"], device="cuda") for t in ex.info["inputs"]]
    outs = [torch.empty(t["dims"], device="cuda") for t in ex.info["outputs"]]
    ex.run(ins, outs, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    print(p, [(k["name"], k["block"], k["grid"], k["scheme"]) for k in ex.info["kernels"]], flush=True)
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'fusion|dbias' -o gpurun_out/$out python /tmp/run_graphs.py "$@" > gpurun_out/$out.log 2>&1
echo "ncu rc=$?"
grep -v '^==' gpurun_out/$out.log | tail -20
