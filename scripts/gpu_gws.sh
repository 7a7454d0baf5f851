#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_executor_gpu.py -m gpu -q -x -k "gws or gru or small_parity or ragged" > gpurun_out/pytest_gws.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gws.log
timeout 600 python bench.py --configs gru,layernorm --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_gws.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open("gpurun_out/bench_gws.log") if x.startswith("{")]
d=json.loads(l[-1])
for k,v in d["config"]["suite"].items(): print(k, v["GBps"], v["frac_of_hbm"], v["ms"], v.get("speedup_vs_unfused"), v["kernel_us"] if len(v["kernel_us"])<4 else "")
print("roofline", d["roofline"])
PY
