#!/bin/bash
mkdir -p gpurun_out
cd tests/cuda && ./gws_2_fast 4096 | head -3; cd ../..
timeout 600 python bench.py --configs gru --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-unfused --no-model-plan > gpurun_out/bench_gws.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open("gpurun_out/bench_gws.log") if x.startswith("{")]
d=json.loads(l[-1])
for k,v in d["config"]["suite"].items(): print(k, v["GBps"], v["frac_of_hbm"], v["ms"], v["kernel_us"])
PY
timeout 600 python scripts/time_graph.py --help 2>&1 | head -5
timeout 900 python -m pytest tests/test_executor_gpu.py -m gpu -q -x -k "gws or gru" > gpurun_out/pytest_gws.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gws.log
