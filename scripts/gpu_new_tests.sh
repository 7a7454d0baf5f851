#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_executor_gpu.py -m gpu -q -k "anchored or sinking or gws or bert" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_new.log
timeout 900 python bench.py --configs bert --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-unfused > gpurun_out/bench_bert.log 2>&1; echo "bench rc=$?"
python -c "
import json
l=[x for x in open('gpurun_out/bench_bert.log') if x.startswith('{')]
d=json.loads(l[-1]); v=d['config']['suite']['bert']; print('bert', v['GBps'], v['frac_of_hbm'], v['ms'], v['kernels'])"
