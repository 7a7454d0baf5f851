#!/bin/bash
# split_cross (column-reduction fold as its own kernel): GPU parity, BERT A/B, bench line.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python scripts/step_ab.py bert '[{"split_cross": false}, {}, {"split_cross": false, "concurrent_lanes": 1}, {"concurrent_lanes": 1}, {"concurrent_lanes": 4}]' 5 > gpurun_out/ab_split.log 2>&1; echo "ab rc=$?"
tail -5 gpurun_out/ab_split.log
timeout 900 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], {k: (v['GBps'], v['ms']) for k, v in d['config']['suite'].items()})"
