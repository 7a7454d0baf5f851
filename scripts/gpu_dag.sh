#!/bin/bash
# Dataflow (multi-lane) launch: bit-identity tests, BERT step A/B against the
# serial order, and the bench's BERT line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_executor_gpu.py -q -x -k "dataflow or random_dag_parity or host_path or chunked" > gpurun_out/pytest_dag.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_dag.log
timeout 900 python scripts/step_ab.py bert '[{"concurrent_lanes": 1}, {"concurrent_lanes": 8}, {"concurrent_lanes": 4}, {"concurrent_lanes": 16}, {"concurrent_lanes": 8, "pdl": false}]' 5 > gpurun_out/ab_dag.log 2>&1; echo "ab rc=$?"
cat gpurun_out/ab_dag.log | tail -6
timeout 900 python bench.py --configs bert --no-cpu-baseline --no-e2e --out gpurun_out/bench_bert.json > gpurun_out/bench_bert.log 2>&1; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_bert.json')); b=d['config']['suite']['bert']; print(d['value'], b['ms'], b['frac_of_hbm'])"
