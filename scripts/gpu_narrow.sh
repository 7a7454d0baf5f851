#!/bin/bash
# Narrow rows + dataflow: GPU parity suite, BERT A/B, bench line.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python scripts/step_ab.py bert '[{"concurrent_lanes": 1, "narrow_rows": false}, {"concurrent_lanes": 1}, {"concurrent_lanes": 3, "narrow_rows": false}, {"concurrent_lanes": 3}, {"concurrent_lanes": 4}, {"concurrent_lanes": 8}]' 5 > gpurun_out/ab_narrow.log 2>&1; echo "ab rc=$?"
tail -6 gpurun_out/ab_narrow.log
timeout 900 python scripts/step_ab.py softmax '[{"narrow_rows": false}, {}]' 3 > gpurun_out/ab_narrow_softmax.log 2>&1; tail -2 gpurun_out/ab_narrow_softmax.log
