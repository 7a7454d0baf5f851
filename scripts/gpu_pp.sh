#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_executor_gpu.py -q -x > gpurun_out/pytest_pp.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_pp.log
timeout 900 python scripts/step_ab.py bert '[{}, {"pp_reduce": false}]' 10 | tail -2
for c in layernorm encoder softmax; do timeout 600 python scripts/step_ab.py $c '[{}, {"pp_reduce": false}]' 4 | tail -2; done
