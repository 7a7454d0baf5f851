#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_executor_gpu.py -q -x -k "discard or dataflow or anchored" > gpurun_out/pytest_discard.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_discard.log
timeout 900 python scripts/step_ab.py bert '[{"l2_discard": false}, {}]' 6 | tail -2
for o in '{"l2_discard": false}' '{}'; do
  timeout 600 ncu --replay-mode app-range --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum \
    python scripts/step_range.py bert "$o" 2>&1 | grep -E "dram__" ; done
