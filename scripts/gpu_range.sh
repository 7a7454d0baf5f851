#!/bin/bash
mkdir -p gpurun_out
for o in '{"concurrent_lanes": 1}' '{"concurrent_lanes": 3}'; do
  timeout 600 ncu --replay-mode app-range --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum \
    python scripts/step_range.py bert "$o" > gpurun_out/range_$(echo $o | tr -dc '0-9').log 2>&1; echo "rc=$?"
  grep -E "dram__|gpu__time|lts__|algo" gpurun_out/range_$(echo $o | tr -dc '0-9').log
done
