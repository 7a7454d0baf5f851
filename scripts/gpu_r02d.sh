#!/bin/bash
# GEMM scheme tests + timing; ncu launch list and --set full of the top
# kernels of the exact BERT plan; default bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_executor_gpu.py -q -k "gemm" > gpurun_out/pytest_gemm.log 2>&1; echo "pytest gemm rc=$?"
tail -2 gpurun_out/pytest_gemm.log
timeout 600 python scripts/gemm_perf.py gpurun_out/gemm_perf.json > gpurun_out/gemm_perf.log 2>&1; echo "gemm perf rc=$?"
cat gpurun_out/gemm_perf.log | tail -5
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python scripts/profile_configs.py --iters 1 > gpurun_out/launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(fusion_40|fusion_6|fusion_62)$' -c 3 \
  -o gpurun_out/r02_bert_top python scripts/profile_configs.py --configs bert --iters 1 > gpurun_out/ncu_bert.log 2>&1; echo "ncu bert rc=$?"
timeout 900 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
