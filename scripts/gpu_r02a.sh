#!/bin/bash
# Round-2 first GPU call: smoke, GPU parity, bench, ncu --set full of the
# kernels the verdict names (GRU fusion_0, BERT fusion_5 / fusion_38).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^fusion_0$' -c 2 \
  -o gpurun_out/r02_gru_full python scripts/profile_configs.py --configs gru --iters 1 > gpurun_out/ncu_gru.log 2>&1; echo "ncu gru rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(fusion_5|fusion_38)$' -c 2 \
  -o gpurun_out/r02_bert_full python scripts/profile_configs.py --configs bert --iters 1 > gpurun_out/ncu_bert.log 2>&1; echo "ncu bert rc=$?"
ls -la gpurun_out
