#!/bin/bash
# One gpurun call: smoke, GPU parity tests, bench, ncu launch list and a
# --set full capture of the stitched kernels. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python scripts/profile_configs.py --unfused --iters 2 > gpurun_out/launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'fusion|dbias' -c 12 \
  -o gpurun_out/prof_full python scripts/profile_configs.py --iters 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 --out gpurun_out/bench_ref.json > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
