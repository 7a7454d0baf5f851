#!/bin/bash
# Re-entry check after the container was recreated: smoke, GPU parity suite,
# default bench on the current commit.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.log
