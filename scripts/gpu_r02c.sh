#!/bin/bash
# Exact whole-graph BERT plan (135 groups): re-tune its per-group variants,
# then the GPU suite and the default bench with the new table.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py --configs bert --out gpurun_out/bench_bert_untuned.json > gpurun_out/bench_bert_untuned.log 2>&1; echo "bench bert untuned rc=$?"
timeout 2400 python scripts/tune_variants.py bert --out gpurun_out/kv_bert.json > gpurun_out/tune_bert.log 2>&1; echo "tune rc=$?"
tail -3 gpurun_out/tune_bert.log
cp gpurun_out/kv_bert.json paper_1911_11576_b200/data/kernel_variants/bert.json
timeout 900 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
