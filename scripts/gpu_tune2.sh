#!/bin/bash
mkdir -p gpurun_out
timeout 2200 python scripts/tune_variants.py bert --out gpurun_out/bert_variants.json > gpurun_out/tune_bert.log 2>&1; echo "tune rc=$?"
tail -7 gpurun_out/tune_bert.log
timeout 2400 python -m pytest tests/test_executor_gpu.py -q -x -k "variants_parity or anchored or dataflow" > gpurun_out/pytest_var.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_var.log
