#!/bin/bash
# Round-2 GPU call b: new parity tests (reference sketches, advice regressions).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_ref_sketches.py tests/test_executor_gpu.py -m gpu -q -x \
  -k "ref_sketch or fixture_gpu or chunked_segment or colred_output or own_device" > gpurun_out/pytest_r02b.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_r02b.log
