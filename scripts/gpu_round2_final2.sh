#!/bin/bash
# Round-2 evidence pass on the final tree (dataflow launch, split folds,
# narrow rows, L2 discard): smoke, GPU parity suite, default bench, reference
# arm, ncu launch list, ncu --set full of the bench-cited kernels, whole-step
# DRAM traffic (range replay) for BERT.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --out gpurun_out/bench_ref.json > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python scripts/profile_configs.py --iters 1 > gpurun_out/launches.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^fusion_0$' -c 1 \
  -o gpurun_out/r02_encoder_full python scripts/profile_configs.py --configs encoder --iters 1 > gpurun_out/ncu_enc.log 2>&1; echo "ncu encoder rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^fusion_0$' -c 1 \
  -o gpurun_out/r02_gru_gws python scripts/profile_configs.py --configs gru --iters 1 > gpurun_out/ncu_gru.log 2>&1; echo "ncu gru rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(fusion_62|fusion_6|fusion_6_fold|fusion_123)$' -c 4 \
  -o gpurun_out/r02_bert_top python scripts/profile_configs.py --configs bert --iters 1 > gpurun_out/ncu_bert.log 2>&1; echo "ncu bert rc=$?"
for o in '{"concurrent_lanes": 1, "l2_discard": false}' '{}'; do
  timeout 600 ncu --replay-mode app-range --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum \
    python scripts/step_range.py bert "$o" > gpurun_out/range_$(echo $o | tr -dc 'a-z0-9' | head -c 20).log 2>&1; echo "range rc=$?"; done
timeout 600 python scripts/trace_step.py bert '[{"concurrent_lanes": 1}, {}]' > gpurun_out/trace.log 2>&1; echo "trace rc=$?"
