#!/bin/bash
# Round-2 evidence pass: smoke, GPU parity suite, default bench, reference
# arm, ncu launch list (time + DRAM + L2-write traffic per launch), ncu
# --set full of the bench-cited kernels.
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
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(fusion_5|fusion_38)$' -c 2 \
  -o gpurun_out/r02_bert_top python scripts/profile_configs.py --configs bert --iters 1 > gpurun_out/ncu_bert.log 2>&1; echo "ncu bert rc=$?"
