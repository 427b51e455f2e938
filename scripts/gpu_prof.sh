#!/bin/bash
# ncu --set full of the per-iteration kernels + residual-kernel A/B (run under gpurun)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout=300 -k config1 > gpurun_out/pytest_cfg1.log 2>&1
for v in m3 m4 m3fast m4fast; do
  KF_FLUX_KERNEL=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_residual|k_grad|k_forward|k_backward|k_update" -s 12 -c 8 -o gpurun_out/prof_r1 python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
