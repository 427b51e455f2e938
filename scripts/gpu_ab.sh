#!/bin/bash
# kernel-variant A/B + GPU tests (run under gpurun from the repo root)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=240 -x -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in m3 m4 m3fast m4fast; do
  KF_FLUX_KERNEL=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_residual|k_grad|k_forward" -s 6 -c 5 -o gpurun_out/prof_r3 python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo done
