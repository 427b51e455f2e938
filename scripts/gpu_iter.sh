#!/bin/bash
# build-check iteration on the GPU: tests, bench A/B, ncu of the main kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in ${KF_VARIANTS:-m3 m4fast}; do
  KF_FLUX_KERNEL=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_residual|k_grad|k_forward|k_backward|k_update" -s 12 -c 12 -o gpurun_out/prof_iter python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
