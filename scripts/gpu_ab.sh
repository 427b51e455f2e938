#!/bin/bash
# A/B of kernel variants + tests (run under gpurun from the repo root)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in "lanes2 lanes8" "lanes3 lanes8" "point point" "lanes2 point"; do
  set -- $v
  KF_FLUX_KERNEL=$1 KF_GRAD_KERNEL=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$1_$2.json 2> gpurun_out/bench_$1_$2.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_residual16|k_grad8" -s 4 -c 3 -o gpurun_out/prof_r2 python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo done
