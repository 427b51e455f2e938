#!/bin/bash
# GPU session (run under gpurun from the repo root): smoke, GPU tests (both
# residual-kernel variants), bench, ncu launch list and --set full captures of
# the per-iteration kernels. Every step has its own timeout.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
KF_FLUX_KERNEL=${ALT_FLUX:-m4fast} timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu_alt.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_alt.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
KF_FLUX_KERNEL=${ALT_FLUX:-m4fast} timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_alt.json 2> gpurun_out/bench_alt.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_residual|k_grad|k_forward|k_backward|k_update" -s 12 -c 10 -o gpurun_out/prof_full python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
echo done
