#!/bin/bash
# Evidence part 1 (run under gpurun): smoke, all GPU tests, ncu launch list,
# ncu --set full of every per-iteration kernel, FP64 counts of the flux kernel.
# (Part 2, scripts/gpu_evidence_bench.sh, runs the bench with the FP64 and
# traffic figures summarised from this part.)
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_residual|k_grad|k_forward|k_backward|k_update|k_q_from_u|k_finalize" -s 14 -c 14 -o gpurun_out/prof_full python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
bash scripts/gpu_fp64.sh
echo done
