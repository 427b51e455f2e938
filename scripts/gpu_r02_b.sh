#!/bin/bash
# round-2 pass B (run under gpurun): new GPU tests, ingest/pack timing at
# 40M points, ncu evidence of one config-5 iteration (launch list, FP64
# counts, --set full of the 13 launches)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_orderings.py tests/test_gpu_advice.py tests/test_gpu_tiles.py tests/test_gpu_partition.py -x -q > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b.log
timeout 600 python scripts/time_setup.py 10240:3920 > gpurun_out/setup_c5.log 2>&1
A="python bench.py --profile-only --steps 1 --warmup 3 --no-cpu-baseline"
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum
K='regex:k_grad_t|k_residual_t|k_forward|k_backward|k_update|k_finalize'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $A > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --metrics $M --clock-control none -k "$K" -s 13 -c 13 --csv --log-file gpurun_out/fp64_c5.csv $A > gpurun_out/ncu_fp64.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_fp64.log
timeout 1800 ncu --set full --clock-control none --import-source on -k "$K" -s 13 -c 13 -o gpurun_out/full_c5 $A > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
tail -3 gpurun_out/pytest_b.log; tail -1 gpurun_out/ncu_*.log; cat gpurun_out/setup_c5.log | tail -15
