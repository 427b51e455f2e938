#!/bin/bash
# FP64 instruction counts of the flux-residual kernel (one launch) for roofline.fp64
mkdir -p gpurun_out
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum --clock-control none -k regex:k_residual -s 1 -c 2 --csv --log-file gpurun_out/fp64.csv python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_fp64.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fp64.log
