#!/bin/bash
# FP64 instruction counts (run under gpurun): the flux-residual kernel (one
# launch, for roofline.fp64) and every kernel of one whole iteration (13
# launches, for roofline.iteration)
mkdir -p gpurun_out
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:k_residual -s 1 -c 2 --csv --log-file gpurun_out/fp64.csv python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_fp64.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fp64.log
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_grad_t|k_residual_t|k_forward|k_backward|k_update|k_finalize" -s 13 -c 13 --csv --log-file gpurun_out/fp64_iter.csv python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_fp64_iter.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fp64_iter.log
