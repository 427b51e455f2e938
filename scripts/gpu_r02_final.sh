#!/bin/bash
# round-2 final evidence (run under gpurun): smoke, ncu evidence of one
# config-5 iteration (FP64 counts, --set full DRAM traffic + brief, launch
# list; converted on the box so bench.py reads the current build's counts),
# the bench line and the reference arm, BASELINE configs 2-4, setup timing,
# the full GPU suite. Everything lands in gpurun_out/.
mkdir -p gpurun_out
N5=40140800
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
A="python bench.py --profile-only --steps 1 --warmup 3 --no-cpu-baseline"
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum
K='regex:k_grad_t|k_residual_t|k_forward|k_backward|k_update|k_finalize'
timeout 900 ncu --metrics $M --clock-control none -k "$K" -s 13 -c 13 --csv --log-file gpurun_out/fp64_c5.csv $A > gpurun_out/ncu_fp64.log 2>&1
python scripts/r02_ncu_json.py fp64 gpurun_out/fp64_c5.csv 5 $N5 > /dev/null && cp profiles/r02_fp64_case5.json gpurun_out/
timeout 1800 ncu --set full --clock-control none --import-source on -k "$K" -s 13 -c 13 -o gpurun_out/full_c5 $A > gpurun_out/ncu_full.log 2>&1
python scripts/r02_ncu_json.py traffic gpurun_out/full_c5.ncu-rep 5 $N5 > /dev/null && cp profiles/r02_traffic_case5.json gpurun_out/
python scripts/ncu_brief.py gpurun_out/full_c5.ncu-rep > gpurun_out/r02_ncu_brief_case5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $A > gpurun_out/ncu_launch.log 2>&1
python scripts/r02_ncu_json.py launch gpurun_out/launches_c5.csv gpurun_out/r02_launches_case5.txt > /dev/null
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?" >> gpurun_out/bench_final.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err
for c in 2 3 4; do timeout 900 python bench.py --case $c --no-cpu-baseline --no-extras > gpurun_out/bench_case${c}_final.json 2>/dev/null; done
KF_TIME_INGEST=1 timeout 600 python scripts/time_setup.py 10240:3920 > gpurun_out/setup_c5.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final.log
tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench_final.err; tail -3 gpurun_out/pytest_final.log
python -c "import json;b=json.load(open('gpurun_out/bench_final.json'));print(b['value'], b['e2e']['value'], b['roofline']['fp64'])"
