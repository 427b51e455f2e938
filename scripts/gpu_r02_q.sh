#!/bin/bash
mkdir -p gpurun_out
KF_TIME_INGEST=1 timeout 600 python scripts/time_setup.py 10240:3920 > gpurun_out/setup_c5.log 2>&1; tail -18 gpurun_out/setup_c5.log
for c in 5 2; do timeout 600 python bench.py --case $c --no-cpu-baseline --no-extras --steps 20 > gpurun_out/q_c$c.json 2>/dev/null; python -c "import json;b=json.load(open('gpurun_out/q_c$c.json'));print('case $c', round(b['value'],1), 'ms', round(b['ms_per_step'],3))"; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log; tail -3 gpurun_out/pytest_q.log
