#!/bin/bash
mkdir -p gpurun_out
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 30 $CASEARG > gpurun_out/p.json 2>/dev/null; python -c "import json;b=json.load(open('gpurun_out/p.json'));print('$* $CASEARG', round(b['value'],1), 'ms', round(b['ms_per_step'],3))"; }
for r in 1 2 3; do run KF_PDL=1; run KF_PDL=0; done
CASEARG="--case 4"; for r in 1 2; do run KF_PDL=1; run KF_PDL=0; done
CASEARG="--case 2"; for r in 1 2; do run KF_PDL=1; run KF_PDL=0; done
KF_TIME_INGEST=1 timeout 600 python scripts/time_setup.py 10240:3920 > gpurun_out/setup_c5.log 2>&1; tail -18 gpurun_out/setup_c5.log
