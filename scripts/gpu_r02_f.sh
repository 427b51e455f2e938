#!/bin/bash
# round-2 pass F: overlapped halo exchanges (partitioned transports) -- GPU
# tests of every partitioned path, then the in-process 4-partition bench with
# the overlap on / off (config 2 and config 5)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_partition.py tests/test_gpu_multirank.py tests/test_gpu_parity.py tests/test_gpu_integration.py tests/test_gpu_orderings.py -x -q > gpurun_out/pytest_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f.log
tail -3 gpurun_out/pytest_f.log
for case in 2 5; do
for ov in 1 0; do
  KF_OVERLAP=$ov timeout 900 python bench.py --case $case --parts 4 --no-cpu-baseline --no-extras --steps 10 > gpurun_out/p4_c${case}_ov$ov.json 2> gpurun_out/p4_c${case}_ov$ov.err
  python -c "import json;b=json.load(open('gpurun_out/p4_c${case}_ov$ov.json'));print('case $case parts 4 overlap $ov', round(b['value'],1), 'ms/step', round(b['ms_per_step'],3))"
done
timeout 900 python bench.py --case $case --no-cpu-baseline --no-extras --steps 10 > gpurun_out/p1_c${case}.json 2>/dev/null
python -c "import json;b=json.load(open('gpurun_out/p1_c${case}.json'));print('case $case parts 1', round(b['value'],1), 'ms/step', round(b['ms_per_step'],3))"
done
