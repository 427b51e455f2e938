#!/bin/bash
# Dataflow sweeps (KF_SWEEP_DF): parity tests first (bounded), then the
# bench A/B per-colour launches vs dataflow at configs 5, 4 and 2.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dataflow.py -q -x -p no:cacheprovider > gpurun_out/df_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/df_pytest.log
tail -3 gpurun_out/df_pytest.log
grep -q "pytest rc=0" gpurun_out/df_pytest.log || exit 1
for r in 1 2; do for case in 5 4 2; do for df in 0 1; do
  KF_SWEEP_DF=$df timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/df.json 2>gpurun_out/df_$case_$df.err
  python -c "import json;b=json.load(open('gpurun_out/df.json'));k=b['kernels_ms'];print('df=$df case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])" || tail -5 gpurun_out/df_$case_$df.err
done; done; done 2>&1 | tee gpurun_out/df_ab.txt
