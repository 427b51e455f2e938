#!/bin/bash
# Dataflow sweeps, second build (one release MEMBAR per slice, no acquire
# fence, products read through L2): parity, A/B at configs 5 and 2, spin
# statistics, ncu DRAM bytes of the sweep kernels (per-colour vs dataflow).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dataflow.py -q -x -p no:cacheprovider > gpurun_out/df_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/df_pytest.log
tail -2 gpurun_out/df_pytest.log
grep -q "pytest rc=0" gpurun_out/df_pytest.log || exit 1
for r in 1 2; do for case in 5 2; do for df in 0 1; do
  KF_SWEEP_DF=$df timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/df.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/df.json'));k=b['kernels_ms'];print('df=$df case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])"
done; done; done 2>&1 | tee gpurun_out/df_ab.txt
KF_SWEEP_DF=1 KF_LIB_PATH=$PWD/paper_2406_07441_b200/libkf_dfstats.so timeout 600 python bench.py --case 5 --no-cpu-baseline --no-extras --steps 3 --warmup 3 2>&1 | grep "df epoch" | head -12 > gpurun_out/df_stats.txt
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for df in 0 1; do
KF_SWEEP_DF=$df timeout 900 ncu --metrics $M --clock-control none -k regex:'k_forward|k_backward' -s 14 -c 7 --csv --log-file gpurun_out/df_ncu_$df.csv python bench.py --profile-only --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
cat gpurun_out/df_stats.txt
