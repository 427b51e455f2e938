#!/bin/bash
# round-2 pass V: staged-slot classes for every record (KF_TILE_SLOTS=free)
# vs own slot = lane (round 1) -- A/B, bank conflicts, tile/parity tests
mkdir -p gpurun_out
for r in 1 2; do for sl in free lane; do for case in 5 2; do
  KF_TILE_SLOTS=$sl timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/v.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/v.json'));k=b['kernels_ms'];print('$sl case $case', round(b['value'],1), 'ms', round(b['ms_per_step'],3), 'g1', round(k['grad_pass1']['ms'],3), 'gk', round(k['grad_passk']['ms'],3), 'flux', round(k['flux_residual']['ms'],3))"
done; done; done
for sl in free lane; do
KF_TILE_SLOTS=$sl timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,gpu__time_duration.sum --clock-control none -k regex:"k_grad_t|k_residual_t" -s 4 -c 4 --csv --log-file gpurun_out/bank_$sl.csv python bench.py --case 2 --profile-only --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/bank_$sl.csv') if l.startswith('"'))]
h=rows[0]; ki,mi,vi=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value')
import collections; d=collections.defaultdict(dict)
for r in rows[1:]: d[(r[0],r[ki][:22])][r[mi]]=float(r[vi].replace(',',''))
for (i,k),m in d.items(): print('$sl', k, 'conflicts/wavefronts %.3f' % (m['l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum']/m['l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum']), 'us %.1f' % (m['gpu__time_duration.sum']/1e3))
PY
done
timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py tests/test_gpu_partition.py -x -q 2>&1 | tail -2
