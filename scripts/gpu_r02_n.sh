#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for lanes in bfs id; do
  KF_TILE_LANES=$lanes timeout 600 python bench.py --case 5 --no-cpu-baseline --no-extras --steps 20 > gpurun_out/lanes2_${lanes}_$rep.json 2>/dev/null
  KF_TILE_LANES=$lanes timeout 600 python bench.py --case 5 --restart --no-cpu-baseline --no-extras --steps 20 > gpurun_out/lanes2r_${lanes}_$rep.json 2>/dev/null
  for m in lanes2 lanes2r; do python -c "import json;b=json.load(open('gpurun_out/${m}_${lanes}_$rep.json'));k=b['kernels_ms'];print('$m $lanes rep $rep', round(b['value'],1), 'ms', round(b['ms_per_step'],3), 'sum', round(sum(v['ms'] for v in k.values()),3), 'gk', round(k['grad_passk']['ms'],3), 'flux', round(k['flux_residual']['ms'],3))"; done
done
done
