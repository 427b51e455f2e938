#!/bin/bash
# round-2 pass M: lane order inside the SMEM tiles (bank conflicts) -- A/B
mkdir -p gpurun_out
for lanes in bfs id morton; do
for case in 5 2; do
  KF_TILE_LANES=$lanes timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 10 > gpurun_out/lanes_${lanes}_c$case.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/lanes_${lanes}_c$case.json'));k=b['kernels_ms'];print('$lanes case $case', round(b['value'],1), 'g1', round(k['grad_pass1']['ms'],3), 'gk', round(k['grad_passk']['ms'],3), 'flux', round(k['flux_residual']['ms'],3))"
done
done
KF_TILE_LANES=id timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
