#!/bin/bash
# exp(-s^2) without kf_exp's range selects on the flux kernel's |s|<1 path
# (both endpoint states of a direction under one erf vote): bitwise check vs the previous build, bench A/B, parity tests
mkdir -p gpurun_out
for lib in libkf libkf_prev; do
KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so python - <<PY
import numpy as np, paper_2406_07441_b200 as kf
c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
h = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=200)).run()
np.save("gpurun_out/state_$lib.npy", h.final_state); np.save("gpurun_out/res_$lib.npy", h.residual)
PY
done
python -c "import numpy as np; a=np.load('gpurun_out/state_libkf.npy'); b=np.load('gpurun_out/state_libkf_prev.npy'); print('bitwise state', np.array_equal(a,b), 'residual', np.array_equal(np.load('gpurun_out/res_libkf.npy'), np.load('gpurun_out/res_libkf_prev.npy')))" | tee gpurun_out/split2_ab.txt
for r in 1 2; do for lib in libkf libkf_prev; do for case in 5 2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/e.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/e.json'));k=b['kernels_ms'];print('$lib case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])"
done; done; done 2>&1 | tee -a gpurun_out/split2_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2 | tee -a gpurun_out/split2_ab.txt
