#!/bin/bash
# density exp through a warp vote (KF_EXP_VOTE, per state) or per pair
# (KF_KIN_PAIR) vs the build without (libkf_base): bitwise + bench A/B
mkdir -p gpurun_out
for lib in libkf libkf_pair libkf_base; do
KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so python - <<PY
import numpy as np, paper_2406_07441_b200 as kf
c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
h = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=200)).run()
np.save("gpurun_out/state_$lib.npy", h.final_state); np.save("gpurun_out/res_$lib.npy", h.residual)
PY
done
python -c "
import numpy as np
b=np.load('gpurun_out/state_libkf_base.npy'); rb=np.load('gpurun_out/res_libkf_base.npy')
for l in ('libkf','libkf_pair'): print(l, 'bitwise vs base', np.array_equal(np.load(f'gpurun_out/state_{l}.npy'), b), np.array_equal(np.load(f'gpurun_out/res_{l}.npy'), rb))" | tee gpurun_out/expvote_ab.txt
for r in 1 2; do for lib in libkf libkf_pair libkf_base; do for case in 5 2; do
  KF_LIB_PATH=$PWD/paper_2406_07441_b200/$lib.so timeout 600 python bench.py --case $case --no-cpu-baseline --no-extras --steps 20 > gpurun_out/e.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/e.json'));k=b['kernels_ms'];print('$lib case $case', round(b['value'],1), *[f'{n} {round(v[\"ms\"],4)}' for n,v in k.items()])"
done; done; done 2>&1 | tee -a gpurun_out/expvote_ab.txt
