"""Golden fixtures for the two largest BASELINE clouds, made by the
UNMODIFIED reference (oracle/_ref): config 4 (NACA 0012 5120x1920, 9,830,400
points) and config 5 (10240x3920, 40,140,800 points).

The reference needs ~15 GB / ~60 GB of host memory for them, so this runs on
the GPU box (which has oracle/_ref and 196 GB), writing into gpurun_out/:

    python tests/golden/make_large_golden.py gpurun_out/large_configs.json

and the file is copied to tests/golden/large_configs.json. Per config: the
sha256 of every ingested array (make_golden.ingest_hashes: geometry, the five
CSR stencils, LS weights and classes, ls_one, colours) and a 6-iteration
manish_ad history at M 0.63, AoA 2, CFL 0.2 (residual, CL, CD, first-order
counts, abort record) plus every 9973rd row of the final state.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from make_golden import ingest_hashes, sha  # noqa: E402
from refpy import Reference  # noqa: E402

CLOUDS = {"config4": ("0012", 5120, 1920, 20.0), "config5": ("0012", 10240, 3920, 20.0)}
RUN = dict(variant="manish_ad", n_iterations=6, mach=0.63, aoa_deg=2.0, cfl=0.2)
ROW_STRIDE = 9973


def make(name):
    spec = CLOUDS[name]
    t0 = time.perf_counter()
    ref = Reference.generate(*spec)
    out = {"spec": list(spec), "run": RUN, "row_stride": ROW_STRIDE, "hashes": ingest_hashes(ref)}
    r = ref.run(**RUN)
    out.update(residual=r.residual.tolist(), cl=r.cl.tolist(), cd=r.cd.tolist(),
               first_order=r.first_order.tolist(), diverged=bool(r.diverged), abort_reason=r.abort_reason,
               final_state_sha=sha(r.final_state), final_rows=r.final_state[::ROW_STRIDE].tolist(),
               seconds=(time.perf_counter() - t0))
    return out


def main(path):
    Reference.num_threads(os.cpu_count() or 1)
    data = {}
    for name in sys.argv[2:] or sorted(CLOUDS):
        data[name] = make(name)
        print(name, data[name]["hashes"]["n"], f"{data[name]['seconds']:.0f}s", flush=True)
    with open(path, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "large_configs.json"))
