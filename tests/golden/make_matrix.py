"""Golden fixtures of a configuration matrix, from the UNMODIFIED reference.

    python tests/golden/make_matrix.py     (build container: needs oracle/_ref)

Covers the SolverConfig knobs the other fixtures keep fixed: n_inner 1, 2, 4,
the CFL ramp (driver.cpp:222-227), free-stream BCs (driver.hpp:25), a
cambered section, the convergence stop and the divergence stop
(driver.cpp:263-275), a pressure abort, an explicit partial-update abort
(driver.cpp:97-112) and an abort in the first iteration (no record). Writes config_matrix.npz: per case the residual, CL,
CD and first-order histories, the stop flags/reason and the final state.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from refpy import Reference  # noqa: E402

# name: (cloud (digits, n_wall, n_radial, radius), SolverConfig fields)
CASES = {
    "cambered_n1": (("2412", 65, 9, 11.0),
                    dict(variant="manish_ad", n_inner=1, mach=0.5, aoa_deg=4.0, cfl=0.2, n_iterations=40)),
    "ramp_n2": (("0012", 48, 12, 12.0),
                dict(variant="anandh", n_inner=2, mach=0.63, aoa_deg=2.0, cfl=0.3, cfl_ramp_iters=10,
                     cfl_start=0.05, n_iterations=40)),
    "freestream_bc_n4": (("0012", 48, 12, 12.0),
                         dict(variant="manish", n_inner=4, mach=0.7, aoa_deg=1.5, cfl=0.2,
                              bc_mode="freestream", n_iterations=40)),
    "explicit_ramp": (("0012", 48, 12, 12.0),
                      dict(variant="explicit", mach=0.63, aoa_deg=2.0, cfl=0.05, cfl_ramp_iters=5,
                           n_iterations=30)),
    "converge_stop": (("0012", 64, 16, 12.0),
                      dict(variant="manish_ad", mach=0.5, aoa_deg=1.0, cfl=0.2, convergence_decades=0.25,
                           n_iterations=400)),
    "diverge_stop": (("0012", 48, 12, 12.0),
                     dict(variant="manish_ad", mach=0.63, aoa_deg=2.0, cfl=0.5, divergence_factor=1.2,
                          n_iterations=80)),
    "pressure_abort": (("0012", 48, 12, 12.0),
                       dict(variant="manish_ad", mach=0.63, aoa_deg=2.0, cfl=0.5, divergence_factor=5.0,
                            n_iterations=80)),
    "explicit_abort": (("0012", 48, 12, 12.0),
                       dict(variant="explicit", mach=0.63, aoa_deg=2.0, cfl=0.5, divergence_factor=5.0,
                            n_iterations=80)),
    "first_iteration_abort": (("0012", 48, 12, 12.0),
                              dict(variant="explicit", mach=0.63, aoa_deg=2.0, cfl=2.0, n_iterations=10)),
}


def main():
    out, meta = {}, {}
    for name, (cl, cfg) in CASES.items():
        ref = Reference.generate(*cl)
        r = ref.run(**cfg)
        out[name + "_residual"] = r.residual
        out[name + "_cl"] = r.cl
        out[name + "_cd"] = r.cd
        out[name + "_first_order"] = r.first_order
        out[name + "_final"] = r.final_state
        meta[name] = {"cloud": cl, "cfg": cfg, "iters": int(len(r.residual)), "diverged": bool(r.diverged),
                      "reason": r.abort_reason}
        print(name, len(r.residual), r.diverged, repr(r.abort_reason))
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "config_matrix.npz"), **out)


if __name__ == "__main__":
    main()
