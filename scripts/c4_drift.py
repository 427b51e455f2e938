"""Evidence (GPU box): where the config-4 whole run (9.8M points, 116
iterations to the reference's own abort) drifts from the reference, per
iteration, for the default flux kernel and for the libdevice-exact one
(KF_FLUX_KERNEL=m3), against ONE reference run. Writes JSON (argv[1])."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
N_IT = 140


def gpu_history(env):
    code = ("import sys,json; sys.path.insert(0, %r); import paper_2406_07441_b200 as kf; "
            "c = kf.generate_naca_ogrid('0012', 5120, 1920, 20.0); "
            "h = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, "
            "cfl=0.2, n_iterations=%d)).run(); "
            "print(json.dumps({'res': list(h.residual), 'cl': list(h.cl), 'abort': h.abort_reason}))" % (ROOT, N_IT))
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                         check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


import refpy  # noqa: E402

refpy.Reference.num_threads(os.cpu_count() or 1)
r = refpy.Reference.generate("0012", 5120, 1920, 20.0).run(variant="manish_ad", n_iterations=N_IT, mach=0.63,
                                                            aoa_deg=2.0, cfl=0.2)
out = {"ref_iterations": len(r.residual), "ref_abort": r.abort_reason, "ref_residual": list(map(float, r.residual))}
for tag, env in [("default", {}), ("m3", {"KF_FLUX_KERNEL": "m3"})]:
    g = gpu_history(env)
    n = min(len(g["res"]), len(r.residual))
    rel = np.abs(np.array(g["res"][:n]) - r.residual[:n]) / np.abs(r.residual[:n])
    out[tag] = {"iterations": len(g["res"]), "abort": g["abort"], "rel": list(map(float, rel)),
                "first_above_1e-10": int(np.argmax(rel > 1e-10)) + 1 if (rel > 1e-10).any() else None,
                "max": float(rel.max())}
    print(tag, out[tag]["iterations"], out[tag]["abort"], "max", out[tag]["max"], "first >1e-10 at",
          out[tag]["first_above_1e-10"], flush=True)
with open(sys.argv[1], "w") as f:
    json.dump(out, f)
