"""Diagnostic: where does the GPU config-1 trajectory leave the reference?"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import paper_2406_07441_b200 as kf
from util import oracle_for, normrel

h = np.load(os.path.join(ROOT, "tests/golden/config1_history.npz"))
c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
o = oracle_for(c)
mk = lambda n: kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=n)
r = kf.Solver(c, mk(1000)).run()
res = r.residual
m = min(len(res), len(h["residual"]))
rel = np.abs(res[:m] - h["residual"][:m]) / np.abs(h["residual"][:m])
print("iters", len(res), "reason", r.abort_reason, "point", r.abort_point)
for t in (1e-14, 1e-12, 1e-10, 1e-8, 1e-4):
    idx = np.flatnonzero(rel > t)
    print(f"first iter rel>{t:g}:", idx[0] + 1 if len(idx) else None)
print("rel at", [(k, float(rel[k-1])) for k in (1, 10, 50, 100, 200, 300, 400, 420, m) if k <= m])
for n in (100, 300, 420, 422):
    rg = kf.Solver(c, mk(n)).run()
    ro = o.run(variant="manish_ad", n_iterations=n, mach=0.63, aoa_deg=2.0, cfl=0.2)
    d = np.abs(rg.final_state - ro.final_state).max(1)
    top = np.argsort(-d)[:5]
    print(n, "state normrel", normrel(rg.final_state, ro.final_state), "top", [(int(p), float(d[p])) for p in top])
# iteration 423 stage by stage from the oracle's 422 state (host stage hooks)
ro = o.run(variant="manish_ad", n_iterations=422, mach=0.63, aoa_deg=2.0, cfl=0.2)
U = ro.final_state
s = kf.Solver(c, mk(10))
q = o.q(U); qx, qy = o.grads(q, 3); R, _ = o.residual(q, qx, qy)
print("q", normrel(s.q(U), q))
gx, gy = s.grads(q); print("grads", normrel(gx, qx), normrel(gy, qy))
Rg, _ = s.residual(q, qx, qy); print("R", normrel(Rg, R))
# dU_prev of iteration 422: rerun 421 and take the difference of states is not exact; use zero and S check
try:
    out = s.lusgs(U, R, np.zeros_like(U), 0.2)
    print("lusgs ok", float(np.abs(out["dU"]).max()))
except Exception as e:
    print("lusgs error", e)
