"""Probe: two ranks of the NCCL transport on ONE GPU (NCCL normally refuses
duplicate devices in a communicator; this records what it does here)."""
import os, sys, json
import multiprocessing as mp
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def worker(rank, world, nid, q):
    try:
        import numpy as np
        import paper_2406_07441_b200 as kf
        c = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
        cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2,
                              n_iterations=40, device=0)
        s = kf.Solver.for_rank(c, cfg, world, rank, nid)
        r = s.run()
        q.put((rank, "ok", [float(x) for x in r.residual[:3]], len(r.iters), r.final_state.tolist()))
    except Exception as e:
        q.put((rank, "error", repr(e), 0, None))

if __name__ == "__main__":
    import paper_2406_07441_b200 as kf
    nid = kf.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, nid, q)) for r in range(2)]
    for p in ps: p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in ps: p.join(timeout=60)
    import numpy as np
    out = {"ranks": [(r[0], r[1], r[2], r[3]) for r in res]}
    if all(r[1] == "ok" for r in res):
        c = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
        one = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0,
                                           cfl=0.2, n_iterations=40)).run()
        owner = kf.partition_plan(c, 2, "angular")
        st = np.zeros_like(one.final_state)
        for r in res:
            f = np.array(r[4]); m = owner == r[0]; st[m] = f[m]
        out["state_bitwise_equal"] = bool(np.array_equal(st, one.final_state))
        out["residual_single"] = [float(x) for x in one.residual[:3]]
    print(json.dumps(out))
