"""Where does a NaN first appear (debug-build triage, dev tool)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2312_07725_b200 as pkg  # noqa: E402

for m in [int(a) for a in sys.argv[1:]] or [64, 128]:
    g = pkg.GpuSolver(pkg.SolverConfig(p=4, m=m, c1d=0.5 * 4.67e-5))
    jac, cof = g.metrics()
    r = {"m": m, "metrics_finite": bool(np.isfinite(jac).all() and np.isfinite(cof).all())}
    g.init_case()
    uq = g.get_state_q()
    r["uq_finite"] = bool(np.isfinite(uq).all())
    u = g.get_state()
    r["u_finite"] = bool(np.isfinite(u).all())
    d = g.rhs()
    bad = ~np.isfinite(d)
    r["rhs_nonfinite"] = int(bad.sum())
    if bad.any():
        e = np.nonzero(bad.any(axis=(1, 2)))[0]
        r["bad_elems"] = [int(e.min()), int(e.max()), int(len(e))]
    tr = g.traces()
    r["traces_nonfinite"] = int((~np.isfinite(tr)).sum())
    print(r, flush=True)
    g.close()
