"""Exact call sequence of test_config5_oracle_parity_on_planes (debug triage)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2312_07725_b200 as pkg  # noqa: E402

for m in [int(a) for a in sys.argv[1:]]:
    g = pkg.GpuSolver(pkg.SolverConfig(p=4, m=m, c1d=0.5 * 4.67e-5))
    g.init_case()
    lam = g.max_wavespeed()
    u = g.get_state()
    d = g.rhs()
    bad = ~np.isfinite(d)
    r = {"m": m, "lam": lam, "u_finite": bool(np.isfinite(u).all()), "rhs_nonfinite": int(bad.sum())}
    if bad.any():
        e = np.nonzero(bad.any(axis=(1, 2)))[0]
        r["bad_elems"] = [int(e.min()), int(e.max()), int(len(e))]
        r["bad_states"] = np.nonzero(bad.any(axis=(0, 2)))[0].tolist()
    d2 = g.rhs()
    r["rhs2_nonfinite"] = int((~np.isfinite(d2)).sum())
    print(r, flush=True)
    g.close()
