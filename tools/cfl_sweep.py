"""Maximum-CFL sweep (SPEC.md cfl_sweep; PAPER.md:1604-1673 procedure) with the
GPU solver: run to t_f = 1.0 at CFL 0.1, then raise the CFL by 0.01 and rerun
until the pressure L2 error at t_f differs from the CFL 0.1 value in its
seventh significant digit (relative change > 5e-7) or the run fails.

The paper sweeps its manufactured solution (not part of this build); this
uses the isentropic vortex on the same warped 4^3 grid, so the numbers are
this case's, and the claim checked is the ordering maxCFL(c_+) >= maxCFL(c_DG).

    python tools/cfl_sweep.py [m]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07725_b200 as nsfr  # noqa: E402


def pressure_error(cfg, cfl):
    g = nsfr.GpuSolver(cfg)
    try:
        g.init_case()
        t = g.advance(100000, cfl=cfl, t_final=1.0)
        if abs(t - 1.0) > 1e-12:
            return None
        e = g.l2_error()[1]
        return e if e == e else None
    except nsfr.NsfrError:
        return None
    finally:
        g.close()


def max_cfl(cfg):
    e0 = pressure_error(cfg, 0.1)
    best, cfl = 0.1, 0.11
    while cfl < 1.0:
        e = pressure_error(cfg, cfl)
        if e is None or abs(e - e0) > 5e-7 * abs(e0):
            break
        best, cfl = cfl, round(cfl + 0.01, 2)
    return best, e0


m = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for p in (3, 4, 5):
    for quad in (0, 1):
        for name, c in (("c_DG", 0.0), ("c_+", nsfr.C_PLUS[p])):
            cfg = nsfr.SolverConfig(p=p, m=m, c1d=c, quad_kind=quad, case="vortex", roe=True)
            best, e0 = max_cfl(cfg)
            print(json.dumps({"p": p, "m": m, "quad": "GL" if quad == 0 else "LGL", "scheme": f"NSFR {name}",
                              "max_cfl": best, "pressure_l2_at_cfl_0.1": e0}), flush=True)
