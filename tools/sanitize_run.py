"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of libnsfr_b200.so on small boxes.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Covers k_metrics/k_init (setup), k_project (K1), k_residual (K2, KM 0/1/2),
k_update (K3: RK stages, entropy diagnostic, c_DG identity path, streamed
OUT variant), k_convert(_lines), the streamed host step, k_l2/k_reduce, the
DG kernels and a z-slab context in external-halo mode. Degrees p = 3, 4, 5.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2312_07725_b200 as pkg  # noqa: E402

C_PLUS = {3: 0.5 * 3.80e-3, 4: 0.5 * 4.67e-5, 5: 0.5 * 4.28e-7}


def run(p, m, c1d, **kw):
    g = pkg.GpuSolver(pkg.SolverConfig(p=p, m=m, c1d=c1d, entropy_diag=True, **kw))
    g.init_case()
    g.rhs(entropy=True)
    g.advance(2, cfl=0.1)
    g.rk4_step(0.1)
    g.l2_error()
    g.conserved_totals()
    g.entropy_total()
    if kw.get("scheme", "nsfr") == "nsfr":
        g.ke_volume()
        g.ke_total()
    u = g.get_state()
    g.rk4_step_host(u, u, dt=0.0, cfl=0.1)
    g.rk4_step_host(u, u, dt=1e-3, cfl=0.1)
    g.close()


def slabs(p, m, nranks):
    ranks = [pkg.GpuSolver(pkg.SolverConfig(p=p, m=m, rank=r, nranks=nranks)) for r in range(nranks)]
    for g in ranks:
        g.init_case()
        g.project()
    for s in range(1, 5):
        sends = [g.halo_get() for g in ranks]
        for r, g in enumerate(ranks):
            g.halo_set(sends[(r - 1) % nranks][1], sends[(r + 1) % nranks][0])
        for g in ranks:
            g.stage(s, 1e-3)
    for g in ranks:
        g.close()


if __name__ == "__main__":
    for p in (3, 4, 5):
        run(p, 3, 0.0)
        run(p, 3, C_PLUS[p])
    run(4, 3, 0.0, quad_kind=1)
    run(3, 3, 0.0, scheme="dg")
    run(4, 2, 0.0, scheme="dg", overint=1)
    slabs(3, 4, 2)
    print("sanitize_run: ok")
