"""Bitwise fingerprint of every kernel family's outputs (dev tool for
tools/debug_checks.sh): run once against the release library and once against
the -DNSFR_DEBUG_CHECKS build (NSFR_B200_LIB=...); the two JSON outputs must be
identical. The debug build poisons shared memory and fresh device arrays with
NaN, delays each warp's start pseudo-randomly and runs CTAs in reverse order,
so equal bits mean no uninitialised read, no missing barrier and no
inter-CTA dependence on these paths."""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07725_b200 as pkg  # noqa: E402

C_PLUS = {3: 0.5 * 3.80e-3, 4: 0.5 * 4.67e-5, 5: 0.5 * 4.28e-7}


def h(a):
    a = np.ascontiguousarray(a)
    assert np.isfinite(a).all(), "non-finite output"
    return hashlib.sha256(a.tobytes()).hexdigest()[:16]


def run(name, cfg, out):
    g = pkg.GpuSolver(cfg)
    g.init_case()
    r = {}
    dudt = g.rhs(entropy=cfg.entropy_diag) if cfg.scheme == "nsfr" else g.rhs()
    r["rhs"] = h(dudt[0] if isinstance(dudt, tuple) else dudt)
    if cfg.entropy_diag:
        r["dS"] = float(dudt[1]).hex()
    g.advance(3, cfl=0.1)
    r["uq3"] = h(g.get_state_q())
    r["u3"] = h(g.get_state())
    r["l2"] = [float(x).hex() for x in g.l2_error()]
    r["tot"] = h(g.conserved_totals())
    if cfg.scheme == "nsfr":
        r["ke"] = [float(g.ke_volume()).hex(), float(g.ke_total()).hex()]
    u = g.get_state()
    if cfg.overint == 0:  # (adaptive dt of an overintegrated DG output is not offered)
        dt_next = g.rk4_step_host(u, u, dt=0.0, cfl=0.1)[2]
        r["host"] = h(u)
        g.rk4_step_host(u, u, dt=dt_next, cfl=0.1)
        r["host2"] = h(u)
    # (the host step of an overintegrated DG context is not offered)
    g.close()
    out[name] = r


def slabs(name, p, m, nranks, out):
    ranks = [pkg.GpuSolver(pkg.SolverConfig(p=p, m=m, rank=r, nranks=nranks, c1d=C_PLUS[p]))
             for r in range(nranks)]
    for g in ranks:
        g.init_case()
        g.project()

    def swap():
        sends = [g.halo_get() for g in ranks]
        for r, g in enumerate(ranks):
            g.halo_set(sends[(r - 1) % nranks][1], sends[(r + 1) % nranks][0])

    swap()
    rhs = np.concatenate([g.residual() for g in ranks])
    for g in ranks:
        g.project()
    for s in range(1, 5):
        swap()
        for g in ranks:
            g.stage(s, 1e-3)
    out[name] = {"rhs": h(rhs), "uq": h(np.concatenate([g.get_state_q() for g in ranks]))}


if __name__ == "__main__":
    out = {}
    if len(sys.argv) > 1 and sys.argv[1] == "--quick":  # smoke of the script itself
        run("nsfr_p3_dg", pkg.SolverConfig(p=3, m=2, entropy_diag=True), out)
        print(json.dumps(out, sort_keys=True, indent=1))
        sys.exit(0)
    for p in (2, 3, 4, 5, 6):
        run(f"nsfr_p{p}_dg", pkg.SolverConfig(p=p, m=3, entropy_diag=True), out)
    for p in (3, 4, 5):
        run(f"nsfr_p{p}_plus", pkg.SolverConfig(p=p, m=4, c1d=C_PLUS[p]), out)
    run("nsfr_p4_lgl", pkg.SolverConfig(p=4, m=3, quad_kind=1), out)
    run("nsfr_p3_tgv_ec", pkg.SolverConfig(p=3, m=4, case="tgv", roe=False, entropy_diag=True), out)
    run("nsfr_p4_m17", pkg.SolverConfig(p=4, m=17, c1d=C_PLUS[4]), out)  # odd batch tails, many chunks
    for p, oi in ((3, 0), (4, 1), (5, 2)):
        run(f"dg_p{p}_oi{oi}", pkg.SolverConfig(p=p, m=3, scheme="dg", overint=oi), out)
    slabs("slabs_p3_m6_n3", 3, 6, 3, out)
    slabs("slabs_p4_m5_n2", 4, 5, 2, out)
    print(json.dumps(out, sort_keys=True, indent=1))
