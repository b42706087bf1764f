"""Generate the committed golden vectors from the REFERENCE's own compiled code.

Run here (where /root/reference exists and oracle/_ref/libnsfr_ref.so is
built by `make -C oracle`):  python tests/golden/make_golden.py
Outputs tests/golden/*.npz and golden.json. Everything is produced by
oracle/_ref/libnsfr_ref.so — the reference's proj/src/*.cpp compiled where
they lie, driven by oracle/ref_driver.cpp (the residual glue the reference
specifies but does not ship). Inputs are seeded (numpy MT19937(20231207)).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_lib import C_PLUS, Config, CpuSolver, prim_fn, ptr  # noqa: E402

SEED = 20231207


def rng():
    return np.random.Generator(np.random.MT19937(SEED))


def random_states(r, n, gamma=1.4):
    """Admissible states: rho, p in [0.1, 10], |u| <= 3."""
    rho = r.uniform(0.1, 10.0, n)
    p = r.uniform(0.1, 10.0, n)
    vel = r.uniform(-3.0 / np.sqrt(3), 3.0 / np.sqrt(3), (n, 3))
    u = np.zeros((n, 5))
    u[:, 0] = rho
    u[:, 1:4] = rho[:, None] * vel
    u[:, 4] = p / (gamma - 1) + 0.5 * rho * (vel ** 2).sum(1)
    return u


def perturbed(u, r, amp=1e-3):
    return u * (1.0 + amp * r.uniform(-1.0, 1.0, u.shape))


def primitives():
    r = rng()
    n = 256
    ul = random_states(r, n)
    ur = random_states(r, n)
    # near-equal pairs exercise the log-mean series branch (euler.cpp:94)
    ur[: n // 4] = ul[: n // 4] * (1.0 + r.uniform(-1e-5, 1e-5, (n // 4, 5)))
    ur[n // 4: n // 2] = ul[n // 4: n // 2] * (1.0 + r.uniform(-3e-4, 3e-4, (n // 4, 5)))
    nrm = r.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[:8] = np.eye(3)[np.arange(8) % 3]  # axis normals hit the |n_x| > 0.9 tangent branch
    a = r.uniform(0.1, 10.0, n)
    b = a * (1.0 + r.uniform(-1e-3, 1e-3, n))
    b[n // 2:] = r.uniform(0.1, 10.0, n // 2)
    lm = np.array([prim_fn("ref", "log_mean")(float(x), float(y)) for x, y in zip(a, b)])
    flux = np.zeros((n, 15))
    roe = np.zeros((n, 5))
    ev = np.zeros((n, 5))
    back = np.zeros((n, 5))
    for i in range(n):
        L, R, N = (np.ascontiguousarray(ul[i]), np.ascontiguousarray(ur[i]),
                   np.ascontiguousarray(nrm[i]))
        f = np.zeros(15)
        assert prim_fn("ref", "flux_ec")(1.4, ptr(L), ptr(R), ptr(f)) == 0
        flux[i] = f
        d = np.zeros(5)
        assert prim_fn("ref", "roe")(1.4, ptr(L), ptr(R), ptr(N), ptr(d)) == 0
        roe[i] = d
        v = np.zeros(5)
        assert prim_fn("ref", "entropy_vars")(1.4, ptr(L), ptr(v)) == 0
        ev[i] = v
        w = np.zeros(5)
        assert prim_fn("ref", "entropy_to_cons")(1.4, ptr(v), ptr(w)) == 0
        back[i] = w
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), ul=ul, ur=ur, normal=nrm, lm_a=a,
                        lm_b=b, log_mean=lm, flux_ec=flux, roe=roe, entropy_vars=ev, round_trip=back)


def tables():
    out = {}
    for p in (2, 3, 4, 5):
        for quad in (0, 1):
            for cname, c in (("dg", 0.0), ("plus", C_PLUS[p])):
                s = CpuSolver("ref", Config(p=p, m=1, quad_kind=quad, c1d=c, workers=1))
                for k, v in s.tables().items():
                    out[f"p{p}_q{quad}_{cname}_{k}"] = v
                s.close()
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)


def rhs_cases():
    """Small full-RHS fixtures: perturbed vortex/TGV states through the reference."""
    cases = {
        "vortex_p3_m3_dg_roe": Config(p=3, m=3, c1d=0.0, case="vortex", roe=True, workers=8),
        "vortex_p4_m2_plus_roe": Config(p=4, m=2, c1d=C_PLUS[4], case="vortex", roe=True, workers=8),
        "tgv_p3_m2_dg_ec": Config(p=3, m=2, c1d=0.0, case="tgv", roe=False, workers=8),
        "vortex_p5_m2_dg_roe": Config(p=5, m=2, c1d=0.0, case="vortex", roe=True, workers=8),
    }
    meta = {}
    for name, cfg in cases.items():
        r = rng()
        s = CpuSolver("ref", cfg)
        u0 = s.initial_state()
        u = perturbed(u0, r)
        dudt, ds = s.rhs(u, entropy=True)
        jac, cof = s.metrics()
        np.savez_compressed(os.path.join(HERE, f"rhs_{name}.npz"), u0=u0, u=u, dudt=dudt, jac=jac,
                            cof=cof, x_sol=s.x_sol())
        meta[name] = {"cfg": {k: getattr(cfg, k) for k in ("p", "m", "c1d", "case", "roe")},
                      "entropy_change": ds, "lambda_max": s.max_wavespeed(u)}
        s.close()
    return meta


def scalars():
    """Config 1 (BASELINE.json configs[0]): 20 RK4 steps at CFL 0.1, L2 errors."""
    out = {}
    cfg = Config(p=3, m=8, c1d=0.0, case="vortex", roe=True, workers=os.cpu_count())
    s = CpuSolver("ref", cfg)
    u = s.initial_state()
    out["config1_lambda0"] = s.max_wavespeed(u)
    out["config1_l2_t0"] = s.l2_error(u, 0.0).tolist()
    out["config1_entropy_change_t0"] = s.rhs(u, entropy=True)[1]
    u, t = s.run(u, 20, cfl=0.1)
    out["config1_t20"] = t
    out["config1_l2_t20"] = s.l2_error(u, t).tolist()
    out["config1_state_checksum"] = [float(u[:, k].sum()) for k in range(5)]
    s.close()
    # free stream (Thm 2) with the reference metrics
    for p in (3, 4):
        s = CpuSolver("ref", Config(p=p, m=3, case="free_stream", c1d=C_PLUS[p], workers=8))
        out[f"freestream_p{p}_max"] = float(np.abs(s.rhs(s.initial_state())).max())
        s.close()
    # EC entropy change on TGV with consistent face metrics (grid_degree = p)
    s = CpuSolver("ref", Config(p=3, m=3, case="tgv", roe=False, grid_degree=3, workers=8))
    u = s.initial_state()
    out["tgv_ec_gd3_entropy_change"] = s.rhs(u, entropy=True)[1]
    out["tgv_ec_gd3_entropy_total"] = s.entropy_total(u)
    s.close()
    return out


if __name__ == "__main__":
    primitives()
    tables()
    meta = rhs_cases()
    meta.update(scalars())
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta, indent=1))
