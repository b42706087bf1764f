"""Pin the C oracle against the golden vectors produced by the REFERENCE's own
compiled code (tests/golden/make_golden.py, oracle/_ref). CPU only."""
import json
import os

import numpy as np
import pytest

from oracle_lib import C_PLUS, Config, CpuSolver, prim_fn, ptr

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


def per_state_rel(a, b):
    a = a.reshape(a.shape[0], 5, -1)
    b = b.reshape(b.shape[0], 5, -1)
    return (np.abs(a - b).max(axis=(0, 2)) / np.abs(b).max(axis=(0, 2))).max()


def test_log_mean_golden():
    g = gold("primitives.npz")
    lm = np.array([prim_fn("oracle", "log_mean")(float(a), float(b)) for a, b in zip(g["lm_a"], g["lm_b"])])
    np.testing.assert_allclose(lm, g["log_mean"], rtol=2e-16, atol=0)


def test_flux_roe_entropy_golden():
    g = gold("primitives.npz")
    for i in range(len(g["ul"])):
        L, R, N = (np.ascontiguousarray(g["ul"][i]), np.ascontiguousarray(g["ur"][i]),
                   np.ascontiguousarray(g["normal"][i]))
        f = np.zeros(15)
        assert prim_fn("oracle", "flux_ec")(1.4, ptr(L), ptr(R), ptr(f)) == 0
        np.testing.assert_allclose(f, g["flux_ec"][i], rtol=1e-14, atol=1e-14)
        d = np.zeros(5)
        assert prim_fn("oracle", "roe")(1.4, ptr(L), ptr(R), ptr(N), ptr(d)) == 0
        np.testing.assert_allclose(d, g["roe"][i], rtol=1e-13, atol=1e-13 * np.abs(g["roe"][i]).max())
        v = np.zeros(5)
        assert prim_fn("oracle", "entropy_vars")(1.4, ptr(L), ptr(v)) == 0
        np.testing.assert_allclose(v, g["entropy_vars"][i], rtol=1e-14, atol=1e-14)
        w = np.zeros(5)
        assert prim_fn("oracle", "entropy_to_cons")(1.4, ptr(v), ptr(w)) == 0
        np.testing.assert_allclose(w, g["round_trip"][i], rtol=1e-14, atol=1e-14)
        # SPEC.md:336,358 round trip u -> v -> u within 1e-12 relative
        np.testing.assert_allclose(w, L, rtol=1e-12)


@pytest.mark.parametrize("p", [2, 3, 4, 5])
@pytest.mark.parametrize("quad", [0, 1])
@pytest.mark.parametrize("cname", ["dg", "plus"])
def test_tables_golden(p, quad, cname):
    g = gold("tables.npz")
    c = 0.0 if cname == "dg" else C_PLUS[p]
    s = CpuSolver("oracle", Config(p=p, m=1, quad_kind=quad, c1d=c, workers=1))
    for k, v in s.tables().items():
        np.testing.assert_allclose(v, g[f"p{p}_q{quad}_{cname}_{k}"], rtol=0, atol=1e-15 * max(1.0, np.abs(v).max()))


@pytest.mark.parametrize("name", ["vortex_p3_m3_dg_roe", "vortex_p4_m2_plus_roe", "tgv_p3_m2_dg_ec",
                                  "vortex_p5_m2_dg_roe"])
def test_rhs_fixture_golden(name, meta):
    g = gold(f"rhs_{name}.npz")
    c = meta[name]["cfg"]
    s = CpuSolver("oracle", Config(p=c["p"], m=c["m"], c1d=c["c1d"], case=c["case"], roe=c["roe"]))
    jac, cof = s.metrics()
    np.testing.assert_allclose(jac, g["jac"], rtol=1e-14)
    np.testing.assert_allclose(cof, g["cof"], rtol=0, atol=1e-14 * np.abs(g["cof"]).max())
    np.testing.assert_allclose(s.x_sol(), g["x_sol"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(s.initial_state(), g["u0"], rtol=1e-14, atol=1e-14)
    dudt, ds = s.rhs(g["u"], entropy=True)
    # the oracle restates the reference operation by operation: agreement far
    # below the reference's own 1-ulp sensitivity floor (see test_parity_floor)
    assert per_state_rel(dudt, g["dudt"]) < 1e-13
    assert abs(ds - meta[name]["entropy_change"]) <= 1e-13 * max(1.0, abs(meta[name]["entropy_change"]))
    assert s.max_wavespeed(g["u"]) == pytest.approx(meta[name]["lambda_max"], rel=1e-15)


def test_config1_scalars_golden(meta):
    s = CpuSolver("oracle", Config(p=3, m=8, c1d=0.0, case="vortex", roe=True))
    u = s.initial_state()
    assert s.max_wavespeed(u) == pytest.approx(meta["config1_lambda0"], rel=1e-15)
    np.testing.assert_allclose(s.l2_error(u, 0.0), meta["config1_l2_t0"], rtol=1e-13)
    assert s.rhs(u, entropy=True)[1] == pytest.approx(meta["config1_entropy_change_t0"], rel=1e-11)


@pytest.mark.slow
def test_config1_20_steps_golden(meta):
    """BASELINE configs[0]: 20 RK4 steps at CFL 0.1; final L2 within 1e-10 relative."""
    s = CpuSolver("oracle", Config(p=3, m=8, c1d=0.0, case="vortex", roe=True))
    u, t = s.run(s.initial_state(), 20, cfl=0.1)
    assert t == pytest.approx(meta["config1_t20"], rel=1e-14)
    np.testing.assert_allclose(s.l2_error(u, t), meta["config1_l2_t20"], rtol=1e-10)
