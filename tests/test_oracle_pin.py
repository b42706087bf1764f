"""Pin the C oracle against the reference's OWN compiled primitives
(oracle/_ref/libnsfr_ref.so, built from /root/reference/proj/src by
oracle/Makefile) on configurations beyond the committed fixtures. CPU only."""
import os

import numpy as np
import pytest

from oracle_lib import C_PLUS, LIBS, Config, CpuSolver

pytestmark = pytest.mark.skipif(not os.path.exists(LIBS["ref"][0]), reason="oracle/_ref not built")


def rel(a, b):
    return (np.abs(a - b).max(axis=(0, 2)) / np.abs(b).max(axis=(0, 2))).max()


@pytest.mark.parametrize("cfg", [
    Config(p=3, m=4, c1d=0.0),
    Config(p=4, m=3, c1d=C_PLUS[4]),
    Config(p=5, m=2, c1d=C_PLUS[5]),
    Config(p=3, m=3, case="tgv", roe=False),
    Config(p=3, m=3, quad_kind=1),
    Config(p=4, m=3, grid_degree=4, roe=False),
])
def test_oracle_matches_reference(cfg):
    o, r = CpuSolver("oracle", cfg), CpuSolver("ref", cfg)
    to, tr = o.tables(), r.tables()
    for k in to:
        np.testing.assert_array_equal(to[k], tr[k])
    jo, co = o.metrics()
    jr, cr = r.metrics()
    np.testing.assert_array_equal(jo, jr)
    np.testing.assert_array_equal(co, cr)
    u = o.initial_state()
    np.testing.assert_array_equal(u, r.initial_state())
    np.testing.assert_allclose(o.traces(u), r.traces(u), rtol=1e-15, atol=1e-15)
    do, so = o.rhs(u, entropy=True)
    dr, sr = r.rhs(u, entropy=True)
    assert rel(do, dr) < 1e-13
    assert abs(so - sr) <= 1e-13 * max(1.0, abs(sr))
    assert o.max_wavespeed(u) == r.max_wavespeed(u)
    np.testing.assert_allclose(o.l2_sq(u, 0.0), r.l2_sq(u, 0.0), rtol=1e-14, atol=1e-28)
    assert o.entropy_total(u) == pytest.approx(r.entropy_total(u), rel=1e-14)
    np.testing.assert_array_equal(o.conserved_totals(u), r.conserved_totals(u))
    assert o.ke_volume(u) == r.ke_volume(u)
    kt_o, kt_r = o.ke_total(u), r.ke_total(u)
    assert abs(kt_o - kt_r) <= 1e-11 * max(1.0, abs(kt_r)) + 1e-12


def test_oracle_rk4_matches_reference():
    cfg = Config(p=3, m=3)
    o, r = CpuSolver("oracle", cfg), CpuSolver("ref", cfg)
    uo, to = o.run(o.initial_state(), 3)
    ur, tr = r.run(r.initial_state(), 3)
    assert to == pytest.approx(tr, rel=1e-14)
    assert rel(uo - o.initial_state(), ur - r.initial_state()) < 1e-10  # 1-ulp floor, see test_invariants


def test_slab_halo_matches_whole_box():
    """A z-slab with neighbour traces as halos reproduces the whole-box residual
    bitwise, in both checkers (the partition the multi-GPU path uses)."""
    for kind in ("oracle", "ref"):
        m = 4
        full = CpuSolver(kind, Config(p=3, m=m))
        u = full.initial_state()
        want = full.rhs(u)
        tr = full.traces(u)  # [e][6][5][nf]
        k0, k1 = 1, 3
        part = CpuSolver(kind, Config(p=3, m=m, k0=k0, k1=k1))
        ul = u[m * m * k0:m * m * k1]
        halo_lo = np.ascontiguousarray(tr[m * m * (k0 - 1):m * m * k0, 5])
        halo_hi = np.ascontiguousarray(tr[m * m * k1:m * m * (k1 + 1), 4])
        got = part.rhs(ul, halo_lo, halo_hi)
        np.testing.assert_array_equal(got, want[m * m * k0:m * m * k1])


@pytest.mark.parametrize("cfg", [
    Config(p=3, m=3, scheme="dg"),
    Config(p=3, m=3, scheme="dg", overint=2),
    Config(p=4, m=2, scheme="dg", quad_kind=1),
    Config(p=4, m=2, scheme="dg", overint=1, c1d=C_PLUS[4], roe=False),
])
def test_dg_oracle_matches_reference(cfg):
    """Conservative strong-form DG glue: the C restatement vs
    the same glue over the reference's own physical_flux, CentralConservative
    two-point flux, roe_dissipation, apply_operator_dir(quad_diff),
    apply_tensor_product and weight_adjusted_inverse_apply."""
    o, r = CpuSolver("oracle", cfg), CpuSolver("ref", cfg)
    u = o.initial_state()
    np.testing.assert_allclose(o.traces(u), r.traces(u), rtol=0, atol=1e-15)
    assert rel(o.rhs(u), r.rhs(u)) < 1e-13
    uo, to = o.run(u.copy(), 2)
    ur, tr = r.run(u.copy(), 2)
    assert rel(uo - u, ur - u) < 1e-10
