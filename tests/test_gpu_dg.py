"""GPU parity of the conservative strong-form DG residual (
SPEC.md:457-465): the DG kernels against the C oracle's DG
glue, which tests/test_oracle_pin.py pins to the reference's own primitives.
Same normwise gate as the NSFR tests (max(1e-12, 4 x the oracle's 1-ulp floor))."""
import numpy as np
import pytest

from oracle_lib import Config, CpuSolver
from test_gpu_parity import assert_rhs_parity, floor_of, gpu_cfg, norm_rel, P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,overint,quad,roe", [
    (3, 0, 0, True), (3, 1, 0, True), (3, 2, 0, True),
    (4, 0, 0, True), (4, 1, 0, True), (4, 2, 0, False),
    (5, 0, 0, True), (5, 2, 0, True),
    (4, 0, 1, True), (3, 1, 1, True),
])
def test_dg_rhs_matches_oracle(p, overint, quad, roe):
    """With the oracle's metrics (isolates the kernels, as the NSFR reference
    fixtures do) at the floor gate; with the device-built metrics (~1e-13 apart,
    amplified by the flux divergence) at 1e-10."""
    kw = dict(p=p, m=3, scheme="dg", overint=overint, quad_kind=quad, roe=roe)
    o = CpuSolver("oracle", Config(**kw))
    g = P().GpuSolver(gpu_cfg(**kw), metrics=o.metrics())
    g.init_case()
    u = g.get_state()
    np.testing.assert_allclose(u, o.initial_state(), rtol=1e-13, atol=1e-14)  # u_hat, unconverted
    want = o.rhs(u)
    tr_o = o.traces(u)
    got = g.rhs()
    tr_g = g.traces()
    assert np.abs(tr_g - tr_o).max() <= 1e-14 * np.abs(tr_o).max()
    assert_rhs_parity(got, want, floor_of(o, u))
    native = P().GpuSolver(gpu_cfg(**kw))
    native.set_state(u)
    assert norm_rel(native.rhs(), want) < 1e-10


@pytest.mark.parametrize("p,overint", [(3, 0), (4, 2)])
def test_dg_rk4_steps_match_oracle(p, overint):
    kw = dict(p=p, m=3, scheme="dg", overint=overint)
    o = CpuSolver("oracle", Config(**kw))
    g = P().GpuSolver(gpu_cfg(**kw))
    g.init_case()
    u0 = g.get_state()
    lam = o.max_wavespeed(u0)
    assert g.max_wavespeed() == pytest.approx(lam, rel=1e-14)
    uo, to = o.run(u0.copy(), 3)
    t = g.advance(3, cfl=0.1)
    assert t == pytest.approx(to, rel=1e-13)
    assert norm_rel(g.get_state() - u0, uo - u0) < 1e-10
    np.testing.assert_allclose(g.l2_error(), np.sqrt(o.l2_sq(uo, to)), rtol=1e-10)


@pytest.mark.parametrize("overint", [0, 2])
def test_dg_free_stream(overint):
    g = P().GpuSolver(gpu_cfg(p=4, m=3, scheme="dg", overint=overint, case="free_stream"))
    g.init_case()
    assert np.abs(g.rhs()).max() < 1e-12


def test_dg_conservation():
    """Thm 3 for DG with single-valued face metrics and the exact (n_q = n_p)
    weight-adjusted inverse: totals drift by round-off over 10 steps."""
    g = P().GpuSolver(gpu_cfg(p=3, m=4, scheme="dg", grid_degree=3))
    g.init_case()
    t0 = g.conserved_totals()
    g.advance(10)
    drift = np.abs(g.conserved_totals() - t0) / np.maximum(np.abs(t0), 1.0)
    assert drift.max() < 1e-12, drift


def test_dg_rejects_nsfr_only_calls():
    pkg = P()
    g = pkg.GpuSolver(gpu_cfg(p=3, m=2, scheme="dg"))
    g.init_case()
    with pytest.raises(pkg.ConfigError):
        g.ke_volume()
    with pytest.raises(pkg.DimensionError):
        pkg.GpuSolver(gpu_cfg(p=3, m=2, overint=1))  # NSFR needs n_q = n_p
