"""The streamed host step (nsfr_gpu_rk4_step_host): upload, RK4 step and
download pipelined over element chunks must equal set_state + step +
get_state BITWISE (per-element arithmetic is launch-range independent and
lambda_max is an order-free max), for fixed and adaptive dt, chunk counts
1..32, odd m (chunk bounds off plane boundaries), aliasing buffers, c_DG and
c_+, and leave the device state/time exactly where the plain calls do."""
import numpy as np
import pytest

from oracle_lib import C_PLUS

pytestmark = pytest.mark.gpu


def P():
    import paper_2312_07725_b200 as pkg
    return pkg


def pair(**kw):
    cfg = P().SolverConfig(**kw)
    a, b = P().GpuSolver(cfg), P().GpuSolver(cfg)
    a.init_case()
    b.init_case()
    return a, b


def perturbed(g, seed=5):
    u = g.get_state()
    rng = np.random.default_rng(seed)
    return u * (1 + 1e-3 * rng.uniform(-1, 1, u.shape))


# m -> chunks: 3 -> 1, 4 -> 2, 6 -> 4 (m^2 = 36: bounds off the planes), 7 -> 6, 8 -> 7, 16 -> 15
@pytest.mark.parametrize("p,m", [(3, 3), (3, 4), (4, 6), (3, 8), (4, 16), (2, 7), (5, 4), (6, 3)])
@pytest.mark.parametrize("fixed", [True, False])
def test_streamed_step_equals_plain_calls(p, m, fixed):
    a, b = pair(p=p, m=m, c1d=C_PLUS.get(p, 0.0))
    u = perturbed(a)
    dt = 0.1 * (10.0 / (m * (p + 1))) / 2.5 if fixed else 0.0
    # plain: set_state, step, get_state
    b.set_state(u)
    want_dt = b.rk4_step_dt(dt) if fixed else b.rk4_step(0.1)
    want = b.get_state()
    got, got_dt, _ = a.rk4_step_host(u, dt=dt, cfl=0.1)
    np.testing.assert_array_equal(got, want)
    assert a.time == b.time
    if not fixed:
        assert got_dt == want_dt
    # the device state, its cached projection and lambda carry on identically
    a.rk4_step(0.1)
    b.rk4_step(0.1)
    np.testing.assert_array_equal(a.get_state(), b.get_state())


@pytest.mark.parametrize("c_plus", [False, True])
def test_streamed_step_aliasing_pinned_and_repeated(c_plus):
    import torch
    p, m = 4, 8
    a, b = pair(p=p, m=m, c1d=C_PLUS[p] if c_plus else 0.0)
    host = torch.empty(a.state_shape, dtype=torch.float64, pin_memory=True).numpy()
    host[...] = perturbed(a, seed=9)
    ub = host.copy()
    for _ in range(3):
        a.rk4_step_host(host, host, cfl=0.1)  # u_out aliases u_in
        b.set_state(ub)
        b.rk4_step(0.1)
        b.get_state(out=ub)
    np.testing.assert_array_equal(host, ub)
    assert a.time == b.time


def test_streamed_step_t_final_clip():
    a, b = pair(p=3, m=4)
    u = a.get_state()
    _, dt_a, _ = a.rk4_step_host(u, cfl=0.1, t_final=1e-3)
    b.set_state(u)
    dt_b = b.rk4_step(0.1, t_final=1e-3)
    assert dt_a == dt_b == pytest.approx(1e-3, abs=1e-18)
    assert a.time == b.time


def test_streamed_step_dg_falls_back_to_plain_calls():
    a, b = pair(p=3, m=4, scheme="dg")
    u = a.get_state()
    got, _, _ = a.rk4_step_host(u, cfl=0.1)
    b.set_state(u)
    b.rk4_step(0.1)
    np.testing.assert_array_equal(got, b.get_state())


def test_streamed_step_inadmissible_raises():
    pkg = P()
    a, _ = pair(p=3, m=4)
    u = a.get_state()
    u.reshape(u.shape[0], 5, -1)[7, 0, :] = -1.0  # negative density in one element
    with pytest.raises(pkg.StepFailureError):
        a.rk4_step_host(u, dt=1e-3)
    # the context stays usable after the failed pipeline
    a.init_case()
    b = pkg.GpuSolver(pkg.SolverConfig(p=3, m=4))
    b.init_case()
    u0 = b.get_state()
    got, _, _ = a.rk4_step_host(u0, dt=1e-3)
    b.set_state(u0)
    b.rk4_step_dt(1e-3)
    np.testing.assert_array_equal(got, b.get_state())


@pytest.mark.parametrize("scheme,m", [("nsfr", 8), ("nsfr", 5), ("dg", 4)])
def test_dt_next_chain_equals_adaptive_steps(scheme, m):
    """dt = adaptive_dt(u); u = rk4_step(u, dt) with adaptive_dt taken from the
    previous call's output (no barrier inside the step) reproduces the
    adaptive-dt steps bitwise: same dt sequence, same states, t_final clip."""
    p = 3
    a, b = pair(p=p, m=m, c1d=C_PLUS[p], scheme=scheme)
    u = a.get_state()
    ub = u.copy()
    t_final = 0.0
    _, _, dt = a.rk4_step_host(u, u, dt=0.0, cfl=0.1)  # first step: adaptive with the barrier
    b.set_state(ub)
    b.rk4_step(0.1)
    b.get_state(out=ub)
    t_final = b.time + 2.5 * dt  # the third chained step is clipped
    for _ in range(4):
        _, used, dt = a.rk4_step_host(u, u, dt=dt, cfl=0.1, t_final=t_final)
        b.set_state(ub)
        want = b.rk4_step(0.1, t_final=t_final)
        b.get_state(out=ub)
        assert used == want
        np.testing.assert_array_equal(u, ub)
        assert a.time == b.time
        if dt == 0.0:
            break
    assert a.time == t_final


@pytest.mark.parametrize("m,fixed", [(8, True), (8, False), (5, False)])
def test_streamed_step_slab_with_nccl_halos(m, fixed):
    """The slab form of the pipeline (end chunks fed by NCCL halo planes, one
    grouped send/recv per stage once both end chunks projected) on a 1-rank
    NCCL loopback communicator (its halo is the periodic wrap): bitwise the
    periodic context's plain calls."""
    pkg = P()
    p = 4
    cfg = pkg.SolverConfig(p=p, m=m, c1d=C_PLUS[p])
    a = pkg.GpuSolver(cfg, nccl_id=pkg.nccl_unique_id())
    b = pkg.GpuSolver(cfg)
    a.init_case()
    b.init_case()
    u = perturbed(b, seed=3)
    ub = u.copy()
    dt = 0.1 * (10.0 / (m * (p + 1))) / 2.5 if fixed else 0.0
    for _ in range(2):
        _, used, nxt = a.rk4_step_host(u, u, dt=dt, cfl=0.1)
        b.set_state(ub)
        want = b.rk4_step_dt(dt) if fixed else b.rk4_step(0.1)
        b.get_state(out=ub)
        np.testing.assert_array_equal(u, ub)
        assert a.time == b.time
        if not fixed:
            assert used == want
