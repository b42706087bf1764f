"""Checkpoint text format and diagnostics CSV (paper_2312_07725_b200/runio.py)
on the host: bit-exact 17-digit round trips, header validation. CPU only."""
import math

import numpy as np
import pytest

from paper_2312_07725_b200 import SolverConfig, runio


class FakeSolver:
    """Duck-typed stand-in for GpuSolver's state/time accessors."""

    def __init__(self, cfg, k0=0, k1=None, seed=0):
        self.cfg = cfg
        self.k0, self.k1 = k0, cfg.m if k1 is None else k1
        ne = cfg.m * cfg.m * (self.k1 - self.k0)
        rng = np.random.default_rng(seed)
        self.u = rng.standard_normal((ne, 5, (cfg.p + 1) ** 3)) * 10.0 ** rng.integers(-8, 8, (ne, 5, 1))
        self.uq = self.u * np.pi
        self.time = 0.1 + 1e-17

    def get_state(self):
        return self.u.copy()

    def get_state_q(self):
        return self.uq.copy()

    def set_state(self, u):
        self.u = u.copy()

    def set_state_q(self, u):
        self.uq = u.copy()

    def set_time(self, t):
        self.time = t


@pytest.mark.parametrize("exact", [False, True])
def test_checkpoint_round_trip_bit_exact(tmp_path, exact):
    cfg = SolverConfig(p=3, m=2, c1d=1.9e-3)
    a = FakeSolver(cfg)
    path = runio.write_checkpoint(str(tmp_path / "ck.txt"), a, exact=exact)
    head, u = runio.read_checkpoint(path)
    assert head["p"] == 3 and head["m"] == 2 and head["t"] == a.time
    assert head["nodes"] == ("quadrature" if exact else "solution")
    np.testing.assert_array_equal(u, a.uq if exact else a.u)
    b = FakeSolver(cfg, seed=1)
    runio.load_checkpoint(str(tmp_path / "ck.txt"), b)
    np.testing.assert_array_equal(b.uq if exact else b.u, a.uq if exact else a.u)
    assert b.time == a.time


def test_checkpoint_rejects_mismatch(tmp_path):
    a = FakeSolver(SolverConfig(p=3, m=2))
    runio.write_checkpoint(str(tmp_path / "ck.txt"), a)
    with pytest.raises(ValueError):
        runio.load_checkpoint(str(tmp_path / "ck.txt"), FakeSolver(SolverConfig(p=4, m=2)))
    with pytest.raises(ValueError):
        runio.load_checkpoint(str(tmp_path / "ck.txt"), FakeSolver(SolverConfig(p=3, m=2, c1d=1e-3)))


def test_checkpoint_per_rank_slab(tmp_path):
    cfg = SolverConfig(p=2, m=4, rank=1, nranks=2)
    a = FakeSolver(cfg, k0=2, k1=4)
    path = runio.write_checkpoint(str(tmp_path / "ck.txt"), a)
    assert path.endswith(".rank1")
    head, u = runio.read_checkpoint(path)
    assert (head["k0"], head["k1"], head["elements"]) == (2, 4, 32)
    np.testing.assert_array_equal(u, a.u)


def test_diagnostics_csv_round_trip(tmp_path):
    path = str(tmp_path / "d.csv")
    out = runio.DiagnosticsCSV(path)
    recs = []
    for i in range(3):
        r = {c: (i + 1) / 3.0 * 10.0 ** (-i) for c in runio.COLUMNS}
        r["entropy_change"] = math.nan
        recs.append(r)
        out.write(r)
    out.close()
    back = runio.read_diagnostics(path)
    assert list(back[0].keys()) == list(runio.COLUMNS)
    for r, b in zip(recs, back):
        for c in runio.COLUMNS:
            assert (math.isnan(r[c]) and math.isnan(b[c])) or r[c] == b[c]


def test_checkpoint_records_scheme(tmp_path):
    """The header names the scheme (NSFR-EC / DG-cons, +Roe) and overintegration;
    a checkpoint of one scheme does not load into a solver of the other."""
    a = FakeSolver(SolverConfig(p=3, m=2, scheme="dg", overint=1))
    path = runio.write_checkpoint(str(tmp_path / "ck.txt"), a)
    head, _ = runio.read_checkpoint(path)
    assert head["scheme"] == "DG-cons+Roe" and head["overint"] == 1
    with pytest.raises(ValueError):
        runio.load_checkpoint(path, FakeSolver(SolverConfig(p=3, m=2)))
    runio.load_checkpoint(path, FakeSolver(SolverConfig(p=3, m=2, scheme="dg", overint=1)))


class DiagSolver(FakeSolver):
    """Stand-in with the diagnostics surface; the KE calls fail for DG like the C ABI."""

    def entropy_total(self):
        return -1.0

    def entropy_change(self):
        return -1e-9

    def ke_volume(self):
        if self.cfg.scheme != "nsfr":
            raise RuntimeError("NSFR_E_CONFIG")
        return 0.0

    ke_total = ke_volume

    def conserved_totals(self):
        return np.ones(5)

    def max_wavespeed(self):
        return 1.5

    def l2_error(self):
        return np.array([1e-3, 2e-3])


def test_diagnostics_of_dg_run_have_nan_ke():
    rec = runio.diagnostic_record(DiagSolver(SolverConfig(p=3, m=2, scheme="dg")), -1.0)
    assert math.isnan(rec["ke_change_volume"]) and math.isnan(rec["ke_change_total_minus_pressure_work"])
    assert rec["l2_density"] == 1e-3
    rec = runio.diagnostic_record(DiagSolver(SolverConfig(p=3, m=2)), -1.0)
    assert rec["ke_change_volume"] == 0.0
