"""State I/O and the diagnostics driver around the GPU residual path
(SPEC.md:511 checkpoint, SPEC.md:585-590 DiagnosticRecord,
SPEC.md:654 and 662 CSV schema, SPEC.md:684-691 cmd_run).

* Checkpoint: plain text, a header of `key value` lines (p, m, slab, scheme,
  t, ...) then per element one `element <global id>` line and 5 lines of
  coefficients printed with 17 significant digits, so the text round-trips
  bit-exactly. `nodes solution` stores u_hat (the reference's coefficient
  blocks; restoring it goes through chi^3, ~1 ulp). `nodes quadrature` stores
  the solver's own u_q and restores the device state bit-exactly.
* DiagnosticsCSV: one DiagnosticRecord per output time, header row, 17
  significant digits.
* run_simulation: advance to t_final, recording diagnostics every
  `diag_every` steps (CUDA-graph steps in between), optional final checkpoint.
"""
from __future__ import annotations

import csv
import math

import numpy as np

FORMAT = "nsfr-b200 checkpoint v1"
CASES = ("vortex", "tgv", "free_stream")


def _fmt(x: float) -> str:
    return repr(float(x)) if math.isfinite(x) else ("nan" if math.isnan(x) else repr(x))


def _scheme_label(cfg) -> str:
    """NSFR-EC / NSFR-EC+Roe, or DG-cons / DG-cons+Roe (SolverConfig.scheme)."""
    base = "NSFR-EC" if cfg.scheme == "nsfr" else "DG-cons"
    return base + ("+Roe" if cfg.roe else "")


def checkpoint_path(path: str, rank: int, nranks: int) -> str:
    """One file per rank (its z-slab) when the box is decomposed."""
    return path if nranks <= 1 else f"{path}.rank{rank}"


def write_checkpoint(path: str, solver, exact: bool = False) -> str:
    cfg = solver.cfg
    u = solver.get_state_q() if exact else solver.get_state()
    t = solver.time
    path = checkpoint_path(path, cfg.rank, cfg.nranks)
    head = {
        "p": cfg.p, "m": cfg.m, "k0": solver.k0, "k1": solver.k1,
        "nodes": "quadrature" if exact else "solution",
        "scheme": _scheme_label(cfg), "overint": cfg.overint, "quad_kind": cfg.quad_kind,
        "c1d": _fmt(cfg.c1d), "gamma": _fmt(cfg.gamma), "case": cfg.case, "t": _fmt(t),
        "elements": u.shape[0],
    }
    m2 = cfg.m * cfg.m
    with open(path, "w") as f:
        f.write(f"# {FORMAT}\n")
        for k, v in head.items():
            f.write(f"{k} {v}\n")
        for e in range(u.shape[0]):
            f.write(f"element {e + m2 * solver.k0}\n")
            for s in range(5):
                f.write(" ".join(repr(float(x)) for x in u[e, s]))
                f.write("\n")
    return path


def read_checkpoint(path: str):
    """-> (header dict, u [elements][5][n^3]); values parse back bit-exactly."""
    with open(path) as f:
        first = f.readline().strip()
        if first != f"# {FORMAT}":
            raise ValueError(f"{path}: not an {FORMAT} file")
        head = {}
        while True:
            pos = f.tell()
            line = f.readline()
            if not line or line.split(None, 1)[0] == "element":
                f.seek(pos)
                break
            k, v = line.split(None, 1)
            head[k] = v.strip()
        head.setdefault("overint", "0")
        for k in ("p", "m", "k0", "k1", "quad_kind", "elements", "overint"):
            head[k] = int(head[k])
        for k in ("c1d", "gamma", "t"):
            head[k] = float(head[k])
        n3 = (head["p"] + 1) ** 3  # (the DG state is u_hat in both node modes)
        u = np.empty((head["elements"], 5, n3))
        for e in range(head["elements"]):
            tag = f.readline().split()
            if tag[0] != "element" or int(tag[1]) != e + head["m"] ** 2 * head["k0"]:
                raise ValueError(f"{path}: element block {e} out of order")
            for s in range(5):
                row = np.array(f.readline().split(), dtype=np.float64)
                if row.size != n3:
                    raise ValueError(f"{path}: element {e} state {s}: {row.size} values, want {n3}")
                u[e, s] = row
    return head, u


def load_checkpoint(path: str, solver) -> dict:
    """Restore state and time into a solver of the same discretisation and slab."""
    cfg = solver.cfg
    head, u = read_checkpoint(checkpoint_path(path, cfg.rank, cfg.nranks))
    want = {"p": cfg.p, "m": cfg.m, "k0": solver.k0, "k1": solver.k1, "quad_kind": cfg.quad_kind,
            "overint": cfg.overint, "scheme": _scheme_label(cfg)}
    for k, v in want.items():
        if head[k] != v:
            raise ValueError(f"checkpoint {k}={head[k]} does not match the solver ({v})")
    if head["c1d"] != cfg.c1d or head["gamma"] != cfg.gamma:
        raise ValueError("checkpoint scheme parameters (c1d, gamma) do not match the solver")
    if head["nodes"] == "quadrature":
        solver.set_state_q(u)
    else:
        solver.set_state(u)
    solver.set_time(head["t"])
    return head


COLUMNS = ("t", "entropy_change", "entropy_change_normalized", "ke_change_volume",
           "ke_change_total_minus_pressure_work", "mass",
           "momentum_x", "momentum_y", "momentum_z", "energy", "max_wavespeed", "l2_density",
           "l2_pressure")


def diagnostic_record(solver, u_total0: float | None) -> dict:
    """DiagnosticRecord of the current state; entropy change
    needs entropy_diag=True (else NaN), L2 errors the vortex case (else NaN),
    the kinetic-energy terms the NSFR scheme (else NaN)."""
    cfg = solver.cfg
    rec = {"t": solver.time}
    if cfg.entropy_diag:
        ds = solver.entropy_change()
        rec["entropy_change"] = ds
        rec["entropy_change_normalized"] = ds / abs(u_total0) if u_total0 else math.nan
    else:
        rec["entropy_change"] = rec["entropy_change_normalized"] = math.nan
    nsfr = cfg.scheme == "nsfr"  # the kinetic-energy terms are NSFR diagnostics (NaN for DG)
    rec["ke_change_volume"] = solver.ke_volume() if nsfr else math.nan
    rec["ke_change_total_minus_pressure_work"] = (solver.ke_total() if nsfr and cfg.nranks == 1
                                                  else math.nan)
    tot = solver.conserved_totals()
    for k, v in zip(("mass", "momentum_x", "momentum_y", "momentum_z", "energy"), tot):
        rec[k] = float(v)
    rec["max_wavespeed"] = solver.max_wavespeed()
    if cfg.case == "vortex":
        rec["l2_density"], rec["l2_pressure"] = (float(x) for x in solver.l2_error())
    else:
        rec["l2_density"] = rec["l2_pressure"] = math.nan
    return rec


class DiagnosticsCSV:
    """Header row, one record per output time, 17 significant digits."""

    def __init__(self, path: str):
        self.path = path
        self.f = open(path, "w", newline="")
        self.w = csv.writer(self.f)
        self.w.writerow(COLUMNS)

    def write(self, rec: dict):
        self.w.writerow([_fmt(rec[c]) for c in COLUMNS])
        self.f.flush()

    def close(self):
        self.f.close()


def read_diagnostics(path: str) -> list[dict]:
    with open(path, newline="") as f:
        rows = list(csv.DictReader(f))
    return [{k: float(v) for k, v in r.items()} for r in rows]


def run_simulation(solver, t_final: float, cfl: float = 0.1, diag_every: int = 10,
                   csv_path: str | None = None, checkpoint: str | None = None,
                   exact_checkpoint: bool = False, max_steps: int = 10 ** 7) -> list[dict]:
    """Advance the solver's current state to t_final (RK4, adaptive dt, CUDA
    graph steps) with a DiagnosticRecord every `diag_every` steps and at the
    end. Only rank 0 writes the CSV (records are allreduced)."""
    rank0 = solver.cfg.rank == 0
    u_total0 = solver.entropy_total()
    out = DiagnosticsCSV(csv_path) if (csv_path and rank0) else None
    recs = []
    try:
        rec = diagnostic_record(solver, u_total0)
        recs.append(rec)
        if out:
            out.write(rec)
        steps = 0
        while rec["t"] < t_final and steps < max_steps:
            solver.advance(min(diag_every, max_steps - steps), cfl=cfl, t_final=t_final)
            steps += diag_every
            rec = diagnostic_record(solver, u_total0)
            recs.append(rec)
            if out:
                out.write(rec)
    finally:
        if out:
            out.close()
    if checkpoint:
        write_checkpoint(checkpoint, solver, exact=exact_checkpoint)
    return recs


__all__ = ["write_checkpoint", "read_checkpoint", "load_checkpoint", "checkpoint_path",
           "DiagnosticsCSV", "read_diagnostics", "diagnostic_record", "run_simulation", "COLUMNS"]
