"""ctypes wrapper over the CPU checkers (TEST INFRASTRUCTURE ONLY).

`CpuSolver("oracle")` loads oracle/libnsfr_oracle.so (the C restatement) and
`CpuSolver("ref")` loads oracle/_ref/libnsfr_ref.so (the reference's own
compiled primitives + glue). Both export oracle/nsfr_oracle.h. Only tests,
`__graft_entry__.smoke()` and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBS = {
    "oracle": (os.path.join(ROOT, "oracle", "libnsfr_oracle.so"), "nsfr_oracle_"),
    "ref": (os.path.join(ROOT, "oracle", "_ref", "libnsfr_ref.so"), "nsfr_ref_"),
}

CASES = {"vortex": 0, "tgv": 1, "free_stream": 2}
C_PLUS = {2: 0.5 * 0.206, 3: 0.5 * 3.80e-3, 4: 0.5 * 4.67e-5, 5: 0.5 * 4.28e-7}


class NsfrCfg(C.Structure):
    _fields_ = [
        ("p", C.c_int), ("quad_kind", C.c_int), ("overint", C.c_int), ("c1d", C.c_double),
        ("m", C.c_int), ("k0", C.c_int), ("k1", C.c_int),
        ("x_left", C.c_double), ("x_right", C.c_double), ("beta", C.c_double),
        ("length_scale", C.c_double), ("grid_degree", C.c_int), ("gamma", C.c_double),
        ("roe", C.c_int), ("workers", C.c_int), ("scheme", C.c_int),
    ]


@dataclass
class Config:
    """One NSFR problem (BASELINE.json configs). grid_degree None -> p+1."""
    p: int = 3
    m: int = 4
    c1d: float = 0.0
    quad_kind: int = 0
    case: str = "vortex"
    roe: bool = True
    beta: float = 0.05
    x_left: float | None = None
    x_right: float | None = None
    length_scale: float = 0.0
    grid_degree: int | None = None
    gamma: float = 1.4
    k0: int = 0
    k1: int | None = None
    workers: int = field(default_factory=lambda: os.cpu_count() or 1)
    scheme: str = "nsfr"   # "nsfr" (NSFR-EC) or "dg" (conservative strong-form DG)
    overint: int = 0       # extra quadrature nodes (n_q = p + 1 + overint)

    def domain(self):
        if self.x_left is not None:
            return self.x_left, self.x_right
        return {"vortex": (0.0, 10.0), "tgv": (-np.pi, np.pi),
                "free_stream": (0.0, 2 * np.pi)}[self.case]

    def to_c(self) -> NsfrCfg:
        xl, xr = self.domain()
        return NsfrCfg(self.p, self.quad_kind, self.overint, self.c1d, self.m, self.k0,
                       self.m if self.k1 is None else self.k1, xl, xr, self.beta,
                       self.length_scale,
                       self.p + 1 if self.grid_degree is None else self.grid_degree,
                       self.gamma, int(self.roe), self.workers,
                       {"nsfr": 0, "dg": 1}[self.scheme])


_loaded: dict[str, C.CDLL] = {}


def load(kind: str) -> tuple[C.CDLL, str]:
    path, prefix = LIBS[kind]
    if kind not in _loaded:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        lib = C.CDLL(path)
        P = C.POINTER(C.c_double)
        sig = {
            "create": (C.c_void_p, [C.POINTER(NsfrCfg), C.c_char_p, C.c_int]),
            "destroy": (None, [C.c_void_p]),
            "last_error": (C.c_char_p, [C.c_void_p]),
            "tables": (C.c_int, [C.c_void_p, P, C.c_int]),
            "metrics": (C.c_int, [C.c_void_p, P, P]),
            "x_sol": (C.c_int, [C.c_void_p, P]),
            "x_vol": (C.c_int, [C.c_void_p, P]),
            "initial_state": (C.c_int, [C.c_void_p, C.c_int, P]),
            "boundary_traces": (C.c_int, [C.c_void_p, P, P, P]),
            "traces": (C.c_int, [C.c_void_p, P, P]),
            "rhs": (C.c_int, [C.c_void_p, P, P, P, P, P]),
            "max_wavespeed": (C.c_int, [C.c_void_p, P, P]),
            "rk4_step": (C.c_int, [C.c_void_p, P, C.c_double]),
            "l2_error": (C.c_int, [C.c_void_p, P, C.c_double, C.c_int, P]),
            "entropy_total": (C.c_int, [C.c_void_p, P, P]),
            "conserved_totals": (C.c_int, [C.c_void_p, P, P]),
            "ke_volume": (C.c_int, [C.c_void_p, P, P]),
            "ke_total": (C.c_int, [C.c_void_p, P, P]),
            "log_mean": (C.c_double, [C.c_double, C.c_double]),
            "flux_ec": (C.c_int, [C.c_double, P, P, P]),
            "roe": (C.c_int, [C.c_double, P, P, P, P]),
            "entropy_vars": (C.c_int, [C.c_double, P, P]),
            "entropy_to_cons": (C.c_int, [C.c_double, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, prefix + name)
            fn.restype = res
            fn.argtypes = args
        _loaded[kind] = lib
    return _loaded[kind], prefix


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


class CheckerError(RuntimeError):
    pass


class CpuSolver:
    """CPU checker with the solver-facing surface of the GPU path."""

    def __init__(self, kind: str, cfg: Config):
        self.kind = kind
        self.cfg = cfg
        self.lib, self.prefix = load(kind)
        self._c = cfg.to_c()
        err = C.create_string_buffer(512)
        self.ctx = self._fn("create")(C.byref(self._c), err, 512)
        if not self.ctx:
            raise CheckerError(err.value.decode())
        self.np_ = cfg.p + 1
        self.nq = cfg.p + 1 + cfg.overint
        self.ne = cfg.m * cfg.m * ((cfg.m if cfg.k1 is None else cfg.k1) - cfg.k0)
        self.nsol = self.np_ ** 3
        self.nv = self.nq ** 3
        self.nf = self.nq ** 2

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc:
            raise CheckerError(f"{self.kind}: rc={rc}: {self._fn('last_error')(self.ctx).decode()}")

    def close(self):
        if self.ctx:
            self._fn("destroy")(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- setup products -----------------------------------------------------
    def tables(self) -> dict[str, np.ndarray]:
        np_, nq = self.np_, self.nq
        buf = np.zeros(4096)
        n = self._fn("tables")(self.ctx, ptr(buf), buf.size)
        shapes = [("interp", (nq, np_)), ("proj", (np_, nq)), ("fr_proj", (np_, nq)),
                  ("skew", (nq, nq)), ("bound_flux", (2, nq)), ("bound_sol", (2, np_)),
                  ("wq", (nq,)), ("quad_nodes", (nq,)), ("sol_nodes", (np_,)),
                  ("mmass1d", (np_, np_)), ("quad_diff", (nq, nq))]
        out, pos = {}, 0
        for name, shp in shapes:
            sz = int(np.prod(shp))
            out[name] = buf[pos:pos + sz].reshape(shp).copy()
            pos += sz
        assert pos == n
        return out

    def metrics(self):
        jac = np.zeros((self.ne, self.nv))
        cof = np.zeros((self.ne, self.nv, 9))
        self._check(self._fn("metrics")(self.ctx, ptr(jac), ptr(cof)))
        return jac, cof

    def x_sol(self):
        x = np.zeros((self.ne, self.nsol, 3))
        self._check(self._fn("x_sol")(self.ctx, ptr(x)))
        return x

    def x_vol(self):
        x = np.zeros((self.ne, self.nv, 3))
        self._check(self._fn("x_vol")(self.ctx, ptr(x)))
        return x

    def initial_state(self, case: str | None = None) -> np.ndarray:
        u = np.zeros((self.ne, 5, self.nsol))
        self._check(self._fn("initial_state")(self.ctx, CASES[case or self.cfg.case], ptr(u)))
        return u

    # --- hot path -----------------------------------------------------------
    def rhs(self, u, halo_lo=None, halo_hi=None, entropy=False):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros_like(u)
        ds = np.zeros(1) if entropy else None
        self._check(self._fn("rhs")(self.ctx, ptr(u), ptr(halo_lo), ptr(halo_hi), ptr(out), ptr(ds)))
        return (out, float(ds[0])) if entropy else out

    def traces(self, u):
        tr = np.zeros((self.ne, 6, 5, self.nf))
        self._check(self._fn("traces")(self.ctx, ptr(np.ascontiguousarray(u)), ptr(tr)))
        return tr

    def boundary_traces(self, u):
        m = self.cfg.m
        lo = np.zeros((m * m, 5, self.nf))
        hi = np.zeros((m * m, 5, self.nf))
        self._check(self._fn("boundary_traces")(self.ctx, ptr(np.ascontiguousarray(u)), ptr(lo), ptr(hi)))
        return lo, hi

    def max_wavespeed(self, u):
        lam = np.zeros(1)
        self._check(self._fn("max_wavespeed")(self.ctx, ptr(np.ascontiguousarray(u)), ptr(lam)))
        return float(lam[0])

    def dx(self):
        xl, xr = self.cfg.domain()
        return (xr - xl) / (self.cfg.m * (self.cfg.p + 1))

    def rk4_step(self, u, dt):
        self._check(self._fn("rk4_step")(self.ctx, ptr(u), dt))
        return u

    def l2_sq(self, u, t, case=None):
        out = np.zeros(2)
        self._check(self._fn("l2_error")(self.ctx, ptr(np.ascontiguousarray(u)), t,
                                         CASES[case or self.cfg.case], ptr(out)))
        return out

    def l2_error(self, u, t, case=None):
        return np.sqrt(self.l2_sq(u, t, case))

    def entropy_total(self, u):
        out = np.zeros(1)
        self._check(self._fn("entropy_total")(self.ctx, ptr(np.ascontiguousarray(u)), ptr(out)))
        return float(out[0])

    def conserved_totals(self, u):
        out = np.zeros(5)
        self._check(self._fn("conserved_totals")(self.ctx, ptr(np.ascontiguousarray(u)), ptr(out)))
        return out

    def ke_volume(self, u):
        out = np.zeros(1)
        self._check(self._fn("ke_volume")(self.ctx, ptr(np.ascontiguousarray(u)), ptr(out)))
        return float(out[0])

    def ke_total(self, u):
        out = np.zeros(1)
        self._check(self._fn("ke_total")(self.ctx, ptr(np.ascontiguousarray(u)), ptr(out)))
        return float(out[0])

    def run(self, u, steps, cfl=0.1, t_final=None, t0=0.0):
        """RK4 driver: dt = cfl*dx/lambda_max from u_n each step, clipped to t_final."""
        t = t0
        for _ in range(steps):
            lam = self.max_wavespeed(u)
            dt = cfl * self.dx() / lam if lam > 0 else cfl * self.dx()
            if t_final is not None:
                if t >= t_final:
                    break
                dt = min(dt, t_final - t)
            self.rk4_step(u, dt)
            t += dt
        return u, t


def prim_fn(kind: str, name: str):
    lib, prefix = load(kind)
    return getattr(lib, prefix + name)
