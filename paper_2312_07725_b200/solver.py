"""Python mirror of the NSFR solver API over the C ABI (include/nsfr_gpu.h).

Names and argument meaning follow the reference's solver surface
(SPEC.md:422-518): operator/mesh setup happens in `GpuSolver(...)`
(build_reference_operators + warp_grid_3d + build_metrics_conservative_curl,
proj/src/fr_operators.cpp:89-113, geometry.cpp:62-266), `rhs` is
`nsfr_residual`/`assemble_rhs`, `rk4_step`/`advance` the time-step driver,
`l2_error` the diagnostic. Errors map to the reference's exception taxonomy
(proj/include/nsfr/defs.hpp:12-32).

There is no CPU fallback: constructing a GpuSolver without the built
libnsfr_b200.so or without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NSFR_B200_LIB") or os.path.join(HERE, "libnsfr_b200.so")

CASES = {"vortex": 0, "tgv": 1, "free_stream": 2}
C_PLUS = {2: 0.5 * 0.206, 3: 0.5 * 3.80e-3, 4: 0.5 * 4.67e-5, 5: 0.5 * 4.28e-7}
DOMAINS = {"vortex": (0.0, 10.0), "tgv": (-np.pi, np.pi), "free_stream": (0.0, 2 * np.pi)}

NSFR_OK, NSFR_E_DIM, NSFR_E_MESH, NSFR_E_INADMISSIBLE, NSFR_E_CUDA, NSFR_E_NCCL, NSFR_E_CONFIG = range(7)


class NsfrError(RuntimeError):
    pass


class DimensionError(NsfrError):          # defs.hpp:12-14
    pass


class InvalidMeshError(NsfrError):        # defs.hpp:16-18
    pass


class StepFailureError(NsfrError):        # defs.hpp:24-28 (InadmissibleStateError during a step)
    def __init__(self, what: str, t: float | None = None):
        super().__init__(what)
        self.t = t


class ConfigError(NsfrError):             # defs.hpp:30-32
    pass


class DeviceError(NsfrError):
    pass


_ERRORS = {NSFR_E_DIM: DimensionError, NSFR_E_MESH: InvalidMeshError,
           NSFR_E_INADMISSIBLE: StepFailureError, NSFR_E_CUDA: DeviceError,
           NSFR_E_NCCL: DeviceError, NSFR_E_CONFIG: ConfigError}


class _Tables(C.Structure):
    _fields_ = [(n, C.POINTER(C.c_double)) for n in
                ("interp", "proj", "fr_proj", "skew", "bound_flux", "bound_sol", "wq")]


SCHEMES = {"nsfr": 0, "dg": 1}


def _scheme_id(name: str) -> int:
    if name not in SCHEMES:
        raise ConfigError(f"scheme must be one of {sorted(SCHEMES)}, got {name!r}")
    return SCHEMES[name]


class _Setup(C.Structure):
    _fields_ = [
        ("p", C.c_int), ("quad_kind", C.c_int), ("c1d", C.c_double), ("gamma", C.c_double),
        ("roe", C.c_int), ("m", C.c_int), ("k0", C.c_int), ("k1", C.c_int),
        ("x_left", C.c_double), ("x_right", C.c_double), ("beta", C.c_double),
        ("length_scale", C.c_double), ("grid_degree", C.c_int), ("device", C.c_int),
        ("entropy_diag", C.c_int), ("tables", C.POINTER(_Tables)),
        ("jac_vol", C.POINTER(C.c_double)), ("cof_vol", C.POINTER(C.c_double)),
        ("nccl_id", C.c_void_p), ("rank", C.c_int), ("nranks", C.c_int),
        ("scheme", C.c_int), ("overint", C.c_int),
    ]


class _HaloPlan(C.Structure):
    _fields_ = [("k0", C.c_int), ("k1", C.c_int), ("peer_lo", C.c_int), ("peer_hi", C.c_int),
                ("count", C.c_longlong)]


_lib: C.CDLL | None = None


def load_library() -> C.CDLL:
    """Load the in-tree CUDA library; raises if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                          "(python -m paper_2312_07725_b200.build)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER(C.c_double)
    V = C.c_void_p
    sig = {
        "nsfr_gpu_create": (C.c_int, [C.POINTER(_Setup), C.POINTER(V)]),
        "nsfr_gpu_destroy": (C.c_int, [V]),
        "nsfr_gpu_last_error": (C.c_char_p, [V]),
        "nsfr_gpu_create_error": (C.c_char_p, []),
        "nsfr_gpu_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "nsfr_gpu_halo_plan_for": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_HaloPlan)]),
        "nsfr_gpu_get_tables": (C.c_int, [V, P, C.c_int]),
        "nsfr_gpu_get_metrics": (C.c_int, [V, P, P]),
        "nsfr_gpu_set_state": (C.c_int, [V, P]),
        "nsfr_gpu_get_state": (C.c_int, [V, P]),
        "nsfr_gpu_init_case": (C.c_int, [V, C.c_int]),
        "nsfr_gpu_set_time": (C.c_int, [V, C.c_double]),
        "nsfr_gpu_get_time": (C.c_int, [V, P]),
        "nsfr_gpu_rhs": (C.c_int, [V, P, P]),
        "nsfr_gpu_get_traces": (C.c_int, [V, P]),
        "nsfr_gpu_rk4_step": (C.c_int, [V, C.c_double, C.c_double, P]),
        "nsfr_gpu_advance": (C.c_int, [V, C.c_int, C.c_double, C.c_double, P]),
        "nsfr_gpu_rk4_step_dt": (C.c_int, [V, C.c_double]),
        "nsfr_gpu_rk4_step_host": (C.c_int, [V, P, P, C.c_double, C.c_double, C.c_double, P, P]),
        "nsfr_gpu_max_wavespeed": (C.c_int, [V, P]),
        "nsfr_gpu_l2_error": (C.c_int, [V, C.c_int, P]),
        "nsfr_gpu_entropy_change": (C.c_int, [V, P]),
        "nsfr_gpu_conserved_totals": (C.c_int, [V, P]),
        "nsfr_gpu_entropy_total": (C.c_int, [V, P]),
        "nsfr_gpu_set_state_q": (C.c_int, [V, P]),
        "nsfr_gpu_halo_get": (C.c_int, [V, P, P]),
        "nsfr_gpu_halo_set": (C.c_int, [V, P, P]),
        "nsfr_gpu_project": (C.c_int, [V]),
        "nsfr_gpu_residual": (C.c_int, [V, P, P]),
        "nsfr_gpu_stage": (C.c_int, [V, C.c_int, C.c_double]),
        "nsfr_gpu_get_state_q": (C.c_int, [V, P]),
        "nsfr_gpu_ke_volume": (C.c_int, [V, P]),
        "nsfr_gpu_ke_total": (C.c_int, [V, P]),
        "nsfr_gpu_time_steps": (C.c_int, [V, C.c_int, C.c_double, P, P]),
        "nsfr_gpu_state_device_ptr": (C.c_void_p, [V]),
        "nsfr_gpu_state_count": (C.c_size_t, [V]),
        "nsfr_gpu_sync": (C.c_int, [V]),
        "nsfr_gpu_launch_count": (C.c_longlong, [V]),
        "nsfr_gpu_measure_fp64_peak": (C.c_int, [C.c_int, P]),
        "nsfr_gpu_measure_fp64_peak_ex": (C.c_int, [C.c_int, P, P]),
        "nsfr_gpu_comm_info": (C.c_int, [V, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, "expect C-contiguous float64"
    return a.ctypes.data_as(C.POINTER(C.c_double))


def halo_plan(m: int, p: int, rank: int, nranks: int) -> dict:
    """z-slab partition + exchange peers used by the multi-GPU path (pure host logic)."""
    lib = load_library()
    hp = _HaloPlan()
    rc = lib.nsfr_gpu_halo_plan_for(m, p, rank, nranks, C.byref(hp))
    if rc:
        raise DimensionError(f"halo plan: m={m} nranks={nranks}")
    return {"k0": hp.k0, "k1": hp.k1, "peer_lo": hp.peer_lo, "peer_hi": hp.peer_hi, "count": hp.count}


def measure_fp64_peak(device: int = 0, with_clock: bool = False):
    """FP64 DFMA peak of the device in TFLOP/s (roofline denominator); with
    with_clock, (tflops, sm_mhz) with the SM clock the DFMA loop ran at."""
    out = np.zeros(1)
    mhz = np.zeros(1)
    if load_library().nsfr_gpu_measure_fp64_peak_ex(device, _ptr(out), _ptr(mhz)):
        raise DeviceError("fp64 peak measurement failed")
    return (float(out[0]), float(mhz[0])) if with_clock else float(out[0])


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = load_library().nsfr_gpu_nccl_unique_id(buf)
    if rc:
        raise DeviceError("ncclGetUniqueId failed")
    return buf.raw


@dataclass
class SolverConfig:
    """SolverConfig of SPEC.md:432-438 restricted to the NSFR-EC path."""
    p: int = 3
    m: int = 8
    c1d: float = 0.0
    quad_kind: int = 0              # 0 GL, 1 LGL
    case: str = "vortex"
    roe: bool = True
    beta: float = 0.05
    length_scale: float = 0.0
    grid_degree: int | None = None  # None -> p+1 (geometry.hpp:50-51)
    gamma: float = 1.4
    entropy_diag: bool = False
    device: int = 0
    rank: int = 0
    nranks: int = 1
    x_left: float | None = None
    x_right: float | None = None
    scheme: str = "nsfr"            # "nsfr" (hot path) or "dg" (conservative strong-form DG)
    overint: int = 0                # extra quadrature nodes, n_q = p+1+overint (dg only)

    def domain(self):
        if self.x_left is not None:
            return self.x_left, self.x_right
        return DOMAINS[self.case]


class GpuSolver:
    """One context of the B200 NSFR path (one GPU, one z-slab)."""

    def __init__(self, cfg: SolverConfig, tables: dict | None = None, metrics=None,
                 nccl_id: bytes | None = None):
        self.lib = load_library()
        self.cfg = cfg
        xl, xr = cfg.domain()
        if cfg.nranks > 1:
            plan = halo_plan(cfg.m, cfg.p, cfg.rank, cfg.nranks)
            k0, k1 = plan["k0"], plan["k1"]
        else:
            k0, k1 = 0, cfg.m
        self.k0, self.k1 = k0, k1
        self._keep = []
        tab_ptr = None
        if tables is not None:
            arrs = [np.ascontiguousarray(tables[k], dtype=np.float64) for k in
                    ("interp", "proj", "fr_proj", "skew", "bound_flux", "bound_sol", "wq")]
            self._keep += arrs
            t = _Tables(*[_ptr(a) for a in arrs])
            self._keep.append(t)
            tab_ptr = C.pointer(t)
        jac = cof = None
        if metrics is not None:
            jac = np.ascontiguousarray(metrics[0], dtype=np.float64)
            cof = np.ascontiguousarray(metrics[1], dtype=np.float64)
            self._keep += [jac, cof]
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(nccl_id, 128)
            self._keep.append(idbuf)
        s = _Setup(cfg.p, cfg.quad_kind, cfg.c1d, cfg.gamma, int(cfg.roe), cfg.m, k0, k1, xl, xr,
                   cfg.beta, cfg.length_scale,
                   cfg.p + 1 if cfg.grid_degree is None else cfg.grid_degree, cfg.device,
                   int(cfg.entropy_diag), tab_ptr, _ptr(jac), _ptr(cof),
                   C.cast(idbuf, C.c_void_p) if idbuf is not None else None, cfg.rank, cfg.nranks,
                   _scheme_id(cfg.scheme), cfg.overint)
        h = C.c_void_p()
        rc = self.lib.nsfr_gpu_create(C.byref(s), C.byref(h))
        if rc:
            raise _ERRORS.get(rc, NsfrError)(self.lib.nsfr_gpu_create_error().decode())
        self.ctx = h
        self.n = cfg.p + 1                 # solution nodes per direction
        self.nq = cfg.p + 1 + cfg.overint  # volume quadrature nodes per direction
        self.nquad = self.nq ** 3
        self.ne = cfg.m * cfg.m * (k1 - k0)
        self.nsol = self.n ** 3

    # --- plumbing -------------------------------------------------------------
    def _check(self, rc):
        if rc:
            msg = self.lib.nsfr_gpu_last_error(self.ctx).decode()
            if rc == NSFR_E_INADMISSIBLE:
                t = np.zeros(1)  # the failing stage's step time (StepFailureError{t})
                ok = self.lib.nsfr_gpu_get_time(self.ctx, _ptr(t)) == NSFR_OK
                raise StepFailureError(msg, float(t[0]) if ok else None)
            raise _ERRORS.get(rc, NsfrError)(msg)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.nsfr_gpu_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def state_shape(self):
        return (self.ne, 5, self.nsol)

    def launch_count(self) -> int:
        return int(self.lib.nsfr_gpu_launch_count(self.ctx))

    def comm_info(self) -> dict:
        """The NCCL communicator as NCCL reports it (nranks 0 without one)."""
        n, r, d = C.c_int(), C.c_int(), C.c_int()
        self._check(self.lib.nsfr_gpu_comm_info(self.ctx, C.byref(n), C.byref(r), C.byref(d)))
        return {"nccl_nranks": n.value, "nccl_rank": r.value, "cuda_device": d.value}

    # --- setup products -------------------------------------------------------
    def tables(self) -> dict[str, np.ndarray]:
        n, q = self.n, self.nq
        buf = np.zeros(4096)
        cnt = self.lib.nsfr_gpu_get_tables(self.ctx, _ptr(buf), buf.size)
        shapes = [("interp", (q, n)), ("proj", (n, q)), ("fr_proj", (n, q)), ("skew", (q, q)),
                  ("bound_flux", (2, q)), ("bound_sol", (2, n)), ("wq", (q,)), ("quad_nodes", (q,)),
                  ("sol_nodes", (n,)), ("mmass1d", (n, n)), ("quad_diff", (q, q))]
        out, pos = {}, 0
        for name, shp in shapes:
            sz = int(np.prod(shp))
            out[name] = buf[pos:pos + sz].reshape(shp).copy()
            pos += sz
        assert pos == cnt
        return out

    def metrics(self):
        jac = np.zeros((self.ne, self.nquad))
        cof = np.zeros((self.ne, self.nquad, 9))
        self._check(self.lib.nsfr_gpu_get_metrics(self.ctx, _ptr(jac), _ptr(cof)))
        return jac, cof

    # --- state ----------------------------------------------------------------
    def set_state(self, u: np.ndarray):
        u = np.ascontiguousarray(u, dtype=np.float64)
        assert u.shape == self.state_shape, (u.shape, self.state_shape)
        self._check(self.lib.nsfr_gpu_set_state(self.ctx, _ptr(u)))

    def get_state(self, out: np.ndarray | None = None) -> np.ndarray:
        """Download the state; `out` (e.g. a pinned host buffer) is filled in place."""
        u = np.zeros(self.state_shape) if out is None else out
        assert u.shape == self.state_shape and u.dtype == np.float64 and u.flags.c_contiguous
        self._check(self.lib.nsfr_gpu_get_state(self.ctx, _ptr(u)))
        return u

    def init_case(self, case: str | None = None):
        self._check(self.lib.nsfr_gpu_init_case(self.ctx, CASES[case or self.cfg.case]))

    def set_state_q(self, uq: np.ndarray):
        """Upload the solver's own representation (u at the volume quadrature nodes)."""
        uq = np.ascontiguousarray(uq, dtype=np.float64)
        assert uq.shape == self.state_shape, (uq.shape, self.state_shape)
        self._check(self.lib.nsfr_gpu_set_state_q(self.ctx, _ptr(uq)))

    def get_state_q(self) -> np.ndarray:
        """u at the volume quadrature nodes, exactly as the solver carries it."""
        uq = np.zeros(self.state_shape)
        self._check(self.lib.nsfr_gpu_get_state_q(self.ctx, _ptr(uq)))
        return uq

    def set_time(self, t: float):
        self._check(self.lib.nsfr_gpu_set_time(self.ctx, t))

    @property
    def time(self) -> float:
        t = np.zeros(1)
        self._check(self.lib.nsfr_gpu_get_time(self.ctx, _ptr(t)))
        return float(t[0])

    # --- hot path -------------------------------------------------------------
    def rhs(self, entropy: bool = False):
        """assemble_rhs of the current state -> dU/dt [e][5][np^3] (and the entropy change)."""
        out = np.zeros(self.state_shape)
        ds = np.zeros(1) if entropy else None
        self._check(self.lib.nsfr_gpu_rhs(self.ctx, _ptr(out), _ptr(ds)))
        return (out, float(ds[0])) if entropy else out

    def traces(self) -> np.ndarray:
        tr = np.zeros((self.ne, 6, 5, self.nq * self.nq))
        self._check(self.lib.nsfr_gpu_get_traces(self.ctx, _ptr(tr)))
        return tr

    def max_wavespeed(self) -> float:
        lam = np.zeros(1)
        self._check(self.lib.nsfr_gpu_max_wavespeed(self.ctx, _ptr(lam)))
        return float(lam[0])

    def rk4_step(self, cfl: float = 0.1, t_final: float = 0.0) -> float:
        dt = np.zeros(1)
        self._check(self.lib.nsfr_gpu_rk4_step(self.ctx, cfl, t_final, _ptr(dt)))
        return float(dt[0])

    def rk4_step_dt(self, dt: float):
        self._check(self.lib.nsfr_gpu_rk4_step_dt(self.ctx, dt))

    def rk4_step_host(self, u_in: np.ndarray, u_out: np.ndarray | None = None, dt: float = 0.0,
                      cfl: float = 0.1, t_final: float = 0.0) -> tuple[np.ndarray, float, float]:
        """rk4_step(field, dt) on host state: upload u_in, one RK4
        step (dt if dt > 0, else adaptive_dt(u_in, cfl) clipped to t_final),
        download into u_out (may be u_in; pinned buffers let the copies overlap
        the compute). Returns (u_out, dt used, adaptive_dt(u_out, cfl) clipped to
        t_final): feeding the last back as dt is the reference's
        `dt = adaptive_dt(u); u = rk4_step(u, dt)` loop without a barrier."""
        for a in (u_in,) + ((u_out,) if u_out is not None else ()):
            assert a.shape == self.state_shape and a.dtype == np.float64 and a.flags.c_contiguous
        out = np.zeros(self.state_shape) if u_out is None else u_out
        used, nxt = np.zeros(1), np.zeros(1)
        self._check(self.lib.nsfr_gpu_rk4_step_host(self.ctx, _ptr(u_in), _ptr(out), dt, cfl, t_final,
                                                    _ptr(used), _ptr(nxt)))
        return out, float(used[0]), float(nxt[0])

    def advance(self, nsteps: int, cfl: float = 0.1, t_final: float = 0.0) -> float:
        t = np.zeros(1)
        self._check(self.lib.nsfr_gpu_advance(self.ctx, nsteps, cfl, t_final, _ptr(t)))
        return float(t[0])

    def l2_error(self, case: str | None = None) -> np.ndarray:
        out = np.zeros(2)
        self._check(self.lib.nsfr_gpu_l2_error(self.ctx, CASES[case or self.cfg.case], _ptr(out)))
        return out

    def entropy_change(self) -> float:
        out = np.zeros(1)
        self._check(self.lib.nsfr_gpu_entropy_change(self.ctx, _ptr(out)))
        return float(out[0])

    def entropy_total(self) -> float:
        """sum w J U(u) with U = -rho s/(gamma-1) (entropy-change normaliser)."""
        out = np.zeros(1)
        self._check(self.lib.nsfr_gpu_entropy_total(self.ctx, _ptr(out)))
        return float(out[0])

    def ke_volume(self) -> float:
        """Kinetic-energy volume term (flux minus pressure work, S6 rows . v_KE)."""
        out = np.zeros(1)
        self._check(self.lib.nsfr_gpu_ke_volume(self.ctx, _ptr(out)))
        return float(out[0])

    # --- stage-level driving / external halo transport (nranks > 1, no NCCL id)
    @property
    def halo_shape(self):
        # NTR = 6 values per face node (NSFR: primitives rho,u,v,w,p,rho/p; DG uses 5 of them)
        return (self.cfg.m * self.cfg.m, 6, self.nq * self.nq)

    def halo_get(self):
        """The two send planes (face 4 of plane k0, face 5 of plane k1-1)."""
        lo, hi = np.zeros(self.halo_shape), np.zeros(self.halo_shape)
        self._check(self.lib.nsfr_gpu_halo_get(self.ctx, _ptr(lo), _ptr(hi)))
        return lo, hi

    def halo_set(self, recv_lo: np.ndarray, recv_hi: np.ndarray):
        lo = np.ascontiguousarray(recv_lo, dtype=np.float64)
        hi = np.ascontiguousarray(recv_hi, dtype=np.float64)
        assert lo.shape == self.halo_shape and hi.shape == self.halo_shape
        self._check(self.lib.nsfr_gpu_halo_set(self.ctx, _ptr(lo), _ptr(hi)))

    def project(self):
        self._check(self.lib.nsfr_gpu_project(self.ctx))

    def residual(self, entropy: bool = False):
        """dU/dt of the projected state (after project() and the halo swap)."""
        out = np.zeros(self.state_shape)
        ds = np.zeros(1) if entropy else None
        self._check(self.lib.nsfr_gpu_residual(self.ctx, _ptr(out), _ptr(ds)))
        return (out, float(ds[0])) if entropy else out

    def stage(self, s: int, dt: float):
        self._check(self.lib.nsfr_gpu_stage(self.ctx, s, dt))

    def ke_total(self) -> float:
        """Kinetic-energy change minus pressure work (-v_hat_KE . R of F - P, no Roe)."""
        out = np.zeros(1)
        self._check(self.lib.nsfr_gpu_ke_total(self.ctx, _ptr(out)))
        return float(out[0])

    def conserved_totals(self) -> np.ndarray:
        """sum w J u over the (global) domain: mass, momentum x3, energy."""
        out = np.zeros(5)
        self._check(self.lib.nsfr_gpu_conserved_totals(self.ctx, _ptr(out)))
        return out

    def time_steps(self, nsteps: int, cfl: float = 0.1, per_kernel: bool = False):
        ms = np.zeros(1)
        kms = np.zeros(3) if per_kernel else None
        self._check(self.lib.nsfr_gpu_time_steps(self.ctx, nsteps, cfl, _ptr(ms), _ptr(kms)))
        return (float(ms[0]), kms.copy()) if per_kernel else float(ms[0])
