"""Timing probe: per-kernel launch times at a few sizes (dev tool)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import C_PLUS, GpuSolver, SolverConfig  # noqa: E402

sizes = [(int(a), int(b)) for a, b in (s.split("x") for s in (sys.argv[1:] or ["4x64"]))]
for p, m in sizes:
    # NSFR_PROBE_C: a c value for degrees without a c_+ preset (general K3 variant instead of the c_DG one)
    g = GpuSolver(SolverConfig(p=p, m=m, c1d=C_PLUS.get(p, float(os.environ.get("NSFR_PROBE_C", "0")))))
    g.init_case()
    g.advance(2)
    ms = g.time_steps(4)
    ms_k, kms = g.time_steps(3, per_kernel=True)
    dof = m ** 3 * (p + 1) ** 3 * 5
    print(json.dumps({"lib": os.environ.get("NSFR_B200_LIB", "default"), "p": p, "m": m,
                      "ms_per_step": ms / 4, "dof_updates_per_s": 4 * dof * 4 / (ms / 1e3),
                      "k2_ms": kms[1] / 12, "k3_ms": kms[2] / 12,
                      "ns_per_elem_rhs": (ms / 4 / 4) * 1e6 / m ** 3}), flush=True)
    g.close()
