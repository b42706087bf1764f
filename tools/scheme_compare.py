"""Cost comparison of the paper's schemes on the B200 (PAPER.md:1896-1992,
Table "TGV Comparison for CPU and Wall Clock Times"): NSFR-EC c_DG / c_+ (the
hot path), conservative DG (Roe surface flux) and overintegrated conservative
DG, on the warped TGV grid, RK4 steps timed with CUDA events (graph replay).
Prints one JSON line per (scheme, p) with ms per RK4 step and ns per element-RHS.

    python tools/scheme_compare.py [m] [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import C_PLUS, GpuSolver, SolverConfig  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
runs = []
for p in (3, 4, 5):
    runs += [("NSFR-EC c_DG", dict(p=p, c1d=0.0, roe=False)),
             ("NSFR-EC c_+", dict(p=p, c1d=C_PLUS[p], roe=False)),
             ("DG-cons", dict(p=p, scheme="dg", roe=True)),
             ("DG-cons overint 1", dict(p=p, scheme="dg", overint=1, roe=True)),
             ("DG-cons overint 2", dict(p=p, scheme="dg", overint=2, roe=True))]
for name, kw in runs:
    g = GpuSolver(SolverConfig(m=m, case="tgv", **kw))
    g.init_case()
    g.advance(2, cfl=0.1)
    ms = g.time_steps(steps, cfl=0.1) / steps
    _, kms = g.time_steps(2, cfl=0.1, per_kernel=True)  # [K1 or KD1, K2 or KD2, K3] summed
    ne = m ** 3
    print(json.dumps({"scheme": name, "p": kw["p"], "m": m, "ms_per_rk4_step": ms,
                      "ns_per_element_rhs": ms * 1e6 / (4 * ne),
                      "kernel_ms_per_stage": [round(x / 8, 4) for x in kms],
                      "dof_updates_per_s": 4 * ne * (kw["p"] + 1) ** 3 * 5 / (ms * 1e-3)}), flush=True)
    g.close()
