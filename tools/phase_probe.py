"""K2/K3 phase breakdown (needs tools/libnsfr_phase.so built with -DNSFR_PHASE_PROF):
per-CTA clock64 deltas summed over CTAs, as shares of each kernel."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["NSFR_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnsfr_phase.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import C_PLUS, GpuSolver, SolverConfig, load_library  # noqa: E402

K2 = {0: "staging", 1: "line phase", 2: "volume-row output"}
K3 = {8: "staging", 9: "lift + Pi~^T (M passes)", 10: "Pi~ passes + RK", 11: "v(u_q) + primitives",
      12: "face contraction", 13: "u(v~) at faces + traces"}
lib = load_library()
lib.nsfr_gpu_phase_counters.argtypes = [C.POINTER(C.c_double)]
for spec in (sys.argv[1:] or ["4x64"]):
    p, m = map(int, spec.split("x"))
    g = GpuSolver(SolverConfig(p=p, m=m, c1d=C_PLUS.get(p, 0.0)))
    g.init_case()
    g.advance(1)
    out = np.zeros(16)
    lib.nsfr_gpu_phase_counters(out.ctypes.data_as(C.POINTER(C.c_double)))
    g.advance(2)
    lib.nsfr_gpu_phase_counters(out.ctypes.data_as(C.POINTER(C.c_double)))
    for name, d in (("K2", K2), ("K3", K3)):
        tot = sum(out[i] for i in d)
        print(f"p={p} m={m} {name}: " + ", ".join(f"{n} {100 * out[i] / tot:.1f}%" for i, n in d.items()))
    g.close()
