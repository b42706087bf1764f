"""K2 phase breakdown (needs tools/libnsfr_phase.so built with -DNSFR_PHASE_PROF)."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["NSFR_B200_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnsfr_phase.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import C_PLUS, GpuSolver, SolverConfig, load_library  # noqa: E402

lib = load_library()
lib.nsfr_gpu_phase_counters.argtypes = [C.POINTER(C.c_double)]
for spec in (sys.argv[1:] or ["4x64"]):
    p, m = map(int, spec.split("x"))
    g = GpuSolver(SolverConfig(p=p, m=m, c1d=C_PLUS.get(p, 0.0)))
    g.init_case()
    g.advance(1)
    out = np.zeros(4)
    lib.nsfr_gpu_phase_counters(out.ctypes.data_as(C.POINTER(C.c_double)))
    g.advance(2)
    lib.nsfr_gpu_phase_counters(out.ctypes.data_as(C.POINTER(C.c_double)))
    tot = out.sum()
    names = ["staging", "line", "lift+project", "WA+epilogue"]
    print(f"p={p} m={m}: " + ", ".join(f"{n} {100 * v / tot:.1f}%" for n, v in zip(names, out)))
    g.close()
