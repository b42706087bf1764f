"""Timing probe: repeated RHS evaluations (K1 + K2 + K3 stage 0) of a FIXED
state, no host copies: isolates kernel variants whose results may be wrong
(dev tool; NSFR_B200_LIB selects the library)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import C_PLUS, GpuSolver, SolverConfig  # noqa: E402

p, m = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4x64").split("x"))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = GpuSolver(SolverConfig(p=p, m=m, c1d=C_PLUS.get(p, 0.0)))
g.init_case()
g.advance(2)
lib, ctx = g.lib, g.ctx
for _ in range(3):
    lib.nsfr_gpu_rhs(ctx, None, None)
lib.nsfr_gpu_sync(ctx)
t0 = time.perf_counter()
for _ in range(reps):
    lib.nsfr_gpu_rhs(ctx, None, None)
lib.nsfr_gpu_sync(ctx)
ms = (time.perf_counter() - t0) / reps * 1e3
print(json.dumps({"lib": os.environ.get("NSFR_B200_LIB", "default"), "p": p, "m": m,
                  "rhs_ms": ms}), flush=True)
