"""K1 (k_project) timing probe: wall time of project() on a resident state (dev tool).
    NSFR_B200_LIB=... python tools/k1_probe.py 4x96"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402  (device synchronisation only)
from paper_2312_07725_b200 import C_PLUS, GpuSolver, SolverConfig  # noqa: E402

for p, m in [(int(a), int(b)) for a, b in (s.split("x") for s in (sys.argv[1:] or ["4x96"]))]:
    g = GpuSolver(SolverConfig(p=p, m=m, c1d=C_PLUS.get(p, 0.0)))
    g.init_case()
    u = g.get_state()
    ts = []
    for _ in range(4):
        g.set_state(u)            # invalidates the cached projection
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.project()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps({"lib": os.environ.get("NSFR_B200_LIB", "default"), "p": p, "m": m, "k1_ms": min(ts)}), flush=True)
    g.close()
