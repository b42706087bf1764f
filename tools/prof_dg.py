"""Small driver for ncu on the DG kernels: p, m, overint from argv."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import GpuSolver, SolverConfig  # noqa: E402

p, m, oi = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (4, 32, 0)))
g = GpuSolver(SolverConfig(p=p, m=m, scheme="dg", overint=oi, case="tgv"))
g.init_case()
g.advance(2)
print("ok", g.time)
