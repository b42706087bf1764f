"""Small driver for ncu: p, m from argv; a few RK4 steps on the device."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import C_PLUS, GpuSolver, SolverConfig  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
m = int(sys.argv[2]) if len(sys.argv) > 2 else 32
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = GpuSolver(SolverConfig(p=p, m=m, c1d=C_PLUS.get(p, 0.0)))
g.init_case()
for _ in range(steps):
    g.rk4_step(0.1)
print("ok", g.time)
