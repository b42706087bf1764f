"""Golden L2 errors of BASELINE configs[1] from the REFERENCE's own compiled code.

16^3 isentropic vortex, p = 3, EC + Roe, advanced to t_f = 2 with RK4 at CFL 0.1,
once with c_DG and once with c_+. Run here (needs oracle/_ref):
    python tests/golden/make_golden_config2.py     (~3 min on 8 cores)
Writes tests/golden/config2.json.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_lib import C_PLUS, Config, CpuSolver  # noqa: E402

out = {}
for name, c in (("c_dg", 0.0), ("c_plus", C_PLUS[3])):
    t0 = time.time()
    s = CpuSolver("ref", Config(p=3, m=16, c1d=c, case="vortex", roe=True, workers=os.cpu_count()))
    u = s.initial_state()
    u, t = s.run(u, 100000, cfl=0.1, t_final=2.0)
    out[name] = {"t_final": t, "l2": s.l2_error(u, t).tolist(), "seconds": time.time() - t0}
    print(name, out[name], flush=True)
with open(os.path.join(HERE, "config2.json"), "w") as f:
    json.dump(out, f, indent=1)
