"""Golden L2 errors of BASELINE configs[2] from the REFERENCE's own compiled code.

32^3 isentropic vortex, c_DG, EC + Roe, advanced to t_f = 2 with RK4 at CFL 0.1
(p = 4: ~763 steps; p = 5: ~916 steps). Run here (needs oracle/_ref):
    python tests/golden/make_golden_config3.py 4 [5] [--t-final T]   (hours on 8 cores)
Merges {"p4": {...}, "p5": {...}} into tests/golden/config3.json. The p = 5
entry was made with --t-final 0.2 (~92 steps, ~26 min; the full t_f = 2 run is
~5 h of the reference build on 8 cores); the entry records its own t_target.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_lib import Config, CpuSolver  # noqa: E402

path = os.path.join(HERE, "config3.json")
args = sys.argv[1:]
t_target = 2.0
if "--t-final" in args:
    i = args.index("--t-final")
    t_target = float(args[i + 1])
    del args[i:i + 2]
for p in [int(a) for a in args] or [4]:
    t0 = time.time()
    s = CpuSolver("ref", Config(p=p, m=32, c1d=0.0, case="vortex", roe=True, workers=os.cpu_count()))
    u = s.initial_state()
    u, t = s.run(u, 100000, cfl=0.1, t_final=t_target)
    res = {"t_target": t_target, "t_final": t, "l2": s.l2_error(u, t).tolist(), "seconds": time.time() - t0}
    print(f"p{p}", res, flush=True)
    out = {}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f)
    out[f"p{p}"] = res
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
