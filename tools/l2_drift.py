"""configs[2] p=4 (32^3 vortex, c_DG, EC+Roe) to t_f = 2 against the reference-build
golden: the L2 drift of a library variant (NSFR_B200_LIB), dev tool."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import GpuSolver, SolverConfig  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
key, tf = ("p4", 2.0) if p == 4 else ("p5_t0.2", 0.2)
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "config3.json")))[key]
g = GpuSolver(SolverConfig(p=p, m=32, c1d=0.0, roe=True))
g.init_case()
t = g.advance(3000, cfl=0.1, t_final=tf)
l2 = np.array(g.l2_error())
err = np.abs(l2 - np.array(gold["l2"]))
print(json.dumps({"lib": os.environ.get("NSFR_B200_LIB", "default"), "p": p, "t": t, "dt_t": t - gold["t_final"],
                  "err": err.tolist(), "rel": (err / np.array(gold["l2"])).tolist()}))
