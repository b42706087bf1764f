"""Quick GPU-vs-oracle parity + timing probe (development tool; runs under gpurun)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import Config, CpuSolver  # noqa: E402

from paper_2312_07725_b200 import GpuSolver, SolverConfig  # noqa: E402


def rel(a, b):
    d = np.abs(a - b).reshape(a.shape[0], 5, -1).max(axis=(0, 2))
    r = np.abs(b).reshape(b.shape[0], 5, -1).max(axis=(0, 2))
    return float((d / r).max())


res = {}
for p, m, c1d, roe in ((3, 4, 0.0, True), (4, 4, 2.335e-5, True), (3, 4, 0.0, False)):
    cc = Config(p=p, m=m, c1d=c1d, roe=roe, workers=os.cpu_count())
    o = CpuSolver("oracle", cc)
    g = GpuSolver(SolverConfig(p=p, m=m, c1d=c1d, roe=roe, entropy_diag=True))
    key = f"p{p}_m{m}_c{c1d}_roe{int(roe)}"
    to, tg = o.tables(), g.tables()
    res[key + "_tables"] = max(float(np.abs(to[k] - tg[k]).max()) for k in to)
    jo, co = o.metrics()
    jg, cg = g.metrics()
    res[key + "_jac"] = float(np.abs(jo - jg).max() / np.abs(jo).max())
    res[key + "_cof"] = float(np.abs(co - cg).max() / np.abs(co).max())
    u0 = o.initial_state()
    g.init_case()
    res[key + "_ic"] = float(np.abs(g.get_state() - u0).max())
    g.set_state(u0)
    ro, dso = o.rhs(u0, entropy=True)
    rg, dsg = g.rhs(entropy=True)
    res[key + "_rhs_rel"] = rel(rg, ro)
    res[key + "_dS"] = [dso, dsg]
    lo, lg = o.max_wavespeed(u0), g.max_wavespeed()
    res[key + "_lam"] = [lo, lg]
    # 3 RK4 steps with the adaptive dt
    uo = u0.copy()
    uo, to_ = o.run(uo, 3, cfl=0.1)
    g.set_state(u0)
    g.set_time(0.0)
    for _ in range(3):
        g.rk4_step(0.1)
    ug = g.get_state()
    res[key + "_rk3_rel"] = rel(ug - u0, uo - u0)
    res[key + "_t"] = [to_, g.time]
    lo2 = o.l2_error(uo, to_)
    lg2 = g.l2_error()
    res[key + "_l2"] = [lo2.tolist(), lg2.tolist()]
    g.close()
print(json.dumps(res, indent=1))

# timing: config 3 / 5 style sizes
for p, m in ((3, 16), (4, 32), (4, 64), (5, 32)):
    g = GpuSolver(SolverConfig(p=p, m=m, c1d=0.0))
    g.init_case()
    t0 = time.time()
    g.advance(2)
    ms = g.time_steps(5)
    ms_k, kms = g.time_steps(3, per_kernel=True)
    dof = m ** 3 * (p + 1) ** 3 * 5
    print(json.dumps({"p": p, "m": m, "ms_per_step": ms / 5, "dof_updates_per_s": 4 * dof * 5 / (ms / 1e3),
                      "k1_ms_per_launch": kms[0] / 12, "k2_ms_per_launch": kms[1] / 12}))
    g.close()
