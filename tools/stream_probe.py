"""Streamed host step vs its parts at the bench workload (128^3, p=4, c_+)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2312_07725_b200 as pkg  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = pkg.GpuSolver(pkg.SolverConfig(p=4, m=m, c1d=0.5 * 4.67e-5, case="vortex", roe=True))
g.init_case()
host = torch.empty(g.state_shape, dtype=torch.float64, pin_memory=True).numpy()
g.get_state(out=host)
g.advance(2)


def t(fn, n=3):
    fn()
    g.lib.nsfr_gpu_sync(g.ctx)
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    g.lib.nsfr_gpu_sync(g.ctx)
    return (time.perf_counter() - t0) / n * 1e3


out = {}
out["advance_ms"] = t(lambda: g.advance(1))
out["set_state_ms"] = t(lambda: g.set_state(host))
out["get_state_ms"] = t(lambda: g.get_state(out=host))
out["plain_e2e_ms"] = t(lambda: (g.set_state(host), g.rk4_step(0.1), g.get_state(out=host)))
out["streamed_adaptive_ms"] = t(lambda: g.rk4_step_host(host, host, cfl=0.1))
dt = g.rk4_step_host(host, host, cfl=0.1)[1]
out["streamed_fixed_ms"] = t(lambda: g.rk4_step_host(host, host, dt=dt))
box = [dt]


def chained():
    box[0] = g.rk4_step_host(host, host, dt=box[0], cfl=0.1)[2]


out["streamed_chained_ms"] = t(chained)
print(json.dumps(out))
