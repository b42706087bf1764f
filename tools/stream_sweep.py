"""Streamed host step (the e2e path) over chunk / lane counts at the bench
workload: chained reference loop dt = adaptive_dt(u); u = rk4_step(u, dt) on
pinned host buffers (dev tool)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2312_07725_b200 as pkg  # noqa: E402

g = pkg.GpuSolver(pkg.SolverConfig(p=4, m=128, c1d=0.5 * 4.67e-5, case="vortex", roe=True))
g.init_case()
host = torch.empty(g.state_shape, dtype=torch.float64, pin_memory=True).numpy()
g.get_state(out=host)
box = [g.rk4_step_host(host, host, cfl=0.1)[2]]


def chained():
    box[0] = g.rk4_step_host(host, host, dt=box[0], cfl=0.1)[2]


def t(fn, n=3):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e3


g.advance(1)
print(json.dumps({"advance_ms": t(lambda: g.advance(1))}), flush=True)
for ch in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["16", "32", "64", "128", "256"])]:
    for ln in (1, 2, 4, 8):
        os.environ["NSFR_STREAM_CHUNKS"] = str(ch)
        os.environ["NSFR_STREAM_LANES"] = str(ln)
        print(json.dumps({"chunks": ch, "lanes": ln, "chained_ms": t(chained)}), flush=True)
