"""Does co-scheduling K2 (FP64-latency bound) with K3 (barrier / HBM bound) on
the SMs pay? Times the chunked wavefront schedule of the streamed step with the
host copies switched off (NSFR_STREAM_NOCOPY) over chunk / lane counts,
against the monolithic graph step, at the bench workload (dev tool)."""
import json
import os
import sys
import time

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


print(json.dumps({"advance_ms": t(lambda: g.advance(1))}), flush=True)
dt = g.rk4_step_host(host, host, cfl=0.1)[1]
os.environ["NSFR_STREAM_NOCOPY"] = "1"
for ch in (8, 16, 32, 64, 128):
    for ln in (2, 4, 8):
        os.environ["NSFR_STREAM_CHUNKS"] = str(ch)
        os.environ["NSFR_STREAM_LANES"] = str(ln)
        print(json.dumps({"chunks": ch, "lanes": ln,
                          "nocopy_fixed_ms": t(lambda: g.rk4_step_host(host, host, dt=dt))}), flush=True)
