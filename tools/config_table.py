"""Throughput on every BASELINE config: the B200 path
(CUDA-event timed RK4 graph steps) next to the reference's own compiled
primitives under the residual glue (oracle/_ref, all host threads, one RK4
step after a warm-up step) on the same box. Configs 1-4 run at full size on
both; config 5 (128^3) is bench.py's workload (GPU only here).

    python tools/config_table.py [gpu_steps]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2312_07725_b200 as nsfr  # noqa: E402
from oracle_lib import LIBS, Config, CpuSolver  # noqa: E402  (CPU reference leg only)

CONFIGS = [
    ("1: vortex 8^3 p=3 c_DG EC+Roe", dict(p=3, m=8, c1d=0.0, case="vortex", roe=True)),
    ("2: vortex 16^3 p=3 c_DG EC+Roe", dict(p=3, m=16, c1d=0.0, case="vortex", roe=True)),
    ("2: vortex 16^3 p=3 c_+ EC+Roe", dict(p=3, m=16, c1d=nsfr.C_PLUS[3], case="vortex", roe=True)),
    ("3: vortex 32^3 p=4 c_DG EC+Roe", dict(p=4, m=32, c1d=0.0, case="vortex", roe=True)),
    ("3: vortex 32^3 p=5 c_DG EC+Roe", dict(p=5, m=32, c1d=0.0, case="vortex", roe=True)),
    ("4: TGV 32^3 p=3 c_DG EC", dict(p=3, m=32, c1d=0.0, case="tgv", roe=False)),
    ("5: vortex 128^3 p=4 c_+ EC+Roe", dict(p=4, m=128, c1d=nsfr.C_PLUS[4], case="vortex", roe=True)),
]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
kind = "ref" if os.path.exists(LIBS["ref"][0]) else "oracle"
for name, kw in CONFIGS:
    g = nsfr.GpuSolver(nsfr.SolverConfig(**kw))
    g.init_case()
    g.advance(3, cfl=0.1)
    ms = g.time_steps(steps, cfl=0.1) / steps
    dof = kw["m"] ** 3 * (kw["p"] + 1) ** 3 * 5
    gpu = 4 * dof / (ms * 1e-3)
    g.close()
    cpu = None
    if kw["m"] <= 32:
        s = CpuSolver(kind, Config(workers=os.cpu_count() or 1, **kw))
        u = s.initial_state()
        dt = 0.1 * s.dx() / s.max_wavespeed(u)
        s.rk4_step(u, dt)
        t0 = time.perf_counter()
        s.rk4_step(u, dt)
        cpu = 4 * dof / (time.perf_counter() - t0)
    print(json.dumps({"config": name, "gpu_dof_updates_per_s": gpu, "gpu_ms_per_rk4_step": ms,
                      "cpu_reference_dof_updates_per_s": cpu, "cpu_kind": kind, "cpu_threads": os.cpu_count(),
                      "speedup": gpu / cpu if cpu else None}), flush=True)
