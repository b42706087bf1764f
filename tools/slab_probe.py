"""Per-rank slab work at the strong-scaling partition of bench.py's config
(128^3, p=4, c_+, EC+Roe), measured on ONE GPU (dev tool).

For N = 1, 2, 4, 8 this times rank 0's z-slab [0, m/N) as an external-halo
context (nranks = N, no NCCL id): 4 x (K2 + K3) per RK4 step plus the step
kernels, exactly the kernels rank 0 runs in an N-GPU job. The halo planes are
set once (the slab's own send planes) and not moved between stages, so the
number excludes the NVLink transfer; the transfer per stage is
2 planes x m^2 x 5 x n^2 doubles sent (printed), which in the N-GPU graph runs on its own
stream under the interior planes' K2. Nothing here waits on another rank.

    python tools/slab_probe.py [m] [p] [steps]
prints one JSON line per N and a markdown table on stderr.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_07725_b200 import C_PLUS, GpuSolver, SolverConfig  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 128
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
n = p + 1


def time_slab(nranks):
    cfg = SolverConfig(p=p, m=m, c1d=C_PLUS[p], rank=0, nranks=nranks)
    g = GpuSolver(cfg)
    try:
        g.init_case()
        graph_ms = None
        if nranks == 1:  # whole box: also the captured graph step bench.py times
            g.time_steps(2)
            graph_ms = g.time_steps(steps) / steps
        g.project()
        if nranks > 1:
            lo, hi = g.halo_get()
            g.halo_set(hi, lo)  # valid planes of the right shape (the slab's own)
        dt = 1e-4

        def step():  # K3 of stage 4 leaves the projection of u_{n+1} in place
            for s in range(1, 5):
                g.stage(s, dt)

        for _ in range(2):
            step()
        t0 = time.perf_counter()
        for _ in range(steps):
            step()
        return g.ne, (time.perf_counter() - t0) / steps * 1e3, graph_ms
    finally:
        g.close()


rows = []
base = None
for nr in (1, 2, 4, 8):
    ne, ms, graph_ms = time_slab(nr)
    dof = ne * n ** 3 * 5
    rate = 4 * dof / (ms / 1e3)
    if base is None:
        base = ms
    eff = base / (nr * ms)
    halo_mb = 2 * m * m * 5 * n * n * 8 / 1e6
    row = {"nranks": nr, "elements": ne, "ms_per_step": ms, "dof_updates_per_s_per_gpu": rate,
           "projected_job_dof_updates_per_s": rate * nr, "compute_efficiency": eff,
           "halo_mb_sent_per_stage": halo_mb if nr > 1 else 0.0,
           "graph_ms_per_step": graph_ms}
    rows.append(row)
    print(json.dumps(row), flush=True)

print("| N | rank-0 elements | ms / RK4 step | DOF/s per GPU | projected job DOF/s | efficiency vs N=1 |",
      file=sys.stderr)
print("|---|---|---|---|---|---|", file=sys.stderr)
for r in rows:
    print(f"| {r['nranks']} | {r['elements']} | {r['ms_per_step']:.2f} | {r['dof_updates_per_s_per_gpu']:.3e} | "
          f"{r['projected_job_dof_updates_per_s']:.3e} | {100 * r['compute_efficiency']:.1f}% |", file=sys.stderr)
