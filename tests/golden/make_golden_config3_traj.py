"""Golden L2 trajectories of BASELINE configs[2] from the REFERENCE's own compiled code,
plus the reference's own 1-ulp trajectory floor (TEST INFRASTRUCTURE ONLY).

32^3 isentropic vortex, c_DG, EC + Roe, RK4 at CFL 0.1 to t_f = 2 (p = 5: ~916
steps, ~2.5 h of oracle/_ref on 8 cores). The run records L2(rho), L2(p) and t after
the step counts in CHECKPOINTS and at the final time, so a GPU test can compare at
any checkpoint by running the same number of adaptive steps.

    python tests/golden/make_golden_config3_traj.py P [--perturbed] [--max-steps K]

--perturbed moves every modal coefficient by one ulp in a seeded random direction
(numpy default_rng(20231207)) at the start AND after every RK4 step: the
difference between the two runs is the reference's own trajectory floor, i.e.
how far two fp64 evaluations of the same scheme whose every step differs by
rounding drift apart (a single kick of the initial state underestimates it:
two implementations differ at every RHS, not once).
Results merge into tests/golden/config3_traj.json under "p{P}" / "p{P}_perturbed".
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle_lib import Config, CpuSolver  # noqa: E402

CHECKPOINTS = (1, 10, 20, 50, 92, 100, 200, 300, 400, 500, 600, 700, 800, 900)


def ulp_perturb(u, rng):
    sign = rng.integers(0, 2, size=u.shape) * 2 - 1
    return np.nextafter(u, u + sign * np.inf)


def main():
    args = sys.argv[1:]
    perturbed = "--perturbed" in args
    args = [a for a in args if a != "--perturbed"]
    max_steps = 100000
    if "--max-steps" in args:
        i = args.index("--max-steps")
        max_steps = int(args[i + 1])
        del args[i:i + 2]
    p = int(args[0]) if args else 5
    t_final = 2.0
    path = os.path.join(HERE, "config3_traj.json")
    key = f"p{p}" + ("_perturbed" if perturbed else "")

    s = CpuSolver("ref", Config(p=p, m=32, c1d=0.0, case="vortex", roe=True,
                                workers=int(os.environ.get("NSFR_GOLDEN_WORKERS", os.cpu_count()))))
    u = s.initial_state()
    rng = np.random.default_rng(20231207)
    if perturbed:
        u = ulp_perturb(u, rng)
    t0 = time.time()
    t, step, rec = 0.0, 0, {}

    def save(res):
        # merged into the JSON after every checkpoint, so a cut-off run keeps
        # what it reached ("partial": true until t_f)
        out = {}
        if os.path.exists(path):
            with open(path) as f:
                out = json.load(f)
        out[key] = res
        tmp = path + ".tmp"
        with open(tmp, "w") as f:
            json.dump(out, f, indent=1)
        os.replace(tmp, path)

    while t < t_final and step < max_steps:
        lam = s.max_wavespeed(u)
        dt = min(0.1 * s.dx() / lam, t_final - t)
        s.rk4_step(u, dt)
        t += dt
        step += 1
        if perturbed:
            u[...] = ulp_perturb(u, rng)
        if step in CHECKPOINTS:
            rec[str(step)] = {"t": t, "l2": s.l2_error(u, t).tolist()}
            print(key, step, rec[str(step)], f"{time.time() - t0:.0f}s", flush=True)
            save({"t_target": t_final, "partial": True, "checkpoints": rec,
                  "seconds": time.time() - t0, "perturbed": perturbed})
    res = {"t_target": t_final, "t_final": t, "steps": step, "checkpoints": rec,
           "l2": s.l2_error(u, t).tolist(), "seconds": time.time() - t0,
           "perturbed": perturbed}
    print(key, "final", res["steps"], res["t_final"], res["l2"], flush=True)
    save(res)


if __name__ == "__main__":
    main()
