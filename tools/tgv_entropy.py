"""Long-time TGV entropy conservation with the GPU solver (§7.3,
Fig. "TGV change entropy"; SURVEY §8(d) config 4 physics): EC flux (no Roe),
p = 3, warped [-pi, pi]^3 grid, RK4 at CFL 0.1 to t_f, DiagnosticRecord CSV
every `every` steps via runio.run_simulation.

    python tools/tgv_entropy.py m t_final every grid_degree out.csv
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_07725_b200 as nsfr  # noqa: E402

m, tf, every, gd = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
out = sys.argv[5]
for name, c in (("c_DG", 0.0), ("c_+", nsfr.C_PLUS[3])):
    g = nsfr.GpuSolver(nsfr.SolverConfig(p=3, m=m, c1d=c, case="tgv", roe=False, grid_degree=gd,
                                         entropy_diag=True))
    g.init_case()
    path = out.replace(".csv", f"_{name.replace('+', 'plus')}.csv")
    recs = nsfr.run_simulation(g, t_final=tf, cfl=0.1, diag_every=every, csv_path=path)
    ds = [abs(r["entropy_change_normalized"]) for r in recs]
    mass = [r["mass"] for r in recs]
    print(json.dumps({"scheme": f"NSFR-EC {name}", "m": m, "p": 3, "grid_degree": gd, "t_final": recs[-1]["t"],
                      "records": len(recs), "max_abs_entropy_change_normalized": max(ds),
                      "max_abs_ke_volume": max(abs(r["ke_change_volume"]) for r in recs),
                      "mass_drift_rel": max(abs(x - mass[0]) for x in mass) / abs(mass[0]),
                      "csv": os.path.basename(path)}), flush=True)
    g.close()
