"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_list.py RAW.csv OUT.csv "header comment"

share_of_step = fraction of the RK4 step's kernel time (k_residual, k_update,
k_step_*); setup and prologue kernels are listed with the share blank.
"""
import csv
import sys
from collections import OrderedDict

STEP = ("k_residual", "k_update", "k_step_")


def main():
    raw, out, note = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.reader(l for l in open(raw) if not l.startswith("=="))]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ik].split("(")[0]
        v = float(r[iv].replace(",", ""))
        v = v / 1e6 if r[iu] == "ns" else (v / 1e3 if r[iu] == "us" else v)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + v)
    step = sum(t for k, (n, t) in agg.items() if any(s in k for s in STEP))
    with open(out, "w") as f:
        f.write(f"# {note}\n# gpu__time_duration.sum, --clock-control none; cold-cache + serialised: compare SHARES\n")
        f.write("# share = fraction of the RK4 step kernel time (k_residual + k_update + k_step_*); "
                "setup/prologue kernels have no share\n")
        f.write("kernel,launches,total_ms,avg_ms,share_of_step\n")
        for k, (n, t) in agg.items():
            share = f"{t / step:.4f}" if any(s in k for s in STEP) else ""
            f.write(f"{k},{n},{t:.3f},{t / n:.3f},{share}\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
