"""Shared-memory wavefronts per SASS instruction of one kernel from an .ncu-rep
(ideal vs actual: bank conflicts), by region and per instruction.
    python tools/ncu_smem_wavefronts.py REP [name:lo-hi ...] [--dump lo hi]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr, base, rows = None, None, []
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "Address":
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if hdr is None or not row[0].startswith("0x"):
        continue
    a = int(row[0], 16)
    base = a if base is None else base
    g = lambda k: float(row[hdr[k]] or 0)
    if g("L1 Wavefronts Shared") > 0:
        rows.append((a - base, row[hdr["Source"]].strip()[:44], g("L1 Wavefronts Shared"),
                     g("L1 Wavefronts Shared Ideal"), g("Instructions Executed")))
tw, ti = sum(r[2] for r in rows), sum(r[3] for r in rows)
print(f"total wavefronts {tw:.4g}, ideal {ti:.4g}, ratio {tw / ti:.3f}")
args = sys.argv[2:]
if "--dump" in args:
    j = args.index("--dump")
    lo, hi = int(args[j + 1], 16), int(args[j + 2], 16)
    for r in rows:
        if lo <= r[0] <= hi:
            print(f"{r[0]:05x} {r[1]:44s} per instr: {r[2] / r[4]:5.2f} (ideal {r[3] / r[4]:4.2f})  share {100 * r[2] / tw:4.1f}%")
    args = args[:j]
for spec in args:
    n, rg = spec.split(":")
    lo, hi = (int(x, 16) for x in rg.split("-"))
    s = [r for r in rows if lo <= r[0] <= hi]
    w, i = sum(r[2] for r in s), sum(r[3] for r in s)
    print(f"{n:10s} wavefronts {100 * w / tw:5.1f}% of total, ratio to ideal {w / max(i, 1):.3f}")
