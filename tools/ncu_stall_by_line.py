"""Per CUDA source line: samples of one stall reason (e.g. long_sb, barrier,
wait, short_sb) from an .ncu-rep source page (cuda,sass), top N lines.

    python tools/ncu_stall_by_line.py REP REASON [N]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, reason = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0.0, ""])
fname, hdr, tot = "?", None, 0.0
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] in ("File Name", "File Path"):
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if hdr is None or not row[0]:
        continue
    try:
        v = float(row[hdr["stall_" + reason]] or 0)
    except (ValueError, IndexError):
        continue
    key = f"{fname}:{row[0]}"
    agg[key][0] += v
    agg[key][1] = row[1].strip()[:80]
    tot += v
print(f"stall_{reason}: {tot:.0f} samples")
for k, (v, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v / max(tot, 1):5.1f}%  {k:28s} {src}")
