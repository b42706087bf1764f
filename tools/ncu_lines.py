"""Aggregate an ncu source page (cuda,sass) per source line: stall samples and executed warp-instructions."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""])
fname, line, src = "?", None, ""
hdr = None
tot_s = tot_i = 0
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name",):
        continue
    if row[0] == "Line No":
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if hdr is None:
        continue
    if row[0]:
        line, src = row[0], row[1]
        continue
    try:
        s = int(row[hdr["Warp Stall Sampling (All Samples)"]])
        n = int(row[hdr["Instructions Executed"]])
    except (ValueError, KeyError):
        continue
    k = (fname, line)
    agg[k][0] += s
    agg[k][1] += n
    agg[k][2] = src
    tot_s += s
    tot_i += n
print(f"total samples {tot_s}  warp-instr {tot_i}")
for k, (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*n/tot_i:5.1f}% ins  {k[0]}:{k[1]:5s} {src.strip()[:90]}")
