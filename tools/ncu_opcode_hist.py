"""Dynamic SASS opcode histogram of one kernel from an .ncu-rep source page:
executed warp-instructions per opcode (DFMA / DMUL / DADD / MUFU / LDS /
UBLKCP ...), as counts and shares (the verdict's "SASS instruction histogram")."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hist, hdr = Counter(), None
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if "Source" in row and ("Instructions Executed" in row):
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if hdr is None:
        continue
    try:
        n = int(row[hdr["Instructions Executed"]])
    except (ValueError, KeyError, IndexError):
        continue
    toks = row[hdr["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    hist[op.split(".")[0]] += n
tot = sum(hist.values())
print(f"total executed warp-instructions {tot}")
fp64 = sum(v for k, v in hist.items() if k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "DSET"))
print(f"FP64 (DFMA/DMUL/DADD/DSETP/DMNMX) {fp64} = {100 * fp64 / max(tot, 1):.1f}%")
for op, n in hist.most_common(top):
    print(f"{op:10s} {n:14d} {100 * n / tot:6.2f}%")
