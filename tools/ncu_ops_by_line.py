"""Per source line: executed warp-instructions split into FP64 / other (from an .ncu-rep source page)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kern = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kern:
    cmd += ["-k", f"regex:{kern}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""])
fname, line, src, hdr = "?", None, "", None
tot_f = tot_o = 0
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
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
        n = int(row[hdr["Instructions Executed"]])
    except (ValueError, KeyError):
        continue
    sass = row[3].split()
    op = (sass[1] if sass and sass[0].startswith("@") and len(sass) > 1 else (sass[0] if sass else "?"))
    is64 = op.startswith(("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "DSET", "F2F.F64", "F2F.F32.F64"))
    a = agg[(fname, line)]
    a[0 if is64 else 1] += n
    a[2] = src
    if is64:
        tot_f += n
    else:
        tot_o += n
print(f"fp64 warp-instr {tot_f}  other {tot_o}")
for k, (f, o, s) in sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][1]))[:top]:
    print(f"{100*f/tot_f:5.1f}% fp64 {100*o/tot_o:5.1f}% oth  {k[0]}:{k[1]:5s} {s.strip()[:80]}")
