"""Print the key sections of an .ncu-rep (details page) compactly."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
keep = sys.argv[2:] or None
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    sec, name, unit, val = r[ix["Section Name"]], r[ix["Metric Name"]], r[ix["Metric Unit"]], r[ix["Metric Value"]]
    if keep and not any(k in sec or k in name for k in keep):
        continue
    if len(val) > 90:
        val = val[:90] + "..."
    print(f"{r[ix['Kernel Name']][:28]:28s} | {sec[:26]:26s} | {name[:48]:48s} | {unit[:12]:12s} | {val}")
