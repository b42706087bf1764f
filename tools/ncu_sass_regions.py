"""Per-SASS-instruction samples / executed counts of one kernel from an .ncu-rep
(source page, sass view), summed over address regions given as hex offsets
relative to the kernel start:

    python tools/ncu_sass_regions.py REP name:lo-hi [name:lo-hi ...]
    python tools/ncu_sass_regions.py REP --dump lo hi        # per instruction

A region's samples / warp-instructions executed = cycles one warp spends per
instruction there (each sample is one warp-cycle at the sampling period).
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows, hdr, base = [], None, None
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
    rows.append({"off": a - base, "sass": row[hdr["Source"]].strip(), "smp": g("# Samples"),
                 "exe": g("Instructions Executed"),
                 "st": {k[6:]: g(k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}})
tot_s = sum(r["smp"] for r in rows)
tot_e = sum(r["exe"] for r in rows)
print(f"total samples {tot_s:.0f}, warp-instr {tot_e:.4g}, samples/instr-per-1e6 {1e6 * tot_s / tot_e:.2f}")
if sys.argv[2] == "--dump":
    lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    for r in rows:
        if lo <= r["off"] <= hi:
            top = sorted(r["st"].items(), key=lambda kv: -kv[1])[:2]
            print(f"{r['off']:05x} {r['smp']:7.0f} {r['exe']:.3g}  {r['sass'][:60]:60s} {top}")
    sys.exit()
for spec in sys.argv[2:]:
    name, rng = spec.split(":")
    lo, hi = (int(x, 16) for x in rng.split("-"))
    sel = [r for r in rows if lo <= r["off"] <= hi]
    s = sum(r["smp"] for r in sel)
    e = sum(r["exe"] for r in sel)
    f = sum(r["exe"] for r in sel if r["sass"].split()[0].lstrip("@!UP0123456789 ").startswith(("DFMA", "DMUL", "DADD", "DSETP")))
    st = {}
    for r in sel:
        for k, v in r["st"].items():
            st[k] = st.get(k, 0) + v
    top = ", ".join(f"{k} {100 * v / max(s, 1):.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:6])
    print(f"{name:10s} samples {100 * s / tot_s:5.1f}%  instr {100 * e / tot_e:5.1f}%  fp64 {100 * f / max(e, 1):4.0f}%  "
          f"rel cycles/instr {(s / max(e, 1)) / (tot_s / tot_e):.2f}  | {top}")
