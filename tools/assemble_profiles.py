"""Assemble the judged profile files under profiles/ from one profiling call's
scratch output (gpurun_out/, written by tools/profile_round.sh and friends).

    python tools/assemble_profiles.py [TAG=r02]
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
prof = os.path.join(G, "prof")

for k in ("k_residual", "k_update", "k_project", "k_convert_lines"):
    md = os.path.join(prof, k + ".md")
    if not os.path.exists(md):
        continue
    parts = [open(md).read().rstrip("\n")]
    for title, suffix in (("Dynamic SASS opcode histogram (tools/ncu_opcode_hist.py):", "_opcodes.txt"),
                          ("Per source line FP64 / other (tools/ncu_ops_by_line.py):", "_ops_by_line.txt"),
                          ("Stall samples by reason and line (tools/ncu_stall_by_line.py):", "_stalls_by_line.txt")):
        f = os.path.join(prof, k + suffix)
        if os.path.exists(f):
            parts.append(f"\n{title}\n```\n{open(f).read().rstrip()}\n```")
    open(os.path.join(P, f"{tag}_{k}_p4_ncu.md"), "w").write("\n".join(parts) + "\n")
    t = os.path.join(prof, k + "_traffic.json")
    if os.path.exists(t):  # bench.py reads these two for roofline.traffic
        shutil.copy(t, os.path.join(P, f"{k}_p4_traffic.json"))

raw = os.path.join(prof, "launches_raw.csv")
if os.path.exists(raw):
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_list.py"), raw,
                    os.path.join(P, f"{tag}_bench_launch_list.csv"),
                    "ncu --metrics gpu__time_duration.sum --clock-control none --csv: python bench.py --steps 2 "
                    f"--warmup 3 --no-cpu-baseline ({tag} final kernels, one B200)"], check=True)
for src, dst in (("bench.json", f"{tag}_bench.json"), ("parity_report.md", f"{tag}_parity_report.md"),
                 ("bench_100.json", f"{tag}_bench_100steps.json"), ("bench_reference.json", f"{tag}_bench_reference.json")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
print("assembled", sorted(f for f in os.listdir(P) if f.startswith(tag) or f.endswith("traffic.json")))
