"""Markdown summary of one kernel's `ncu --set full` capture (key metrics, stall
shares, top source lines) for profiles/.

    python tools/ncu_report.py REP "title" "one-line description" OUT.md
"""
import csv
import io
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main():
    rep, title, desc, out = sys.argv[1:5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    lines = [f"# {title}\n", desc + "\n", "| metric | value |", "|---|---|"]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"| {k} | {v[i]} {u[i]} |")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[i].replace(",", ""))))
            except ValueError:
                pass
    tot = sum(x for _, x in st) or 1.0
    st.sort(key=lambda x: -x[1])
    lines.append("\nStall samples (share of PC samples): " + ", ".join(f"{a} {100 * b / tot:.1f}%" for a, b in st[:8]))
    here = os.path.dirname(os.path.abspath(__file__))
    top = subprocess.run([sys.executable, os.path.join(here, "ncu_lines.py"), rep, "14"], capture_output=True,
                         text=True).stdout
    lines += ["\nTop source lines (stall-sample share / executed-instruction share):\n```", top.rstrip(), "```"]
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
