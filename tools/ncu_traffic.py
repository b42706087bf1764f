"""Per-launch DRAM traffic and key counters of one kernel from an .ncu-rep
(--page raw), written as the JSON bench.py reads for roofline.traffic.

    python tools/ncu_traffic.py REP ELEMENTS OUT.json [kernel-substring]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, elements, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    want = sys.argv[4] if len(sys.argv) > 4 else ""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        if want not in name:
            continue
        vals = {}
        for k in KEYS:
            i = hdr.index(k)
            v = float(row[i].replace(",", ""))
            vals[k] = v * SCALE.get(units[i], 1) if units[i] in SCALE else v
        dram = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
        res = {"kernel": name.split("(")[0], "source": os.path.basename(rep), "elements": elements,
               "dram_bytes_per_element": dram / elements, "metrics": vals,
               "note": "ncu --set full, one launch; bench scales by elements per launch"}
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps(res))
        return
    sys.exit("kernel not found")


if __name__ == "__main__":
    main()
