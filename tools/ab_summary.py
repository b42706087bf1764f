"""Mean per (variant, p, m) of tools/ab.sh output (jsonl): ms/step, K2 ms, K3 ms."""
import collections
import json
import sys

agg = collections.defaultdict(list)
order = []
for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        v = r["lib"].split("libnsfr_")[-1].replace(".so", "")
        if v not in order:
            order.append(v)
        agg[(r["p"], r["m"], v)].append((r["ms_per_step"], r["k2_ms"], r["k3_ms"]))
print("| variant | p | m | ms/step | K2 ms | K3 ms |\n|---|---|---|---|---|---|")
for v in order:
    for (p, m, vv), rows in sorted(agg.items(), key=lambda kv: (-kv[0][1] * (kv[0][0] == 4), kv[0][0])):
        if vv == v:
            n = len(rows)
            print(f"| {v} | {p} | {m} | " + " | ".join(f"{sum(x[i] for x in rows) / n:.3f}" if i else f"{sum(x[i] for x in rows) / n:.2f}" for i in range(3)) + " |")
