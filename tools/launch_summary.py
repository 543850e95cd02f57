"""Per-kernel share of the timed step from an ncu launch list (gpu__time_duration.sum),
keeping only complete steps: select_bits_kernel (fused select+route) followed by
(act-quant, qlinear) x 4 (the 120 untimed select_bits history steps have no
qlinear after them).  usage: launch_summary.py launches.csv > out.json"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
rows = [r for r in rows if r[-3] == "gpu__time_duration.sum"]
# keep complete steps only: select_bits (+route), then (act-quant, qlinear) x 4
names = [r[4] for r in rows]
keep = []
i = 0
while i + 9 <= len(rows):
    if "select_bits_kernel" in names[i] and "actquant_dec_kernel" in names[i + 1]:
        keep.extend(rows[i:i + 9])
        i += 9
    else:
        i += 1
rows = keep
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    name = r[4].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[-1])
tot = sum(v[1] for v in agg.values())
out = {"source": sys.argv[1], "unit": rows[0][-2], "launches": len(rows), "steps": len(rows) // 10, "note":
       "ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised launches; shares, not absolute times",
       "kernels": {k: {"launches": v[0], "total": v[1], "mean": v[1] / v[0], "share": round(v[1] / tot, 4)}
                   for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}}
print(json.dumps(out, indent=1))
