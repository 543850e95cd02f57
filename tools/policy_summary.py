"""Per-kernel totals of the LAST policy step in an ncu launch list (starts at the
last select_bits_kernel).  usage: policy_summary.py launches.csv"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID" and r[-3] == "gpu__time_duration.sum"]
last = max(i for i, r in enumerate(rows) if "select_bits_kernel" in r[4])
rows = rows[last:]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    k = r[4].split("(")[0].replace("void ", "")
    if "qlinear_decode" in k or "qlinear_prefill" in k:
        k += f" grid={r[8]}"
    tot[k] += float(r[-1].replace(",", ""))
    cnt[k] += 1
T = sum(tot.values())
out = {"launches": len(rows), "total_us_serialized": round(T / 1e3, 1), "unit": "ns",
       "kernels": {k: {"launches": cnt[k], "total_us": round(v / 1e3, 1), "share": round(v / T, 4)}
                   for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}}
print(json.dumps(out, indent=1))
