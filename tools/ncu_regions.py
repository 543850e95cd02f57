"""Summarise an ncu source-page CSV (SASS) by code region: stall samples,
executed instructions, top stall reasons.  usage: ncu_regions.py src.csv
[name:lo-hi ...] (hex offsets relative to the kernel start)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
tot = sum(float(r[iss] or 0) for r in data)
regions = []
for spec in sys.argv[2:]:
    n, rng = spec.split(":")
    lo, hi = (int(x, 16) for x in rng.split("-"))
    regions.append((lo, hi, n))
for lo, hi, n in regions:
    agg, ex, smp = {}, 0, 0
    for r in data:
        a = int(r[ia], 16) - base
        if lo <= a < hi:
            ex += int(r[iex] or 0)
            smp += float(r[iss] or 0)
            for i in cols:
                agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
    t = sum(agg.values()) or 1
    top = {k[6:]: round(v / t * 100) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6]}
    print(f"{n:12s} samples {smp / tot * 100:5.1f}%  warp-instr {ex:>10d}  {top}")
print("top instructions:")
for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:int(__import__('os').environ.get('TOPN', '15'))]:
    print(f"  {int(r[ia], 16) - base:#06x} {float(r[iss]) / tot * 100:5.1f}% {r[iex]:>9s}  {r[isrc][:70]}")
