"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total
device time and share.  Usage: python scripts/launch_summary.py launches.csv [steps]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) > vi:
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'ms total':>9} {'ms/step':>8} {'share':>6}  kernel   (steps={steps})")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:8d} {v[1] / 1e6:9.3f} {v[1] / 1e6 / steps:8.3f} {100 * v[1] / tot:5.1f}%  {k[:90]}")
print(f"{sum(v[0] for v in agg.values()):8d} {tot / 1e6:9.3f} {tot / 1e6 / steps:8.3f}  all")
