"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count, mean, share."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(list)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("fdg::<unnamed>::", "")[:70]
    agg[name].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'n':>5s} {'mean_us':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} {len(v):5d} {sum(v) / len(v):10.1f} {sum(v) / tot * 100:6.1f}%")
