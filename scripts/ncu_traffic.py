"""Per-kernel duration + DRAM bytes from an ncu CSV (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = defaultdict(dict)
names = {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    names[r[idi]] = r[ki].split("(")[0].replace("fdg::<unnamed>::", "")[:60]
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0)
    a[3] += m.get("dram__bytes_write.sum", 0)
print(f"{'kernel':60s} {'n':>4s} {'us':>8s} {'rd MB':>9s} {'wr MB':>9s} {'GB/s':>8s}")
for k, (n, t, r, w) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {n:4d} {t / n:8.1f} {r / n / 1e6:9.2f} {w / n / 1e6:9.2f} {(r + w) / (t * 1e-6) / 1e9 / 1 if t else 0:8.0f}")
