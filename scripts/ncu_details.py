"""Condense `ncu -i REP --page details --csv` into one row per launch with the metrics we cite."""
import csv
import io
import subprocess
import sys

KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Grid Size", "Block Size", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
launches = {}
for r in rows[1:]:
    d = dict(zip(h, r))
    key = (int(d["ID"]), d["Kernel Name"])
    if d["Metric Name"] in KEEP:
        launches.setdefault(key, {})[f'{d["Metric Name"]} ({d["Metric Unit"]})'] = d["Metric Value"]
cols = sorted({c for v in launches.values() for c in v})
w = csv.writer(sys.stdout)
w.writerow(["id", "kernel"] + cols)
for (i, k), v in sorted(launches.items()):
    w.writerow([i, k[:60]] + [v.get(c, "") for c in cols])
