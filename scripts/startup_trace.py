"""Start of a pipelined run (the driver's bench times 20 batches, so the first batch's
latency matters): per-launch timeline of a K-batch run from its t0 (fdg_trace), first
extraction start / end, and the host enqueue time."""
import csv
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200 import _lib  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer  # noqa: E402

cfgname = os.environ.get("CFG", "papers")
K = int(os.environ.get("K", "20"))
S = int(os.environ.get("S", "8"))
n, dim, avg, fan, B, t_ids, dtype, frac = bench.CONFIGS[cfgname]
L = fd.featdrive.lib()
L.fdg_trace_enable.argtypes = [C.c_int]
L.fdg_trace_dump.argtypes = [C.c_char_p]
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    fd.featdrive.check(L.fdg_set_option(k.encode(), int(v)))
topo = fd.Topology.generate(n, dim, avg, 7, dtype=dtype)
order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, bench.hash_combine(0, 0)))
rng = np.array([L.fdg_batch_seed(0, 0, int(g)) for g in range(K)], np.uint64)
seeds = DeviceBuffer.from_array(np.ascontiguousarray(order[:K * B]))
pipe = fd.Pipeline(topo, fan, B, samplers=S)
pipe.run(seeds.ptr, False, rng)  # warm-up
for rep in range(3):  # untraced: time to the first extraction and host enqueue
    ext = np.zeros(K, np.float32)
    ms = pipe.run(seeds.ptr, False, rng, extract_ms=ext)
    xs, xe = pipe.extract_times(K)
    print(f"untraced run {rep}: {ms:.3f} ms, {ms / K * 1e3:.1f} us/batch, batch 0 extraction {xs[0]:.3f}-{xe[0]:.3f} ms, "
          f"host enqueue {pipe.host_enqueue_ms():.3f} ms")
L.fdg_trace_enable(1)
ext = np.zeros(K, np.float32)
ms = pipe.run(seeds.ptr, False, rng, extract_ms=ext)
path = "gpurun_out/startup_trace.csv"
L.fdg_trace_dump(path.encode())
L.fdg_trace_enable(0)
xs, xe = pipe.extract_times(K)
print(f"{cfgname} K={K} S={S} {sys.argv[1:]}: {ms:.3f} ms total, {ms / K * 1e3:.1f} us/batch, host enqueue "
      f"{pipe.host_enqueue_ms():.3f} ms")
print("  extraction start/end of batches 0-3 (ms from t0):",
      [(round(float(a), 3), round(float(b), 3)) for a, b in zip(xs[:4], xe[:4])])
print(f"  steady extraction spacing (batches 5..K): {np.mean(np.diff(xs[5:])) * 1e3:.1f} us")
rows = list(csv.DictReader(open(path)))
t0 = min(float(r["start_ms"]) for r in rows)
rows.sort(key=lambda r: float(r["start_ms"]))
print("  first launches (name, stream, start, end) in ms from the first traced launch:")
for r in rows[:70]:
    print(f"    {r['name']:10s} {r['stream'][-6:]:>6s} {float(r['start_ms']) - t0:7.3f} {float(r['end_ms']) - t0:7.3f}")
