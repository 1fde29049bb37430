"""Timeline of the pipelined run (fdg_trace): per-kernel mean duration in situ, extract-stream
idle gaps and per-batch sampler chain latency."""
import csv
import os
import ctypes as C
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200 import _lib  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
impl = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n, dim, avg, fan, B, t_ids, dtype, frac = bench.CONFIGS["papers"]
L = fd.featdrive.lib()
L.fdg_trace_enable.argtypes = [C.c_int]
L.fdg_trace_dump.argtypes = [C.c_char_p]
L.fdg_set_gather_impl(impl)
if os.environ.get("BM_OVERLAP"):
    fd.featdrive.check(L.fdg_set_option(b"bm_overlap", int(os.environ["BM_OVERLAP"])))
topo = fd.Topology.generate(n, dim, avg, 7, dtype=dtype)
if os.environ.get("HOST"):  # out-of-core tier: table in pinned host memory
    topo.features_to_host()
order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, bench.hash_combine(0, 0)))
K = int(os.environ.get("K", "200"))
rng = np.array([L.fdg_batch_seed(0, 0, int(g)) for g in range(K)], np.uint64)
nb_epoch = len(order) // B  # wrap at the epoch end (products has 196 batches)
seeds = DeviceBuffer.from_array(np.ascontiguousarray(np.concatenate([order[(b % nb_epoch) * B:(b % nb_epoch + 1) * B] for b in range(K)])))
import os
bm_slots = int(os.environ.get("BM", "0"))
cfg = _lib.PipelineConfig(batch_size=B, n_samplers=S, prefetch_group=16, write_x=1,
                          use_buffer_manager=1 if bm_slots else 0, buffer_slots=bm_slots,
                          flags=int(os.environ.get("FLAGS", "0")))
f = np.ascontiguousarray(fan, np.uint32)
p = C.c_void_p()
fd.featdrive.check(L.fdg_pipeline_create(topo.ctx, f.ctypes.data_as(C.c_void_p), len(f), C.byref(cfg), C.byref(p)))
ms = C.c_float()
if os.environ.get("COLD"):  # warm up on other batches: the traced batches then miss the feature buffer
    rng_w = np.array([L.fdg_batch_seed(0, 1, int(g)) for g in range(K)], np.uint64)
    seeds_w = DeviceBuffer.from_array(np.ascontiguousarray(np.concatenate(
        [order[((b + K) % nb_epoch) * B:((b + K) % nb_epoch + 1) * B] for b in range(K)])))
    fd.featdrive.check(L.fdg_pipeline_run(p, seeds_w.ptr, 0, rng_w.ctypes.data_as(C.c_void_p), K, None, None,
                                          C.byref(ms)))
else:
    fd.featdrive.check(L.fdg_pipeline_run(p, seeds.ptr, 0, rng.ctypes.data_as(C.c_void_p), K, None, None,
                                          C.byref(ms)))
L.fdg_trace_enable(1)
fd.featdrive.check(L.fdg_pipeline_run(p, seeds.ptr, 0, rng.ctypes.data_as(C.c_void_p), K, None, None, C.byref(ms)))
L.fdg_trace_dump(b"gpurun_out/trace.csv")
L.fdg_trace_enable(0)
print(f"S={S} impl={impl}: traced run {ms.value / K * 1e3:.1f} us/batch")
rows = list(csv.DictReader(open("gpurun_out/trace.csv")))
dur = defaultdict(list)
for r in rows:
    dur[r["name"]].append(float(r["end_ms"]) - float(r["start_ms"]))
for k, v in sorted(dur.items(), key=lambda x: -np.mean(x[1]) * len(x[1])):
    print(f"  {k:10s} n={len(v):4d} mean={np.mean(v) * 1e3:8.1f} us  p90={np.percentile(v, 90) * 1e3:8.1f}")
ex = sorted((float(r["start_ms"]), float(r["end_ms"])) for r in rows if r["name"] == "extract")
gaps = [b[0] - a[1] for a, b in zip(ex, ex[1:])]
busy = sum(e - s for s, e in ex)
span = ex[-1][1] - ex[0][0]
print(f"  extract stream busy {busy / span * 100:.1f}% of {span:.2f} ms; mean gap {np.mean(gaps) * 1e3:.1f} us")
# sampler chain latency per batch: 'memset' start -> 'fix_src' end on the same stream, in order
chains = defaultdict(list)
for r in rows:
    chains[r["stream"]].append(r)
lat = []
for st, rs in chains.items():
    cur = None
    for r in rs:
        if r["name"] == "memset":
            cur = float(r["start_ms"])
        elif r["name"] == f"intern{len(fan)}" and cur is not None:
            lat.append(float(r["end_ms"]) - cur)
            cur = None
print(f"  sampler chain latency mean {np.mean(lat) * 1e3:.1f} us (n={len(lat)})")
