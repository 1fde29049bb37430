"""Row-sharded gather over NVLink in ONE process (so ncu may profile it): the Papers-shaped
table split into G row shards, shard s generated on GPU s; GPU 0's context installs all G
bases (peer access enabled) and gathers a batch whose rows are mostly remote. Prints the
gather GB/s, the remote-row share and the NVLink floor (remote bytes / 770 GB/s, the measured
peer-copy bandwidth per direction, B200_PROFILING.md). Needs >= 2 GPUs.

    python scripts/nvlink_gather.py [G]
    ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum -k regex:k_gather \\
        python scripts/nvlink_gather.py 2        (scripts/nvlink_counters.sh)
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer  # noqa: E402

L = fd.featdrive.lib()
G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if fd.device_count() < G:
    print(f"needs {G} GPUs, {fd.device_count()} visible")
    sys.exit(0)
n, dim, avg = 111_059_956, 128, 16
rps = -(-n // G)
ctxs, bases = [], []
for g in range(G):  # shard g on GPU g (each context also holds nothing else)
    t = fd.Topology(g)
    b = C.c_void_p()
    fd.featdrive.check(L.fdg_ctx_generate_feature_shard(t.ctx, 7, n, dim, 0, g, G, C.byref(b)))
    ctxs.append(t)
    bases.append(b.value)
for g in range(1, G):
    fd.featdrive.check(L.fdg_enable_peer_access(0, g))
fd.featdrive.check(L.fdg_set_device(0))
topo = fd.Topology.generate(n, dim, avg, 7, device=0, features=False)
arr = (C.c_void_p * G)(*bases)
fd.featdrive.check(L.fdg_ctx_set_feature_shards(topo.ctx, C.cast(arr, C.c_void_p), G, rps, n, dim * 4, 0))
order = np.concatenate(fd.partition_epoch(np.arange(1_000_000, dtype=np.uint64), 1000, 0x0))
nodes = fd.sample_khop(topo, order[:1000], [10, 10, 10], fd.batch_seed(0, 0, 0)).nodes
remote = float(np.mean(nodes.astype(np.int64) // rps != 0))
nd = DeviceBuffer.from_array(nodes)
out = DeviceBuffer(len(nodes) * dim * 4)
ev = [C.c_void_p(), C.c_void_p()]
for e in ev:
    fd.featdrive.check(L.fdg_event_create(C.byref(e)))
times = []
for rep in range(6):
    fd.featdrive.check(L.fdg_event_record(ev[0], None))
    fd.featdrive.check(L.fdg_gather(topo.ctx, None, nd.ptr, None, len(nodes), out.ptr, None))
    fd.featdrive.check(L.fdg_event_record(ev[1], None))
    fd.featdrive.check(L.fdg_device_sync())
    ms = C.c_float()
    fd.featdrive.check(L.fdg_event_elapsed_ms(ev[0], ev[1], C.byref(ms)))
    times.append(ms.value)
ms = min(times[1:])
rb = dim * 4
remote_bytes = remote * len(nodes) * rb
print(f"G={G}: {len(nodes)} rows, remote share {remote:.3f}; gather {ms * 1e3:.1f} us = "
      f"{2 * len(nodes) * rb / (ms / 1e3) / 1e9:.0f} GB/s (read+write); remote rows {remote_bytes / (ms / 1e3) / 1e9:.0f} GB/s "
      f"over NVLink; NVLink floor {remote_bytes / 770e9 * 1e6:.1f} us (770 GB/s measured peer copy)")
