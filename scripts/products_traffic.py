"""Products-shaped (400-byte rows) standalone gathers for ncu DRAM-traffic captures: the
pipeline's engine (chunk-striped LDG) with the 64-byte L2 fetch hint off / on, and the
row-group engine, and the TMA bulk-copy engine (does cp.async.bulk fill whole 128-byte lines
like LDG misses do?). One launch each on a batch's worth of random rows (875 k)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer, check, lib  # noqa: E402

n, dim = 2_449_029, 100
t = fd.Topology.generate(n, dim, 28, 7)
nodes = np.random.RandomState(0).randint(0, n, 875_461).astype(np.uint64)
nd, out = DeviceBuffer.from_array(nodes), DeviceBuffer(len(nodes) * 400)
import os
combos = ((0, 0, 64), (1, 0, 64), (1, 1, 64), (4, 1, 64)) if os.environ.get('SHORT') else \
    ((1, 0, 128), (1, 1, 128), (4, 0, 128), (4, 1, 128), (1, 0, 32), (4, 0, 32), (1, 0, 64), (0, 0, 64))
for impl, pf, gran in combos:
    fd.set_option("gather_impl", impl)
    fd.set_option("gather_pf64", pf)
    fd.set_option("l2_fetch_granularity", gran)
    print(f"impl {impl} pf64 {pf} granularity {fd.featdrive.get_option('l2_fetch_granularity')}", flush=True)
    for _ in range(2):
        check(lib().fdg_gather(t.ctx, None, nd.ptr, None, len(nodes), out.ptr, None))
    check(lib().fdg_device_sync())
