"""Gather time on a row-sharded table (local shards, one process) vs a single shard."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer, check, lib  # noqa: E402

n, dim = 111_059_956, 128
nodes = np.random.RandomState(0).randint(0, n, 933_000).astype(np.uint64)
nd = DeviceBuffer.from_array(nodes)
for shards, impl in ((1, 1), (1, 3), (1, 4), (2, 3), (2, 4)):
    fd.set_option("gather_impl", impl)
    t = fd.Topology.generate(n, dim, 16, 7, shards=shards)
    out = DeviceBuffer(len(nodes) * 512)
    for _ in range(3):
        check(lib().fdg_gather(t.ctx, None, nd.ptr, None, len(nodes), out.ptr, None))
    check(lib().fdg_device_sync())
    t0 = time.time()
    for _ in range(20):
        check(lib().fdg_gather(t.ctx, None, nd.ptr, None, len(nodes), out.ptr, None))
    check(lib().fdg_device_sync())
    print("shards", shards, "impl", impl, "gather us", (time.time() - t0) / 20 * 1e6, flush=True)
    del t
