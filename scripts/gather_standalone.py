"""Standalone Papers-batch gathers (for ncu captures): 933k random rows of the 111M x 512 B table."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer, check, lib  # noqa: E402

n, dim = 111_059_956, 128
t = fd.Topology.generate(n, dim, 16, 7)
nodes = np.random.RandomState(0).randint(0, n, 933_574).astype(np.uint64)
nd, out = DeviceBuffer.from_array(nodes), DeviceBuffer(len(nodes) * 512)
for _ in range(8):
    check(lib().fdg_gather(t.ctx, None, nd.ptr, None, len(nodes), out.ptr, None))
check(lib().fdg_device_sync())
