"""Out-of-core tier: gather GB/s of random 512-B rows from a pinned, mapped host table by
each gather engine (zero-copy LDG chunk-striped, row-group LDG, TMA bulk copies), against
the measured pinned H2D copy peak."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer  # noqa: E402

L = fd.featdrive.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
dim = 128
if len(sys.argv) > 2:
    fd.set_option("host_tier_thp", int(sys.argv[2]))
print(f"table: {n} rows x {dim * 4} B = {n * dim * 4 / 1e9:.1f} GB in host memory, thp={fd.featdrive.get_option('host_tier_thp')}")
t = fd.Topology.generate(n, dim, 4, 7).features_to_host()
rb = t.row_bytes
nodes = np.random.RandomState(0).randint(0, n, size=900_000).astype(np.uint64)
nd = DeviceBuffer.from_array(nodes)
out = DeviceBuffer(len(nodes) * rb)
h, d = C.c_void_p(), C.c_void_p()
nbytes = 1 << 30
fd.featdrive.check(L.fdg_host_alloc(C.byref(h), nbytes))
fd.featdrive.check(L.fdg_malloc(C.byref(d), nbytes))
C.memset(h.value, 1, nbytes)
best = 0
for _ in range(5):
    t0 = time.perf_counter()
    fd.featdrive.check(L.fdg_memcpy_h2d(d.value, h.value, nbytes, None))
    fd.featdrive.check(L.fdg_device_sync())
    best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
print(f"pinned H2D copy peak: {best:.1f} GB/s")
ev = [C.c_void_p(), C.c_void_p()]
for e in ev:
    fd.featdrive.check(L.fdg_event_create(C.byref(e)))
nd_sorted = DeviceBuffer.from_array(np.sort(nodes))
for name, impl in (("LDG chunk-striped", 1), ("row-group dyn", 4), ("TMA bulk", 0), ("LDG, sorted ids", 1)):
    src = nd_sorted if "sorted" in name else nd
    fd.set_option("gather_impl", impl)
    times = []
    for rep in range(4):
        fd.featdrive.check(L.fdg_event_record(ev[0], None))
        fd.featdrive.check(L.fdg_gather(t.ctx, None, src.ptr, None, len(nodes), out.ptr, None))
        fd.featdrive.check(L.fdg_event_record(ev[1], None))
        fd.featdrive.check(L.fdg_device_sync())
        ms = C.c_float()
        fd.featdrive.check(L.fdg_event_elapsed_ms(ev[0], ev[1], C.byref(ms)))
        times.append(ms.value)
    ms = min(times[1:])
    gbs = len(nodes) * rb / (ms / 1e3) / 1e9
    print(f"{name:20s} {ms:8.3f} ms  {gbs:6.1f} GB/s of rows read over PCIe ({gbs / best:.2f} of the copy peak)")
fd.set_option("gather_impl", 4)

# the buffer manager's extraction from the same host table (all misses: table -> slot and -> X)
nodes_u = np.unique(nodes)[:800_000]
rs = np.random.RandomState(2)
rs.shuffle(nodes_u)
ndu = DeviceBuffer.from_array(nodes_u)
alias = DeviceBuffer(len(nodes_u) * 8)
xo = DeviceBuffer(len(nodes_u) * rb)
for with_x in (True, False):
    times = []
    for rep in range(3):
        bm = fd.BufferManager(t, 2_000_000, max_batch_nodes=len(nodes_u))
        fd.featdrive.check(L.fdg_device_sync())
        fd.featdrive.check(L.fdg_event_record(ev[0], None))
        fd.featdrive.check(L.fdg_bm_extract(bm.ptr, None, ndu.ptr, None, len(nodes_u), alias.ptr,
                                            xo.ptr if with_x else None, None))
        fd.featdrive.check(L.fdg_event_record(ev[1], None))
        fd.featdrive.check(L.fdg_device_sync())
        ms = C.c_float()
        fd.featdrive.check(L.fdg_event_elapsed_ms(ev[0], ev[1], C.byref(ms)))
        times.append(ms.value)
        del bm
    ms = min(times)
    gbs = len(nodes_u) * rb / (ms / 1e3) / 1e9
    print(f"bm_extract (all misses{', + X' if with_x else ''}) {ms:8.3f} ms  {gbs:6.1f} GB/s of miss rows ({gbs / best:.2f} of the copy peak)")
