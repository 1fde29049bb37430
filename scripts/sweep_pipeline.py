"""Sweep pipeline variants (gather impl, samplers, flags) on a config; prints us/batch."""
import ctypes as C
import itertools
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200 import _lib  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "papers"
n, dim, avg, fan, B, t_ids, dtype, frac = bench.CONFIGS[cfgname]
L = fd.featdrive.lib()
topo = fd.Topology.generate(n, dim, avg, 7, dtype=dtype)
order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, bench.hash_combine(0, 0)))
K = 300
rng = np.array([L.fdg_batch_seed(0, 0, int(g)) for g in range(K)], np.uint64)
seeds = DeviceBuffer.from_array(np.ascontiguousarray(order[:K * B]))
f = np.ascontiguousarray(fan, np.uint32)
impls = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1"])]
Ss = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["2", "3"])]
flagsets = [int(x) for x in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["0", "4", "8", "12"])]
for impl, S, flags in itertools.product(impls, Ss, flagsets):
    L.fdg_set_gather_impl(impl)
    cfg = _lib.PipelineConfig(batch_size=B, n_samplers=S, prefetch_group=16, write_x=1, flags=flags)
    p = C.c_void_p()
    fd.featdrive.check(L.fdg_pipeline_create(topo.ctx, f.ctypes.data_as(C.c_void_p), len(f), C.byref(cfg), C.byref(p)))
    ms = C.c_float()
    res = []
    for rep in range(3):
        fd.featdrive.check(L.fdg_pipeline_run(p, seeds.ptr, 0, rng.ctypes.data_as(C.c_void_p), K, None, None, C.byref(ms)))
        res.append(ms.value / K * 1e3)
    L.fdg_pipeline_destroy(p)
    print(f"impl={'TMA' if impl == 0 else 'LDG'} S={S} flags={flags:2d}: {min(res[1:]):7.1f} us/batch "
          f"({K / min(res[1:]) * 1e3:6.0f} batches/s)", flush=True)
