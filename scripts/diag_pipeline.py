"""Pipeline diagnostics on the Papers100M shape: full / sample-only / extract-only throughput
for several sampler counts, with host enqueue time (is the CPU or the GPU the bound?)."""
import ctypes as C
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
K = 400
ids = np.arange(K)
rng = np.array([L.fdg_batch_seed(0, 0, int(g)) for g in ids], np.uint64)
seeds = DeviceBuffer.from_array(np.ascontiguousarray(order[:K * B]))
for flags, name in [(0, "full"), (1, "sample-only"), (2, "extract-only")]:
    for S in (1, 2, 3, 4):
        cfg = _lib.PipelineConfig(batch_size=B, n_samplers=S, prefetch_group=16, write_x=1, flags=flags)
        f = np.ascontiguousarray(fan, np.uint32)
        p = C.c_void_p()
        fd.featdrive.check(L.fdg_pipeline_create(topo.ctx, f.ctypes.data_as(C.c_void_p), len(f), C.byref(cfg), C.byref(p)))
        ms = C.c_float()
        for rep in range(2):
            fd.featdrive.check(L.fdg_pipeline_run(p, seeds.ptr, 0, rng.ctypes.data_as(C.c_void_p), K, None, None, C.byref(ms)))
        out = _lib.PipelineConfig()
        L.fdg_pipeline_get_config(p, C.byref(out))
        print(f"{name:13s} S={S}: {ms.value / K * 1e3:7.1f} us/batch  ({K / ms.value * 1e3:7.0f} batches/s)  "
              f"host enqueue {out.host_enqueue_ms / K * 1e3:6.1f} us/batch", flush=True)
        L.fdg_pipeline_destroy(p)
        if flags == 2:
            break
