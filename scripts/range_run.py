"""One pipelined run under FDG_PROFILE_RANGE for ncu range replay: python scripts/range_run.py <mode> [G] [S]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_13984_b200 as fd  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "full"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 1
S = int(sys.argv[3]) if len(sys.argv) > 3 else 2
fd.set_option("gather_impl", 1)
n, dim, avg, fan, B, t_ids, dtype, frac = bench.CONFIGS["papers"]
L = fd.featdrive.lib()
topo = fd.Topology.generate(n, dim, avg, 7)
order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, bench.hash_combine(0, 0)))
K = 60
rng = np.array([L.fdg_batch_seed(0, 0, int(g)) for g in range(K)], np.uint64)
seeds = fd.DeviceBuffer.from_array(np.ascontiguousarray(order[:K * B]))
flags = {"full": 0, "sample": 1, "extract": 2}[mode]
p = fd.Pipeline(topo, fan, B, samplers=S, group_batches=G, flags=flags)
ms = p.run(seeds.ptr, False, rng)  # warm (the library reads the env var once, at first run)
print(f"{mode} G={G} S={S}: {ms / K * 1e3:.1f} us/batch", flush=True)
