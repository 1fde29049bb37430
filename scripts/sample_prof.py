"""A few Papers-shape sample_khop calls (for ncu on the sampler kernels)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_13984_b200 as fd  # noqa: E402

n, dim, avg, fan, B, t_ids, dtype, frac = bench.CONFIGS["papers"]
topo = fd.Topology.generate(n, dim, avg, 7, features=False)
order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, bench.hash_combine(0, 0)))
s = fd.Sampler(topo, fan, B)
for b in range(3):
    r = s.sample(order[b * B:(b + 1) * B], fd.batch_seed(0, 0, b))
print("nodes", len(r.nodes))
