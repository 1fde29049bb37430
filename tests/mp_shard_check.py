"""Launched by tests/test_dist.py under torchrun (2 ranks): IPC row-sharded gather check."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch.distributed as dist  # noqa: E402

import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200 import dist as fdist  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
dev = fdist.local_device(int(os.environ.get("LOCAL_RANK", "0")))
n, dim = 50_003, 64
dtype = os.environ.get("MP_SHARD_DTYPE", "f32")  # f16: the MAG240M-style table
topo = fd.Topology.generate(n, dim, 8, 7, device=dev, features=False)
sh = fdist.ShardedFeatures(topo, rank, world, 7, n, dim, dtype=dtype)
ref = fd.Topology.generate(n, dim, 8, 7, dtype=dtype, device=dev)  # the full table, single process
nodes = np.random.RandomState(rank).randint(0, n, size=20_000).astype(np.uint64)
x, cs = fd.gather(topo, nodes, checksum=True)
want, want_cs = fd.gather(ref, nodes, checksum=True)
assert topo.info().n_shards == world
assert np.array_equal(x, want), "sharded gather differs"
assert cs == want_cs, "sharded checksum differs"
# the full pipeline over a sharded table
pipe = fd.Pipeline(topo, [5, 5], 100, checksum=True)
rng = np.arange(6, dtype=np.uint64) + 3
seeds = np.random.RandomState(9).randint(0, n, size=600).astype(np.uint64)
recs = pipe.run_batches(seeds, rng)
pipe.close()
for b in range(6):
    batch = fd.sample_khop(topo, seeds[b * 100:(b + 1) * 100], [5, 5], int(rng[b]))
    assert int(recs["checksum"][b]) == fd.gather(ref, batch.nodes, checksum=True)[1]
dist.barrier()
sh.close()
print(f"shard-ok rank {rank}", flush=True)
dist.destroy_process_group()
