"""Launched by tests/test_dist.py under torchrun (2 ranks): data-parallel train stage.
Each rank takes its own batch; after allreduce_grads both ranks hold the mean of the two
batches' gradients and take identical SGD steps."""
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
fd.featdrive.check(fd.featdrive.lib().fdg_set_device(dev))
t = fd.Topology.generate(30_000, 16, 8, 4, device=dev)
fan = [5, 5]
seeds = [np.arange(r, 30_000, 211, dtype=np.uint64)[:100] for r in range(world)]
batches = [fd.sample_khop(t, s, fan, 17 + r) for r, s in enumerate(seeds)]
model = fd.GraphSAGE(t, [16, 16, 8], fan, max_seeds=100, seed=3)
model.train_step(batches[rank], label_seed=1, lr=0.0, allreduce=fdist.allreduce_grads)
got = [model.layer(i, grads=True) for i in range(2)]
# single-process reference: the mean of both batches' gradients
ref = fd.GraphSAGE(t, [16, 16, 8], fan, max_seeds=100, seed=3)
acc = None
for b in batches:
    ref.train_step(b, label_seed=1, lr=0.0)
    g = [ref.layer(i, grads=True) for i in range(2)]
    acc = g if acc is None else [tuple(x + y for x, y in zip(a, c)) for a, c in zip(acc, g)]
for i in range(2):
    for u, v in zip(got[i], acc[i]):
        np.testing.assert_allclose(u, v / world, rtol=1e-5, atol=1e-7)
model.sgd(0.1)
w = np.concatenate([a.ravel() for i in range(2) for a in model.layer(i)])
all_w = [None] * world
dist.all_gather_object(all_w, w.tobytes())
assert all(x == all_w[0] for x in all_w), "ranks diverged after the averaged step"
dist.barrier()
print(f"train-ok rank {rank}", flush=True)
dist.destroy_process_group()
