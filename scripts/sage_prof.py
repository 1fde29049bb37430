"""Train-stage kernels on one Papers-shaped batch (1000 seeds, fanout 10,10,10, 128-dim,
hidden 256, 172 classes) for ncu: `python scripts/sage_prof.py [train]`."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402

t = fd.Topology.generate(20_000_000, 128, 16, 7)
s = np.random.RandomState(1).choice(20_000_000, 1000, replace=False).astype(np.uint64)
batch = fd.sample_khop(t, s, [10, 10, 10], fd.batch_seed(0, 0, 0))
print("layer_nodes", batch.layer_nodes, "edges", len(batch.edges), flush=True)
m = fd.GraphSAGE(t, [128, 256, 256, 172], [10, 10, 10], max_seeds=1000, seed=0)
train = len(sys.argv) > 1 and sys.argv[1] == "train"
for _ in range(5):
    print(m.train_step(batch, lr=0.0) if train else m.forward(batch)[0], flush=True)
m.close()
