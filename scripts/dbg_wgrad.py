"""Debug: tensor-core vs CUDA-core weight gradients of the train stage on a tiny model."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2406_13984_b200 as fd  # noqa: E402

t = fd.Topology.generate(60_000, 32, 12, 5)
s = np.random.RandomState(33).randint(0, 60_000, 300).astype(np.uint64)
batch = fd.sample_khop(t, s, [10, 10, 10], fd.batch_seed(0, 1, 32))
print("layer_nodes", batch.layer_nodes, "edges", len(batch.edges))
res = {}
for eng in (0, 1):
    fd.set_option("sage_gemm", eng)
    m = fd.GraphSAGE(t, [32, 64, 64, 12], [10, 10, 10], max_seeds=300, seed=33)
    loss = m.train_step(batch, label_seed=11, lr=0.0)
    res[eng] = [m.layer(i, grads=True) for i in range(3)]
    print("engine", eng, "loss", loss)
for i in range(3):
    for name, a, b in zip(("wn", "ws", "b"), res[0][i], res[1][i]):
        print(i, name, "cuda-core |g|", float(np.abs(a).max()), "tc |g|", float(np.abs(b).max()),
              "max diff", float(np.abs(a - b).max()))
