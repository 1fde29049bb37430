import sys, numpy as np
sys.path.insert(0, '.')
import oracle, paper_2406_13984_b200 as fd
P = oracle.Port()
t = fd.Topology.generate(200_000, 8, 16, 3, features=False)
ip, ix = t.download_topology()
for ns in [37, 300, 1000]:
    for fan in ([10, 10, 10], [10, 10]):
        seeds = np.random.RandomState(ns).randint(0, 200_000, size=ns).astype(np.uint64)
        b = fd.sample_khop(t, seeds, fan, 12345)
        o = P.sample_khop(ip, ix, seeds, fan, 12345)
        print(ns, fan, 'gpu', b.layer_nodes.tolist(), b.layer_edges.tolist(), 'port', o['layer_nodes'].tolist(), o['layer_edges'].tolist(),
              'nodes_eq_prefix', np.array_equal(b.nodes[:len(b.nodes)], o['nodes'][:len(b.nodes)]))
