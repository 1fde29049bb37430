import sys, numpy as np
sys.path.insert(0, '.')
import oracle, paper_2406_13984_b200 as fd
g = dict(np.load('tests/golden/golden.npz'))
P = oracle.Port()
t = fd.Topology.generate(5000, 16, 12, 7)
off = g["bm_off"].astype(np.int64)
batches = [g["bm_nodes"][off[b]:off[b + 1]] for b in range(len(off) - 1)]
print('sizes', [len(x) for x in batches], 'S', g['bm_S'])
bm = fd.BufferManager(t, int(g["bm_S"][0]), max_batch_nodes=max(len(x) for x in batches))
ob = oracle.PortBufferManager(P, 5000, int(g['bm_S'][0]))
for b, nodes in enumerate(batches):
    try:
        a = bm.extract(nodes)
    except Exception as e:
        print('extract fail', b, e); break
    oa, _ = ob.extract(nodes)
    print(b, 'alias eq', np.array_equal(a, oa), bm.stats(), ob.stats().tolist())
    if b >= 1:
        bm.release_batch(batches[b - 1]); ob.release(batches[b - 1])
