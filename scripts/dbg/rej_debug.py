"""Debug: pipeline rejection hooks -- print per-batch status / rejections / counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2406_13984_b200 import _lib
if os.environ.get("FDG_DBG_LIB"):
    _lib.LIB_PATH = os.environ["FDG_DBG_LIB"]
    _lib.load.__defaults__ = (_lib.LIB_PATH,)
import paper_2406_13984_b200 as fd
import oracle

port = oracle.Port()
n, B, fan, nb, target, pos = 300_000, 256, [10, 5, 5], 12, 5, 3
t = fd.Topology.generate(n, 32, 12, 3)
ip, ix = t.download_topology()
order = np.concatenate(fd.partition_epoch(np.arange(nb * B, dtype=np.uint64), B, 4321))
rng = np.array([fd.batch_seed(0, 0, b) for b in range(nb)], np.uint64)
for key, val in (("debug_zero_word", (target << 24) | pos), ("debug_reject_batch", target)):
    fd.set_option(key, val)
    pipe = fd.Pipeline(t, fan, B, checksum=True, samplers=2)
    recs = pipe.run_batches(order, rng)
    pipe.close()
    fd.set_option(key, -1)
    print(key, "status", recs["status"].tolist(), "rej", recs["rejections"].tolist(), "words", recs["words_used"].tolist())
    seeds = order[target * B:(target + 1) * B]
    words = fd.mt_stream(int(rng[target]), 400_000)
    w0 = words.copy()
    words[pos] = 0
    o = port.sample_khop(ip, ix, seeds, fan, int(rng[target]), words=words)
    p0 = port.sample_khop(ip, ix, seeds, fan, int(rng[target]), words=w0)
    print(" port modified words_used", o["words_used"], "nodes", len(o["nodes"]), "plain", p0["words_used"], len(p0["nodes"]),
          "gpu nodes", int(recs["n_nodes"][target]))
s = fd.Sampler(t, fan, max_seeds=B)
seeds = order[target * B:(target + 1) * B]
words = fd.mt_stream(int(rng[target]), s.max_edges + 4096)
words[pos] = 0
nodes, edges, used = s.sample_words(seeds, words)
o = port.sample_khop(ip, ix, seeds, fan, 0, words=words)
print("host api:", used, o["words_used"], np.array_equal(nodes, o["nodes"]))
