"""Soak check: a long pipelined run (plain and buffer-manager) on the Papers shape; every
batch record must be status 0, and the checksums of 40 random batches must equal the
synchronous host API (sample_khop + gather) on the same seeds."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_13984_b200 as fd  # noqa: E402

n, dim, avg, fan, B, t_ids, dtype, frac = bench.CONFIGS["papers"]
topo = fd.Topology.generate(n, dim, avg, 7, dtype=dtype)
order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, bench.hash_combine(0, 0)))
K = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
nb = t_ids // B
ids = np.arange(K) % nb
rng = np.array([fd.batch_seed(0, 0, int(g)) for g in ids], np.uint64)
seeds = np.concatenate([order[g * B:(g + 1) * B] for g in ids])
pick = np.random.RandomState(0).choice(K, 40, replace=False)
want = {}
for k in pick:
    batch = fd.sample_khop(topo, seeds[k * B:(k + 1) * B], fan, int(rng[k]))
    want[k] = fd.gather(topo, batch.nodes, checksum=True)[1]
for slots in (None, int(n * 0.1)):
    pipe = fd.Pipeline(topo, fan, B, buffer_slots=slots, checksum=True, samplers=8)
    recs = pipe.run_batches(seeds, rng)
    pipe.close()
    bad = int(np.sum(recs["status"] != 0))
    miss = [int(k) for k in pick if int(recs["checksum"][k]) != want[k]]
    print(f"buffer={slots} batches={K} bad_status={bad} checksum_mismatch={miss}", flush=True)
    assert bad == 0 and not miss
print("soak-ok")
