"""Generate tests/golden/golden.npz from the REFERENCE ITSELF.

Runs the unmodified featdrive headers compiled into oracle/_ref/libfdref.so
(`make -C oracle ref`, needs /root/reference) -- generator, sample_khop,
partition_epoch, BufferManager, the real Extractor and the sync-reference
pipeline -- and records their outputs as small fixtures. The GPU tests and the
C restatement are checked against these vectors; this script only runs in the
build container (the reference does not exist on the GPU box).

    python tests/golden/make_golden.py
"""
import hashlib
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "golden.npz")

# generator parameter sets: (num_nodes, dim, avg_degree, seed)
GEN_SETS = [(2000, 16, 12, 7), (1, 3, 5, 7), (2, 1, 4, 3), (500, 7, 30, 11), (3000, 4, 1, 5), (4096, 100, 28, 7)]
SAMPLE_DS = (5000, 16, 12, 7)      # sampling / buffer dataset
SPARSE_DS = (3000, 4, 1, 5)        # avg_degree 1 -> many zero / low degree nodes


def sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 22), b""):
            h.update(chunk)
    return h.hexdigest()


def main():
    R = oracle.Ref()
    g = {}
    rs = np.random.RandomState(1234)

    # --- common.hpp hashing + batch_seed --------------------------------------
    xs = rs.randint(0, 2**63, size=64, dtype=np.int64).astype(np.uint64)
    g["sm_in"] = xs
    g["sm_out"] = np.array([R.splitmix64(int(x)) for x in xs], np.uint64)
    g["hc_out"] = np.array([R.hash_combine(int(a), int(b)) for a, b in zip(xs[:32], xs[32:])], np.uint64)
    g["bs_in"] = np.array([[0, 0, 0], [0, 0, 1], [0, 1, 7], [42, 3, 999], [7, 0, 123456]], np.uint64)
    g["bs_out"] = np.array([R.batch_seed(*map(int, r)) for r in g["bs_in"]], np.uint64)
    blob = rs.randint(0, 256, size=4096, dtype=np.int64).astype(np.uint8)
    lens = np.array([0, 1, 3, 7, 8, 9, 15, 16, 17, 63, 64, 100, 400, 512, 1024, 1536], np.uint64)
    g["hash_blob"] = blob
    g["hash_lens"] = lens
    g["hash_out"] = np.array([R.hash_bytes64(blob[: int(n)]) for n in lens], np.uint64)

    # --- MT19937-64 stream and libstdc++ uniform_int_distribution ------------
    seeds = np.array([R.batch_seed(0, 0, 0), R.batch_seed(0, 0, 1), 0, 2**64 - 1], np.uint64)
    g["mt_seeds"] = seeds
    g["mt_words"] = np.stack([R.mt_stream(int(s), 2000) for s in seeds])
    js = rs.randint(1, 200, size=3000).astype(np.uint64)
    js[::97] = np.uint64(2**64 - 2)
    g["uni_js"] = js
    g["uni_out"] = R.uniform_seq(int(seeds[0]), js)

    # --- generator: file digests + a few raw arrays -----------------------------
    tmp = tempfile.mkdtemp(prefix="fd_golden_")
    digests = []
    for k, (n, dim, avg, seed) in enumerate(GEN_SETS):
        d = os.path.join(tmp, f"gen{k}")
        ne = R.generate_dataset(d, n, dim, avg, seed)
        digests.append([sha(os.path.join(d, f)) for f in ("features.bin", "indptr.bin", "indices.bin")])
        g[f"gen{k}_params"] = np.array([n, dim, avg, seed, ne], np.uint64)
    g["gen_digests"] = np.array(digests)
    d0 = os.path.join(tmp, "gen0")
    g["gen0_indptr"] = np.fromfile(os.path.join(d0, "indptr.bin"), np.uint64)
    g["gen0_indices"] = np.fromfile(os.path.join(d0, "indices.bin"), np.uint64)
    g["gen0_features"] = np.fromfile(os.path.join(d0, "features.bin"), np.uint8)
    g["gen0_rows"] = np.stack([R.synthetic_row(7, v, 16) for v in (0, 1, 1999)])

    # --- sampling -----------------------------------------------------------------
    n, dim, avg, seed = SAMPLE_DS
    ds = os.path.join(tmp, "sample")
    R.generate_dataset(ds, n, dim, avg, seed)
    topo = oracle.RefTopology(R, ds)
    train = np.arange(1000, dtype=np.uint64)
    order = R.partition_epoch(train, 20, R.hash_combine(0, 0))
    g["part_order"] = order
    g["part_small"] = R.partition_epoch(np.arange(100, dtype=np.uint64), 7, 99)
    cases = []
    # (name, seeds, fanouts, rng_seed)
    for b in range(4):
        cases.append((order[b * 20:(b + 1) * 20], [5, 5, 5], R.batch_seed(0, 0, b)))
    cases.append((order[:20], [10, 10, 10], R.batch_seed(0, 0, 0)))
    cases.append((order[:50], [3], R.batch_seed(0, 0, 9)))
    cases.append((order[:8], [25, 2], R.batch_seed(1, 2, 3)))
    cases.append((np.array([5, 5, 17, 5, 17, 4999], np.uint64), [4, 4], R.batch_seed(0, 5, 5)))  # dup seeds
    cases.append((np.array([], np.uint64), [3, 3], 1))
    sparse = os.path.join(tmp, "sparse")
    R.generate_dataset(sparse, *SPARSE_DS[:3], SPARSE_DS[3])
    stopo = oracle.RefTopology(R, sparse)
    sp_indptr = np.fromfile(os.path.join(sparse, "indptr.bin"), np.uint64)
    deg = np.diff(sp_indptr)
    zero = np.nonzero(deg == 0)[0][:5].astype(np.uint64)
    low = np.nonzero((deg > 0) & (deg <= 2))[0][:5].astype(np.uint64)
    g["sparse_seeds"] = np.concatenate([zero, low])
    sparse_out = stopo.sample_khop(g["sparse_seeds"], [2, 2, 2], 77)
    g["sparse_nodes"] = sparse_out["nodes"]
    g["sparse_edges"] = sparse_out["edges"]
    g["zero_seed_nodes"] = stopo.sample_khop(zero[:1], [3, 3], 5)["nodes"]

    all_nodes, all_edges, meta = [], [], []
    seed_cat, seed_off = [], [0]
    fan_cat, fan_off = [], [0]
    for s, f, r in cases:
        out = topo.sample_khop(s, f, r)
        meta.append([len(out["nodes"]), len(out["edges"]), r])
        all_nodes.append(out["nodes"])
        all_edges.append(out["edges"])
        seed_cat.append(np.asarray(s, np.uint64))
        seed_off.append(seed_off[-1] + len(s))
        fan_cat.append(np.asarray(f, np.uint32))
        fan_off.append(fan_off[-1] + len(f))
    g["smp_meta"] = np.array(meta, np.uint64)
    g["smp_nodes"] = np.concatenate(all_nodes)
    g["smp_edges"] = np.concatenate(all_edges)
    g["smp_seeds"] = np.concatenate(seed_cat)
    g["smp_seed_off"] = np.array(seed_off, np.uint64)
    g["smp_fan"] = np.concatenate(fan_cat)
    g["smp_fan_off"] = np.array(fan_off, np.uint64)
    try:
        topo.sample_khop(np.array([3, 5000, 7, 6000], np.uint64), [2], 1)
        g["oor_code"] = np.array([0])
    except oracle.OracleError as e:
        g["oor_code"] = np.array([e.code])

    # --- buffer manager: sequential schedule (acquire b, release b-1) ---------------
    S = 900
    bm = oracle.RefBufferManager(R, n, S, 0, 1)
    batches = [topo.sample_khop(order[b * 20:(b + 1) * 20], [3, 3], R.batch_seed(0, 0, b))["nodes"] for b in range(12)]
    aliases, stats = [], []
    for b, nodes in enumerate(batches):
        aliases.append(bm.extract(nodes))
        if b >= 1:
            bm.release(batches[b - 1])
        stats.append(bm.stats())
    bm.validate()
    entries = np.array([bm.entry(v) for v in range(0, n, 7)], np.int64)
    g["bm_S"] = np.array([S])
    g["bm_nodes"] = np.concatenate(batches)
    g["bm_off"] = np.cumsum([0] + [len(x) for x in batches]).astype(np.uint64)
    g["bm_alias"] = np.concatenate(aliases)
    g["bm_stats"] = np.array(stats, np.uint64)
    g["bm_entries"] = entries

    # --- real Extractor + trainer_step checksum, and the sync-reference pipeline ------
    ex = oracle.RefExtractor(R, ds, 2 * max(len(x) for x in batches) + 50)
    ex_alias, ex_cs = [], []
    for b in range(4):
        a, rows, cs = ex.extract(batches[b], dim * 4)
        ex_alias.append(a)
        ex_cs.append(cs)
        if b >= 1:
            ex.release(batches[b - 1])
    g["ex_alias"] = np.concatenate(ex_alias)
    g["ex_checksum"] = np.array(ex_cs, np.uint64)
    recs, _ = R.run_epoch(ds, np.arange(200, dtype=np.uint64), 0, 0, 50, [4, 4], sync=True)
    g["sync_records"] = recs
    recs2, _ = R.run_epoch(ds, np.arange(200, dtype=np.uint64), 0, 0, 50, [4, 4], sync=False)
    g["async_records"] = recs2
    # PipelineSession epochs with a short last chunk (1050 ids, batch 100) and a
    # nonzero seed, for the featdrive-gpu CLI / C++ session parity test
    for e in (0, 1):
        r, _ = R.run_epoch(ds, np.arange(1050, dtype=np.uint64), e, 3, 100, [5, 5], sync=True)
        g[f"session_e{e}"] = r

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
