"""CPU: pin the C restatement (oracle/fd_oracle.c) against the reference.

Two anchors: the committed golden vectors (produced by the reference itself,
tests/golden/make_golden.py) and -- where oracle/_ref is built -- the reference
run live on fresh random inputs.
"""
import hashlib
import os
import tempfile

import numpy as np
import pytest

import oracle


def _sample_cases(g):
    meta, so, fo = g["smp_meta"], g["smp_seed_off"], g["smp_fan_off"]
    no = np.concatenate([[0], np.cumsum(meta[:, 0])]).astype(np.int64)
    eo = np.concatenate([[0], np.cumsum(meta[:, 1])]).astype(np.int64)
    for k in range(len(meta)):
        yield (g["smp_seeds"][so[k]:so[k + 1]], g["smp_fan"][fo[k]:fo[k + 1]], int(meta[k, 2]),
               g["smp_nodes"][no[k]:no[k + 1]], g["smp_edges"][eo[k]:eo[k + 1]])


def test_hashing_golden(port, golden):
    g = golden
    assert [port.splitmix64(int(x)) for x in g["sm_in"]] == [int(x) for x in g["sm_out"]]
    assert [port.hash_combine(int(a), int(b)) for a, b in zip(g["sm_in"][:32], g["sm_in"][32:])] == \
        [int(x) for x in g["hc_out"]]
    assert [port.batch_seed(*map(int, r)) for r in g["bs_in"]] == [int(x) for x in g["bs_out"]]
    blob = g["hash_blob"]
    assert [port.hash_bytes64(blob[: int(n)]) for n in g["hash_lens"]] == [int(x) for x in g["hash_out"]]


def test_mt_and_lemire_golden(port, golden):
    for s, words in zip(golden["mt_seeds"], golden["mt_words"]):
        np.testing.assert_array_equal(port.mt_stream(int(s), words.shape[0]), words)
    # uniform_int_distribution(0, j) over the first seed's stream (Lemire, may reject for huge j)
    words = port.mt_stream(int(golden["mt_seeds"][0]), 10000)
    pos = np.zeros(1, np.uint64)
    out = []
    for j in golden["uni_js"]:
        out.append(port.lib.fdo_uniform_0_j(oracle._p(words), len(words), oracle._p(pos), int(j)))
    np.testing.assert_array_equal(np.array(out, np.uint64), golden["uni_out"])


def test_generator_golden(port, golden):
    for k in range(len(golden["gen_digests"])):
        n, dim, avg, seed, ne = map(int, golden[f"gen{k}_params"])
        indptr, indices = port.generate_topology(seed, n, avg)
        assert int(indptr[-1]) == ne
        assert hashlib.sha256(indptr.tobytes()).hexdigest() == golden["gen_digests"][k][1]
        assert hashlib.sha256(indices.tobytes()).hexdigest() == golden["gen_digests"][k][2]
        if n * dim <= 500_000:
            feats = port.generate_features(seed, n, dim)
            header = bytearray(512)
            header[0:8] = b"FEATDRV1"
            header[8:12] = (1).to_bytes(4, "little")
            header[16:24] = n.to_bytes(8, "little")
            header[24:28] = dim.to_bytes(4, "little")
            header[32:36] = (dim * 4).to_bytes(4, "little")
            header[40:48] = (512).to_bytes(8, "little")
            digest = hashlib.sha256(bytes(header) + feats.tobytes()).hexdigest()
            assert digest == golden["gen_digests"][k][0]
    np.testing.assert_array_equal(port.generate_topology(7, 2000, 12)[1], golden["gen0_indices"])


def test_sample_khop_golden(port, golden):
    indptr, indices = port.generate_topology(7, 5000, 12)
    for seeds, fan, rs, nodes, edges in _sample_cases(golden):
        o = port.sample_khop(indptr, indices, seeds, fan, rs)
        np.testing.assert_array_equal(o["nodes"], nodes)
        np.testing.assert_array_equal(o["edges"], edges)
        o32 = port.sample_khop(indptr, indices.astype(np.uint32), seeds, fan, rs)
        np.testing.assert_array_equal(o32["nodes"], nodes)
    sp, sx = port.generate_topology(5, 3000, 1)
    o = port.sample_khop(sp, sx, golden["sparse_seeds"], [2, 2, 2], 77)
    np.testing.assert_array_equal(o["nodes"], golden["sparse_nodes"])
    np.testing.assert_array_equal(o["edges"], golden["sparse_edges"])
    with pytest.raises(oracle.OracleError) as e:
        port.sample_khop(indptr, indices, np.array([3, 5000, 7, 6000], np.uint64), [2], 1)
    assert e.value.code == int(golden["oor_code"][0]) == 1
    with pytest.raises(oracle.OracleError) as e:
        port.sample_khop(indptr, indices, np.array([3], np.uint64), [2, 0], 1)
    assert e.value.code == 2


def test_buffer_manager_golden(port, golden):
    g = golden
    off = g["bm_off"].astype(np.int64)
    bm = oracle.PortBufferManager(port, 5000, int(g["bm_S"][0]))
    batches = [g["bm_nodes"][off[b]:off[b + 1]] for b in range(len(off) - 1)]
    aliases = []
    for b, nodes in enumerate(batches):
        a, _ = bm.extract(nodes)
        aliases.append(a)
        if b >= 1:
            bm.release(batches[b - 1])
        np.testing.assert_array_equal(bm.stats(), g["bm_stats"][b])
    np.testing.assert_array_equal(np.concatenate(aliases), g["bm_alias"])
    ent = np.array([bm.entry(v) for v in range(0, 5000, 7)], np.int64)
    np.testing.assert_array_equal(ent, g["bm_entries"])


def test_checksum_golden(port, golden):
    """trainer_step checksums of the reference's sync pipeline = sum of row hashes."""
    indptr, indices = port.generate_topology(7, 5000, 12)
    feats = port.generate_features(7, 5000, 16)
    order = np.array(oracle.Ref().partition_epoch(np.arange(200, dtype=np.uint64), 50, port.hash_combine(0, 0))) \
        if oracle.ref_available() else None
    for rec in golden["sync_records"]:
        b = int(rec[0])
        if order is None:
            pytest.skip("partition needs libstdc++ shuffle (reference or product host library)")
        o = port.sample_khop(indptr, indices, order[b * 50:(b + 1) * 50], [4, 4], port.batch_seed(0, 0, b))
        assert len(o["nodes"]) == int(rec[2])
        _, cs = port.gather(feats, o["nodes"])
        assert cs == int(rec[3])
    np.testing.assert_array_equal(golden["sync_records"], golden["async_records"])


# ---------------------------------------------------------------- live vs ref --
def test_port_vs_ref_live_sampling(port, ref):
    rs = np.random.RandomState(7)
    d = tempfile.mkdtemp(prefix="fd_live_")
    ref.generate_dataset(d, 20000, 8, 16, 3)
    topo = oracle.RefTopology(ref, d)
    indptr = np.fromfile(os.path.join(d, "indptr.bin"), np.uint64)
    indices = np.fromfile(os.path.join(d, "indices.bin"), np.uint64)
    for t in range(12):
        seeds = rs.randint(0, 20000, size=rs.randint(1, 200)).astype(np.uint64)
        fan = list(rs.randint(1, 30, size=rs.randint(1, 4)))
        r = int(rs.randint(0, 2**63))
        a = topo.sample_khop(seeds, fan, r)
        b = port.sample_khop(indptr, indices, seeds, fan, r)
        np.testing.assert_array_equal(a["nodes"], b["nodes"])
        np.testing.assert_array_equal(a["edges"], b["edges"])


def test_port_vs_ref_live_buffer(port, ref):
    rs = np.random.RandomState(11)
    n, S = 3000, 700
    a = oracle.RefBufferManager(ref, n, S, 0, 1)
    b = oracle.PortBufferManager(port, n, S)
    hist = []
    for it in range(40):
        nodes = np.unique(rs.randint(0, n, size=rs.randint(1, 300))).astype(np.uint64)
        rs.shuffle(nodes)
        np.testing.assert_array_equal(a.extract(nodes), b.extract(nodes)[0])
        hist.append(nodes)
        lag = rs.randint(0, 3)
        while len(hist) > lag:
            old = hist.pop(0)
            a.release(old)
            b.release(old)
        np.testing.assert_array_equal(a.stats(), b.stats())
    a.validate()


def _torch_sage(x, nodes, edges, layer_nodes, weights, label_seed):
    """Independent formulation of the train stage (torch fp64, index_add_ scatter-mean
    per layer over the dst-sorted block edges) used to pin oracle/sage.py."""
    import torch
    L = len(weights)
    ln = [int(v) for v in layer_nodes]
    D = [min(max(ln[: j + 2]), len(nodes)) for j in range(L + 1)]
    h = torch.tensor(np.asarray(x, np.float64))
    e = torch.tensor(np.asarray(edges, np.int64)).reshape(-1, 2)
    for k in range(1, L + 1):
        rows = D[L - k]
        wn, ws, b = (torch.tensor(np.asarray(a, np.float64)) for a in weights[k - 1])
        m = e[:, 1] < rows
        s = torch.zeros(rows, h.shape[1], dtype=torch.float64).index_add_(0, e[m, 1], h[e[m, 0]])
        c = torch.zeros(rows, dtype=torch.float64).index_add_(0, e[m, 1], torch.ones(int(m.sum()), dtype=torch.float64))
        out = (s / c.clamp(min=1).unsqueeze(1)) @ wn + h[:rows] @ ws + b
        h = torch.relu(out) if k < L else out
    from oracle import sage
    y = torch.tensor(sage.labels(nodes[: len(h)], label_seed, h.shape[1]))
    return float(torch.nn.functional.cross_entropy(h, y)), h.numpy()


@pytest.mark.parametrize("fan,dims", [([10, 10, 10], [16, 32, 32, 12]), ([5, 3], [8, 8, 4]), ([25], [12, 20])])
def test_sage_oracle_matches_torch(port, fan, dims):
    """oracle/sage.py (numpy fp64) against an independent torch fp64 formulation on blocks
    sampled by the C restatement of sample_khop (parity for the train stage is pinned here:
    the reference has no model)."""
    from oracle import sage
    n = 5000
    indptr, indices = port.generate_topology(3, n, 6)
    x = np.random.RandomState(1).standard_normal((n, dims[0])).astype(np.float32)
    seeds = np.random.RandomState(2).randint(0, n, 300).astype(np.uint64)
    b = port.sample_khop(indptr, indices, seeds, fan, 77)
    w = [(np.random.RandomState(10 + i).standard_normal((a, c)) * 0.2, np.random.RandomState(20 + i).standard_normal((a, c)) * 0.2,
          np.random.RandomState(30 + i).standard_normal(c) * 0.1) for i, (a, c) in enumerate(zip(dims[:-1], dims[1:]))]
    xb = x[b["nodes"].astype(np.int64)]
    l1, g1 = sage.sage_forward(xb, b["nodes"], b["edges"], b["layer_nodes"], w, 5)
    l2, g2 = _torch_sage(xb, b["nodes"], b["edges"], b["layer_nodes"], w, 5)
    assert abs(l1 - l2) <= 1e-12 * abs(l2)
    np.testing.assert_allclose(g1, g2, rtol=1e-12, atol=1e-12)
    assert g1.shape == (len(np.unique(seeds)), dims[-1])


def test_ref_config3_baseline_checksums(ref):
    """bench.py's config-3 CPU baseline (batches in order through the reference
    BufferManager, rows hashed from the region via the alias list) yields the same
    per-batch trainer checksums as the plain extraction path, across two calls that share
    the warm buffer (lag-1 release carried over)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    d = tempfile.mkdtemp(prefix="fd_c3_")
    n, dim = 300_000, 8
    feats, _ = ref.stage_dataset(d, n, dim, 10, 7, 4)
    order = ref.partition_epoch(np.arange(8000, dtype=np.uint64), 500, ref.hash_combine(0, 0))
    bench.CONFIGS["c3_test"] = (n, dim, 10, [5, 5, 5], 500, 8000, "f32", 0.5)
    bm = bench.RefBuffer(n, n // 2, dim * 4)
    try:
        _, cs0, nc0 = bench.cpu_reference("c3_test", (d, feats), order, np.arange(0, 10), 4)
        _, cs1, nc1 = bench.cpu_reference("c3_test", (d, feats), order, np.arange(0, 5), 4, bm)
        _, cs2, nc2 = bench.cpu_reference("c3_test", (d, feats), order, np.arange(5, 10), 4, bm)
        st = np.zeros(7, np.uint64)
        ref.lib.fdref_bm_stats(bm.h, st.ctypes.data)
    finally:
        bm.close()
        del bench.CONFIGS["c3_test"]
        import shutil
        shutil.rmtree(d, ignore_errors=True)
    np.testing.assert_array_equal(cs0, np.concatenate([cs1, cs2]))
    np.testing.assert_array_equal(nc0, np.concatenate([nc1, nc2]))
    assert int(st[1]) > 0 and int(st[3]) > 0 and int(st[5]) == 9  # loads, evictions, 9 lag-1 releases
