"""GPU parity of the train stage (fdg_sage_*): GraphSAGE forward + loss on sampled
blocks, fp32 on the GPU against the fp64 restatement oracle/sage.py. Tolerance:
loss within 1e-5 relative (BASELINE.json north_star), logits within 1e-4 relative /
1e-5 absolute."""
import numpy as np
import pytest

from oracle import sage

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-5


def _rows(t, nodes, dtype):
    table = t.download_rows(0, t.num_nodes)
    return table.view(dtype)[nodes.astype(np.int64)]


def _check(model, t, batch, dtype, label_seed):
    loss, logits = model.forward(batch, label_seed)
    want, want_logits = sage.sage_forward(_rows(t, batch.nodes, dtype), batch.nodes, batch.edges,
                                          batch.layer_nodes, model.weights, label_seed)
    assert abs(loss - want) <= LOSS_RTOL * abs(want), (loss, want)
    np.testing.assert_allclose(logits, want_logits, rtol=1e-4, atol=1e-5)
    return loss


@pytest.fixture(params=[1, 0], ids=["tcgen05", "cudacore"])
def gemm(request, fd):
    """Both GEMM engines: tcgen05 kind::tf32 with 3xTF32 splitting, and CUDA-core fp32."""
    old = fd.featdrive.get_option("sage_gemm")
    fd.set_option("sage_gemm", request.param)
    yield request.param
    fd.set_option("sage_gemm", old)


def test_tf32_truncation_check(fd):
    """The 3xTF32 split relies on kind::tf32 ignoring the low 13 mantissa bits of an fp32
    operand (A_hi is then the TMA-landed block itself). fdg_sage_tc.cu checks this once per
    device -- the same GEMM with and without the explicit A_hi write must agree bit for bit
    and be fp32-accurate -- and writes A_hi when it does not hold (option "tc_write_hi").
    B200 truncates: the check must find that (a 1 here would mean a slower but still exact
    split, and that the hardware model in DESIGN.md is wrong)."""
    assert fd.featdrive.get_option("tc_write_hi") == 0


@pytest.mark.parametrize("dim,dims,fan,seeds", [
    (32, [32, 64, 64, 12], [10, 10, 10], 300),
    (128, [128, 256, 256, 172], [10, 10, 10], 200),   # the paper's Papers100M model shape
    (64, [64, 132, 40], [15, 10], 257),               # ragged GEMM tiles (N = 132, 40)
    (16, [16, 8], [25], 1000),
    (4, [4, 12, 8], [3, 3], 50),                      # K = 8 / 24: no tensor-core tiling -> CUDA cores
])
def test_sage_forward_vs_oracle(fd, gemm, dim, dims, fan, seeds):
    t = fd.Topology.generate(60_000, dim, 12, 5)
    s = np.random.RandomState(dim).randint(0, 60_000, seeds).astype(np.uint64)
    batch = fd.sample_khop(t, s, fan, fd.batch_seed(0, 0, dim))
    model = fd.GraphSAGE(t, dims, fan, max_seeds=seeds, seed=dim)
    _check(model, t, batch, np.float32, 0x1234)
    _check(model, t, batch, np.float32, 99)  # a second forward reuses the workspace


def test_sage_forward_fp16_table(fd, gemm):
    """MAG240M-style f16 feature rows: aggregation upconverts to fp32."""
    t = fd.Topology.generate(40_000, 96, 8, 11, dtype="f16")
    s = np.arange(0, 40_000, 97, dtype=np.uint64)
    batch = fd.sample_khop(t, s, [10, 5], 31)
    model = fd.GraphSAGE(t, [96, 64, 20], [10, 5], max_seeds=len(s), seed=3)
    _check(model, t, batch, np.float16, 7)


def test_sage_zero_degree_and_early_stop(fd, gemm):
    """Seeds without in-edges (mean aggregates 0), duplicate seeds and a frontier that
    empties before the last hop (D_j of unreached hops = all nodes)."""
    n = 2000
    rs = np.random.RandomState(4)
    indptr = [0]
    indices = []
    for v in range(n):
        nb = [] if v < 1000 else sorted(set(rs.randint(1000, n, rs.randint(1, 6)).tolist()) - {v})
        indices += nb
        indptr.append(len(indices))
    feats = rs.standard_normal((n, 8)).astype(np.float32)
    t = fd.Topology.from_arrays(np.array(indptr, np.uint64), np.array(indices, np.uint64), feats)
    seeds = np.array([5, 5, 17, 1500, 1999, 3, 1200], np.uint64)
    batch = fd.sample_khop(t, seeds, [4, 4, 4], 9)
    model = fd.GraphSAGE(t, [8, 12, 4, 8], [4, 4, 4], max_seeds=len(seeds), seed=1)
    _check(model, t, batch, np.float32, 3)
    only_isolated = fd.sample_khop(t, np.array([1, 2, 3], np.uint64), [4, 4, 4], 9)
    assert len(only_isolated.edges) == 0
    _check(model, t, only_isolated, np.float32, 3)


def test_sage_bad_config(fd):
    t = fd.Topology.generate(1000, 16, 4, 1)
    with pytest.raises(fd.InvalidArgument):
        fd.GraphSAGE(t, [32, 8], [5])       # dims[0] != feature width
    with pytest.raises(fd.InvalidArgument):
        fd.GraphSAGE(t, [16, 6], [5])       # not a multiple of 4
    with pytest.raises(fd.InvalidArgument):
        fd.GraphSAGE(t, [16, 8, 4], [5])    # one layer per hop


@pytest.mark.parametrize("bm", [False, True])
def test_pipeline_train_stage(fd, bm):
    """The runner's train stage: per-batch losses equal the standalone forward on the
    same batch (same kernels, same bytes -> bitwise) and the fp64 oracle (1e-5)."""
    n, B, fan = 200_000, 256, [10, 5, 5]
    t = fd.Topology.generate(n, 32, 12, 3)
    order = np.concatenate(fd.partition_epoch(np.arange(12 * B, dtype=np.uint64), B, 77))
    nb = 12
    rng = np.array([fd.batch_seed(0, 0, b) for b in range(nb)], np.uint64)
    model = fd.GraphSAGE(t, [32, 64, 64, 16], fan, max_seeds=B, seed=2)
    pipe = fd.Pipeline(t, fan, B, buffer_slots=(150_000 if bm else None), checksum=True, samplers=2)
    pipe.set_model(model, label_seed=5)
    recs = pipe.run_batches(order, rng)
    losses = pipe.losses(nb)
    pipe.close()
    assert np.all(recs["status"] == 0)
    for b in range(nb):
        batch = fd.sample_khop(t, order[b * B:(b + 1) * B], fan, int(rng[b]))
        loss, _ = model.forward(batch, 5)
        assert losses[b] == np.float32(loss), b
        if b < 3:
            want, _ = sage.sage_forward(_rows(t, batch.nodes, np.float32), batch.nodes, batch.edges,
                                        batch.layer_nodes, model.weights, 5)
            assert abs(loss - want) <= LOSS_RTOL * abs(want)


# ------------------------------------------------------------------ backward --
def _grads_close(model, want, rtol=2e-4):
    for layer, w in enumerate(want):
        got = model.layer(layer, grads=True)
        for g, t in zip(got, w):
            scale = max(np.abs(t).max(), 1e-12)
            np.testing.assert_allclose(g, t, rtol=rtol, atol=rtol * scale)


@pytest.mark.parametrize("dim,dims,fan,seeds", [
    (32, [32, 64, 64, 12], [10, 10, 10], 300),
    (128, [128, 256, 256, 172], [10, 10, 10], 200),   # the paper's model shape (d_out 172: K % 8 = 4)
    (16, [16, 8], [25], 500),
])
def test_sage_backward_vs_autograd(fd, gemm, dim, dims, fan, seeds):
    """fdg_sage_backward: every layer's W_neigh / W_self / b gradient against torch fp64
    autograd of the same model (fp32 + atomics: 2e-4 relative to each tensor's scale)."""
    t = fd.Topology.generate(60_000, dim, 12, 5)
    s = np.random.RandomState(dim + 1).randint(0, 60_000, seeds).astype(np.uint64)
    batch = fd.sample_khop(t, s, fan, fd.batch_seed(0, 1, dim))
    model = fd.GraphSAGE(t, dims, fan, max_seeds=seeds, seed=dim + 1)
    loss = model.train_step(batch, label_seed=11, lr=0.0)
    want_loss, want = sage.sage_grads(_rows(t, batch.nodes, np.float32), batch.nodes, batch.edges,
                                      batch.layer_nodes, model.weights, 11)
    assert abs(loss - want_loss) <= LOSS_RTOL * abs(want_loss)
    _grads_close(model, want)


def test_sage_sgd_step_and_descent(fd, gemm):
    """SGD: W' = W - lr * grad exactly as the host computes it, the derived (tensor-core /
    CUDA-core) copies follow, and repeated steps on one batch reduce its loss."""
    t = fd.Topology.generate(40_000, 32, 10, 2)
    s = np.arange(0, 40_000, 157, dtype=np.uint64)
    batch = fd.sample_khop(t, s, [10, 5], 3)
    model = fd.GraphSAGE(t, [32, 64, 16], [10, 5], max_seeds=len(s), seed=4)
    before = [model.layer(i) for i in range(2)]
    l0 = model.train_step(batch, label_seed=1, lr=0.0)
    grads = [model.layer(i, grads=True) for i in range(2)]
    model.sgd(0.5)
    for i in range(2):
        for w, g, now in zip(before[i], grads[i], model.layer(i)):
            np.testing.assert_allclose(now, w.astype(np.float64) - 0.5 * g.astype(np.float64), rtol=1e-6, atol=1e-7)
    loss1, _ = model.forward(batch, 1)
    assert loss1 < l0
    losses = [model.train_step(batch, label_seed=1, lr=0.5) for _ in range(5)]
    assert losses[-1] < losses[0] < l0


def test_sage_backward_zero_degree(fd):
    """Isolated seeds / an early-stopped frontier: zero-degree destinations scatter nothing."""
    n = 2000
    rs = np.random.RandomState(4)
    indptr, indices = [0], []
    for v in range(n):
        nb = [] if v < 1000 else sorted(set(rs.randint(1000, n, rs.randint(1, 6)).tolist()) - {v})
        indices += nb
        indptr.append(len(indices))
    feats = rs.standard_normal((n, 8)).astype(np.float32)
    t = fd.Topology.from_arrays(np.array(indptr, np.uint64), np.array(indices, np.uint64), feats)
    batch = fd.sample_khop(t, np.array([5, 5, 17, 1500, 1999, 3, 1200], np.uint64), [4, 4, 4], 9)
    model = fd.GraphSAGE(t, [8, 12, 4, 8], [4, 4, 4], max_seeds=7, seed=1)
    model.train_step(batch, label_seed=3)
    _, want = sage.sage_grads(_rows(t, batch.nodes, np.float32), batch.nodes, batch.edges, batch.layer_nodes,
                              model.weights, 3)
    _grads_close(model, want)


def test_pipeline_training_matches_host_loop(fd):
    """The runner in training mode (forward + backward + SGD per batch) reproduces a host
    loop of train_step over the same batches: losses and final weights."""
    n, B, fan = 100_000, 128, [5, 5]
    t = fd.Topology.generate(n, 32, 10, 6)
    order = np.concatenate(fd.partition_epoch(np.arange(6 * B, dtype=np.uint64), B, 5))
    rng = np.array([fd.batch_seed(0, 0, b) for b in range(6)], np.uint64)
    a = fd.GraphSAGE(t, [32, 32, 8], fan, max_seeds=B, seed=9)
    b = fd.GraphSAGE(t, [32, 32, 8], fan, max_seeds=B, seed=9)
    pipe = fd.Pipeline(t, fan, B, samplers=2)
    pipe.set_model(a, label_seed=2)
    pipe.set_training(0.3)
    pipe.run_batches(order, rng)
    losses = pipe.losses(6)
    pipe.close()
    for j in range(6):
        batch = fd.sample_khop(t, order[j * B:(j + 1) * B], fan, int(rng[j]))
        lj = b.train_step(batch, label_seed=2, lr=0.3)
        assert abs(losses[j] - lj) <= 1e-5 * abs(lj), j
    for i in range(2):
        for u, v in zip(a.layer(i), b.layer(i)):
            np.testing.assert_allclose(u, v, rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("R,Kin,N,Z", [(64, 128, 128, 1), (1000, 256, 256, 4), (777, 512, 172, 5), (33, 64, 12, 3),
                                       (5000, 24, 8, 7)])
def test_weight_gradient_engines(fd, gemm, R, Kin, N, Z):
    """A^T . B (+ column sums of B) through the backward's weight-gradient engines: the
    tcgen05 MN-major split-K kernel (128B / 32B-atom swizzle) and the CUDA-core one, with
    ragged rows / columns and empty row slices, against fp64."""
    from paper_2406_13984_b200.featdrive import DeviceBuffer, check, lib
    rs = np.random.RandomState(R + Kin)
    A = rs.standard_normal((R, Kin)).astype(np.float32)
    B = rs.standard_normal((R, N)).astype(np.float32)
    da, db, out = DeviceBuffer.from_array(A), DeviceBuffer.from_array(B), DeviceBuffer((Kin + 1) * N * 4)
    check(lib().fdg_sage_wgrad_test(da.ptr, db.ptr, R, Kin, N, Z, out.ptr))
    got = out.download(np.float32, (Kin + 1) * N)
    want = A.astype(np.float64).T @ B.astype(np.float64)
    scale = np.abs(want).max()
    np.testing.assert_allclose(got[:Kin * N].reshape(Kin, N), want, rtol=1e-5, atol=1e-5 * scale)
    np.testing.assert_allclose(got[Kin * N:], B.astype(np.float64).sum(0), rtol=1e-5, atol=1e-4)
