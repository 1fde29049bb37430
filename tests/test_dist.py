"""Multi-process (world_size 2, gloo) coverage of the N>1 host logic on CPU, and the
IPC row-sharded gather with two processes on one GPU."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2406_13984_b200 import dist as fdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # contiguous segments of the epoch's batches, as PipelineSession::run_epoch_multi
        lo, hi = fdist.segment(1001, world, rank)
        segs = [None] * world
        dist.all_gather_object(segs, (lo, hi))
        # IPC handle exchange protocol (fake 64-byte handles)
        mine = bytes([rank + 1]) * 64
        handles = fdist.exchange_handles(mine, rank, world, fdist.torch_allgather())
        # bench's max-over-ranks timing reduction
        os.environ["WORLD_SIZE"], os.environ["RANK"], os.environ["LOCAL_RANK"] = str(world), str(rank), str(rank)
        import bench
        d = bench.Dist.__new__(bench.Dist)
        d.world, d.rank, d.local, d.dist = world, rank, rank, dist
        mx = d.reduce(float(10 + rank), "max")
        sm = d.reduce(1.0, "sum")
        q.put((rank, segs, [h[0] for h in handles], mx, sm))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_host_logic():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    (r0, segs0, h0, mx0, sm0), (r1, segs1, h1, mx1, sm1) = res
    assert segs0 == segs1 == [(0, 501), (501, 1001)]  # contiguous, sizes differ by <= 1
    assert h0 == h1 == [1, 2]
    assert mx0 == mx1 == 11.0 and sm0 == sm1 == 2.0


def test_shard_geometry_and_segments():
    sys.path.insert(0, ROOT)
    from paper_2406_13984_b200 import dist as fdist
    rps, blocks = fdist.shard_geometry(10_001, 4)
    assert rps == 2501 and blocks[-1] == (7503, 10_001)
    owner = np.arange(10_001) // rps
    for s, (lo, hi) in enumerate(blocks):
        assert np.all(owner[lo:hi] == s)
    for world in (1, 2, 3, 8):
        covered = np.concatenate([fdist.rank_batches(1000, world, r) for r in range(world)])
        np.testing.assert_array_equal(covered, np.arange(1000))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_two_process_ipc_sharded_gather(dtype):
    """Two ranks (torchrun, one GPU): each generates its half of the table, the halves
    are exchanged over CUDA IPC, and every rank's sharded gather equals the rows of
    the full single-process table."""
    port = _free_port()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(ROOT, "tests", "mp_shard_check.py")],
                         capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=dict(os.environ, MP_SHARD_DTYPE=dtype))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert out.stdout.count("shard-ok") == 2


@pytest.mark.gpu
def test_two_process_data_parallel_train_stage():
    """Two ranks (torchrun, one GPU): per-rank backward, gradient all-reduce
    (paper_2406_13984_b200.dist.allreduce_grads), identical SGD steps."""
    port = _free_port()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(ROOT, "tests", "mp_train_check.py")],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert out.stdout.count("train-ok") == 2


def _a2a_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2406_13984_b200 import dist as fdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, d = 1001, 6
        table = np.random.RandomState(5).randn(n, d).astype(np.float32)
        rps, blocks = fdist.shard_geometry(n, world)
        lo, hi = blocks[rank]
        local = torch.from_numpy(table[lo:hi].copy())
        g = fdist.AllToAllGather(rps, rank, world, lambda ids: local[ids])
        rs = np.random.RandomState(100 + rank)
        cases = [rs.randint(0, n, 700), np.arange(lo, hi)[::-1], np.zeros(0, np.int64),
                 np.array([n - 1, 0, n - 1, 500])]
        ok = []
        for nodes in cases:
            x = g(torch.from_numpy(np.ascontiguousarray(nodes, np.int64)))
            ok.append(bool(np.array_equal(x.numpy(), table[np.asarray(nodes, np.int64)])))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_all_to_all_gather_protocol_two_ranks():
    """SURVEY §8e's all-to-allv baseline (dist.AllToAllGather) with two gloo ranks: each
    rank's rows, in batch order, equal the full table's -- random, own-shard-only, empty
    and repeated-id batches (the ranks' batches differ, so the exchange is asymmetric)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res == [(0, [True] * 4), (1, [True] * 4)]


@pytest.mark.gpu
def test_all_to_all_gather_nccl_one_rank():
    """The device path of the all-to-allv baseline: NCCL collectives (one rank) around
    fdg_gather on a single-shard context (dist.LocalShardGather) reproduce the gather."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2406_13984_b200 as fd
    from paper_2406_13984_b200 import dist as fdist
    t = fd.Topology.generate(5000, 32, 8, 3)
    info = t.info()
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1)
    try:
        lg = fdist.LocalShardGather(0, info.table_dev, 5000, t.row_bytes)
        g = fdist.AllToAllGather(5000, 0, 1, lg)
        nodes = np.random.RandomState(9).randint(0, 5000, 3000).astype(np.int64)
        x = g(torch.from_numpy(nodes).cuda())
        torch.cuda.synchronize()
        np.testing.assert_array_equal(x.cpu().numpy(), t.download_rows(0, 5000).view(np.float32)[nodes])
        lg.close()
    finally:
        dist.destroy_process_group()
