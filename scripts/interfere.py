"""Diagnostic: how much does a concurrent random-access (or streaming) load slow the
feature gather? Runs fdg_gather in a loop on one stream while torch kernels with a
known access pattern run on another; prints gather time/launch and the load's rate."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2406_13984_b200 as fd  # noqa: E402

fd.set_option("gather_impl", 1)
n, dim, avg, fan, B, t_ids, dtype, frac = bench.CONFIGS["papers"]
L = fd.featdrive.lib()
topo = fd.Topology.generate(n, dim, avg, 7)
rows = 934_000
g = torch.Generator(device="cuda").manual_seed(1)
nodes = torch.randint(0, n, (rows,), device="cuda", generator=g, dtype=torch.int64)
out = torch.empty(rows * topo.row_bytes, dtype=torch.uint8, device="cuda")
big = torch.empty(6 << 30, dtype=torch.uint8, device="cuda").view(torch.int64)
ridx = torch.randint(0, big.numel(), (1 << 20,), device="cuda", generator=g)
seq_src = big[: (32 << 20) // 8]
seq_dst = torch.empty_like(seq_src)
rnd_out = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
small = torch.zeros(2_200_000, dtype=torch.int64, device="cuda")  # hash-sized (17.6 MB)
sidx = torch.randint(0, small.numel(), (1 << 20,), device="cuda", generator=g)
ones = torch.ones(1 << 20, dtype=torch.int64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def gather_loop(k):
    for _ in range(k):
        fd.featdrive.check(L.fdg_gather(topo.ctx, C.c_void_p(sa.cuda_stream), C.c_void_p(nodes.data_ptr()), None,
                                        rows, C.c_void_p(out.data_ptr()), None))


loads = {
    "none": None,
    "rand_read_8B": lambda: torch.index_select(big, 0, ridx, out=rnd_out),
    "seq_copy_32MB": lambda: seq_dst.copy_(seq_src),
    "rand_atomic_L2": lambda: small.index_add_(0, sidx, ones),
}
K = 40
alone = {}
for name, fn in loads.items():
    if fn is None:
        continue
    torch.cuda.synchronize()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0.record()
    for _ in range(200):
        fn()
    b1.record()
    torch.cuda.synchronize()
    alone[name] = b0.elapsed_time(b1) / 200 * 1e3
    print(f"{name:16s} alone: {alone[name]:7.1f} us/op")
for name, fn in loads.items():
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nops = 0
    if fn is not None:  # enqueue ~12 ms of load first (the gather call may block the host)
        nops = int(12000 / alone[name])
        with torch.cuda.stream(sb):
            b0.record(sb)
            for _ in range(nops):
                fn()
            b1.record(sb)
    with torch.cuda.stream(sa):
        e0.record(sa)
        gather_loop(K)
        e1.record(sa)
    torch.cuda.synchronize()
    gt = e0.elapsed_time(e1) / K * 1e3
    gbs = 2 * rows * topo.row_bytes / (gt * 1e-6) / 1e9
    msg = f"{name:16s} gather {gt:7.1f} us/launch ({gbs:6.0f} GB/s)"
    if fn is not None:
        lt = b0.elapsed_time(b1)
        msg += f"   load: {nops} ops in {lt:.2f} ms ({lt * 1e3 / nops:.1f} us/op vs {alone[name]:.1f} alone)"
    print(msg, flush=True)
