"""Multi-GPU plumbing: one process per GPU (torchrun), batches split into contiguous
segments like PipelineSession::run_epoch_multi (pipeline.hpp:185-203), and an
optional row-sharded feature table whose remote rows the gather reads through
CUDA IPC peer mappings over NVLink (no collective on the data path).

torch.distributed is used only as the control plane (barriers, max-over-ranks
timing, IPC handle exchange); the data path is libfdg.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import featdrive as fdm


def segment(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous chunk range of `rank`; sizes differ by at most one (pipeline.hpp:192-203)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def shard_geometry(num_nodes: int, n_shards: int) -> tuple[int, list[tuple[int, int]]]:
    """Row blocks of ceil(N / n_shards): owner(node) = node // rows_per_shard."""
    rps = -(-num_nodes // n_shards)
    return rps, [(min(s * rps, num_nodes), min((s + 1) * rps, num_nodes)) for s in range(n_shards)]


def exchange_handles(my_handle: bytes, rank: int, world: int, allgather) -> list[bytes]:
    """All ranks' IPC handles in rank order; `allgather(obj) -> list` is e.g.
    torch.distributed.all_gather_object over a gloo group."""
    got = allgather(bytes(my_handle))
    if len(got) != world or bytes(got[rank]) != bytes(my_handle):
        raise fdm.InvariantViolation("IPC handle exchange returned an inconsistent view")
    return [bytes(h) for h in got]


def torch_allgather(group=None):
    import torch.distributed as dist

    def ag(obj):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, obj, group=group)
        return out

    return ag


class ShardedFeatures:
    """This rank's shard of the synthetic table + the peers' shards mapped over IPC."""

    def __init__(self, topo: fdm.Topology, rank: int, world: int, seed: int, num_nodes: int, dim: int,
                 dtype: str = "f32", allgather=None):
        L = fdm.lib()
        self.topo, self.rank, self.world = topo, rank, world
        base = C.c_void_p()
        dt = 0 if dtype == "f32" else 1
        fdm.check(L.fdg_ctx_generate_feature_shard(topo.ctx, seed, num_nodes, dim, dt, rank, world, C.byref(base)))
        h = (C.c_ubyte * 64)()
        fdm.check(L.fdg_ipc_get_handle(base.value, h))
        handles = exchange_handles(bytes(h), rank, world, allgather or torch_allgather())
        self.opened = []
        bases = []
        for r, hb in enumerate(handles):
            if r == rank:
                bases.append(base.value)
                continue
            p = C.c_void_p()
            fdm.check(L.fdg_ipc_open_handle((C.c_ubyte * 64).from_buffer_copy(hb), C.byref(p)))
            self.opened.append(p.value)
            bases.append(p.value)
        rps, _ = shard_geometry(num_nodes, world)
        arr = (C.c_void_p * world)(*bases)
        row_bytes = dim * (4 if dt == 0 else 2)
        fdm.check(L.fdg_ctx_set_feature_shards(topo.ctx, C.cast(arr, C.c_void_p), world, rps, num_nodes, row_bytes,
                                               dt))
        self.rows_per_shard = rps

    def close(self):
        L = fdm.lib()
        for p in self.opened:
            L.fdg_ipc_close_handle(p)
        self.opened = []


def local_device(local_rank: int) -> int:
    """GPU of this process (several ranks may share one GPU in tests)."""
    n = fdm.device_count()
    return local_rank % max(n, 1)


def rank_batches(n_batches: int, world: int, rank: int) -> np.ndarray:
    lo, hi = segment(n_batches, world, rank)
    return np.arange(lo, hi, dtype=np.int64)


class _DeviceArray:
    """A libfdg device buffer viewed through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def allreduce_grads(model: "fdm.GraphSAGE", group=None) -> None:
    """Data-parallel train stage: average the model's contiguous gradient block over the
    ranks (call between fdg_sage_backward and fdg_sage_sgd, e.g. as
    GraphSAGE.train_step(..., allreduce=allreduce_grads)). With NCCL the block is reduced
    in place on the device (torch wraps the pointer); other backends stage through host
    memory."""
    import torch
    import torch.distributed as dist
    _, gp, n = model.buffers()
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        t = torch.as_tensor(_DeviceArray(gp, n), device="cuda")
        dist.all_reduce(t, group=group)
        t.div_(world)
        torch.cuda.synchronize()
        return
    host = np.empty(n, np.float32)
    fdm.check(fdm.lib().fdg_memcpy_d2h(host.ctypes.data, gp, n * 4, None))
    fdm.check(fdm.lib().fdg_device_sync())
    t = torch.from_numpy(host)
    dist.all_reduce(t, group=group)
    t.div_(world)
    fdm.check(fdm.lib().fdg_memcpy_h2d(gp, host.ctypes.data, n * 4, None))
    fdm.check(fdm.lib().fdg_device_sync())


class AllToAllGather:
    """The comparison baseline of SURVEY §8e for a row-sharded table: rows move by two
    all-to-allv collectives instead of the gather kernel's one-sided NVLink loads
    (ShardedFeatures). Per batch:

      1. bucket the batch's node ids by owner (owner = node // rows_per_shard), stable, so
         every bucket keeps batch order;
      2. all_to_all_single of the per-owner counts, then of the ids;
      3. every owner gathers the requested rows from its local shard (`local_gather`, e.g.
         LocalShardGather = fdg_gather on the shard alone);
      4. all_to_all_single of the rows back; X = the received rows in batch order.

    With the NCCL backend steps 2 and 4 are the grouped ncclSend/ncclRecv all-to-allv the
    one-sided design avoids (pipeline.hpp:193-203 splits batches, not rows, so the
    reference has no such exchange). Tensors live wherever the backend wants them (CUDA
    for NCCL, CPU for gloo: tests/test_dist.py runs the protocol with two gloo ranks)."""

    def __init__(self, rows_per_shard: int, rank: int, world: int, local_gather, group=None):
        self.rps, self.rank, self.world = int(rows_per_shard), rank, world
        self.local_gather, self.group = local_gather, group

    def plan(self, nodes):
        """(order, send_counts): the stable owner-major permutation of the batch and the
        number of ids bound for each rank."""
        import torch
        owner = torch.div(nodes, self.rps, rounding_mode="floor")
        if len(nodes) and int(owner.max()) >= self.world:
            raise fdm.OutOfRange("AllToAllGather: node id beyond the sharded table")
        order = torch.argsort(owner, stable=True)
        return order, torch.bincount(owner, minlength=self.world)

    def __call__(self, nodes):
        import torch
        import torch.distributed as dist
        nodes = nodes.to(torch.int64)
        order, send_counts = self.plan(nodes)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        want = torch.empty(sum(rc), dtype=torch.int64, device=nodes.device)
        dist.all_to_all_single(want, nodes[order], rc, sc, group=self.group)
        rows = self.local_gather(want - self.rank * self.rps)  # [sum(rc), row elems], request order
        back = torch.empty((len(nodes),) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
        dist.all_to_all_single(back, rows, sc, rc, group=self.group)
        x = torch.empty_like(back)
        x[order] = back
        return x


class LocalShardGather:
    """fdg_gather over this rank's shard alone (local row ids): the owner-side step of
    AllToAllGather on the GPU. `base` is the shard's device pointer (e.g. from
    fdg_ctx_generate_feature_shard), `rows` its row count."""

    def __init__(self, device: int, base: int, rows: int, row_bytes: int, dtype: str = "f32"):
        L = fdm.lib()
        self.ctx = C.c_void_p()
        fdm.check(L.fdg_ctx_create(device, C.byref(self.ctx)))
        arr = (C.c_void_p * 1)(base)
        self.dt = 0 if dtype == "f32" else 1
        fdm.check(L.fdg_ctx_set_feature_shards(self.ctx, C.cast(arr, C.c_void_p), 1, rows, rows, row_bytes, self.dt))
        self.row_bytes = row_bytes

    def __call__(self, ids):
        import torch
        tdt = torch.float32 if self.dt == 0 else torch.float16
        elems = self.row_bytes // (4 if self.dt == 0 else 2)
        ids = ids.to(torch.int64).contiguous()
        out = torch.empty((len(ids), elems), dtype=tdt, device=ids.device)
        if len(ids):
            stream = torch.cuda.current_stream(ids.device).cuda_stream
            fdm.check(fdm.lib().fdg_gather(self.ctx, C.c_void_p(stream), C.c_void_p(ids.data_ptr()), None, len(ids),
                                           C.c_void_p(out.data_ptr()), None))
        return out

    def close(self):
        if self.ctx:
            fdm.lib().fdg_ctx_destroy(self.ctx)
            self.ctx = None
