"""Python mirror of the reference's sample -> extract interface, backed by libfdg.

Names, argument meaning and error behaviour follow featdrive
(/root/reference/proj/include/featdrive):

=============================  ==============================================
reference                      here
=============================  ==============================================
graph::Topology                Topology (device-resident CSC; generate / files)
graph::Fanouts                 Fanouts
graph::SampledBatch            SampledBatch (nodes u64, edges [E,2] u32)
graph::sample_khop             sample_khop (GPU, bit-exact)
graph::partition_epoch         partition_epoch (libstdc++ std::shuffle, host)
PipelineSession::batch_seed    batch_seed
featbuf::BufferManager         BufferManager (GPU mapping table / standby ring)
featbuf::FeatureRegion         BufferManager.region (HBM slot pool)
extract::Extractor             Extractor.extract_batch -> NodeAliasList
pipeline::trainer_step         trainer_step (GPU hash_bytes64 checksum)
=============================  ==============================================

Exceptions: std::out_of_range -> OutOfRange (IndexError), std::invalid_argument
-> InvalidArgument (ValueError), InvariantViolation -> InvariantViolation,
StandbyTimeout -> StandbyTimeout. There is no CPU fallback: every operation
runs on the GPU through libfdg.so or raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import BatchCounts, BmStats, CtxInfo


class FeatdriveError(RuntimeError):
    pass


class OutOfRange(FeatdriveError, IndexError):
    pass


class InvalidArgument(FeatdriveError, ValueError):
    pass


class InvariantViolation(FeatdriveError):
    pass


class StandbyTimeout(FeatdriveError):
    pass


class CudaError(FeatdriveError):
    pass


class DatasetError(FeatdriveError):
    """A dataset file is missing or malformed (the reference's std::runtime_error from
    Topology / FeatureTable / DatasetHeader::validate). `errno` is set (non-zero) where the
    reference throws std::system_error from a failed system call."""

    def __init__(self, msg: str, errno: int = 0):
        super().__init__(msg if not errno else f"{msg}: {os.strerror(errno)}")
        self.errno = errno


_ERRORS = {1: OutOfRange, 2: InvalidArgument, 3: InvariantViolation, 4: StandbyTimeout, 5: CudaError}


def check(rc: int) -> None:
    if rc == 8:
        raise DatasetError(_lib.last_error(), lib().fdg_last_errno())
    if rc != 0:
        raise _ERRORS.get(rc, FeatdriveError)(_lib.last_error() or f"fdg status {rc}")


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def lib():
    return _lib.load()


# ------------------------------------------------------------------ plumbing --
class DeviceBuffer:
    """Raw HBM allocation owned by Python."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        p = C.c_void_p()
        check(lib().fdg_malloc(C.byref(p), max(self.nbytes, 1)))
        self.ptr = p.value

    @classmethod
    def from_array(cls, a: np.ndarray, stream=None) -> "DeviceBuffer":
        a = np.ascontiguousarray(a)
        b = cls(a.nbytes)
        b.upload(a, stream)
        return b

    def upload(self, a: np.ndarray, stream=None, offset: int = 0):
        a = np.ascontiguousarray(a)
        check(lib().fdg_memcpy_h2d(self.ptr + offset, _p(a), a.nbytes, stream))
        if stream is None:
            check(lib().fdg_stream_sync(None))

    def download(self, dtype, count: int | None = None, offset: int = 0, stream=None) -> np.ndarray:
        dt = np.dtype(dtype)
        if count is None:
            count = (self.nbytes - offset) // dt.itemsize
        out = np.empty(count, dt)
        check(lib().fdg_memcpy_d2h(_p(out), self.ptr + offset, out.nbytes, stream))
        check(lib().fdg_stream_sync(stream))
        return out

    def zero(self, stream=None):
        check(lib().fdg_memset(self.ptr, 0, self.nbytes, stream))

    def free(self):
        if getattr(self, "ptr", None):
            lib().fdg_free(self.ptr)
            self.ptr = None

    __del__ = free


class Stream:
    def __init__(self):
        p = C.c_void_p()
        check(lib().fdg_stream_create(C.byref(p)))
        self.ptr = p.value

    def sync(self):
        check(lib().fdg_stream_sync(self.ptr))

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().fdg_stream_destroy(self.ptr)
            self.ptr = None


class Event:
    def __init__(self):
        p = C.c_void_p()
        check(lib().fdg_event_create(C.byref(p)))
        self.ptr = p.value

    def record(self, stream: "Stream | None" = None):
        check(lib().fdg_event_record(self.ptr, stream.ptr if stream else None))

    def synchronize(self):
        check(lib().fdg_event_sync(self.ptr))

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        check(lib().fdg_event_elapsed_ms(self.ptr, end.ptr, C.byref(ms)))
        return ms.value

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().fdg_event_destroy(self.ptr)
            self.ptr = None


def set_option(key: str, value: int) -> None:
    """Process-wide tuning knob (fdg_set_option): gather_impl, gather_evict_first, ..."""
    check(lib().fdg_set_option(key.encode(), int(value)))


def get_option(key: str) -> int:
    v = C.c_int64()
    check(lib().fdg_get_option(key.encode(), C.byref(v)))
    return v.value


def device_count() -> int:
    n = C.c_int()
    check(lib().fdg_device_count(C.byref(n)))
    return n.value


# -------------------------------------------------------------------- helpers --
def batch_seed(seed: int, epoch: int, global_batch: int) -> int:
    """PipelineSession::batch_seed (pipeline.hpp:295-298)."""
    return lib().fdg_batch_seed(seed, epoch, global_batch)


def partition_epoch(train_ids, batch_size: int, shuffle_seed: int) -> list[np.ndarray]:
    """graph::partition_epoch (sampling.hpp:57-70)."""
    if batch_size < 1:
        raise InvalidArgument("partition_epoch: batch_size must be >= 1")
    ids = np.ascontiguousarray(train_ids, np.uint64)
    out = np.empty_like(ids)
    check(lib().fdg_partition_epoch(_p(ids), len(ids), batch_size, shuffle_seed, _p(out)))
    return [out[i:i + batch_size] for i in range(0, len(out), batch_size)]


# ------------------------------------------------------------------- topology --
class Topology:
    """Device-resident CSC topology + feature table (graph::Topology, topology.hpp:33-193,
    plus the FeatureTable rows, feature_file.hpp:25-107)."""

    def __init__(self, device: int = 0):
        self.device = device
        p = C.c_void_p()
        check(lib().fdg_ctx_create(device, C.byref(p)))
        self.ctx = p.value

    # constructors -----------------------------------------------------------
    @classmethod
    def from_dataset(cls, dataset_dir: str, device: int = 0, features: bool = True) -> "Topology":
        t = cls(device)
        check(lib().fdg_ctx_load_topology_files(t.ctx, dataset_dir.encode()))
        if features:
            check(lib().fdg_ctx_load_features_file(t.ctx, f"{dataset_dir}/features.bin".encode()))
        return t

    @classmethod
    def from_arrays(cls, indptr, indices, features: np.ndarray | None = None, device: int = 0) -> "Topology":
        t = cls(device)
        ip = np.ascontiguousarray(indptr, np.uint64)
        ix = np.ascontiguousarray(indices, np.uint64)
        check(lib().fdg_ctx_load_topology(t.ctx, _p(ip), len(ip) - 1, _p(ix), len(ix)))
        if features is not None:
            f = np.ascontiguousarray(features)
            dtype = 1 if f.dtype == np.float16 else 0
            check(lib().fdg_ctx_load_features(t.ctx, _p(f), f.shape[0], f.shape[1] * f.itemsize, dtype))
        return t

    @classmethod
    def generate(cls, num_nodes: int, dim: int, avg_degree: int, seed: int = 7, dtype: str = "f32",
                 device: int = 0, shards: int = 1, features: bool = True) -> "Topology":
        """GPU port of storage::create_synthetic_dataset (generator.hpp:187-267), HBM-resident."""
        t = cls(device)
        check(lib().fdg_ctx_generate_topology(t.ctx, seed, num_nodes, avg_degree))
        if features:
            check(lib().fdg_ctx_generate_features(t.ctx, seed, num_nodes, dim, 0 if dtype == "f32" else 1, shards))
        return t

    # introspection ----------------------------------------------------------
    def info(self) -> CtxInfo:
        i = CtxInfo()
        check(lib().fdg_ctx_info_get(self.ctx, C.byref(i)))
        return i

    @property
    def num_nodes(self) -> int:
        return self.info().num_nodes

    @property
    def num_edges(self) -> int:
        return self.info().num_edges

    @property
    def row_bytes(self) -> int:
        return self.info().row_bytes

    def download_topology(self):
        i = self.info()
        indptr = np.empty(i.num_nodes + 1, np.uint64)
        indices = np.empty(i.num_edges, np.uint32 if i.idx_bytes == 4 else np.uint64)
        check(lib().fdg_ctx_download_topology(self.ctx, _p(indptr), _p(indices)))
        return indptr, indices

    def features_to_host(self) -> "Topology":
        """Out-of-core tier: keep the feature table in pinned host memory (mapped); the
        gather and buffer-manager misses read it over PCIe / C2C."""
        check(lib().fdg_ctx_features_to_host(self.ctx))
        return self

    @property
    def features_on_host(self) -> bool:
        return bool(lib().fdg_ctx_features_on_host(self.ctx))

    def download_rows(self, first: int, count: int) -> np.ndarray:
        rb = self.row_bytes
        out = np.empty((count, rb), np.uint8)
        check(lib().fdg_ctx_download_rows(self.ctx, first, count, _p(out)))
        return out

    def __del__(self):
        if getattr(self, "ctx", None):
            lib().fdg_ctx_destroy(self.ctx)
            self.ctx = None


# -------------------------------------------------------------------- sampling --
@dataclass
class Fanouts:
    """graph::Fanouts (sampling.hpp:21-41)."""
    per_layer: list = field(default_factory=lambda: [10, 10, 10])

    def validate(self):
        if not self.per_layer:
            raise InvalidArgument("fanouts: need at least one layer")
        if any(int(f) < 1 for f in self.per_layer):
            raise InvalidArgument("fanouts: every entry must be >= 1")

    def max_batch_nodes(self, batch_size: int) -> int:
        total, layer = 1, 1
        for f in self.per_layer:
            layer *= int(f)
            total += layer
        return batch_size * total


@dataclass
class SampledBatch:
    """graph::SampledBatch (sampling.hpp:48-54) + per-layer block offsets."""
    batch_id: int = 0
    epoch: int = 0
    seeds: np.ndarray = None
    nodes: np.ndarray = None        # u64, deduplicated, seeds first
    edges: np.ndarray = None        # [E, 2] u32 {src_local, dst_local}
    layer_nodes: np.ndarray = None  # [L+2]
    layer_edges: np.ndarray = None  # [L+1]


class Sampler:
    """A GPU sampling workspace (one stream at a time)."""

    def __init__(self, topo: Topology, fanouts: Fanouts | list, max_seeds: int = 1000):
        self.topo = topo
        self.fanouts = fanouts if isinstance(fanouts, Fanouts) else Fanouts(list(fanouts))
        f = np.ascontiguousarray(self.fanouts.per_layer, np.uint32)
        p = C.c_void_p()
        check(lib().fdg_sampler_create(topo.ctx, max_seeds, _p(f), len(f), C.byref(p)))
        self.ptr = p.value
        self.max_seeds = max_seeds
        mn, me = C.c_uint64(), C.c_uint64()
        check(lib().fdg_sampler_capacity(self.ptr, C.byref(mn), C.byref(me)))
        self.max_nodes, self.max_edges = mn.value, me.value
        self.cap = max(self.max_nodes, self.max_edges, 1)

    def sample(self, seeds, rng_seed: int) -> SampledBatch:
        seeds = np.ascontiguousarray(seeds, np.uint64)
        L = len(self.fanouts.per_layer)
        nodes = np.empty(self.cap, np.uint64)
        edges = np.empty((self.cap, 2), np.uint32)
        nn, ne = C.c_uint64(), C.c_uint64()
        ln = np.zeros(L + 2, np.uint64)
        le = np.zeros(L + 1, np.uint64)
        check(lib().fdg_sample_khop_host(self.ptr, _p(seeds), len(seeds), rng_seed, _p(nodes), _p(edges), self.cap,
                                         C.byref(nn), C.byref(ne), _p(ln), _p(le)))
        return SampledBatch(seeds=seeds.copy(), nodes=nodes[: nn.value].copy(), edges=edges[: ne.value].copy(),
                            layer_nodes=ln, layer_edges=le)

    def sample_words(self, seeds, words):
        """Test hook: draw from an explicit word stream instead of MT19937-64."""
        seeds = np.ascontiguousarray(seeds, np.uint64)
        w = np.ascontiguousarray(words, np.uint64)
        nodes = np.empty(self.cap, np.uint64)
        edges = np.empty((self.cap, 2), np.uint32)
        nn, ne, wu = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().fdg_sample_khop_words_host(self.ptr, _p(seeds), len(seeds), _p(w), len(w), _p(nodes), _p(edges),
                                               self.cap, C.byref(nn), C.byref(ne), C.byref(wu)))
        return nodes[: nn.value].copy(), edges[: ne.value].copy(), wu.value

    def sample_async(self, stream: Stream, seeds_dev: DeviceBuffer, n_seeds: int, rng_seed: int,
                     nodes_dev: DeviceBuffer, edges_dev: DeviceBuffer, counts_dev: DeviceBuffer):
        check(lib().fdg_sample_khop(self.ptr, stream.ptr if stream else None, seeds_dev.ptr, n_seeds, rng_seed,
                                    nodes_dev.ptr, edges_dev.ptr, self.cap, counts_dev.ptr))

    def prefetch(self, stream: Stream, rng_seeds):
        s = np.ascontiguousarray(rng_seeds, np.uint64)
        check(lib().fdg_sampler_prefetch(self.ptr, stream.ptr if stream else None, _p(s), len(s)))

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().fdg_sampler_destroy(self.ptr)
            self.ptr = None


def sample_khop(topo: Topology, seeds, fanouts: Fanouts | list, rng_seed: int) -> SampledBatch:
    """graph::sample_khop (sampling.hpp:72-134), on the GPU, bit-exact."""
    fan = fanouts if isinstance(fanouts, Fanouts) else Fanouts(list(fanouts))
    fan.validate()
    seeds = np.ascontiguousarray(seeds, np.uint64)
    key = (tuple(int(f) for f in fan.per_layer), max(len(seeds), 1))
    cache = topo.__dict__.setdefault("_samplers", {})
    s = cache.get(key)
    if s is None:
        s = cache[key] = Sampler(topo, fan, max(len(seeds), 1))
    return s.sample(seeds, rng_seed)


def mt_stream(rng_seed: int, n: int) -> np.ndarray:
    """std::mt19937_64(splitmix64(rng_seed)) words generated on the GPU."""
    buf = DeviceBuffer(8 * n)
    check(lib().fdg_mt_stream(None, rng_seed, n, buf.ptr))
    check(lib().fdg_device_sync())
    return buf.download(np.uint64, n)


# ------------------------------------------------------------------- gather --
def gather(topo: Topology, nodes, checksum: bool = False):
    """Mini-batch tensor X[i] = row(nodes[i]) (+ trainer_step checksum)."""
    nodes = np.ascontiguousarray(nodes, np.uint64)
    rb = topo.row_bytes
    nd = DeviceBuffer.from_array(nodes)
    out = DeviceBuffer(len(nodes) * rb)
    cs = DeviceBuffer(8) if checksum else None
    if cs:
        cs.zero()
    check(lib().fdg_gather(topo.ctx, None, nd.ptr, None, len(nodes), out.ptr, cs.ptr if cs else None))
    check(lib().fdg_device_sync())
    x = out.download(np.uint8).reshape(len(nodes), rb)
    return (x, int(cs.download(np.uint64)[0])) if cs else x


# ----------------------------------------------------------- buffer manager --
class BufferManager:
    """featbuf::BufferManager (buffer_manager.hpp:222-527) + FeatureRegion
    (device_region.hpp:24-50) on the GPU. Operations are stream-ordered batches:
    extract = acquire_for_batch + (get_standby_slot + bind_slot) per miss in batch
    order + row copies + publish_valid; release = release_batch."""

    def __init__(self, topo: Topology, slot_count: int, min_reserved: int = 0, max_batch_nodes: int | None = None):
        self.topo = topo
        self.slot_count = int(slot_count)
        self.row_bytes = topo.row_bytes
        mb = int(max_batch_nodes if max_batch_nodes is not None else min(slot_count, topo.num_nodes))
        p = C.c_void_p()
        check(lib().fdg_bm_create(topo.ctx, slot_count, min_reserved, mb, C.byref(p)))
        self.ptr = p.value
        self.max_batch_nodes = mb

    @property
    def region_ptr(self) -> int:
        return lib().fdg_bm_region(self.ptr)

    def _status(self):
        rc = lib().fdg_bm_status(self.ptr)
        if rc == 4:
            raise StandbyTimeout("get_standby_slot: standby list exhausted; feature buffer is undersized")
        if rc == 3:
            raise InvariantViolation("buffer manager invariant violated (device-detected)")
        check(rc)

    def extract(self, nodes, want_rows: bool = False, checksum: bool = False):
        """Returns alias (NodeAliasList) [, X rows] [, checksum]."""
        nodes = np.ascontiguousarray(nodes, np.uint64)
        n = len(nodes)
        nd = DeviceBuffer.from_array(nodes) if n else DeviceBuffer(8)
        al = DeviceBuffer(max(n, 1) * 8)
        x = DeviceBuffer(max(n, 1) * self.row_bytes) if want_rows else None
        cs = DeviceBuffer(8) if checksum else None
        if cs:
            cs.zero()
        check(lib().fdg_bm_extract(self.ptr, None, nd.ptr, None, n, al.ptr, x.ptr if x else None,
                                   cs.ptr if cs else None))
        self._status()
        out = [al.download(np.int64, n)]
        if x:
            out.append(x.download(np.uint8, n * self.row_bytes).reshape(n, self.row_bytes))
        if cs:
            out.append(int(cs.download(np.uint64)[0]))
        return out[0] if len(out) == 1 else tuple(out)

    def release_batch(self, nodes):
        nodes = np.ascontiguousarray(nodes, np.uint64)
        nd = DeviceBuffer.from_array(nodes) if len(nodes) else DeviceBuffer(8)
        check(lib().fdg_bm_release(self.ptr, None, nd.ptr, None, len(nodes)))
        self._status()

    def stats(self) -> dict:
        s = BmStats()
        check(lib().fdg_bm_stats_get(self.ptr, C.byref(s)))
        return {k: getattr(s, k) for k, _ in BmStats._fields_}

    def mapping_entry(self, node: int):
        slot, ref, valid = C.c_int64(), C.c_uint32(), C.c_uint32()
        check(lib().fdg_bm_entry(self.ptr, node, C.byref(slot), C.byref(ref), C.byref(valid)))
        return slot.value, ref.value, valid.value

    def reverse_mapping(self, slot: int) -> int:
        v = C.c_int64()
        check(lib().fdg_bm_reverse(self.ptr, slot, C.byref(v)))
        return v.value

    def validate(self):
        check(lib().fdg_bm_validate(self.ptr))

    def ring_info(self) -> dict:
        """Standby ring positions [head, tail), capacity and tombstone compactions so far."""
        v = [C.c_uint64() for _ in range(4)]
        check(lib().fdg_bm_ring_info(self.ptr, *[C.byref(x) for x in v]))
        return dict(zip(("head", "tail", "capacity", "compactions"), (x.value for x in v)))

    def region_slots(self, slots) -> np.ndarray:
        """Bytes of FeatureRegion slots (device_region.hpp:36-44), for tests."""
        rb = self.row_bytes
        out = np.empty((len(slots), rb), np.uint8)
        for k, s in enumerate(slots):
            check(lib().fdg_memcpy_d2h(_p(out[k]), self.region_ptr + int(s) * rb, rb, None))
        check(lib().fdg_stream_sync(None))
        return out

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().fdg_bm_destroy(self.ptr)
            self.ptr = None


COUNTS_DTYPE = np.dtype([("status", "<u4"), ("n_nodes", "<u4"), ("n_edges", "<u4"), ("rejections", "<u4"),
                         ("bad_seed", "<u8"), ("checksum", "<u8"), ("bad_seed_pos", "<u4"), ("n_layers", "<u4"),
                         ("layer_nodes", "<u4", (_lib.MAX_LAYERS + 2,)),
                         ("layer_edges", "<u4", (_lib.MAX_LAYERS + 1,)),
                         ("layer_draws", "<u4", (_lib.MAX_LAYERS + 1,)), ("words_used", "<u4"), ("replays", "<u4")])


class Pipeline:
    """Native SET-loop runner (fdg_pipeline_*): PipelineSession's sampler ->
    extractor (-> trainer checksum -> releaser) stages for one GPU
    (pipeline.hpp:325-543), batches pipelined across CUDA streams."""

    def __init__(self, topo: Topology, fanouts, batch_size: int = 1000, buffer_slots: int | None = None,
                 checksum: bool = False, samplers: int = 6, group_batches: int = 1, prefetch_group: int = 16,
                 flags: int = 0, write_x: bool = True):
        self.topo = topo
        cfg = _lib.PipelineConfig(batch_size=batch_size, n_samplers=samplers, prefetch_group=prefetch_group,
                                  use_buffer_manager=1 if buffer_slots else 0, buffer_slots=buffer_slots or 0,
                                  write_x=1 if write_x else 0, checksum=1 if checksum else 0, flags=flags,
                                  group_batches=group_batches)
        f = np.ascontiguousarray(list(fanouts.per_layer if isinstance(fanouts, Fanouts) else fanouts), np.uint32)
        p = C.c_void_p()
        check(lib().fdg_pipeline_create(topo.ctx, _p(f), len(f), C.byref(cfg), C.byref(p)))
        self.ptr = p.value
        self.batch_size = batch_size

    def run(self, seeds_ptr: int, on_host: bool, rng_seeds, records_ptr: int | None = None,
            extract_ms: np.ndarray | None = None, n_seeds: int | None = None) -> float:
        """Run len(rng_seeds) batches; returns the device time of the run in ms. n_seeds
        (default len(rng_seeds) * batch_size) lets the last batch be short."""
        rng = np.ascontiguousarray(rng_seeds, np.uint64)
        ms = C.c_float()
        total = len(rng) * self.batch_size if n_seeds is None else int(n_seeds)
        check(lib().fdg_pipeline_run_ragged(self.ptr, seeds_ptr, 1 if on_host else 0, total, _p(rng), len(rng),
                                            records_ptr, _p(extract_ms), C.byref(ms)))
        return ms.value

    def set_model(self, model: "GraphSAGE | None", label_seed: int = 0):
        """Run the train stage (GraphSAGE forward + loss) after every extraction."""
        self.model = model
        check(lib().fdg_pipeline_set_model(self.ptr, model.ptr if model else None, label_seed))

    def set_training(self, lr: float):
        """lr != 0: the train stage also runs backward + SGD after every forward."""
        check(lib().fdg_pipeline_set_training(self.ptr, lr))

    def bm_stats(self) -> dict:
        """Cumulative counters of the runner's buffer manager (BufferManager::stats())."""
        s = BmStats()
        check(lib().fdg_pipeline_bm_stats(self.ptr, C.byref(s)))
        return {k: getattr(s, k) for k, _ in BmStats._fields_}

    def losses(self, n: int, first: int = 0) -> np.ndarray:
        out = np.empty(n, np.float32)
        check(lib().fdg_pipeline_losses(self.ptr, first, n, _p(out)))
        return out

    def sample_busy_ms(self) -> float:
        """Sampling-stage busy time of the last run (run with extract_ms)."""
        ms = C.c_float()
        check(lib().fdg_pipeline_sample_times(self.ptr, None, C.byref(ms)))
        return ms.value

    def run_batches(self, seeds: np.ndarray, rng_seeds, checksum_records: bool = True) -> np.ndarray:
        """Convenience: host seeds (batch j = seeds[j*B:(j+1)*B], the last may be short)
        -> per-batch records (COUNTS_DTYPE)."""
        seeds = np.ascontiguousarray(seeds, np.uint64)
        dev = DeviceBuffer.from_array(seeds)
        self.run(dev.ptr, False, rng_seeds, n_seeds=len(seeds))
        return self.records(len(rng_seeds))

    def records(self, n: int) -> np.ndarray:
        out = np.zeros(n, COUNTS_DTYPE)
        check(lib().fdg_pipeline_records(self.ptr, 0, n, _p(out)))
        return out

    def extract_times(self, n: int) -> tuple[np.ndarray, np.ndarray]:
        """(start_ms, end_ms) of each batch's extraction in the last run (run with extract_ms)."""
        a, b = np.zeros(n, np.float32), np.zeros(n, np.float32)
        check(lib().fdg_pipeline_extract_times(self.ptr, 0, n, _p(a), _p(b)))
        return a, b

    def host_enqueue_ms(self) -> float:
        cfg = _lib.PipelineConfig()
        check(lib().fdg_pipeline_get_config(self.ptr, C.byref(cfg)))
        return cfg.host_enqueue_ms

    def close(self):
        if getattr(self, "ptr", None):
            lib().fdg_pipeline_destroy(self.ptr)
            self.ptr = None

    __del__ = close


class Extractor:
    """extract::Extractor (extractor.hpp:75-113): extract_batch -> NodeAliasList."""

    def __init__(self, buffer: BufferManager):
        self.buffer = buffer

    def extract_batch(self, batch: SampledBatch) -> np.ndarray:
        return self.buffer.extract(batch.nodes)


def trainer_step(batch: SampledBatch, alias: np.ndarray, buffer: BufferManager) -> int:
    """pipeline::trainer_step (pipeline.hpp:103-124): sum of hash_bytes64 of each
    node's row read through its alias slot, computed on the GPU."""
    alias = np.ascontiguousarray(alias, np.int64)
    if len(alias) != len(batch.nodes):
        raise InvalidArgument("trainer_step: alias list length != batch nodes")
    if len(alias) and alias.min() < 0:
        raise InvariantViolation("trainer saw an unassigned alias")
    ad = DeviceBuffer.from_array(alias) if len(alias) else DeviceBuffer(8)
    cs = DeviceBuffer(8)
    cs.zero()
    check(lib().fdg_checksum_alias(buffer.topo.ctx, None, buffer.region_ptr, ad.ptr, None, len(alias), cs.ptr))
    check(lib().fdg_device_sync())
    return int(cs.download(np.uint64)[0])


# -------------------------------------------------------------- train stage --
class GraphSAGE:
    """The train stage behind fdg_sage_* (include/fdg.h): GraphSAGE forward + loss over a
    sampled batch's blocks, fed from the mini-batch tensor X. The reference's trainer is
    the checksum above (pipeline.hpp:103-124); the paper's model is a 3-layer GraphSAGE,
    hidden 256. Layer k computes local nodes [0, D_{L-k}),
    D_j = layer_nodes[j+1]: h_v = W_neigh . mean_{u->v} h_u + W_self . h_v + b (ReLU
    between layers); loss = mean softmax cross-entropy over the unique seeds with
    label(v) = splitmix64(v ^ label_seed) % dims[-1]. fp32 on the GPU."""

    def __init__(self, topo: Topology, dims, fanouts, max_seeds: int = 1000, seed: int = 0, weights=None):
        self.topo = topo
        self.dims = [int(d) for d in dims]
        fan = list(fanouts.per_layer if isinstance(fanouts, Fanouts) else fanouts)
        if len(fan) != len(self.dims) - 1:
            raise InvalidArgument("GraphSAGE: one layer per sampling hop (len(dims) == len(fanouts) + 1)")
        d = np.ascontiguousarray(self.dims, np.uint32)
        f = np.ascontiguousarray(fan, np.uint32)
        p = C.c_void_p()
        check(lib().fdg_sage_create(topo.ctx, _p(d), len(f), _p(f), max_seeds, C.byref(p)))
        self.ptr = p.value
        self.weights = weights if weights is not None else GraphSAGE.init_weights(self.dims, seed)
        for layer, (wn, ws, b) in enumerate(self.weights):
            wn, ws, b = (np.ascontiguousarray(a, np.float32) for a in (wn, ws, b))
            check(lib().fdg_sage_set_layer(self.ptr, layer, _p(wn), _p(ws), _p(b)))

    @staticmethod
    def init_weights(dims, seed: int = 0):
        """Glorot-uniform W_neigh / W_self ([d_in, d_out], input-major) and small biases."""
        rng = np.random.default_rng(seed)
        out = []
        for din, dout in zip(dims[:-1], dims[1:]):
            a = np.sqrt(6.0 / (din + dout))
            out.append((rng.uniform(-a, a, (din, dout)).astype(np.float32),
                        rng.uniform(-a, a, (din, dout)).astype(np.float32),
                        rng.uniform(-0.1, 0.1, dout).astype(np.float32)))
        return out

    def forward_async(self, stream, x_ptr: int, nodes_ptr: int, edges_ptr: int, counts_ptr: int, label_seed: int,
                      loss_ptr: int, logits_ptr: int | None = None):
        check(lib().fdg_sage_forward(self.ptr, stream.ptr if stream else None, x_ptr, nodes_ptr, edges_ptr,
                                     counts_ptr, label_seed, loss_ptr, logits_ptr))

    def _upload(self, batch: SampledBatch):
        """Device copies of a host batch: nodes, edges, the batch record and X (gathered)."""
        n, e = len(batch.nodes), len(batch.edges)
        cnt = _lib.BatchCounts()
        cnt.n_nodes, cnt.n_edges, cnt.n_layers = n, e, len(batch.layer_nodes) - 2
        for i, v in enumerate(batch.layer_nodes):
            cnt.layer_nodes[i] = int(v)
        for i, v in enumerate(batch.layer_edges):
            cnt.layer_edges[i] = int(v)
        cd = DeviceBuffer(C.sizeof(cnt))
        check(lib().fdg_memcpy_h2d(cd.ptr, C.addressof(cnt), C.sizeof(cnt), None))
        nd = DeviceBuffer.from_array(batch.nodes) if n else DeviceBuffer(8)
        ed = DeviceBuffer.from_array(np.ascontiguousarray(batch.edges, np.uint32)) if e else DeviceBuffer(8)
        x = DeviceBuffer(max(n, 1) * self.topo.row_bytes)
        if n:
            check(lib().fdg_gather(self.topo.ctx, None, nd.ptr, None, n, x.ptr, None))
        return nd, ed, cd, x

    def forward(self, batch: SampledBatch, label_seed: int = 0):
        """Host convenience: X gathered on the device from the batch's nodes, then the
        forward; returns (loss, logits of the unique seeds)."""
        nd, ed, cd, x = self._upload(batch)
        loss = DeviceBuffer(4)
        seeds = int(max(batch.layer_nodes[:2])) if len(batch.layer_nodes) > 1 else 0
        logits = DeviceBuffer(max(seeds, 1) * self.dims[-1] * 4)
        self.forward_async(None, x.ptr, nd.ptr, ed.ptr, cd.ptr, label_seed, loss.ptr, logits.ptr)
        check(lib().fdg_device_sync())
        return (float(loss.download(np.float32)[0]),
                logits.download(np.float32, seeds * self.dims[-1]).reshape(seeds, self.dims[-1]))

    def train_step(self, batch: SampledBatch, label_seed: int = 0, lr: float = 0.0, allreduce=None) -> float:
        """forward + backward (+ allreduce(grads) for data parallelism) + SGD; returns the
        pre-update loss. lr = 0 leaves the weights unchanged (gradients only)."""
        nd, ed, cd, x = self._upload(batch)
        loss = DeviceBuffer(4)
        self.forward_async(None, x.ptr, nd.ptr, ed.ptr, cd.ptr, label_seed, loss.ptr, None)
        check(lib().fdg_sage_backward(self.ptr, None, nd.ptr, ed.ptr, cd.ptr, label_seed))
        if allreduce is not None:
            check(lib().fdg_device_sync())
            allreduce(self)
        if lr:
            check(lib().fdg_sage_sgd(self.ptr, None, lr))
        check(lib().fdg_device_sync())
        return float(loss.download(np.float32)[0])

    def sgd(self, lr: float):
        check(lib().fdg_sage_sgd(self.ptr, None, lr))
        check(lib().fdg_device_sync())

    def layer(self, layer: int, grads: bool = False):
        """(W_neigh, W_self, b) of a layer -- or their gradients from the last backward."""
        din, dout = self.dims[layer], self.dims[layer + 1]
        wn, ws, b = np.empty((din, dout), np.float32), np.empty((din, dout), np.float32), np.empty(dout, np.float32)
        check(lib().fdg_sage_get_layer(self.ptr, layer, 1 if grads else 0, _p(wn), _p(ws), _p(b)))
        return wn, ws, b

    def buffers(self):
        """(params_dev_ptr, grads_dev_ptr, n_floats): the contiguous parameter / gradient blocks."""
        pp, gp, n = C.c_void_p(), C.c_void_p(), C.c_uint64()
        check(lib().fdg_sage_buffers(self.ptr, C.byref(pp), C.byref(gp), C.byref(n)))
        return pp.value, gp.value, n.value

    def close(self):
        if getattr(self, "ptr", None):
            lib().fdg_sage_destroy(self.ptr)
            self.ptr = None

    __del__ = close
