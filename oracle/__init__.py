"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

* ``port``  -- oracle/libfdoracle.so, the plain-C restatement (fd_oracle.c).
* ``ref``   -- oracle/_ref/libfdref.so, the unmodified reference headers
  (/root/reference/proj/include/featdrive) compiled behind a C driver
  (ref_driver.cpp). Present wherever `make -C oracle ref` ran (this container;
  the built .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline legs may
import this package; the product (paper_2406_13984_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "libfdoracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libfdref.so")

u64, u32, i64, vp = C.c_uint64, C.c_uint32, C.c_int64, C.c_void_p


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build(ref: bool = True) -> None:
    import subprocess
    targets = ["liboracle"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/include") else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


# ----------------------------------------------------------------- the port --
class Port:
    def __init__(self, path: str = PORT_PATH):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.fdo_splitmix64.restype = u64; L.fdo_splitmix64.argtypes = [u64]
        L.fdo_hash_combine.restype = u64; L.fdo_hash_combine.argtypes = [u64, u64]
        L.fdo_hash_bytes64.restype = u64; L.fdo_hash_bytes64.argtypes = [vp, C.c_size_t]
        L.fdo_batch_seed.restype = u64; L.fdo_batch_seed.argtypes = [u64, u64, u64]
        L.fdo_mt_stream.argtypes = [u64, u64, vp]
        L.fdo_uniform_0_j.restype = u64; L.fdo_uniform_0_j.argtypes = [vp, u64, vp, u64]
        L.fdo_synthetic_row.argtypes = [u64, u64, u32, vp]
        L.fdo_synthetic_in_degree.restype = u64
        L.fdo_synthetic_in_degree.argtypes = [u64, u64, u32, u64]
        L.fdo_synthetic_in_neighbors.restype = u64
        L.fdo_synthetic_in_neighbors.argtypes = [u64, u64, u32, u64, vp]
        L.fdo_generate_indptr.argtypes = [u64, u64, u32, vp]
        L.fdo_generate_indices.argtypes = [u64, u64, u32, vp, vp]
        L.fdo_sample_khop.restype = C.c_int
        L.fdo_sample_khop.argtypes = [vp, vp, C.c_int, u64, vp, u64, vp, u32, u64, vp, u64,
                                      vp, u64, vp, u64, vp, vp, vp, vp, vp, vp]
        L.fdo_max_batch_nodes.restype = u64; L.fdo_max_batch_nodes.argtypes = [vp, u32, u64]
        L.fdo_bm_create.restype = vp; L.fdo_bm_create.argtypes = [u64, u64, u64]
        L.fdo_bm_destroy.argtypes = [vp]
        L.fdo_bm_extract.restype = C.c_int; L.fdo_bm_extract.argtypes = [vp, vp, u64, vp, vp, vp]
        L.fdo_bm_release.restype = C.c_int; L.fdo_bm_release.argtypes = [vp, vp, u64]
        L.fdo_bm_stats.argtypes = [vp, vp]
        L.fdo_bm_entry.argtypes = [vp, u64, vp, vp, vp]
        L.fdo_bm_reverse.restype = i64; L.fdo_bm_reverse.argtypes = [vp, u64]
        L.fdo_bm_standby.restype = u64; L.fdo_bm_standby.argtypes = [vp, vp, u64]
        L.fdo_gather.restype = u64; L.fdo_gather.argtypes = [vp, u32, vp, u64, vp]
        L.fdo_checksum_rows.restype = u64; L.fdo_checksum_rows.argtypes = [vp, u32, u64]

    # scalar helpers
    def splitmix64(self, x): return self.lib.fdo_splitmix64(x)
    def hash_combine(self, a, b): return self.lib.fdo_hash_combine(a, b)
    def batch_seed(self, s, e, b): return self.lib.fdo_batch_seed(s, e, b)

    def hash_bytes64(self, data: bytes | np.ndarray) -> int:
        a = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        a = np.ascontiguousarray(a)
        return self.lib.fdo_hash_bytes64(_p(a), a.nbytes)

    def mt_stream(self, rng_seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.fdo_mt_stream(rng_seed, n, _p(out))
        return out

    def synthetic_row(self, seed, node, dim) -> np.ndarray:
        out = np.empty(dim + 1, np.float32)
        self.lib.fdo_synthetic_row(seed, node, dim, _p(out))
        return out[:dim]

    def synthetic_in_degree(self, seed, node, avg, n):
        return self.lib.fdo_synthetic_in_degree(seed, node, avg, n)

    def synthetic_in_neighbors(self, seed, node, avg, n) -> np.ndarray:
        out = np.empty(max(4 * avg, 1) + 1, np.uint64)
        d = self.lib.fdo_synthetic_in_neighbors(seed, node, avg, n, _p(out))
        return out[:d].copy()

    def generate_topology(self, seed, n, avg):
        indptr = np.empty(n + 1, np.uint64)
        self.lib.fdo_generate_indptr(seed, n, avg, _p(indptr))
        indices = np.empty(int(indptr[-1]), np.uint64)
        self.lib.fdo_generate_indices(seed, n, avg, _p(indptr), _p(indices))
        return indptr, indices

    def generate_features(self, seed, n, dim) -> np.ndarray:
        out = np.empty((n, dim + (dim & 1)), np.float32)
        for v in range(n):
            self.lib.fdo_synthetic_row(seed, v, dim, _p(out[v]))
        return np.ascontiguousarray(out[:, :dim])

    def max_batch_nodes(self, fanouts, b):
        f = np.asarray(fanouts, np.uint32)
        return self.lib.fdo_max_batch_nodes(_p(f), len(f), b)

    def sample_khop(self, indptr, indices, seeds, fanouts, rng_seed, words=None):
        """Returns dict(nodes, edges[E,2], layer_nodes, layer_edges, words_used) or raises OracleError."""
        indptr = np.ascontiguousarray(indptr, np.uint64)
        assert indices.dtype in (np.uint32, np.uint64)
        seeds = np.ascontiguousarray(seeds, np.uint64)
        f = np.ascontiguousarray(fanouts, np.uint32)
        n = len(indptr) - 1
        cap = self.max_batch_nodes(f, max(len(seeds), 1)) + 1
        ecap = cap
        nodes = np.empty(cap, np.uint64)
        edges = np.empty((ecap, 2), np.uint32)
        nn, ne, wu, bad = (np.zeros(1, np.uint64) for _ in range(4))
        ln = np.zeros(len(f) + 2, np.uint64)
        le = np.zeros(len(f) + 1, np.uint64)
        w = None if words is None else np.ascontiguousarray(words, np.uint64)
        rc = self.lib.fdo_sample_khop(_p(indptr), _p(indices), indices.dtype.itemsize, n,
                                      _p(seeds), len(seeds), _p(f), len(f), rng_seed,
                                      _p(w), 0 if w is None else len(w),
                                      _p(nodes), cap, _p(edges), ecap, _p(nn), _p(ne), _p(ln), _p(le),
                                      _p(wu), _p(bad))
        if rc != 0:
            raise OracleError(rc, f"bad_seed={int(bad[0])}")
        return dict(nodes=nodes[: int(nn[0])].copy(), edges=edges[: int(ne[0])].copy(),
                    layer_nodes=ln, layer_edges=le, words_used=int(wu[0]))

    def gather(self, table: np.ndarray, nodes: np.ndarray):
        table = np.ascontiguousarray(table)
        rb = table.shape[1] * table.itemsize
        nodes = np.ascontiguousarray(nodes, np.uint64)
        out = np.empty((len(nodes), table.shape[1]), table.dtype)
        s = self.lib.fdo_gather(_p(table), rb, _p(nodes), len(nodes), _p(out))
        return out, s

    def checksum_rows(self, rows: np.ndarray) -> int:
        rows = np.ascontiguousarray(rows)
        rb = rows.shape[1] * rows.itemsize
        return self.lib.fdo_checksum_rows(_p(rows), rb, rows.shape[0])


class PortBufferManager:
    """fd_oracle.c restatement of featbuf::BufferManager (sequential schedule)."""

    def __init__(self, port: Port, num_nodes, slots, min_reserved=0):
        self.L = port.lib
        self.h = self.L.fdo_bm_create(num_nodes, slots, min_reserved)
        if not self.h:
            raise OracleError(3, "bad buffer config")

    def extract(self, nodes):
        nodes = np.ascontiguousarray(nodes, np.uint64)
        alias = np.empty(len(nodes), np.int64)
        lp = np.empty(max(len(nodes), 1), np.uint32)
        nl = np.zeros(1, np.uint64)
        rc = self.L.fdo_bm_extract(self.h, _p(nodes), len(nodes), _p(alias), _p(lp), _p(nl))
        if rc:
            raise OracleError(rc)
        return alias, lp[: int(nl[0])].copy()

    def release(self, nodes):
        nodes = np.ascontiguousarray(nodes, np.uint64)
        rc = self.L.fdo_bm_release(self.h, _p(nodes), len(nodes))
        if rc:
            raise OracleError(rc)

    def stats(self):
        out = np.zeros(7, np.uint64)
        self.L.fdo_bm_stats(self.h, _p(out))
        return out

    def standby(self, cap):
        out = np.empty(cap, np.int64)
        n = self.L.fdo_bm_standby(self.h, _p(out), cap)
        return out[:n].copy()

    def entry(self, node):
        s, r, v = np.zeros(1, np.int64), np.zeros(1, np.uint32), np.zeros(1, np.uint32)
        self.L.fdo_bm_entry(self.h, node, _p(s), _p(r), _p(v))
        return int(s[0]), int(r[0]), int(v[0])

    def reverse(self, slot):
        return self.L.fdo_bm_reverse(self.h, slot)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.fdo_bm_destroy(self.h)
            self.h = None


# ------------------------------------------------------------ the reference --
def ref_available() -> bool:
    return os.path.exists(REF_PATH)


class Ref:
    def __init__(self, path: str = REF_PATH):
        L = self.lib = C.CDLL(path)
        L.fdref_last_error.restype = C.c_char_p
        L.fdref_last_error_kind.restype = C.c_int
        L.fdref_last_errno.restype = C.c_int
        L.fdref_feature_table_check.restype = C.c_int; L.fdref_feature_table_check.argtypes = [C.c_char_p]
        L.fdref_splitmix64.restype = u64; L.fdref_splitmix64.argtypes = [u64]
        L.fdref_hash_combine.restype = u64; L.fdref_hash_combine.argtypes = [u64, u64]
        L.fdref_hash_bytes64.restype = u64; L.fdref_hash_bytes64.argtypes = [vp, u64]
        L.fdref_batch_seed.restype = u64; L.fdref_batch_seed.argtypes = [u64, u64, u64]
        L.fdref_mt_stream.argtypes = [u64, u64, vp]
        L.fdref_uniform_seq.argtypes = [u64, vp, u64, vp]
        L.fdref_synthetic_row.argtypes = [u64, u64, u32, vp]
        L.fdref_synthetic_in_degree.restype = u64
        L.fdref_synthetic_in_degree.argtypes = [u64, u64, u32, u64]
        L.fdref_synthetic_in_neighbors.restype = u64
        L.fdref_synthetic_in_neighbors.argtypes = [u64, u64, u32, u64, vp]
        L.fdref_generate_dataset.restype = C.c_int
        L.fdref_generate_dataset.argtypes = [C.c_char_p, u64, u32, u32, u64, vp]
        L.fdref_topology_open.restype = vp; L.fdref_topology_open.argtypes = [C.c_char_p]
        L.fdref_topology_close.argtypes = [vp]
        L.fdref_topology_num_nodes.restype = u64; L.fdref_topology_num_nodes.argtypes = [vp]
        L.fdref_sample_khop.restype = C.c_int
        L.fdref_sample_khop.argtypes = [vp, vp, u64, vp, u32, u64, vp, u64, vp, u64, vp, vp]
        L.fdref_partition_epoch.restype = C.c_int
        L.fdref_partition_epoch.argtypes = [vp, u64, u64, u64, vp]
        L.fdref_bm_create.restype = vp; L.fdref_bm_create.argtypes = [u64, u64, u64, C.c_int]
        L.fdref_bm_destroy.argtypes = [vp]
        L.fdref_bm_extract.restype = C.c_int; L.fdref_bm_extract.argtypes = [vp, vp, u64, vp]
        L.fdref_bm_release.restype = C.c_int; L.fdref_bm_release.argtypes = [vp, vp, u64]
        L.fdref_bm_stats.argtypes = [vp, vp]
        L.fdref_bm_entry.argtypes = [vp, u64, vp, vp, vp]
        L.fdref_bm_reverse.restype = i64; L.fdref_bm_reverse.argtypes = [vp, u64]
        L.fdref_bm_standby_mru.restype = i64; L.fdref_bm_standby_mru.argtypes = [vp]
        L.fdref_bm_validate.restype = C.c_int; L.fdref_bm_validate.argtypes = [vp]
        L.fdref_extractor_open.restype = vp
        L.fdref_extractor_open.argtypes = [C.c_char_p, u64, u64, C.c_int]
        L.fdref_extractor_close.argtypes = [vp]
        L.fdref_extractor_extract.restype = C.c_int
        L.fdref_extractor_extract.argtypes = [vp, vp, u64, vp, vp, vp]
        L.fdref_extractor_release.restype = C.c_int
        L.fdref_extractor_release.argtypes = [vp, vp, u64]
        L.fdref_extractor_stats.argtypes = [vp, vp]
        L.fdref_run_epoch.restype = i64
        L.fdref_run_epoch.argtypes = [C.c_char_p, vp, u64, u64, u64, u64, vp, u32, C.c_int, u32, u32,
                                      vp, u64, vp]
        L.fdref_gen_indptr.argtypes = [u64, u64, u32, u32, vp]
        L.fdref_gen_indices.argtypes = [u64, u64, u32, u32, vp, vp]
        L.fdref_gen_features.argtypes = [u64, u64, u32, u32, vp]
        L.fdref_bench_sample_extract.restype = C.c_double
        L.fdref_bench_sample_extract.argtypes = [vp, vp, u32, vp, u64, u64, vp, u32, u64, u64, u64, u32,
                                                 vp, vp]
        L.fdref_bench_sample_extract_bm.restype = C.c_double
        L.fdref_bench_sample_extract_bm.argtypes = [vp, vp, u32, vp, u64, u64, vp, u32, u64, u64, u64, u32,
                                                    vp, vp, vp, vp]

    def err(self):
        return self.lib.fdref_last_error().decode()

    def err_kind(self):
        """(category, errno) of the last recorded reference exception: 1 std::system_error,
        2 std::runtime_error, 3 invalid_argument, 4 out_of_range, 5 logic_error, 9 other."""
        return int(self.lib.fdref_last_error_kind()), int(self.lib.fdref_last_errno())

    def open_topology(self, dataset_dir):
        """graph::Topology(dataset_dir): None on success, else (message, category, errno)."""
        h = self.lib.fdref_topology_open(dataset_dir.encode())
        if h:
            self.lib.fdref_topology_close(h)
            return None
        return (self.err(),) + self.err_kind()

    def open_feature_table(self, path):
        """storage::FeatureTable(path): None on success, else (message, category, errno)."""
        if self.lib.fdref_feature_table_check(path.encode()) == 0:
            return None
        return (self.err(),) + self.err_kind()

    def check(self, rc):
        if rc:
            raise OracleError(rc, self.err())

    def splitmix64(self, x): return self.lib.fdref_splitmix64(x)
    def hash_combine(self, a, b): return self.lib.fdref_hash_combine(a, b)
    def batch_seed(self, s, e, b): return self.lib.fdref_batch_seed(s, e, b)

    def hash_bytes64(self, data) -> int:
        a = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else data)
        return self.lib.fdref_hash_bytes64(_p(a), a.nbytes)

    def mt_stream(self, rng_seed, n):
        out = np.empty(n, np.uint64)
        self.lib.fdref_mt_stream(rng_seed, n, _p(out))
        return out

    def uniform_seq(self, rng_seed, js):
        js = np.ascontiguousarray(js, np.uint64)
        out = np.empty(len(js), np.uint64)
        self.lib.fdref_uniform_seq(rng_seed, _p(js), len(js), _p(out))
        return out

    def synthetic_row(self, seed, node, dim):
        out = np.empty(dim, np.float32)
        self.lib.fdref_synthetic_row(seed, node, dim, _p(out))
        return out

    def synthetic_in_degree(self, seed, node, avg, n):
        return self.lib.fdref_synthetic_in_degree(seed, node, avg, n)

    def synthetic_in_neighbors(self, seed, node, avg, n):
        out = np.empty(max(4 * avg, 1) + 1, np.uint64)
        d = self.lib.fdref_synthetic_in_neighbors(seed, node, avg, n, _p(out))
        return out[:d].copy()

    def generate_dataset(self, out_dir, num_nodes, dim, avg, seed):
        ne = np.zeros(1, np.uint64)
        self.check(self.lib.fdref_generate_dataset(out_dir.encode(), num_nodes, dim, avg, seed, _p(ne)))
        return int(ne[0])

    def stage_dataset(self, out_dir, num_nodes, dim, avg, seed, threads, features=True):
        """Reference generator run multi-threaded straight into indptr.bin / indices.bin
        under out_dir (a tmpfs such as /dev/shm keeps it in RAM). Returns (features
        array in host memory or None, num_edges). The feature file itself is not
        written: the CPU baseline extracts from host memory (SSD staging is out of scope)."""
        os.makedirs(out_dir, exist_ok=True)
        indptr = np.lib.format.open_memmap(os.path.join(out_dir, "indptr.npy"), mode="w+", dtype=np.uint64,
                                           shape=(num_nodes + 1,))
        self.lib.fdref_gen_indptr(seed, num_nodes, avg, threads, _p(indptr))
        ne = int(indptr[-1])
        indptr.tofile(os.path.join(out_dir, "indptr.bin"))
        del indptr
        os.remove(os.path.join(out_dir, "indptr.npy"))
        ip = np.fromfile(os.path.join(out_dir, "indptr.bin"), np.uint64)
        indices = np.memmap(os.path.join(out_dir, "indices.bin"), mode="w+", dtype=np.uint64, shape=(max(ne, 1),))
        self.lib.fdref_gen_indices(seed, num_nodes, avg, threads, _p(ip), _p(indices))
        indices.flush()
        del indices
        if ne == 0:
            open(os.path.join(out_dir, "indices.bin"), "wb").close()
        feats = None
        if features:
            feats = np.empty((num_nodes, dim), np.float32)
            self.lib.fdref_gen_features(seed, num_nodes, dim, threads, _p(feats))
        return feats, ne

    def bench_sample_extract(self, topo, table, seeds, n_batches, batch_size, fanouts, seed, epoch, first_batch,
                             threads):
        table = np.ascontiguousarray(table)
        rb = table.shape[1] * table.itemsize
        seeds = np.ascontiguousarray(seeds, np.uint64)
        f = np.ascontiguousarray(fanouts, np.uint32)
        cs = np.zeros(n_batches, np.uint64)
        nc = np.zeros(n_batches, np.uint64)
        secs = self.lib.fdref_bench_sample_extract(topo.h, _p(table), rb, _p(seeds), n_batches, batch_size, _p(f),
                                                   len(f), seed, epoch, first_batch, threads, _p(cs), _p(nc))
        if secs < 0:
            raise OracleError(9, self.err())
        return secs, cs, nc

    def bench_sample_extract_bm(self, topo, table, seeds, n_batches, batch_size, fanouts, seed, epoch, first_batch,
                                threads, bm, region):
        """Config 3: sampling on threads - 1 workers, extraction in batch order through the
        reference BufferManager `bm` (fdref_bm_create) into `region` (slots x row bytes)."""
        table = np.ascontiguousarray(table)
        rb = table.shape[1] * table.itemsize
        seeds = np.ascontiguousarray(seeds, np.uint64)
        f = np.ascontiguousarray(fanouts, np.uint32)
        cs = np.zeros(n_batches, np.uint64)
        nc = np.zeros(n_batches, np.uint64)
        secs = self.lib.fdref_bench_sample_extract_bm(topo.h, _p(table), rb, _p(seeds), n_batches, batch_size,
                                                      _p(f), len(f), seed, epoch, first_batch, threads, bm,
                                                      _p(region), _p(cs), _p(nc))
        if secs < 0:
            raise OracleError(9, self.err())
        return secs, cs, nc

    def partition_epoch(self, ids, batch, shuffle_seed):
        ids = np.ascontiguousarray(ids, np.uint64)
        out = np.empty_like(ids)
        self.check(self.lib.fdref_partition_epoch(_p(ids), len(ids), batch, shuffle_seed, _p(out)))
        return out

    def run_epoch(self, dataset_dir, train_ids, epoch, seed, batch, fanouts, sync=True, samplers=2,
                  extractors=2):
        ids = np.ascontiguousarray(train_ids, np.uint64)
        f = np.ascontiguousarray(fanouts, np.uint32)
        cap = (len(ids) + batch - 1) // batch
        out = np.zeros((cap, 4), np.uint64)
        bs = np.zeros(4, np.uint64)
        k = self.lib.fdref_run_epoch(dataset_dir.encode(), _p(ids), len(ids), epoch, seed, batch, _p(f), len(f),
                                     1 if sync else 0, samplers, extractors, _p(out), cap, _p(bs))
        if k < 0:
            raise OracleError(9, self.err())
        recs = out[:k]
        return recs[np.argsort(recs[:, 0], kind="stable")], bs


class RefTopology:
    def __init__(self, ref: Ref, dataset_dir: str):
        self.ref = ref
        self.h = ref.lib.fdref_topology_open(dataset_dir.encode())
        if not self.h:
            raise OracleError(9, ref.err())

    @property
    def num_nodes(self):
        return self.ref.lib.fdref_topology_num_nodes(self.h)

    def sample_khop(self, seeds, fanouts, rng_seed, cap=None):
        seeds = np.ascontiguousarray(seeds, np.uint64)
        f = np.ascontiguousarray(fanouts, np.uint32)
        if cap is None:
            cap = Port().max_batch_nodes(f, max(len(seeds), 1)) + 1
        nodes = np.empty(cap, np.uint64)
        edges = np.empty((cap, 2), np.uint32)
        nn, ne = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        self.ref.check(self.ref.lib.fdref_sample_khop(self.h, _p(seeds), len(seeds), _p(f), len(f), rng_seed,
                                                      _p(nodes), cap, _p(edges), cap, _p(nn), _p(ne)))
        return dict(nodes=nodes[: int(nn[0])].copy(), edges=edges[: int(ne[0])].copy())

    def close(self):
        if self.h:
            self.ref.lib.fdref_topology_close(self.h)
            self.h = None

    __del__ = close


class RefBufferManager:
    def __init__(self, ref: Ref, num_nodes, slots, min_reserved=0, mapping=0):
        self.ref = ref
        self.h = ref.lib.fdref_bm_create(num_nodes, slots, min_reserved, mapping)
        if not self.h:
            raise OracleError(3, ref.err())

    def extract(self, nodes):
        nodes = np.ascontiguousarray(nodes, np.uint64)
        alias = np.empty(len(nodes), np.int64)
        self.ref.check(self.ref.lib.fdref_bm_extract(self.h, _p(nodes), len(nodes), _p(alias)))
        return alias

    def release(self, nodes):
        nodes = np.ascontiguousarray(nodes, np.uint64)
        self.ref.check(self.ref.lib.fdref_bm_release(self.h, _p(nodes), len(nodes)))

    def stats(self):
        out = np.zeros(7, np.uint64)
        self.ref.lib.fdref_bm_stats(self.h, _p(out))
        return out

    def entry(self, node):
        s, r, v = np.zeros(1, np.int64), np.zeros(1, np.uint32), np.zeros(1, np.uint32)
        self.ref.lib.fdref_bm_entry(self.h, node, _p(s), _p(r), _p(v))
        return int(s[0]), int(r[0]), int(v[0])

    def reverse(self, slot):
        return self.ref.lib.fdref_bm_reverse(self.h, slot)

    def validate(self):
        self.ref.check(self.ref.lib.fdref_bm_validate(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.fdref_bm_destroy(self.h)
            self.h = None


class RefExtractor:
    """The reference's real extract::Extractor over an on-disk dataset."""

    def __init__(self, ref: Ref, dataset_dir, slots, min_reserved=0, mapping=0):
        self.ref = ref
        self.h = ref.lib.fdref_extractor_open(dataset_dir.encode(), slots, min_reserved, mapping)
        if not self.h:
            raise OracleError(9, ref.err())

    def extract(self, nodes, row_bytes):
        nodes = np.ascontiguousarray(nodes, np.uint64)
        alias = np.empty(len(nodes), np.int64)
        rows = np.empty((len(nodes), row_bytes), np.uint8)
        cs = np.zeros(1, np.uint64)
        self.ref.check(self.ref.lib.fdref_extractor_extract(self.h, _p(nodes), len(nodes), _p(alias), _p(rows),
                                                            _p(cs)))
        return alias, rows, int(cs[0])

    def release(self, nodes):
        nodes = np.ascontiguousarray(nodes, np.uint64)
        self.ref.check(self.ref.lib.fdref_extractor_release(self.h, _p(nodes), len(nodes)))

    def stats(self):
        out = np.zeros(7, np.uint64)
        self.ref.lib.fdref_extractor_stats(self.h, _p(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.fdref_extractor_close(self.h)
            self.h = None
