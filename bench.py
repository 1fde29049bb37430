#!/usr/bin/env python3
"""Benchmark: GNNDrive sample -> extract mini-batches/s on B200 (+ gather GB/s vs HBM).

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--config papers|products|friendster|papers_bm] [--impl ours|reference]

A step is one mini-batch through the hot path: graph::sample_khop (3-hop CSR
neighbour sampling + first-occurrence dedup/reindex, bit-exact) followed by
feature extraction into the mini-batch tensor X (an HBM gather; with
--config papers_bm through the GPU feature-buffer manager at a 10 % cap). The
native runner (fdg_pipeline_run, the PipelineSession counterpart) pipelines the
batches: MT19937-64 streams are generated ahead, two sampler workspaces sample
batches j+1, j+2 while batch j is extracted.

Workload (default, BASELINE.json configs[1]): synthetic Papers100M-shaped graph
(111,059,956 nodes, 1,613,492,860 edges, 128-dim f32 rows) built bit-exactly in
HBM by the GPU port of the reference generator (seed 7), fanout (10,10,10),
batch 1000, train ids 0..999,999, epoch-0 partition (partition_epoch) and
per-batch rng seeds batch_seed(0, 0, b) -- exactly the reference pipeline's keying.

--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from the /root/reference headers): sample_khop + row extraction + the
trainer checksum, one batch per host thread, on the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (num_nodes, dim, avg_degree, fanouts, batch, train_ids, dtype, buffer_fraction)
    "products": (2_449_029, 100, 28, [10, 10, 10], 1000, 196_000, "f32", None),
    "papers": (111_059_956, 128, 16, [10, 10, 10], 1000, 1_000_000, "f32", None),
    "papers_bm": (111_059_956, 128, 16, [10, 10, 10], 1000, 1_000_000, "f32", 0.10),
    "friendster": (65_608_366, 256, 30, [15, 10, 5], 1000, 1_000_000, "f32", None),
    # config 4: 768-dim fp16 table (375 GB) only fits row-sharded over >= 3 GPUs (--shard)
    "mag": (244_160_499, 768, 8, [10, 10, 10], 1000, 1_000_000, "f16", None),
    # out-of-core tier: table in pinned host memory, GPU feature buffer (10 %) in front of it
    "products_host_bm": (2_449_029, 100, 28, [10, 10, 10], 1000, 196_000, "f32", 0.80),
    "papers_host_bm": (111_059_956, 128, 16, [10, 10, 10], 1000, 1_000_000, "f32", 0.10),
}
HOST_TIER = {"products_host_bm", "papers_host_bm"}
DESCR = {
    "products": "synthetic ogbn-products-shaped graph (2,449,029 nodes, 100-dim f32), fanout (10,10,10), batch 1000",
    "papers": "synthetic Papers100M-shaped graph (111,059,956 nodes, 1,613,492,860 edges, 128-dim f32), "
              "fanout (10,10,10), batch 1000",
    "papers_bm": "Papers100M-shaped graph, feature buffer capped at 10% of the table (11,105,995 slots)",
    "friendster": "synthetic Friendster-shaped graph (65,608,366 nodes, 256-dim f32), fanout (15,10,5), batch 1000",
    "mag": "synthetic MAG240M-shaped graph (244,160,499 nodes, 1,720,983,565 edges, 768-dim fp16), feature "
           "table row-sharded over the GPUs, remote rows read over NVLink P2P",
    "products_host_bm": "ogbn-products shape, feature table in pinned host memory (out-of-core tier), GPU feature "
                        "buffer at 80% (1,959,223 slots: two live batches of ~875 k nodes must fit)",
    "papers_host_bm": "Papers100M shape, feature table in pinned host memory (out-of-core tier), GPU feature buffer "
                      "at 10% (11,105,995 slots)",
}
GEN_SEED = 7
METRIC = "sample+extract mini-batches/sec (Papers100M-shape); gather GB/s vs HBM peak"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def hash_combine(a, b):
    """common.hpp:77-86 in Python integers (the epoch shuffle seed)."""
    M = (1 << 64) - 1

    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    return sm(a ^ ((b + 0x9E3779B97F4A7C15 + (a << 6) + (a >> 2)) & M))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of the SM clock + clock-event reasons during the timed region."""

    REASONS = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("clock sampling unavailable:", e)
            self.nv, self.max_mhz = None, None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons.update(name for bit, name in self.REASONS.items() if r & bit)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop_ev.set()
        if self.nv:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


class Dist:
    """One process per GPU (torchrun env); gloo for the barrier and max-over-ranks."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def reduce(self, x: float, op: str) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def gather(self, x: float) -> list:
        """x of every rank, in rank order."""
        if self.world == 1:
            return [x]
        import torch
        t = torch.zeros(self.world, dtype=torch.float64)
        t[self.rank] = x
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return [float(v) for v in t.tolist()]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def segment(total: int, world: int, rank: int):
    """Contiguous chunk ranges per worker, sizes differing by at most one (pipeline.hpp:192-203)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def counts_dtype():
    from paper_2406_13984_b200._lib import MAX_LAYERS
    return np.dtype([("status", "<u4"), ("n_nodes", "<u4"), ("n_edges", "<u4"), ("rejections", "<u4"),
                     ("bad_seed", "<u8"), ("checksum", "<u8"), ("bad_seed_pos", "<u4"), ("n_layers", "<u4"),
                     ("layer_nodes", "<u4", (MAX_LAYERS + 2,)), ("layer_edges", "<u4", (MAX_LAYERS + 1,)),
                     ("layer_draws", "<u4", (MAX_LAYERS + 1,)), ("words_used", "<u4"), ("replays", "<u4")])


EDGES = {"products": 63_177_558, "papers": 1_613_492_860, "papers_bm": 1_613_492_860, "friendster": 1_813_633_279,
         "mag": 1_720_983_565, "products_host_bm": 63_177_558, "papers_host_bm": 1_613_492_860}


def bench_config(cfg, world, layout):
    """The workload description both arms print as `config` (identical for the same
    --config / --gpus): what is computed, not how (that goes under "execution")."""
    n, dim, avg, fan, B, t_ids, dtype, frac = CONFIGS[cfg]
    rb = dim * (4 if dtype == "f32" else 2)
    return {"workload": DESCR[cfg], "config": cfg, "nodes": n, "edges": EDGES[cfg], "row_bytes": rb,
            "fanouts": fan, "batch": B, "global_batch": B * world, "train_ids": t_ids,
            "parallelism": f"dp{world}" + ({"sharded": " (replicated CSR, feature table row-sharded, remote rows "
                                                       "over NVLink P2P)",
                                            "replicas": " (replicated CSR + table)",
                                            "local": ""}[layout]),
            "l2_policy": "inputs > L2 (the table and ~0.5 GB of X per batch); no flush",
            "table_tier": "pinned host memory (mapped)" if cfg in HOST_TIER else "HBM",
            "buffer_slots": int(n * frac) if frac else None}


def host_cpu():
    """nproc and the lscpu model name of this host."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


# ------------------------------------------------------------ reference (CPU) ----
def stage_reference_dataset(cfg, threads):
    """The reference generator (oracle/_ref), multi-threaded, into /dev/shm + host RAM."""
    import oracle
    n, dim, avg = CONFIGS[cfg][:3]
    R = oracle.Ref()
    d = f"/dev/shm/fd_bench_ref_{cfg}_{os.getpid()}"
    t0 = time.time()
    feats, ne = R.stage_dataset(d, n, dim, avg, GEN_SEED, threads)
    log(f"[ref] staged {cfg} with the reference generator in {time.time() - t0:.1f}s ({ne} edges)")
    return d, feats


def cpu_reference(cfg, staged, order, batch_ids, threads, bm=None):
    """The reference's sample_khop -> row extraction -> trainer checksum for `batch_ids`
    (contiguous), one batch per host thread. With `bm` (RefBuffer, config 3) the batches
    go in order through the reference BufferManager into its region (samplers on the other
    threads). Returns (secs, checksums, node_counts)."""
    import oracle
    n, dim, avg, fan, b, t_ids, dtype, _ = CONFIGS[cfg]
    R = oracle.Ref()
    d, feats = staged
    topo = oracle.RefTopology(R, d)
    first = int(batch_ids[0])
    seeds = np.ascontiguousarray(order[first * b:(first + len(batch_ids)) * b])
    if bm is not None:
        secs, cs, nc = R.bench_sample_extract_bm(topo, feats, seeds, len(batch_ids), b, fan, 0, 0, first, threads,
                                                 bm.h, bm.region)
    else:
        secs, cs, nc = R.bench_sample_extract(topo, feats, seeds, len(batch_ids), b, fan, 0, 0, first, threads)
    topo.close()
    return secs, cs, nc


class RefBuffer:
    """The reference's featbuf::BufferManager (default mapping: dense below 32 M nodes,
    sparse above) + a host region of `slots` rows, persisting across cpu_reference calls."""

    def __init__(self, num_nodes, slots, row_bytes):
        import oracle
        self.R = oracle.Ref()
        self.h = self.R.lib.fdref_bm_create(num_nodes, slots, 0, 0)
        if not self.h:
            raise RuntimeError("fdref_bm_create: " + self.R.err())
        self.region = np.empty(slots * row_bytes, np.uint8)

    def close(self):
        if self.h:
            self.R.lib.fdref_bm_destroy(self.h)
            self.h = None


def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref) on all host threads, timed in
    whole waves: every timed call runs a multiple of `threads` batches (one batch per
    thread, and >= 4 waves), so no thread idles through a partial last wave."""
    dist = Dist()
    if dist.rank != 0:  # rank 0 alone runs the CPU reference
        dist.close()
        return
    import shutil

    import oracle
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfdref.so not built"}), flush=True)
        return
    cfg = args.config
    n, dim, avg, fan, b, t_ids, dtype, frac = CONFIGS[cfg]
    threads = os.cpu_count()
    staged = stage_reference_dataset(cfg, threads)
    R = oracle.Ref()
    order = R.partition_epoch(np.arange(t_ids, dtype=np.uint64), b, R.hash_combine(0, 0))
    nb = t_ids // b
    bm = RefBuffer(n, int(n * frac), dim * (4 if dtype == "f32" else 2)) if frac else None
    W, K = args.warmup, args.steps
    # buffer configs extract in batch order through one BufferManager (its mutex serialises
    # the reference anyway): K batches; otherwise whole waves of `threads` batches.
    total = K if frac else -(-max(K, 4 * threads) // threads) * threads
    try:
        cpu_reference(cfg, staged, order, np.arange(min(W, nb)) % nb, threads, bm)
        ids = (W + np.arange(total)) % nb
        secs, nodes = 0.0, 0
        at = 0
        while at < total:
            run = int(min(total - at, nb - ids[at]))
            sc, cs, nc = cpu_reference(cfg, staged, order, ids[at:at + run], threads, bm)
            secs += sc
            nodes += int(nc.sum())
            at += run
    finally:
        shutil.rmtree(staged[0], ignore_errors=True)
        if bm:
            bm.close()
    value = total / secs
    cpu = host_cpu()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "batches/s", "n_gpus": args.gpus,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * secs / total, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (reference generator, seed 7)",
        "config": bench_config(cfg, args.gpus, "local" if args.gpus == 1 else "replicas"),
        "execution": {"threads": threads, "cpu": cpu, "batches_timed": total, "batches_per_step": total / K,
                      "path": ("graph::sample_khop on threads-1 workers; batches in order through "
                               "featbuf::BufferManager (acquire, get_standby_slot + bind_slot + row copy per miss, "
                               "publish_valid, lag-1 release_batch) + trainer_step hash over region[alias] (oracle/_ref)"
                               if frac else
                               "graph::sample_khop + per-row extraction copy + trainer_step hash (oracle/_ref), one "
                               "batch per host thread, whole waves"),
                      "mean_nodes_per_batch": nodes / total},
        "cpu_baseline": {"value": value, "unit": "batches/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu["model"],
                         "sample": f"{total} batches of the epoch-0 partition "
                                   + ("sampled on threads - 1 workers, extracted in order through one "
                                      "reference BufferManager (warm after the warm-up batches)" if frac
                                      else f"in {total // threads} whole waves of one batch per thread")},
        "e2e": {"value": value, "unit": "batches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.sync_reference:
        line["sync_reference"] = _sync_reference(cfg, args)
    print(json.dumps(line), flush=True)
    dist.close()


def _sync_reference(cfg, args):
    """the reference PipelineSession::run_sync_reference
    (pipeline.hpp:261-293) on a dataset written by the reference generator (features.bin
    included), over a bounded prefix of the epoch's train ids."""
    import shutil

    import oracle
    n, dim, avg, fan, b, t_ids, dtype, frac = CONFIGS[cfg]
    R = oracle.Ref()
    d = f"/dev/shm/fd_sync_ref_{cfg}_{os.getpid()}"
    try:
        t0 = time.time()
        R.generate_dataset(d, n, dim, avg, GEN_SEED)
        log(f"[ref] wrote the {cfg} dataset (features.bin included) in {time.time() - t0:.1f}s")
        ids = np.arange(args.sync_batches * b, dtype=np.uint64)
        t0 = time.perf_counter()
        recs, _ = R.run_epoch(d, ids, 0, 0, b, fan, sync=True)
        secs = time.perf_counter() - t0
    finally:
        shutil.rmtree(d, ignore_errors=True)
    return {"value": len(recs) / secs, "unit": "batches/s", "batches": int(len(recs)), "threads": 1,
            "path": "PipelineSession::run_sync_reference (sample, blocking row reads, trainer checksum, verify on)",
            "sample": f"train ids 0..{len(ids) - 1} of the {cfg} shape, epoch 0"}


# ------------------------------------------------------------------ our arm ----
def Pipeline(fd, topo, fan, B, bm_slots=None, checksum=False, samplers=6, group=1):
    return fd.Pipeline(topo, fan, B, buffer_slots=bm_slots, checksum=checksum, samplers=samplers,
                       group_batches=group)


def run_ours(args):
    import paper_2406_13984_b200 as fd
    from paper_2406_13984_b200 import dist as fdist
    from paper_2406_13984_b200.featdrive import DeviceBuffer

    dist = Dist()
    dev = fdist.local_device(dist.local)
    L = fd.featdrive.lib()
    for kv in args.option:
        k, v = kv.split("=", 1)
        fd.set_option(k, int(v))
    fd.featdrive.check(L.fdg_set_device(dev))
    cfg = args.config
    n, dim, avg, fan, B, t_ids, dtype, frac = CONFIGS[cfg]
    # North-star layout at N > 1: the table row-sharded over the GPUs, remote rows read by
    # one-sided P2P loads inside the gather. The buffer-manager and host-tier configs keep
    # one table per GPU (their miss source is a single table).
    layout = args.layout
    if layout == "auto":
        layout = "sharded" if dist.world > 1 and not frac and cfg not in HOST_TIER else (
            "replicas" if dist.world > 1 else "local")
    proxy = cfg == "mag" and dist.world < 3  # the 375 GB fp16 table needs >= 3 GPUs
    if proxy:
        layout = "proxy"
    t0 = time.time()
    topo = fd.Topology.generate(n, dim, avg, GEN_SEED, dtype=dtype, device=dev,
                                features=layout in ("local", "replicas"))
    sharded, rps, shard_of = None, None, dist.rank
    if layout == "sharded":  # own rows generated locally, peers' rows read over NVLink (IPC)
        sharded = fdist.ShardedFeatures(topo, dist.rank, dist.world, GEN_SEED, n, dim, dtype)
        rps = sharded.rows_per_shard
    elif layout == "proxy":
        rps, shard_of = _c4_proxy_table(fd, L, topo, n, dim, dtype, shards=8)
    if cfg in HOST_TIER:
        t1 = time.time()
        topo.features_to_host()
        log(f"[rank {dist.rank}] feature table moved to pinned host memory in {time.time() - t1:.1f}s")
    info = topo.info()
    rb = info.row_bytes
    log(f"[rank {dist.rank}] generated {cfg} ({layout}) on GPU {dev}: {info.num_edges} edges, {rb} B rows, "
        f"{time.time() - t0:.1f}s")
    order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, hash_combine(0, 0)))
    nb = t_ids // B
    lo, hi = segment(nb, dist.world, dist.rank)  # this rank's contiguous batch segment
    W, K = args.warmup, args.steps
    seg = np.arange(lo, hi)
    ids_warm = seg[np.arange(W) % len(seg)]
    ids = seg[(W + np.arange(K)) % len(seg)]
    rng_of = lambda ids_: np.array([L.fdg_batch_seed(0, 0, int(g)) for g in ids_], np.uint64)  # noqa: E731

    def seeds_for(ids_):
        return np.ascontiguousarray(np.concatenate([order[g * B:(g + 1) * B] for g in ids_]))

    bm_slots = int(n * frac) if frac else None
    timed = _timed_run(fd, topo, fan, B, bm_slots, seeds_for, rng_of, ids, ids_warm, args, dist, dev, extract=True)
    n_nodes, value, max_ms, ext_ms, busy_ms, clk = (timed[k] for k in ("n_nodes", "value", "max_ms", "ext_ms",
                                                                      "busy_ms", "clocks"))
    gather_bytes = 2 * n_nodes * rb
    if frac:  # buffer manager: a miss also fills its slot (the reference Extractor's region write)
        gather_bytes = gather_bytes + int(round(timed["loads_per_batch"])) * rb
    achieved = float(gather_bytes.sum()) / (busy_ms / 1e3) / 1e9
    hbm, hbm_kind = peaks()
    try:  # explanatory extra: never let it cost the bench line
        alone = None if (frac or layout != "local") else _gather_alone(fd, L, topo, fan, seeds_for, rng_of, ids[:3],
                                                                      hbm)
    except Exception as e:  # noqa: BLE001
        alone = {"error": repr(e)}

    # ---------------- end to end through the C ABI with host buffers ----------------
    # every step: H2D of the batch's seeds from pinned memory, sample, extract with the
    # fused trainer checksum, D2H of the batch record (counts + checksum) into pinned memory.
    # Timed on the host wall clock around the call (enqueue + final synchronisation included).
    e2e = Pipeline(fd, topo, fan, B, bm_slots=bm_slots, checksum=True, samplers=args.samplers, group=args.group)
    csz = counts_dtype().itemsize
    pins = []

    def pinned(nbytes):
        p = C.c_void_p()
        fd.featdrive.check(L.fdg_host_alloc(C.byref(p), nbytes))
        pins.append(p.value)
        return p.value

    hw, ht = seeds_for(ids_warm), seeds_for(ids)
    pw, pt = pinned(hw.nbytes), pinned(ht.nbytes)
    C.memmove(pw, hw.ctypes.data, hw.nbytes)
    C.memmove(pt, ht.ctypes.data, ht.nbytes)
    rec_w, rec_t = pinned(W * csz), pinned(K * csz)
    rng_w, rng_t = rng_of(ids_warm), rng_of(ids)
    e2e.run(pw, True, rng_w, rec_w)
    dist.barrier()
    h0 = time.perf_counter()
    dev_ms = e2e.run(pt, True, rng_t, rec_t)
    wall_ms = (time.perf_counter() - h0) * 1e3
    e2e_ms = dist.reduce(wall_ms, "max")
    dist.barrier()
    host_recs = np.frombuffer((C.c_uint8 * (K * csz)).from_address(rec_t), counts_dtype()).copy()
    e2e.close()
    if np.any(host_recs["status"] != 0):
        raise RuntimeError("e2e batch status errors")
    total = dist.reduce(K, "sum")
    e2e_value = total / (e2e_ms / 1e3)
    gpu_cs = {int(g): int(c) for g, c in zip(ids, host_recs["checksum"])}
    gpu_nn = {int(g): int(c) for g, c in zip(ids, host_recs["n_nodes"])}
    for p in pins:
        L.fdg_host_free(p)

    kernel = ("k_move_hash_rb<HASH=false> (buffer-manager row move, 32-row groups: misses table -> slot and X, "
              "hits slot -> X; its launches timed "
              "alone, the metadata chain runs before them on the other stream)") if frac else (
        "k_gather_rb_dyn<SHARDED> (row groups; remote rows loaded through the peers' IPC mappings)"
        if layout in ("sharded", "proxy") else "k_gather16_dyn")
    line = {
        "metric": METRIC, "value": value, "unit": "batches/s", "n_gpus": dist.world, "steps": K, "warmup": W,
        "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (bit-exact GPU port of the reference generator, seed 7)",
        "config": bench_config(cfg, dist.world, "sharded" if layout == "proxy" else layout),
        "execution": {"layout": layout, "samplers": args.samplers, "group_batches": args.group,
                      "mean_nodes_per_batch": float(n_nodes.mean()), "gpus_visible": fd.device_count(),
                      "device_of_rank0": dev},
        "gather_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "pipeline_gbs": float(gather_bytes.sum()) / (max_ms / 1e3) / 1e9,
                     "traffic": (_traffic(cfg) or {}).get("bytes"), "traffic_detail": _traffic(cfg),
                     "peak_kind": hbm_kind, "kernel": kernel,
                     "launch_ms_mean": busy_ms / K, "launch_ms_mean_per_stream": float(ext_ms.mean()),
                     "bytes_per_launch": float(gather_bytes.mean()),
                     "note": ("algorithmic bytes = (2 x nodes + misses) x row_bytes per launch (a miss is read "
                              "from the table and written to its slot and to X; a hit is read from its slot "
                              "and written to X); " if frac else "algorithmic bytes = 2 x nodes x row_bytes "
                              "per launch; ") + "launch duration = CUDA "
                             "events around each extraction launch on its stream inside the timed pipelined "
                             "run; consecutive gathers alternate between two streams and can overlap, so the "
                             "average launch duration is the union of the launch intervals / launches; "
                             "pipeline_gbs = all gather bytes / whole timed region"},
        "step_roofline": _step_roofline(cfg, max_ms / K, hbm) if layout == "local" else None,
        "gather_alone": alone,
        "gpu_launches": _launch_count(K, len(fan), frac is not None, args.samplers),
        "e2e": {"value": e2e_value, "unit": "batches/s", "h2d_bytes_per_step": B * 8, "d2h_bytes_per_step": csz,
                "timing": "host wall clock around fdg_pipeline_run (enqueue + final synchronisation), max over ranks",
                "device_ms": dev_ms, "wall_ms": wall_ms,
                "includes": "seed H2D, sample, extract, fused trainer checksum, batch-record D2H"},
        "clocks": clk,
    }
    if dist.world > 1:
        line["per_rank_gather_gbs"] = dist.gather(achieved)
    if layout in ("sharded", "proxy"):
        line["sharding"] = _shard_stats(fd, topo, fan, seeds_for, rng_of, ids[:3], rps, shard_of, rb,
                                        max_ms / K, proxy=layout == "proxy")
    if layout == "proxy":
        line["unavailable_full"] = ("the 375 GB fp16 MAG240M table needs >= 3 GPUs; this line is the 1-GPU C4 proxy: "
                                    "the MAG-shaped CSR + one 1/8 fp16 shard, all 8 shard pointers aliasing it, so "
                                    "the per-GPU sampling and gather bytes are real and remote rows read local HBM")
        line["value_kind"] = "c4_proxy"
    if sharded is not None:
        dist.barrier()  # peers read this rank's shard until every rank is done
        sharded.close()
        dist.barrier()
        if cfg != "mag":  # the same batches with a full table copy per GPU (replicas)
            fd.featdrive.check(L.fdg_ctx_generate_features(topo.ctx, GEN_SEED, n, dim, 0 if dtype == "f32" else 1, 1))
            rep = _timed_run(fd, topo, fan, B, bm_slots, seeds_for, rng_of, ids, ids_warm, args, dist, dev,
                             extract=False)
            line["replicas"] = {"value": rep["value"], "unit": "batches/s", "ms_per_step": rep["max_ms"] / K,
                                "layout": "replicated CSR + full table per GPU (no data-path exchange)"}
    if cfg in HOST_TIER:
        line["host_tier"] = _host_tier_link(fd, L, timed, rb, max_ms / K)
    if bm_slots:
        line["alias_only"] = _alias_only(fd, topo, fan, B, bm_slots, seeds_for, rng_of, ids, ids_warm, args, dist)
    if args.train and layout == "local":
        line["train_stage"] = _train_stage(fd, topo, fan, B, bm_slots, seeds_for, rng_of, ids, ids_warm, args, dist)
    if not args.no_per_call and layout == "local" and cfg in ("papers", "products"):
        try:
            line["per_call"] = _per_call(cfg)
        except Exception as e:  # noqa: BLE001
            line["per_call"] = {"error": repr(e)}
    if dist.world == 1 and not args.no_cpu_baseline and layout == "local":
        try:
            line["cpu_baseline"], line["checksum_match_vs_reference"] = _cpu_baseline(cfg, topo, order, args, gpu_cs,
                                                                                    gpu_nn)
            line["cpu_baseline"]["cpu_model"] = host_cpu()["model"]
        except Exception as e:  # pragma: no cover
            log("cpu baseline failed:", repr(e))
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.close()


def _timed_run(fd, topo, fan, B, bm_slots, seeds_for, rng_of, ids, ids_warm, args, dist, dev, extract):
    """The device-resident timed region: W warm-up batches, then exactly K batches between
    barriers, CUDA events on the runner's streams, max over ranks."""
    from paper_2406_13984_b200.featdrive import DeviceBuffer
    K = len(ids)
    pipe = Pipeline(fd, topo, fan, B, bm_slots=bm_slots, checksum=False, samplers=args.samplers, group=args.group)
    warm_dev = DeviceBuffer.from_array(seeds_for(ids_warm))
    timed_dev = DeviceBuffer.from_array(seeds_for(ids))
    pipe.run(warm_dev.ptr, False, rng_of(ids_warm))
    loads_warm = bm_loads(pipe) if bm_slots else None
    dist.barrier()
    ext_ms = np.zeros(K, np.float32)
    with ClockSampler(dev) as clk:
        ms = pipe.run(timed_dev.ptr, False, rng_of(ids), extract_ms=ext_ms)
    dist.barrier()
    recs = pipe.records(K)
    xs, xe = pipe.extract_times(K)
    loads = bm_loads(pipe) if bm_slots else None
    pipe.close()
    if np.any(recs["status"] != 0):
        raise RuntimeError(f"batch status errors in the timed region: {np.unique(recs['status'])}")
    max_ms = dist.reduce(ms, "max")
    return {"n_nodes": recs["n_nodes"].astype(np.int64), "max_ms": max_ms,
            "loads_per_batch": (loads - loads_warm) / K if loads is not None else None,
            "value": dist.reduce(K, "sum") / (max_ms / 1e3), "ext_ms": ext_ms, "busy_ms": _union_ms(xs, xe),
            "clocks": clk.summary()}


def bm_loads(pipe):
    """Cumulative buffer-manager loads (misses) of a runner."""
    import paper_2406_13984_b200 as fd
    from paper_2406_13984_b200._lib import BmStats
    st = BmStats()
    fd.featdrive.check(fd.featdrive.lib().fdg_pipeline_bm_stats(pipe.ptr, C.byref(st)))
    return st.loads


def _c4_proxy_table(fd, L, topo, n, dim, dtype, shards):
    """C4 on one GPU: shard 0 of the 8-way fp16 table (30.5 M rows x 1536 B = 46.9 GB), installed
    as all 8 shard bases. Returns (rows_per_shard, this GPU's shard index)."""
    base = C.c_void_p()
    dt = 0 if dtype == "f32" else 1
    fd.featdrive.check(L.fdg_ctx_generate_feature_shard(topo.ctx, GEN_SEED, n, dim, dt, 0, shards, C.byref(base)))
    rps = -(-n // shards)
    arr = (C.c_void_p * shards)(*([base.value] * shards))
    fd.featdrive.check(L.fdg_ctx_set_feature_shards(topo.ctx, C.cast(arr, C.c_void_p), shards, rps, n,
                                                    dim * (4 if dt == 0 else 2), dt))
    return rps, 0


def _shard_stats(fd, topo, fan, seeds_for, rng_of, ids, rps, shard, rb, ms_per_step, proxy):
    """Remote-row share of this rank's batches (node lists of 3 timed batches through the
    host API) and the NVLink-bound time per batch it implies."""
    remote, total = 0, 0
    for g, r in zip(ids, rng_of(ids)):
        nodes = fd.sample_khop(topo, seeds_for([g]), fan, int(r)).nodes.astype(np.int64)
        remote += int(np.count_nonzero(nodes // rps != shard))
        total += len(nodes)
    share = remote / max(total, 1)
    remote_bytes = share * (total / max(len(ids), 1)) * rb
    nvl = 770e9  # measured NVLink 5 peer copy per direction per GPU (B200_PROFILING.md; 900 nominal)
    return {"rows_per_shard": int(rps), "remote_row_share": share, "remote_bytes_per_batch": remote_bytes,
            "nvlink_floor_ms_per_batch": remote_bytes / nvl * 1e3, "nvlink_gbs_basis": "770 GB/s measured peer copy", "ms_per_step": ms_per_step,
            "note": ("proxy: remote rows are read from the aliased local shard (HBM), so ms_per_step is the "
                     "sampling + gather cost with remote reads at HBM speed; the NVLink floor is what the remote "
                     "share costs on 8 B200s" if proxy else
                     "remote rows are loaded one-sided through CUDA IPC peer mappings (NVLink when the ranks own "
                     "different GPUs)")}


def _host_tier_link(fd, L, timed, rb, ms_per_step):
    """The out-of-core tier against its link: the measured pinned host -> device copy peak
    (1 GiB cudaMemcpy, best of 5) vs the miss rows the buffer manager pulled over it."""
    nbytes = 1 << 30
    h, d = C.c_void_p(), C.c_void_p()
    fd.featdrive.check(L.fdg_host_alloc(C.byref(h), nbytes))
    fd.featdrive.check(L.fdg_malloc(C.byref(d), nbytes))
    C.memset(h.value, 1, nbytes)
    best = 0.0
    for _ in range(5):
        t0 = time.perf_counter()
        fd.featdrive.check(L.fdg_memcpy_h2d(d.value, h.value, nbytes, None))
        fd.featdrive.check(L.fdg_device_sync())
        best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
    L.fdg_free(d.value)
    L.fdg_host_free(h.value)
    loads = timed.get("loads_per_batch")
    out = {"pcie_h2d_peak_gbs": best, "peak_how": "1 GiB pinned cudaMemcpy H2D, best of 5"}
    if loads:
        gbs = loads * rb / (ms_per_step / 1e3) / 1e9
        out.update({"miss_rows_per_batch": loads, "miss_gbs": gbs, "frac_of_link": gbs / best})
    return out


def _per_call(cfg, batches=200):
    """The reference's per-call SET loop (tests/cpp/set_loop.cpp: sample_khop -> Extractor::
    extract_batch -> trainer_step -> release_batch, one batch at a time, host vectors in and
    out) through the C++ drop-in (include/featdrive_gpu.hpp), at this config's shape, in a
    separate process (tools/set_loop) on a dataset generated in HBM."""
    import re
    import subprocess
    n, dim, avg, fan, B, t_ids, dtype, frac = CONFIGS[cfg]
    exe = os.path.join(ROOT, "tools", "set_loop")
    if not os.path.exists(exe):
        return {"error": "tools/set_loop not built"}
    slots = 4 * min(B * (1 + 10 + 100 + 1000), n)  # the reference default N_e * M_b (N_e = 4)
    p = subprocess.run([exe, "--generate", f"{n}:{dim}:{avg}:{GEN_SEED}", str(slots), str(batches)],
                       capture_output=True, text=True, timeout=600)
    m = re.search(r"per_call ([0-9.]+) batches/s", p.stdout)
    if p.returncode != 0 or not m:
        return {"error": (p.stderr or p.stdout)[-300:]}
    return {"value": float(m.group(1)), "unit": "batches/s", "batches": batches, "buffer_slots": slots,
            "path": "reference-shaped SET loop through the C++ drop-in, one batch per call: graph::sample_khop, "
                    "extract::Extractor::extract_batch (GPU BufferManager), pipeline::trainer_step, "
                    "BufferManager::release_batch; host vectors in and out, synchronous"}


def _alias_only(fd, topo, fan, B, bm_slots, seeds_for, rng_of, ids, ids_warm, args, dist):
    """Config 3 in the reference's own form: extraction produces the NodeAliasList and fills
    the FeatureRegion slots of the misses (extractor.hpp:88-113); the trainer reads rows
    through the aliases (pipeline.hpp:103-124), so no separate mini-batch tensor is written."""
    from paper_2406_13984_b200.featdrive import DeviceBuffer
    pipe = fd.Pipeline(topo, fan, B, buffer_slots=bm_slots, checksum=False, samplers=args.samplers,
                       group_batches=args.group, write_x=False)
    warm = DeviceBuffer.from_array(seeds_for(ids_warm))
    timed = DeviceBuffer.from_array(seeds_for(ids))
    pipe.run(warm.ptr, False, rng_of(ids_warm))
    dist.barrier()
    ms = dist.reduce(pipe.run(timed.ptr, False, rng_of(ids)), "max")
    recs = pipe.records(len(ids))
    pipe.close()
    if np.any(recs["status"] != 0):
        raise RuntimeError("alias-only run: batch status errors")
    K = len(ids)
    return {"value": dist.reduce(K, "sum") / (ms / 1e3), "unit": "batches/s", "ms_per_step": ms / K,
            "note": "extraction = NodeAliasList + region slot fill of the misses (the reference's Extractor "
                    "output); the headline value above also materialises X[i] = slot(alias[i])"}


def _train_stage(fd, topo, fan, B, bm_slots, seeds_for, rng_of, ids, ids_warm, args, dist):
    """sample -> extract -> GraphSAGE forward + loss (the paper's 3-layer model, hidden 256,
    PAPER.md:405, 1122-1125) per batch through the same runner, device-resident seeds."""
    from paper_2406_13984_b200.featdrive import DeviceBuffer
    dim = topo.row_bytes // 4
    classes = 172  # ogbn-papers100M label count
    dims = [dim] + [256] * (len(fan) - 1) + [classes]
    model = fd.GraphSAGE(topo, dims, fan, max_seeds=B, seed=0)
    pipe = Pipeline(fd, topo, fan, B, bm_slots=bm_slots, checksum=False, samplers=args.samplers, group=args.group)
    pipe.set_model(model, label_seed=0)
    warm = DeviceBuffer.from_array(seeds_for(ids_warm))
    timed = DeviceBuffer.from_array(seeds_for(ids))
    pipe.run(warm.ptr, False, rng_of(ids_warm))
    dist.barrier()
    ms = dist.reduce(pipe.run(timed.ptr, False, rng_of(ids)), "max")
    losses = pipe.losses(len(ids))
    # training mode: + backward (ReLU masks, transposed scatter-mean, weight gradients) + SGD
    pipe.set_training(0.01)
    pipe.run(warm.ptr, False, rng_of(ids_warm))
    dist.barrier()
    ms_train = dist.reduce(pipe.run(timed.ptr, False, rng_of(ids)), "max")
    train_losses = pipe.losses(len(ids))
    pipe.close()
    model.close()
    K = len(ids)
    return {"value": dist.reduce(K, "sum") / (ms / 1e3), "unit": "batches/s", "ms_per_step": ms / K,
            "train_step": {"value": dist.reduce(K, "sum") / (ms_train / 1e3), "unit": "batches/s",
                           "ms_per_step": ms_train / K, "lr": 0.01,
                           "loss_first_last": [float(train_losses[0]), float(train_losses[-1])],
                           "includes": "forward + loss + backward + SGD per batch (data-parallel gradient "
                                       "all-reduce not included: one GPU)"},
            "model": "GraphSAGE mean-aggregator " + "-".join(map(str, dims)) + (
                ", layer GEMMs on tcgen05 (kind::tf32, 3xTF32 fp32-accurate)" if fd.featdrive.get_option("sage_gemm")
                else ", fp32 CUDA-core GEMMs"),
            "mean_loss": float(np.mean(losses)), "finite": bool(np.all(np.isfinite(losses))),
            "includes": "sample + extract + per-layer scatter-mean + GEMM + bias/ReLU + softmax cross-entropy"}


def _union_ms(starts, ends):
    """Total length of the union of [start, end) intervals (ms)."""
    tot, cur_s, cur_e = 0.0, None, None
    for a, b in sorted(zip(starts.tolist(), ends.tolist())):
        if cur_e is None or a > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def _launch_count(K, layers, bm, samplers, prefetch=16):
    # per batch: 2 k_fill_ones (early and last-layer hash clears), k_seeds, k_intern_s x (layers + 1),
    # k_expand x layers, k_replay (a no-op unless the batch saw a Lemire rejection), then the
    # gather (k_gather16_dyn) -- or, with the buffer manager, 5 extract kernels (reset, acquire,
    # select + bind, bind_finish, move) + k_status_to + 4 release kernels (reset, release,
    # compact, finish). Plus two k_mt_stream launches (the stream's two pieces) per prefetch
    # request of each sampler: one chunk of `prefetch` streams up front, then one stream per batch.
    per_batch = 2 + 1 + (layers + 1) + layers + 1 + (1 if not bm else 10)
    per_sampler = -(-K // samplers)
    return K * per_batch + samplers * 2 * (1 + max(per_sampler - prefetch, 0))


def _gather_alone(fd, L, topo, fan, seeds_for, rng_of, ids, peak_gbs, reps=10):
    """The standalone fdg_gather (default engine) on three of the timed batches' node lists,
    nothing else running: CUDA events around each launch on its stream, batches alternating
    so consecutive launches read different rows. Explains the in-pipeline roofline fraction
    (the same bytes next to the sampler chains)."""
    from paper_2406_13984_b200.featdrive import DeviceBuffer
    rb = topo.row_bytes
    lists = [fd.sample_khop(topo, seeds_for([g]), fan, int(r)).nodes for g, r in zip(ids, rng_of(ids))]
    bufs = [DeviceBuffer.from_array(np.ascontiguousarray(x, np.uint64)) for x in lists]
    out = DeviceBuffer(max(len(x) for x in lists) * rb)
    evs = []
    for _ in range(2 * reps + 2):
        e = C.c_void_p()
        fd.featdrive.check(L.fdg_event_create(C.byref(e)))
        evs.append(e)
    times, nbytes = [], []
    for i in range(reps + 1):
        b = i % len(bufs)
        fd.featdrive.check(L.fdg_event_record(evs[2 * i], None))
        fd.featdrive.check(L.fdg_gather(topo.ctx, None, bufs[b].ptr, None, len(lists[b]), out.ptr, None))
        fd.featdrive.check(L.fdg_event_record(evs[2 * i + 1], None))
        if i:  # the first launch warms the engine up
            nbytes.append(2 * len(lists[b]) * rb)
    fd.featdrive.check(L.fdg_device_sync())
    for i in range(1, reps + 1):
        ms = C.c_float()
        fd.featdrive.check(L.fdg_event_elapsed_ms(evs[2 * i], evs[2 * i + 1], C.byref(ms)))
        times.append(ms.value)
    for e in evs:
        L.fdg_event_destroy(e)
    us = float(np.mean(times)) * 1e3
    gbs = float(np.sum(nbytes)) / (float(np.sum(times)) / 1e3) / 1e9
    return {"engine": "fdg_gather default (k_gather_rb_dyn, 32-row groups, 256-byte chunks)", "us_per_launch": us,
            "achieved": gbs, "peak": peak_gbs, "unit": "GB/s", "frac": gbs / peak_gbs, "launches": reps,
            "note": "same algorithmic bytes (2 x nodes x row_bytes) as roofline.achieved, gather alone on the GPU"}


def _step_roofline(cfg, ms_per_step, peak_gbs):
    """Whole pipelined step against the DRAM roofline: profiled DRAM bytes per batch
    (ncu range replay, profiles/ncu_traffic.json '<cfg>_step') / peak vs the live step time."""
    t = _traffic(cfg + "_step")
    if not t:
        return None
    floor_ms = t["bytes"] / (peak_gbs * 1e9) * 1e3
    return {"bytes_per_step": t["bytes"], "floor_ms": floor_ms, "ms_per_step": ms_per_step,
            "frac": floor_ms / ms_per_step, "source": t["source"]}


def _traffic(cfg):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(cfg)
    except Exception:
        return None


def _cpu_baseline(cfg, topo, order, args, gpu_cs, gpu_nn):
    """Stage the GPU-generated dataset (bit-identical to the reference generator's
    files, SHA-256-checked in tests) in /dev/shm + host RAM, time the reference's CPU
    sample -> extract -> checksum on a bounded sample of the same epoch, and compare
    its per-batch trainer checksums with the GPU e2e records of the same batches."""
    import shutil

    from paper_2406_13984_b200.featdrive import _p, check, lib
    n = CONFIGS[cfg][0]
    d = f"/dev/shm/fd_cpu_{cfg}_{os.getpid()}"
    os.makedirs(d, exist_ok=True)
    t0 = time.time()
    ip, ix = topo.download_topology()
    ip.tofile(os.path.join(d, "indptr.bin"))
    mm = np.memmap(os.path.join(d, "indices.bin"), mode="w+", dtype=np.uint64, shape=(max(len(ix), 1),))
    for a in range(0, len(ix), 1 << 27):
        mm[a:a + (1 << 27)] = ix[a:a + (1 << 27)]
    mm.flush()
    del mm, ix, ip
    feats = np.empty((n, topo.row_bytes), np.uint8)
    for a in range(0, n, 1 << 22):
        k = min(1 << 22, n - a)
        check(lib().fdg_ctx_download_rows(topo.ctx, a, k, _p(feats[a:a + k])))
    log(f"[cpu] staged the dataset in host memory in {time.time() - t0:.1f}s")
    threads = os.cpu_count()
    first = min(gpu_cs) if gpu_cs else 0
    frac = CONFIGS[cfg][7]
    nbat = args.cpu_batches or (16 if frac else 4 * threads)  # config 3 extracts batch after batch
    bm = RefBuffer(n, int(n * frac), topo.row_bytes) if frac else None
    try:
        secs, cs, nc = cpu_reference(cfg, (d, feats), order, np.arange(first, first + nbat), threads, bm)
    finally:
        shutil.rmtree(d, ignore_errors=True)
        if bm:
            bm.close()
    compared = [b for b in range(nbat) if first + b in gpu_cs]
    equal = all(gpu_cs[first + b] == int(cs[b]) and gpu_nn[first + b] == int(nc[b]) for b in compared)
    return ({"value": nbat / secs, "unit": "batches/s", "cores": threads, "kind": "reference",
             "sample": f"batches {first}..{first + nbat - 1} of the epoch-0 partition (sample_khop + "
                       + ("reference BufferManager extraction into a cold buffer" if frac else "row extraction")
                       + f" + trainer checksum), {secs:.1f}s on {threads} threads"},
            {"batches_compared": len(compared), "all_equal": bool(equal)})


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under
    torch.distributed.run with N local ranks (rank 0 prints the line)."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] spawning {n} ranks: {' '.join(cmd[1:])}")
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="papers", choices=sorted(CONFIGS))
    ap.add_argument("--samplers", type=int, default=8,
                    help="concurrent sampler streams (measured: Papers flat at 6-10, products 155 -> 132 us/batch from 6 to 8)")
    ap.add_argument("--group", type=int, default=1, help="batches sampled per launch chain")
    ap.add_argument("--layout", default="auto", choices=["auto", "local", "sharded", "replicas"],
                    help="N>1: 'sharded' (default: table row-sharded, remote rows over NVLink P2P) or 'replicas'")
    ap.add_argument("--shard", action="store_true", help="alias of --layout sharded")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--train", action="store_true",
                    help="also time sample -> extract -> GraphSAGE forward + loss (key train_stage)")
    ap.add_argument("--no-per-call", action="store_true", help="skip the reference-shaped per-call SET loop")
    ap.add_argument("--sync-reference", action="store_true",
                    help="--impl reference: also time PipelineSession::run_sync_reference (BASELINE.md 2 iii)")
    ap.add_argument("--sync-batches", type=int, default=4)
    ap.add_argument("--cpu-batches", type=int, default=0)
    ap.add_argument("--option", action="append", default=[], metavar="KEY=VALUE",
                    help="fdg_set_option before the run (repeatable), e.g. host_tier_thp=1")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.shard:
        args.layout = "sharded"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
