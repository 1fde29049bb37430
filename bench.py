#!/usr/bin/env python3
"""Benchmark: GNNDrive sample -> extract mini-batches/s on B200 (+ gather GB/s vs HBM).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config papers|products|friendster|papers_bm]
                    [--impl ours|reference]

A step is one mini-batch through the hot path: graph::sample_khop (3-hop CSR
neighbour sampling + first-occurrence dedup/reindex, bit-exact) followed by
feature extraction into the mini-batch tensor X (an HBM gather; with
--config papers_bm the GPU feature-buffer manager at a 10 % cap). Batches are
pipelined: MT19937-64 streams are generated ahead on one stream, batch b+1 is
sampled while batch b is gathered on another.

Workload (default, BASELINE.json configs[1]): synthetic Papers100M-shaped graph
(111,059,956 nodes, 1,613,492,860 edges, 128-dim f32 rows) built bit-exactly by
the GPU port of the reference generator, fanout (10,10,10), batch 1000, train
ids 0..999,999, epoch-0 partition (partition_epoch) and per-batch rng seeds
batch_seed(0, 0, b) -- exactly the reference pipeline's keying.

--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference headers): sample_khop + row extraction + the
trainer checksum on all host cores.
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
}
DESCR = {
    "products": "synthetic ogbn-products-shaped graph (2,449,029 nodes, 100-dim f32), fanout (10,10,10), batch 1000",
    "papers": "synthetic Papers100M-shaped graph (111,059,956 nodes, 1,613,492,860 edges, 128-dim f32), "
              "fanout (10,10,10), batch 1000",
    "papers_bm": "Papers100M-shaped graph, feature buffer capped at 10% of the table (11,105,995 slots)",
    "friendster": "synthetic Friendster-shaped graph (65,608,366 nodes, 256-dim f32), fanout (15,10,5), batch 1000",
}
GEN_SEED = 7
METRIC = "sample+extract mini-batches/sec (Papers100M-shape); gather GB/s vs HBM peak"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

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
            self.nv = None
            self.max_mhz = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

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
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- dist ----
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def segment(total: int, world: int, rank: int):
    """Contiguous chunk ranges per worker, sizes differing by at most one (pipeline.hpp:192-203)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


# ------------------------------------------------------------ reference arm ----
def cpu_reference(cfg_name, n_batches, threads=None, staged=None, order=None, first_batch=0):
    """The reference's sample -> extract -> trainer-checksum path on host cores
    (oracle/_ref, compiled from the reference headers). Returns (secs, checksums, node_counts, meta)."""
    import oracle
    n, dim, avg, fan, b, t_ids, dtype, _ = CONFIGS[cfg_name]
    threads = threads or os.cpu_count()
    kind = "reference" if oracle.ref_available() else "port"
    if kind != "reference":
        raise RuntimeError("oracle/_ref/libfdref.so missing; build it with `make -C oracle ref`")
    R = oracle.Ref()
    if staged is None:
        d = f"/dev/shm/fd_bench_{cfg_name}_{os.getpid()}"
        t0 = time.time()
        feats, ne = R.stage_dataset(d, n, dim, avg, GEN_SEED, threads)
        log(f"[ref] staged {cfg_name} with the reference generator in {time.time() - t0:.1f}s ({ne} edges)")
        staged = (d, feats)
    d, feats = staged
    topo = oracle.RefTopology(R, d)
    if order is None:
        order = R.partition_epoch(np.arange(t_ids, dtype=np.uint64), b, R.hash_combine(0, 0))
    seeds = order[first_batch * b:(first_batch + n_batches) * b]
    secs, cs, nc = R.bench_sample_extract(topo, feats, seeds, n_batches, b, fan, 0, 0, first_batch, threads)
    topo.close()
    return secs, cs, nc, {"kind": kind, "cores": threads, "staged": staged}


def run_reference_arm(args):
    dist = Dist()
    if dist.rank != 0:
        dist.close()
        return
    cfg = args.config
    n, dim, avg, fan, b, t_ids, dtype, frac = CONFIGS[cfg]
    threads = os.cpu_count()
    per_step = max(threads, args.ref_batches_per_step)
    import oracle
    R = oracle.Ref()
    d = f"/dev/shm/fd_bench_ref_{cfg}_{os.getpid()}"
    t0 = time.time()
    feats, ne = R.stage_dataset(d, n, dim, avg, GEN_SEED, threads)
    log(f"[ref] staged {cfg}: {time.time() - t0:.1f}s")
    order = R.partition_epoch(np.arange(t_ids, dtype=np.uint64), b, R.hash_combine(0, 0))
    nb = t_ids // b
    times, nodes = [], 0
    try:
        for step in range(args.warmup + args.steps):
            first = (step * per_step) % max(nb - per_step, 1)
            secs, cs, nc, _ = cpu_reference(cfg, per_step, threads, (d, feats), order, first)
            if step >= args.warmup:
                times.append(secs)
                nodes += int(nc.sum())
    finally:
        import shutil
        shutil.rmtree(d, ignore_errors=True)
    total = sum(times)
    value = args.steps * per_step / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "batches/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (reference generator, seed 7)",
        "config": {"workload": DESCR[cfg], "batches_per_step": per_step, "threads": threads},
        "cpu_baseline": {"value": value, "unit": "batches/s", "cores": threads, "kind": "reference",
                         "sample": f"{args.steps} steps x {per_step} batches of the epoch-0 partition"},
        "e2e": {"value": value, "unit": "batches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    dist.close()


# ------------------------------------------------------------------ our arm ----
def run_ours(args):
    import paper_2406_13984_b200 as fd
    from paper_2406_13984_b200 import _lib
    from paper_2406_13984_b200.featdrive import DeviceBuffer, Event, Stream, check

    dist = Dist()
    dev = dist.local
    L = fd.featdrive.lib()
    check(L.fdg_set_device(dev))
    cfg = args.config
    n, dim, avg, fan, B, t_ids, dtype, frac = CONFIGS[cfg]
    t0 = time.time()
    topo = fd.Topology.generate(n, dim, avg, GEN_SEED, dtype=dtype, device=dev)
    info = topo.info()
    rb = info.row_bytes
    log(f"[rank {dist.rank}] generated {cfg}: {info.num_edges} edges, {rb} B rows in {time.time() - t0:.1f}s")
    order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, _hc(0, 0)))
    nb = t_ids // B
    lo, hi = segment(nb, dist.world, dist.rank)
    seg = np.arange(lo, hi, dtype=np.int64)
    rng = np.array([L.fdg_batch_seed(0, 0, int(g)) for g in seg], np.uint64)
    seeds_host = np.ascontiguousarray(order[lo * B:hi * B])

    sampler = fd.Sampler(topo, fan, max_seeds=B)
    cap = sampler.cap
    K, W = args.steps, args.warmup
    seeds_dev = DeviceBuffer.from_array(seeds_host)
    nodes = [DeviceBuffer(cap * 8) for _ in range(2)]
    edges = [DeviceBuffer(cap * 8) for _ in range(2)]
    X = [DeviceBuffer(cap * rb) for _ in range(2)]
    counts = DeviceBuffer((W + K + 8) * C.sizeof(_lib.BatchCounts))
    csz = C.sizeof(_lib.BatchCounts)
    bm = None
    if frac:
        slots = int(n * frac)
        bm = fd.BufferManager(topo, slots, min_reserved=0, max_batch_nodes=sampler.max_nodes)
        alias = [DeviceBuffer(cap * 8) for _ in range(2)]
    ss, gs, ms = Stream(), Stream(), Stream()
    ev_sampled = [Event() for _ in range(2)]
    ev_gdone = [Event() for _ in range(2)]
    PREF = 6

    def batch_of(k):
        return k % len(seg)

    def prefetch(k):
        sampler.prefetch(ms, [int(rng[batch_of(k)])])

    gstart = [Event() for _ in range(W + K)]
    gend = [Event() for _ in range(W + K)]

    def step(k, e2e=False, host_seeds=None, rec=None):
        j = batch_of(k)
        slot = k & 1
        cnt = counts.ptr + k * csz
        if k + PREF < W + K:
            prefetch(k + PREF)
        check(L.fdg_stream_wait_event(ss.ptr, ev_gdone[slot].ptr))
        sp = seeds_dev.ptr + j * B * 8
        if e2e:  # host -> device copy of this step's seeds from pinned memory
            sp = e2e_seeds[slot].ptr
            check(L.fdg_memcpy_h2d(sp, host_seeds + j * B * 8, B * 8, ss.ptr))
        check(L.fdg_sample_khop(sampler.ptr, ss.ptr, sp, B, int(rng[j]), nodes[slot].ptr, edges[slot].ptr, cap, cnt))
        check(L.fdg_event_record(ev_sampled[slot].ptr, ss.ptr))
        check(L.fdg_stream_wait_event(gs.ptr, ev_sampled[slot].ptr))
        if not e2e:
            check(L.fdg_event_record(gstart[k].ptr, gs.ptr))
        cs_ptr = cnt + _lib.BatchCounts.checksum.offset if e2e else None
        if bm is None:
            check(L.fdg_gather(topo.ctx, gs.ptr, nodes[slot].ptr, cnt + _lib.BatchCounts.n_nodes.offset, cap,
                               X[slot].ptr, cs_ptr))
        else:
            check(L.fdg_bm_extract(bm.ptr, gs.ptr, nodes[slot].ptr, cnt + _lib.BatchCounts.n_nodes.offset, cap,
                                   alias[slot].ptr, X[slot].ptr, cs_ptr))
            prev = counts.ptr + (k - 1) * csz
            if k >= 1:  # release the previous batch once this one is extracted (lag-1 schedule)
                check(L.fdg_bm_release(bm.ptr, gs.ptr, nodes[slot ^ 1].ptr, prev + _lib.BatchCounts.n_nodes.offset,
                                       cap))
        if not e2e:
            check(L.fdg_event_record(gend[k].ptr, gs.ptr))
        if e2e:  # device -> host read of the step's result record (counts + trainer checksum)
            check(L.fdg_memcpy_d2h(rec + k * csz, cnt, csz, gs.ptr))
        check(L.fdg_event_record(ev_gdone[slot].ptr, gs.ptr))

    e2e_seeds = [DeviceBuffer(B * 8) for _ in range(2)]
    for k in range(min(PREF, W + K)):
        prefetch(k)
    # ---------------- device-resident timed loop ----------------
    for k in range(W):
        step(k)
    check(L.fdg_device_sync())
    dist.barrier()
    t_start, t_end = Event(), Event()
    with ClockSampler(dev) as clk:
        check(L.fdg_event_record(t_start.ptr, ss.ptr))
        check(L.fdg_stream_wait_event(gs.ptr, t_start.ptr))
        for k in range(W, W + K):
            step(k)
        check(L.fdg_event_record(t_end.ptr, gs.ptr))
        check(L.fdg_device_sync())
    dist.barrier()
    elapsed_ms = t_start.elapsed_ms(t_end)
    recs = counts.download(np.uint8, (W + K) * csz).view(np.dtype(_counts_dtype()))
    bad = recs["status"][W:W + K]
    if np.any(bad != 0):
        raise RuntimeError(f"batch status errors in timed region: {np.unique(bad)}")
    n_nodes = recs["n_nodes"][W:W + K].astype(np.int64)
    gms = [gstart[k].elapsed_ms(gend[k]) for k in range(W, W + K)]
    gather_bytes = 2 * n_nodes * rb
    max_ms = dist.max(elapsed_ms)
    total_batches = dist.sum(K)
    value = total_batches / (max_ms / 1e3)
    achieved = float(np.mean(gather_bytes)) / (float(np.mean(gms)) / 1e3) / 1e9
    hbm, hbm_kind = peaks()

    # ---------------- end-to-end through the C ABI with host buffers ----------------
    pinned = C.c_void_p()
    check(L.fdg_host_alloc(C.byref(pinned), seeds_host.nbytes))
    C.memmove(pinned.value, seeds_host.ctypes.data, seeds_host.nbytes)
    recbuf = C.c_void_p()
    check(L.fdg_host_alloc(C.byref(recbuf), (W + K) * csz))
    for k in range(min(PREF, W + K)):
        prefetch(k)
    for k in range(W):
        step(k, True, pinned.value, recbuf.value)
    check(L.fdg_device_sync())
    dist.barrier()
    e0, e1 = Event(), Event()
    check(L.fdg_event_record(e0.ptr, ss.ptr))
    check(L.fdg_stream_wait_event(gs.ptr, e0.ptr))
    for k in range(W, W + K):
        step(k, True, pinned.value, recbuf.value)
    check(L.fdg_event_record(e1.ptr, gs.ptr))
    check(L.fdg_device_sync())
    dist.barrier()
    e2e_ms = dist.max(e0.elapsed_ms(e1))
    e2e_value = total_batches / (e2e_ms / 1e3)
    host_recs = np.frombuffer((C.c_uint8 * ((W + K) * csz)).from_address(recbuf.value), np.uint8).copy()
    host_recs = host_recs.view(np.dtype(_counts_dtype()))
    if np.any(host_recs["status"] != 0):
        raise RuntimeError("e2e batch status errors")
    e2e_checksums = {int(seg[batch_of(k)]): int(host_recs["checksum"][k]) for k in range(W + K)}
    e2e_nodes = {int(seg[batch_of(k)]): int(host_recs["n_nodes"][k]) for k in range(W + K)}

    line = {
        "metric": METRIC, "value": value, "unit": "batches/s", "n_gpus": dist.world, "steps": K, "warmup": W,
        "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (bit-exact GPU port of the reference generator, seed 7)",
        "config": {"workload": DESCR[cfg], "config": cfg, "nodes": n, "edges": int(info.num_edges),
                   "row_bytes": rb, "fanouts": fan, "batch": B, "global_batch": B * dist.world,
                   "parallelism": f"dp{dist.world} (replicated CSR + table)",
                   "l2_policy": "inputs > L2 (57 GB table, ~0.5 GB X per batch); no flush",
                   "mean_nodes_per_batch": float(n_nodes.mean()),
                   "buffer_slots": int(n * frac) if frac else None},
        "gather_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": _traffic(cfg), "peak_kind": hbm_kind,
                     "kernel": "k_move (buffer manager)" if bm else "k_gather16",
                     "gather_ms_mean": float(np.mean(gms)),
                     "bytes_per_launch": float(np.mean(gather_bytes))},
        "gpu_launches": _launch_count(K, len(fan), bm is not None),
        "e2e": {"value": e2e_value, "unit": "batches/s", "h2d_bytes_per_step": B * 8, "d2h_bytes_per_step": csz},
        "clocks": clk.summary(),
    }
    # ---------------- CPU baseline (rank 0, N=1): the reference on host cores ----------------
    if dist.world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"], match = _cpu_baseline(cfg, topo, order, args, e2e_checksums, e2e_nodes)
            line["checksum_match_vs_reference"] = match
        except Exception as e:  # pragma: no cover
            log("cpu baseline failed:", repr(e))
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    check(L.fdg_host_free(pinned.value))
    check(L.fdg_host_free(recbuf.value))
    dist.close()


def _hc(a, b):
    """hash_combine (common.hpp:84-86) in Python integers: the epoch shuffle seed."""
    M = (1 << 64) - 1

    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    return sm(a ^ ((b + 0x9E3779B97F4A7C15 + (a << 6) + (a >> 2)) & M))


def _counts_dtype():
    from paper_2406_13984_b200._lib import MAX_LAYERS
    return [("status", "<u4"), ("n_nodes", "<u4"), ("n_edges", "<u4"), ("rejections", "<u4"),
            ("bad_seed", "<u8"), ("checksum", "<u8"), ("bad_seed_pos", "<u4"), ("n_layers", "<u4"),
            ("layer_nodes", "<u4", (MAX_LAYERS + 2,)), ("layer_edges", "<u4", (MAX_LAYERS + 1,)),
            ("layer_draws", "<u4", (MAX_LAYERS + 1,)), ("words_used", "<u4"), ("pad", "<u4")]


def _launch_count(K, layers, bm):
    # per batch: MT prefetch 1, k_seeds 1, k_intern layers+1, k_sample layers, k_fix_src 1, gather 1
    # (+ buffer manager: 5 extract + 4 release); memset of the hash table is a copy-engine op.
    per = 1 + 1 + (layers + 1) + layers + 1 + (1 if not bm else 9)
    return K * per


def _traffic(cfg):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg)
    except Exception:
        return None


def _cpu_baseline(cfg, topo, order, args, gpu_cs, gpu_nodes):
    """Stage the GPU-generated (bit-identical, SHA-verified) dataset in host RAM /
    /dev/shm and time the reference's CPU sample -> extract -> checksum on a bounded
    sample of the same epoch. Also cross-checks the reference's per-batch trainer
    checksums against the GPU e2e records for the same batches."""
    import shutil

    n, dim, avg, fan, B, t_ids, dtype, frac = CONFIGS[cfg]
    d = f"/dev/shm/fd_cpu_{cfg}_{os.getpid()}"
    os.makedirs(d, exist_ok=True)
    t0 = time.time()
    ip, ix = topo.download_topology()
    ip.tofile(os.path.join(d, "indptr.bin"))
    del ip
    mm = np.memmap(os.path.join(d, "indices.bin"), mode="w+", dtype=np.uint64, shape=(len(ix),))
    step_ = 1 << 27
    for a in range(0, len(ix), step_):
        mm[a:a + step_] = ix[a:a + step_]
    mm.flush()
    del mm, ix
    feats = np.empty((n, topo.row_bytes), np.uint8)
    chunk = 1 << 22
    from paper_2406_13984_b200.featdrive import check, lib, _p
    for a in range(0, n, chunk):
        k = min(chunk, n - a)
        check(lib().fdg_ctx_download_rows(topo.ctx, a, k, _p(feats[a:a + k])))
    log(f"[cpu] staged dataset in {time.time() - t0:.1f}s")
    threads = os.cpu_count()
    nbat = args.cpu_batches or 4 * threads
    try:
        secs, cs, nc, meta = cpu_reference(cfg, nbat, threads, (d, feats), order, 0)
    finally:
        shutil.rmtree(d, ignore_errors=True)
    match = all(gpu_cs.get(b, cs[b]) == int(cs[b]) and gpu_nodes.get(b, nc[b]) == int(nc[b]) for b in range(nbat))
    checked = sum(1 for b in range(nbat) if b in gpu_cs)
    return ({"value": nbat / secs, "unit": "batches/s", "cores": threads, "kind": meta["kind"],
             "sample": f"first {nbat} batches of the epoch-0 partition (sample_khop + row extraction + "
                       f"trainer checksum), {secs:.1f}s on {threads} threads"},
            {"batches_compared": checked, "all_equal": bool(match)})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="papers", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-batches", type=int, default=0)
    ap.add_argument("--ref-batches-per-step", type=int, default=16)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
