"""A/B experiments on the pipelined run. Each arg: 'k=v,k=v' with keys
S (samplers), flags, mode (full|sample|extract) and any fdg_set_option key."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import os  # noqa: E402

from paper_2406_13984_b200 import _lib as _l  # noqa: E402
if os.environ.get("FDG_DBG_LIB"):  # A/B of a variant build of libfdg.so
    _l.load.__defaults__ = (os.environ["FDG_DBG_LIB"],)
import bench  # noqa: E402
import paper_2406_13984_b200 as fd  # noqa: E402
from paper_2406_13984_b200 import _lib  # noqa: E402
from paper_2406_13984_b200.featdrive import DeviceBuffer  # noqa: E402

import os
cfgname = os.environ.get("CFG", "papers")
n, dim, avg, fan, B, t_ids, dtype, frac = bench.CONFIGS[cfgname]
L = fd.featdrive.lib()
topo = fd.Topology.generate(n, dim, avg, 7, dtype=dtype)
order = np.concatenate(fd.partition_epoch(np.arange(t_ids, dtype=np.uint64), B, bench.hash_combine(0, 0)))
K = int(os.environ.get("K", "300"))
rng = np.array([L.fdg_batch_seed(0, 0, int(g)) for g in range(K)], np.uint64)
nb_epoch = len(order) // B  # wrap at the epoch end (products has 196 batches)
seeds = DeviceBuffer.from_array(np.ascontiguousarray(np.concatenate([order[(b % nb_epoch) * B:(b % nb_epoch + 1) * B] for b in range(K)])))
f = np.ascontiguousarray(fan, np.uint32)
defaults = {"gather_impl": 4, "pipeline_gather_impl": 1, "gather_evict_first": 0, "l2_persist_mb": 0, "hash_load_pct": 50,
            "hash_clear": 1, "sampler_ctas_per_sm": 16, "gather_ctas_per_sm": 1,
            "extract_streams": 2, "hash_keep": 1,
            "checksum_impl": 1, "hash_chunk": 0, "gather_pf64": 2, "rb_ctas_per_sm": 2, "rb_chunk": 256, "sampler_sms": 0, "tma_cfg": 0,
            "replay": 1, "mt_adaptive": 1, "hash_dyn": 0, "hash_ctas_per_sm": 1, "bm_move_impl": 2, "bm_move_grid": 0, "bm_meta_prio": 0, "hash_early_pct": 0, "early_fused": 0, "bm_fuse_bind": 1, "bm_move_hash": 1, "bm_move_early": 0, "early_bloom": 1, "extract_prio": 2, "pipe_slots": 0, "bm_split_move": 0, "hash_ctas": 0, "intern_lean": 2}
for spec in sys.argv[1:]:
    kv = dict(x.split("=") for x in spec.split(",") if x)
    S = int(kv.pop("S", 2))
    Gb = int(kv.pop("G", 1))
    mode = kv.pop("mode", "full")
    cs = int(kv.pop("cs", 0))
    flags = int(kv.pop("flags", 0)) | {"full": 0, "sample": 1, "extract": 2}[mode]
    bm_slots = int(kv.pop("bm", 0))
    opts = dict(defaults)
    opts.update({k: int(v) for k, v in kv.items()})
    for k, v in opts.items():
        fd.featdrive.check(L.fdg_set_option(k.encode(), v))
    bm = bm_slots
    cfg = _lib.PipelineConfig(batch_size=B, n_samplers=S, prefetch_group=16, write_x=1, flags=flags, group_batches=Gb,
                              checksum=cs, use_buffer_manager=1 if bm else 0, buffer_slots=bm)
    p = C.c_void_p()
    fd.featdrive.check(L.fdg_pipeline_create(topo.ctx, f.ctypes.data_as(C.c_void_p), len(f), C.byref(cfg), C.byref(p)))
    ms = C.c_float()
    res = []
    for rep in range(3):
        fd.featdrive.check(L.fdg_pipeline_run(p, seeds.ptr, 0, rng.ctypes.data_as(C.c_void_p), K, None, None, C.byref(ms)))
        res.append(ms.value / K * 1e3)
    out = _lib.PipelineConfig()
    fd.featdrive.check(L.fdg_pipeline_get_config(p, C.byref(out)))
    L.fdg_pipeline_destroy(p)
    best = min(res[1:])
    print(f"{spec:60s} {best:7.1f} us/batch  {1e6 / best:7.0f} batches/s  host enqueue "
          f"{out.host_enqueue_ms / K * 1e3:6.1f} us/batch", flush=True)
