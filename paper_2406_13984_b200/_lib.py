"""ctypes loader for libfdg.so (the C-ABI declared in include/fdg.h).

The library is built in-tree (paper_2406_13984_b200/libfdg.so) by
`make -C paper_2406_13984_b200/csrc` / __graft_entry__.build(). There is no
fallback: if the library or a GPU is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfdg.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "fdg.h")

u64, u32, i64, vp, ci = C.c_uint64, C.c_uint32, C.c_int64, C.c_void_p, C.c_int
MAX_LAYERS = 8

FDG_OK, FDG_OUT_OF_RANGE, FDG_INVALID_ARG, FDG_INVARIANT, FDG_CAPACITY, FDG_CUDA_ERROR, FDG_NOT_LOADED, \
    FDG_REJECTION = range(8)


class BatchCounts(C.Structure):
    _fields_ = [("status", u32), ("n_nodes", u32), ("n_edges", u32), ("rejections", u32),
                ("bad_seed", u64), ("checksum", u64), ("bad_seed_pos", u32), ("n_layers", u32),
                ("layer_nodes", u32 * (MAX_LAYERS + 2)), ("layer_edges", u32 * (MAX_LAYERS + 1)),
                ("layer_draws", u32 * (MAX_LAYERS + 1)), ("words_used", u32), ("replays", u32)]


class CtxInfo(C.Structure):
    _fields_ = [("num_nodes", u64), ("num_edges", u64), ("idx_bytes", u32), ("row_bytes", u32),
                ("dtype", u32), ("n_shards", u32), ("indptr_dev", vp), ("indices_dev", vp),
                ("table_dev", vp), ("rows_per_shard", u64), ("device", ci), ("pad", ci)]


class PipelineConfig(C.Structure):
    _fields_ = [("batch_size", u32), ("n_samplers", u32), ("prefetch_group", u32), ("use_buffer_manager", u32),
                ("buffer_slots", u64), ("write_x", u32), ("checksum", u32), ("flags", u32),
                ("host_enqueue_ms", C.c_float), ("group_batches", u32)]


class BmStats(C.Structure):
    _fields_ = [(k, u64) for k in ("hits", "loads", "waits", "evictions", "takeovers", "releases", "standby_len")]


# name -> (restype, argtypes)
SIGNATURES = {
    "fdg_last_error": (C.c_char_p, []),
    "fdg_last_errno": (ci, []),
    "fdg_version": (ci, []),
    "fdg_device_count": (ci, [C.POINTER(ci)]),
    "fdg_set_device": (ci, [ci]),
    "fdg_enable_peer_access": (ci, [ci, ci]),
    "fdg_malloc": (ci, [C.POINTER(vp), u64]),
    "fdg_free": (ci, [vp]),
    "fdg_host_alloc": (ci, [C.POINTER(vp), u64]),
    "fdg_host_free": (ci, [vp]),
    "fdg_memcpy_h2d": (ci, [vp, vp, u64, vp]),
    "fdg_memcpy_d2h": (ci, [vp, vp, u64, vp]),
    "fdg_memcpy_d2d": (ci, [vp, vp, u64, vp]),
    "fdg_memset": (ci, [vp, ci, u64, vp]),
    "fdg_stream_create": (ci, [C.POINTER(vp)]),
    "fdg_stream_destroy": (ci, [vp]),
    "fdg_stream_sync": (ci, [vp]),
    "fdg_device_sync": (ci, []),
    "fdg_event_create": (ci, [C.POINTER(vp)]),
    "fdg_event_destroy": (ci, [vp]),
    "fdg_event_record": (ci, [vp, vp]),
    "fdg_stream_wait_event": (ci, [vp, vp]),
    "fdg_event_elapsed_ms": (ci, [vp, vp, C.POINTER(C.c_float)]),
    "fdg_event_sync": (ci, [vp]),
    "fdg_mem_info": (ci, [C.POINTER(u64), C.POINTER(u64)]),
    "fdg_ctx_create": (ci, [ci, C.POINTER(vp)]),
    "fdg_ctx_destroy": (ci, [vp]),
    "fdg_ctx_info_get": (ci, [vp, C.POINTER(CtxInfo)]),
    "fdg_ctx_load_topology": (ci, [vp, vp, u64, vp, u64]),
    "fdg_ctx_load_topology_files": (ci, [vp, C.c_char_p]),
    "fdg_ctx_generate_topology": (ci, [vp, u64, u64, u32]),
    "fdg_ctx_load_features": (ci, [vp, vp, u64, u32, u32]),
    "fdg_ctx_load_features_file": (ci, [vp, C.c_char_p]),
    "fdg_ctx_generate_features": (ci, [vp, u64, u64, u32, u32, u32]),
    "fdg_ctx_set_feature_shards": (ci, [vp, vp, u32, u64, u64, u32, u32]),
    "fdg_ctx_download_topology": (ci, [vp, vp, vp]),
    "fdg_ctx_generate_feature_shard": (ci, [vp, u64, u64, u32, u32, u32, u32, C.POINTER(vp)]),
    "fdg_ipc_get_handle": (ci, [vp, vp]),
    "fdg_ipc_open_handle": (ci, [vp, C.POINTER(vp)]),
    "fdg_ipc_close_handle": (ci, [vp]),
    "fdg_ctx_download_rows": (ci, [vp, u64, u64, vp]),
    "fdg_ctx_features_to_host": (ci, [vp]),
    "fdg_ctx_features_on_host": (ci, [vp]),
    "fdg_sampler_create": (ci, [vp, u32, vp, u32, C.POINTER(vp)]),
    "fdg_sampler_destroy": (ci, [vp]),
    "fdg_sampler_capacity": (ci, [vp, C.POINTER(u64), C.POINTER(u64)]),
    "fdg_sample_khop": (ci, [vp, vp, vp, u32, u64, vp, vp, u64, vp]),
    "fdg_sampler_prefetch": (ci, [vp, vp, vp, u32]),
    "fdg_sample_khop_host": (ci, [vp, vp, u32, u64, vp, vp, u64, vp, vp, vp, vp]),
    "fdg_sample_khop_words_host": (ci, [vp, vp, u32, vp, u64, vp, vp, u64, vp, vp, vp]),
    "fdg_mt_stream": (ci, [vp, u64, u64, vp]),
    "fdg_gather": (ci, [vp, vp, vp, vp, u64, vp, vp]),
    "fdg_checksum_alias": (ci, [vp, vp, vp, vp, vp, u64, vp]),
    "fdg_set_gather_impl": (ci, [ci]),
    "fdg_set_option": (ci, [C.c_char_p, C.c_int64]),
    "fdg_get_option": (ci, [C.c_char_p, C.POINTER(C.c_int64)]),
    "fdg_bm_create": (ci, [vp, u64, u64, u32, C.POINTER(vp)]),
    "fdg_bm_destroy": (ci, [vp]),
    "fdg_bm_extract": (ci, [vp, vp, vp, vp, u64, vp, vp, vp]),
    "fdg_bm_release": (ci, [vp, vp, vp, vp, u64]),
    "fdg_bm_stats_get": (ci, [vp, C.POINTER(BmStats)]),
    "fdg_bm_status": (ci, [vp]),
    "fdg_bm_region": (vp, [vp]),
    "fdg_bm_entry": (ci, [vp, u64, C.POINTER(i64), C.POINTER(u32), C.POINTER(u32)]),
    "fdg_bm_reverse": (ci, [vp, u64, C.POINTER(i64)]),
    "fdg_bm_validate": (ci, [vp]),
    "fdg_bm_ring_info": (ci, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)]),
    "fdg_pipeline_create": (ci, [vp, vp, u32, C.POINTER(PipelineConfig), C.POINTER(vp)]),
    "fdg_pipeline_destroy": (ci, [vp]),
    "fdg_pipeline_run": (ci, [vp, vp, ci, vp, u64, vp, vp, C.POINTER(C.c_float)]),
    "fdg_pipeline_records": (ci, [vp, u64, u64, vp]),
    "fdg_pipeline_extract_times": (ci, [vp, u64, u64, vp, vp]),
    "fdg_pipeline_run_ragged": (ci, [vp, vp, ci, u64, vp, u64, vp, vp, vp]),
    "fdg_pipeline_sample_times": (ci, [vp, vp, vp]),
    "fdg_pipeline_bm_stats": (ci, [vp, C.POINTER(BmStats)]),
    "fdg_pipeline_get_config": (ci, [vp, C.POINTER(PipelineConfig)]),
    "fdg_sage_create": (ci, [vp, vp, u32, vp, u32, C.POINTER(vp)]),
    "fdg_sage_destroy": (ci, [vp]),
    "fdg_sage_set_layer": (ci, [vp, u32, vp, vp, vp]),
    "fdg_sage_forward": (ci, [vp, vp, vp, vp, vp, vp, u64, vp, vp]),
    "fdg_sage_get_layer": (ci, [vp, u32, ci, vp, vp, vp]),
    "fdg_sage_buffers": (ci, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(u64)]),
    "fdg_sage_backward": (ci, [vp, vp, vp, vp, vp, u64]),
    "fdg_sage_sgd": (ci, [vp, vp, C.c_float]),
    "fdg_sage_wgrad_test": (ci, [vp, vp, u32, u32, u32, u32, vp]),
    "fdg_pipeline_set_model": (ci, [vp, vp, u64]),
    "fdg_pipeline_set_training": (ci, [vp, C.c_float]),
    "fdg_pipeline_losses": (ci, [vp, u64, u64, vp]),
    "fdg_partition_epoch": (ci, [vp, u64, u64, u64, vp]),
    "fdg_batch_seed": (u64, [u64, u64, u64]),
}

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libfdg.so; raises if it was not built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libfdg.so not built at {path}; run __graft_entry__.build() "
                          f"or `make -C {os.path.join(HERE, 'csrc')}`")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError = a declared symbol is missing
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def header_symbols(header: str = HEADER) -> list[str]:
    import re
    src = open(header).read()
    return sorted(set(re.findall(r"\b(fdg_[a-z0-9_]+)\s*\(", src)))


def last_error() -> str:
    return load().fdg_last_error().decode(errors="replace")
