/*
 * fdg.h -- C ABI of the B200-native GNNDrive sample -> extract path.
 *
 * This is the drop-in boundary: the reference (featdrive, header-only C++20)
 * has no FFI of its own, so each entry point below replaces one concrete
 * reference interface (cited file:line, relative to
 * /root/reference/proj/include/featdrive). Plain pointers and sizes only.
 * Pointers suffixed `_dev` are device (HBM) pointers; `stream` is a
 * cudaStream_t passed as void* (NULL = the legacy default stream).
 *
 * Error convention: every function returns an fdg_status; on failure a
 * thread-local message is available from fdg_last_error(). Reference exception
 * types map as: std::out_of_range -> FDG_OUT_OF_RANGE, std::invalid_argument ->
 * FDG_INVALID_ARG, InvariantViolation -> FDG_INVARIANT, StandbyTimeout ->
 * FDG_CAPACITY, dataset-file std::runtime_error / std::system_error -> FDG_IO_ERROR
 * (+ fdg_last_errno). The C++ shim (include/featdrive_gpu.hpp) rethrows those types.
 * Asynchronous calls report device-detected errors through fdg_batch_counts.status.
 */
#ifndef FDG_H
#define FDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDG_MAX_LAYERS 8

typedef enum {
    FDG_OK = 0,
    FDG_OUT_OF_RANGE = 1, /* seed / node id >= num_nodes   (sampling.hpp:90-91, feature_file.hpp:74-76) */
    FDG_INVALID_ARG = 2,  /* bad fanouts / config          (sampling.hpp:24-28, pipeline.hpp:56-65)    */
    FDG_INVARIANT = 3,    /* buffer-manager invariant      (common.hpp:57-65, buffer_manager.hpp:478)  */
    FDG_CAPACITY = 4,     /* standby list / arena exhausted (buffer_manager.hpp:274-279)               */
    FDG_CUDA_ERROR = 5,
    FDG_NOT_LOADED = 6,   /* topology / features not resident yet                                        */
    FDG_REJECTION = 7,    /* internal: Lemire rejection seen, batch re-run exactly (never user visible) */
    FDG_IO_ERROR = 8      /* dataset file missing / malformed: std::runtime_error, or std::system_error when
                             fdg_last_errno() != 0 (topology.hpp:76-113, feature_file.hpp:27-51, format.hpp:54-64) */
} fdg_status;

typedef struct fdg_ctx fdg_ctx;         /* device + resident CSC topology + feature table (shards)   */
typedef struct fdg_sampler fdg_sampler; /* per-stream sampling workspace                             */
typedef struct fdg_bm fdg_bm;           /* GPU feature-buffer manager                                */

/* Device-written per-batch record (the async counterpart of SampledBatch sizes,
 * pipeline/stats.hpp:19-25 BatchRecord, plus per-layer block offsets). */
typedef struct {
    uint32_t status;        /* fdg_status of the batch (device-detected)                         */
    uint32_t n_nodes;       /* SampledBatch.nodes.size()                                          */
    uint32_t n_edges;       /* SampledBatch.edges.size()                                          */
    uint32_t rejections;    /* Lemire rejections observed (0 in practice)                         */
    uint64_t bad_seed;      /* first out-of-range seed when status == FDG_OUT_OF_RANGE             */
    uint64_t checksum;      /* trainer_step checksum when a fused gather ran (pipeline.hpp:103-124) */
    uint32_t bad_seed_pos;
    uint32_t n_layers;
    uint32_t layer_nodes[FDG_MAX_LAYERS + 2]; /* nodes before layer l's new nodes; [1] = #unique seeds */
    uint32_t layer_edges[FDG_MAX_LAYERS + 1]; /* edges before layer l                               */
    uint32_t layer_draws[FDG_MAX_LAYERS + 1]; /* MT19937-64 words before layer l                    */
    uint32_t words_used;
    uint32_t replays;       /* in-stream exact re-runs of the batch (a Lemire rejection, or more MT
                               words drawn than the prefetched estimate); results are unaffected   */
} fdg_batch_counts;

typedef struct {
    uint64_t num_nodes;
    uint64_t num_edges;
    uint32_t idx_bytes;     /* 4 when num_nodes < 2^32 (indices stored as u32), else 8 */
    uint32_t row_bytes;     /* feature row bytes (0 if no features)                    */
    uint32_t dtype;         /* 0 = f32 (reference format, format.hpp:58-61), 1 = f16   */
    uint32_t n_shards;
    const void* indptr_dev; /* u64[num_nodes+1]                                         */
    const void* indices_dev;
    const void* table_dev;  /* shard 0 base (row-major, no header)                       */
    uint64_t rows_per_shard;
    int device;
    int pad;
} fdg_ctx_info;

const char* fdg_last_error(void);
/* errno of the failed system call behind the last FDG_IO_ERROR on this thread (0: a format
 * error). The reference throws std::system_error(errno, generic_category(), context) there. */
int fdg_last_errno(void);
int fdg_version(void);

/* ---- device plumbing (so callers need no CUDA runtime of their own) ---------- */
int fdg_device_count(int* n);
int fdg_set_device(int device);
/* Loads and stores of `device` may address `peer`'s memory directly (NVLink); used by a
 * single process that installs another GPU's shard with fdg_ctx_set_feature_shards. */
int fdg_enable_peer_access(int device, int peer);
int fdg_malloc(void** ptr_dev, uint64_t bytes);
int fdg_free(void* ptr_dev);
int fdg_host_alloc(void** ptr, uint64_t bytes); /* pinned */
int fdg_host_free(void* ptr);
int fdg_memcpy_h2d(void* dst_dev, const void* src, uint64_t bytes, void* stream);
int fdg_memcpy_d2h(void* dst, const void* src_dev, uint64_t bytes, void* stream);
int fdg_memcpy_d2d(void* dst_dev, const void* src_dev, uint64_t bytes, void* stream);
int fdg_memset(void* dst_dev, int value, uint64_t bytes, void* stream);
int fdg_stream_create(void** stream);
int fdg_stream_destroy(void* stream);
int fdg_stream_sync(void* stream);
int fdg_device_sync(void);
int fdg_event_create(void** ev);
int fdg_event_destroy(void* ev);
int fdg_event_record(void* ev, void* stream);
int fdg_stream_wait_event(void* stream, void* ev);
int fdg_event_elapsed_ms(void* start, void* end, float* ms);
int fdg_event_sync(void* ev);
int fdg_mem_info(uint64_t* free_bytes, uint64_t* total_bytes);

/* ---- context: replaces graph::Topology (topology.hpp:33-193) and the feature
 *      table reader storage::FeatureTable (feature_file.hpp:25-107) ------------- */
int fdg_ctx_create(int device, fdg_ctx** out);
int fdg_ctx_destroy(fdg_ctx* ctx);
int fdg_ctx_info_get(const fdg_ctx* ctx, fdg_ctx_info* out);
/* Host CSC arrays as in indptr.bin / indices.bin (format.hpp:9-12); validated like
 * Topology::load_indptr (topology.hpp:76-105). */
int fdg_ctx_load_topology(fdg_ctx* ctx, const uint64_t* indptr, uint64_t num_nodes,
                          const uint64_t* indices, uint64_t num_edges);
int fdg_ctx_load_topology_files(fdg_ctx* ctx, const char* dataset_dir);
/* Bit-exact GPU port of storage::synthetic_in_degree / synthetic_in_neighbors
 * (generator.hpp:85-121) building the CSC directly in HBM. */
int fdg_ctx_generate_topology(fdg_ctx* ctx, uint64_t seed, uint64_t num_nodes, uint32_t avg_degree);
/* Feature rows, packed by node id (format.hpp:42). */
int fdg_ctx_load_features(fdg_ctx* ctx, const void* rows, uint64_t num_nodes, uint32_t row_bytes, uint32_t dtype);
int fdg_ctx_load_features_file(fdg_ctx* ctx, const char* features_bin);
/* Bit-exact GPU port of storage::synthetic_row (generator.hpp:65-81); dtype 1
 * stores RN(f32 -> f16) of the same values. n_shards > 1 splits rows into
 * contiguous blocks of ceil(N / n_shards) (owner = node / rows_per_shard). */
int fdg_ctx_generate_features(fdg_ctx* ctx, uint64_t seed, uint64_t num_nodes, uint32_t dim, uint32_t dtype,
                              uint32_t n_shards);
/* Row-sharded table: shard s lives at bases[s] (local or NVLink peer pointer). */
int fdg_ctx_set_feature_shards(fdg_ctx* ctx, const void* const* bases_dev, uint32_t n_shards,
                               uint64_t rows_per_shard, uint64_t num_nodes, uint32_t row_bytes, uint32_t dtype);
int fdg_ctx_download_topology(const fdg_ctx* ctx, uint64_t* indptr, void* indices /* idx_bytes each */);
/* Out-of-core tier (the paper's host-resident feature store): move the
 * context's single-shard table to pinned host memory mapped into the device address space.
 * fdg_gather and the buffer manager's misses then read rows over PCIe / C2C with the same
 * kernels; put a buffer manager (fdg_bm_* / use_buffer_manager) in front of it so hits are
 * served from HBM slots. fdg_ctx_features_on_host returns 1 when the table lives on the host. */
int fdg_ctx_features_to_host(fdg_ctx* ctx);
int fdg_ctx_features_on_host(const fdg_ctx* ctx);

/* ---- multi-GPU: one process per GPU, row-sharded feature table read over NVLink ----
 * Rank r generates only its block of rows (owner = node / ceil(N / n_shards)) into a
 * fresh allocation owned by the context, exports it with a CUDA IPC handle, opens
 * the peers' handles, and installs all bases with fdg_ctx_set_feature_shards; the
 * gather then loads remote rows directly through the peer mappings (one-sided, no
 * collective). */
int fdg_ctx_generate_feature_shard(fdg_ctx* ctx, uint64_t seed, uint64_t num_nodes, uint32_t dim, uint32_t dtype,
                                   uint32_t shard, uint32_t n_shards, void** base_dev);
#define FDG_IPC_HANDLE_BYTES 64
int fdg_ipc_get_handle(const void* base_dev, unsigned char* handle /* FDG_IPC_HANDLE_BYTES */);
int fdg_ipc_open_handle(const unsigned char* handle, void** base_dev);
int fdg_ipc_close_handle(void* base_dev);
int fdg_ctx_download_rows(const fdg_ctx* ctx, uint64_t first, uint64_t count, void* out);

/* ---- sampler: replaces graph::sample_khop (sampling.hpp:72-134) --------------- */
/* Workspace for batches of <= max_seeds seeds with the given fanouts; fanouts are
 * validated as Fanouts::validate (sampling.hpp:23-29). */
int fdg_sampler_create(fdg_ctx* ctx, uint32_t max_seeds, const uint32_t* fanouts, uint32_t n_layers,
                       fdg_sampler** out);
int fdg_sampler_destroy(fdg_sampler* s);
/* Fanouts::max_batch_nodes (sampling.hpp:32-40) clamped to N (pipeline.hpp:69-71), and the edge bound. */
int fdg_sampler_capacity(const fdg_sampler* s, uint64_t* max_nodes, uint64_t* max_edges);
/* Asynchronous sample on `stream`. seeds_dev: u64[n_seeds]. Outputs: nodes_dev u64[cap],
 * edges_dev u32[2*cap] as {src_local, dst_local} (LocalEdge, sampling.hpp:43-46),
 * counts_dev: device fdg_batch_counts. cap must be >= fdg_sampler_capacity. */
int fdg_sample_khop(fdg_sampler* s, void* stream, const uint64_t* seeds_dev, uint32_t n_seeds,
                    uint64_t rng_seed, uint64_t* nodes_dev, uint32_t* edges_dev, uint64_t cap,
                    fdg_batch_counts* counts_dev);
/* Pre-generate the MT19937-64 streams of upcoming batches on `stream` (off the
 * critical path); a later fdg_sample_khop with the same rng_seed consumes them. */
int fdg_sampler_prefetch(fdg_sampler* s, void* stream, const uint64_t* rng_seeds, uint32_t n);
/* Synchronous convenience with host buffers and the reference's exact error
 * behaviour (first out-of-range seed in order -> FDG_OUT_OF_RANGE). A batch that
 * hit a Lemire rejection is transparently re-run in the exact (serialised
 * offset) mode. layer_nodes[L+2] / layer_edges[L+1] may be NULL. */
int fdg_sample_khop_host(fdg_sampler* s, const uint64_t* seeds, uint32_t n_seeds, uint64_t rng_seed,
                         uint64_t* nodes, uint32_t* edges, uint64_t cap, uint64_t* n_nodes, uint64_t* n_edges,
                         uint64_t* layer_nodes, uint64_t* layer_edges);
/* Test hook: as fdg_sample_khop_host but drawing from an explicit word stream
 * instead of MT19937-64 (exercises the Lemire rejection path exactly). */
int fdg_sample_khop_words_host(fdg_sampler* s, const uint64_t* seeds, uint32_t n_seeds, const uint64_t* words,
                               uint64_t n_words, uint64_t* nodes, uint32_t* edges, uint64_t cap,
                               uint64_t* n_nodes, uint64_t* n_edges, uint64_t* words_used);
/* MT19937-64 words of std::mt19937_64(splitmix64(rng_seed)) (sampling.hpp:78), on device. */
int fdg_mt_stream(void* stream, uint64_t rng_seed, uint64_t n, uint64_t* out_dev);

/* ---- extraction: the mini-batch gather -------------------------------------- */
/* out_dev[i, :] = row(nodes_dev[i]) for i < n (n = *n_dev when n_dev != NULL, else
 * n_host). When checksum_dev != NULL it also accumulates trainer_step's
 * order-insensitive checksum sum_i hash_bytes64(row) (pipeline.hpp:103-124,
 * common.hpp:88-105) into *checksum_dev (caller zeroes it). */
int fdg_gather(fdg_ctx* ctx, void* stream, const uint64_t* nodes_dev, const uint32_t* n_dev, uint64_t n_host,
               void* out_dev, uint64_t* checksum_dev);
/* Gather engines. fdg_gather (standalone) defaults to FDG_GATHER_RB_DYN (32-row groups
 * claimed dynamically, 256-byte row chunks; other row sizes fall back to the 16-byte LDG/STG
 * kernels); the pipeline runner uses option "pipeline_gather_impl" (default FDG_GATHER_LDG,
 * chunk-striped with dynamic claiming). Sharded tables always take the row-group kernel.
 * The fused-checksum gather uses option "checksum_impl" (default LDG: compile-time row-size
 * kernels for the benchmarked rows, a software-pipelined kernel for other 16-byte multiples,
 * a generic one otherwise). FDG_GATHER_TMA moves rows with cp.async.bulk (the TMA). */
#define FDG_GATHER_TMA 0
#define FDG_GATHER_LDG 1
#define FDG_GATHER_RB_DYN 4 /* 32-row groups claimed dynamically from a per-launch counter */
int fdg_set_gather_impl(int impl);
/* Tuning knobs (process-wide; fdg_api.cu lists all, with their ranges). Main ones:
 * "gather_impl" / "pipeline_gather_impl" / "checksum_impl" (FDG_GATHER_*),
 * "gather_evict_first" (0-3: L2 evict-first hints on the gather stream), "l2_persist_mb"
 * (L2 set-aside for the samplers' hash tables; 0 = off), "hash_load_pct" (hash table
 * sizing), "extract_streams" (1/2), "sage_gemm" (1 tcgen05 3xTF32, 0 CUDA cores),
 * "bm_overlap" (buffer-manager row move on its own stream), "sampler_sms" (> 0: pipeline
 * samplers on a green-context SM partition of that size, extraction on the rest; measured
 * slower than sharing, default 0), "tma_cfg" (TMA gather ring shape 0-3).
 * Round 2: "early_bloom" (Bloom filter before the last layer's early-table lookups, 1),
 * "intern_lean" (lean next-frontier intern passes: 0 never, 1 always, 2 pipelines without the
 * checksum), "early_fused" (seeds + layer 0 in one shared-memory CTA, 0), "bm_fuse_bind" (1),
 * "bm_move_impl" (0 LDG, 1 TMA, 2 row groups), "bm_move_hash" (move + checksum in one pass, 1),
 * "bm_split_move" (0), "extract_prio" (0, 1, 2 = with the buffer manager), "records_stream" (1),
 * "hash_ctas_per_sm" (1) / "hash_ctas" (0), "pipe_slots" (0 = 2 x samplers x group),
 * "tc_write_hi" (read-only: the kind::tf32 truncation check), "force_idx64" (test hook).
 * Loading the library sets CUDA_DEVICE_MAX_CONNECTIONS=32 unless the process already did. */
int fdg_set_option(const char* key, int64_t value);
int fdg_get_option(const char* key, int64_t* value);
/* Checksum of rows already resident (region slot payloads addressed by alias). */
int fdg_checksum_alias(fdg_ctx* ctx, void* stream, const void* region_dev, const int64_t* alias_dev,
                       const uint32_t* n_dev, uint64_t n_host, uint64_t* checksum_dev);

/* ---- buffer manager: replaces featbuf::BufferManager (buffer_manager.hpp:222-527),
 *      FeatureRegion (device_region.hpp:24-50) and Extractor::extract_batch
 *      (extractor.hpp:88-113) ---------------------------------------------------- */
typedef struct {
    uint64_t hits, loads, waits, evictions, takeovers, releases, standby_len;
} fdg_bm_stats;

/* slot_count >= min_reserved (N_e * M_b rule, buffer_manager.hpp:229-231). */
int fdg_bm_create(fdg_ctx* ctx, uint64_t slot_count, uint64_t min_reserved, uint32_t max_batch_nodes,
                  fdg_bm** out);
int fdg_bm_destroy(fdg_bm* bm);
/* Algorithm 1 for one batch, stream-ordered: acquire_for_batch (241-269), LRU
 * standby pops with eviction (274-294), bind (297-310), table -> slot row copies
 * for the misses, publish (313-324). alias_dev: i64[n] (NodeAliasList). When
 * out_dev != NULL the mini-batch tensor X[i] = slot(alias[i]) is also written. */
int fdg_bm_extract(fdg_bm* bm, void* stream, const uint64_t* nodes_dev, const uint32_t* n_dev, uint64_t n_host,
                   int64_t* alias_dev, void* out_dev, uint64_t* checksum_dev);
/* release_batch (352-364): ref--, MRU append at 0 with the mapping left valid. */
int fdg_bm_release(fdg_bm* bm, void* stream, const uint64_t* nodes_dev, const uint32_t* n_dev, uint64_t n_host);
int fdg_bm_stats_get(fdg_bm* bm, fdg_bm_stats* out); /* synchronises the bm stream */
int fdg_bm_status(fdg_bm* bm);                       /* sticky device-detected status */
void* fdg_bm_region(fdg_bm* bm);                     /* FeatureRegion base: slot s at s*row_bytes */
/* Introspection for tests (mapping_entry / reverse_mapping, buffer_manager.hpp:420-429). */
int fdg_bm_entry(fdg_bm* bm, uint64_t node, int64_t* slot, uint32_t* ref, uint32_t* valid);
int fdg_bm_reverse(fdg_bm* bm, uint64_t slot, int64_t* node);
/* Full invariant sweep (validate_locked, buffer_manager.hpp:488-515) on a host copy. Mapping
 * entries are invalidated lazily (an entry is live while its slot still names the node); a
 * buffer manager created with option "bm_eager_invalidate" = 1 clears the previous owner's entry
 * on every eviction as the reference does (buffer_manager.hpp:284-287), and its validate then
 * treats any stale entry as a corruption. */
int fdg_bm_validate(fdg_bm* bm);
/* ---- the reference's object split and per-node protocol (the C++ drop-in) ----------
 * featbuf::BufferManager(BufferConfig) holds no table: a standalone buffer manager has its
 * metadata on `device` and gets its miss source and its FeatureRegion (slot_count x
 * row_bytes device bytes owned by the caller, e.g. a featbuf::FeatureRegion; NULL = allocated
 * by the buffer manager) when an Extractor binds them (ExtractorEnv, extractor.hpp:58-66). */
int fdg_bm_create_standalone(int device, uint64_t num_nodes, uint64_t slot_count, uint32_t row_bytes,
                             uint64_t min_reserved, uint32_t max_batch_nodes, void* region_dev, fdg_bm** out);
int fdg_bm_bind_table(fdg_bm* bm, const fdg_ctx* table, void* region_dev);
/* acquire_for_batch (buffer_manager.hpp:241-269): alias_dev[i] = slot of a hit, -1 otherwise;
 * to_load_dev[0..*n_load_dev) = positions to load, in batch order (device outputs). Misses
 * take their reference when bound. */
int fdg_bm_acquire(fdg_bm* bm, void* stream, const uint64_t* nodes_dev, uint64_t n, int64_t* alias_dev,
                   uint32_t* to_load_dev, uint32_t* n_load_dev);
/* get_standby_slot x count (274-294): the LRU slots, previous owners evicted, in pop order. */
int fdg_bm_pop_standby(fdg_bm* bm, void* stream, uint32_t count, int64_t* slots_dev);
/* bind_slot (297-310) and publish_valid (313-324) for n (node, slot) pairs / nodes. */
int fdg_bm_bind(fdg_bm* bm, void* stream, const uint64_t* nodes_dev, const int64_t* slots_dev, uint32_t n);
int fdg_bm_publish(fdg_bm* bm, void* stream, const uint64_t* nodes_dev, uint32_t n);
/* unwind_bound (372-388) and release_ref (392-400) of one node. */
int fdg_bm_unwind_bound(fdg_bm* bm, void* stream, uint64_t node);
int fdg_bm_release_ref(fdg_bm* bm, void* stream, uint64_t node);
/* The load + transfer of planned misses: table rows -> region slots. */
int fdg_bm_load_rows(fdg_bm* bm, void* stream, const uint64_t* nodes_dev, const int64_t* slots_dev, uint32_t n);
/* trainer_step over a FeatureRegion (pipeline.hpp:103-124): *checksum_dev += sum_i
 * hash_bytes64(region[alias[i]]); and its verify: *first_bad_dev = the smallest i whose
 * region row differs from the table row of nodes[i] (~0 when all equal). */
int fdg_region_checksum(void* stream, const void* region_dev, uint32_t row_bytes, const int64_t* alias_dev, uint64_t n,
                        uint64_t* checksum_dev);
int fdg_region_verify(const fdg_ctx* table, void* stream, const void* region_dev, const int64_t* alias_dev,
                      const uint64_t* nodes_dev, uint64_t n, uint64_t* first_bad_dev);
/* Standby-ring geometry for tests: positions [head, tail) of capacity `capacity`, and the number
 * of tombstone compactions so far. */
int fdg_bm_ring_info(fdg_bm* bm, uint64_t* head, uint64_t* tail, uint64_t* capacity, uint64_t* compactions);

/* ---- native SET-loop runner: PipelineSession's sampler / extractor / trainer /
 *      releaser stages for one worker = one GPU (pipeline.hpp:325-543) ------------ */
typedef struct fdg_pipeline fdg_pipeline;
typedef struct {
    uint32_t batch_size;          /* seeds per batch (PipelineConfig::batch_size, pipeline.hpp:37)       */
    uint32_t n_samplers;          /* concurrent sampler workspaces/streams (0 -> 2)                      */
    uint32_t prefetch_group;      /* MT19937-64 streams generated per launch, per sampler (0 -> 16)     */
    uint32_t use_buffer_manager;  /* extract through the GPU BufferManager (config 3)                    */
    uint64_t buffer_slots;        /* S when use_buffer_manager                                           */
    uint32_t write_x;             /* materialise the mini-batch tensor X (always on for the plain gather) */
    uint32_t checksum;            /* fuse trainer_step's checksum (pipeline.hpp:103-124)                 */
    uint32_t flags;               /* diagnostics: FDG_PIPE_SAMPLE_ONLY / FDG_PIPE_EXTRACT_ONLY           */
    float host_enqueue_ms;        /* out: host time spent enqueueing the last run                        */
    uint32_t group_batches;       /* batches sampled per launch chain (0 -> 4, max 8)                    */
} fdg_pipeline_config;
#define FDG_PIPE_SAMPLE_ONLY 1u   /* skip extraction (sampler throughput)                                 */
#define FDG_PIPE_EXTRACT_ONLY 2u  /* sample each slot once, then only extract (extraction throughput)    */
#define FDG_PIPE_NO_L2_PERSIST 4u /* do not pin the samplers' hash tables in L2                          */
#define FDG_PIPE_NO_PRIORITY 8u   /* equal stream priorities for sampling and extraction                 */
/* Current configuration (including host_enqueue_ms of the last run). */
int fdg_pipeline_get_config(const fdg_pipeline* p, fdg_pipeline_config* out);

int fdg_pipeline_create(fdg_ctx* ctx, const uint32_t* fanouts, uint32_t n_layers, const fdg_pipeline_config* cfg,
                        fdg_pipeline** out);
int fdg_pipeline_destroy(fdg_pipeline* p);
/* Runs n_batches batches; batch j uses seeds[j*batch_size ...] (device memory, or
 * pinned host memory copied per batch when seeds_on_host) and rng_seeds[j] (host).
 * records_host (nullable, pinned for async) receives each batch's fdg_batch_counts
 * by an in-stream D2H copy; extract_ms (nullable) per-batch extraction kernel time;
 * elapsed_ms = device time of the whole run. Synchronises before returning. */
int fdg_pipeline_run(fdg_pipeline* p, const uint64_t* seeds, int seeds_on_host, const uint64_t* rng_seeds,
                     uint64_t n_batches, fdg_batch_counts* records_host, float* extract_ms, float* elapsed_ms);
/* As fdg_pipeline_run, but the seed list holds n_seeds_total seeds: batch j takes
 * [j*batch_size, min((j+1)*batch_size, n_seeds_total)) -- the last chunk of
 * partition_epoch (sampling.hpp:57-70) may be short. */
int fdg_pipeline_run_ragged(fdg_pipeline* p, const uint64_t* seeds, int seeds_on_host, uint64_t n_seeds_total,
                            const uint64_t* rng_seeds, uint64_t n_batches, fdg_batch_counts* records_host,
                            float* extract_ms, float* elapsed_ms);
/* Sampling stage time of the last run (which must have passed extract_ms): the sum over
 * launch groups of the sampler stream's busy interval (sample_busy of EpochStats). */
int fdg_pipeline_sample_times(fdg_pipeline* p, uint64_t* n_groups, float* busy_ms);
/* Buffer-manager counters of a pipeline created with use_buffer_manager (cumulative
 * over its runs; FDG_NOT_LOADED without a buffer manager). */
int fdg_pipeline_bm_stats(fdg_pipeline* p, fdg_bm_stats* out);
/* Device batch records of the last run, [first, first+n). */
int fdg_pipeline_records(fdg_pipeline* p, uint64_t first, uint64_t n, fdg_batch_counts* out);
/* Extraction intervals of the last run (which must have passed extract_ms): start/end of
 * batch j's extraction launches in ms from the start of the run (one device timeline, so
 * launches alternating over the two extraction streams can be unioned). */
int fdg_pipeline_extract_times(fdg_pipeline* p, uint64_t first, uint64_t n, float* start_ms, float* end_ms);

/* ---- train stage: GraphSAGE forward + loss on a sampled batch --------------------------
 * The consumer of the mini-batch tensor. The reference's trainer is a checksum
 * (trainer_step, pipeline.hpp:103-124); the paper trains a 3-layer GraphSAGE on these
 * blocks. Model (PyG SAGEConv, mean aggregator): layer
 * k = 1..L computes local nodes [0, D_{L-k}), D_j = layer_nodes[j+1] (nodes within j
 * hops), as h_v = W_neigh . mean_{(u->v) in edges} h_u + W_self . h_v + b, ReLU between
 * layers, h^0 = X; loss = mean softmax cross-entropy over the unique seeds with
 * label(v) = splitmix64(node_id ^ label_seed) % dims[L]. fp32 (CUDA-core FMA).
 * dims: L+1 widths, dims[0] = feature width of the context's table (f32 or f16), every
 * dim a multiple of 4; fanouts / max_seeds bound the block sizes (sampling.hpp:32-40). */
typedef struct fdg_sage fdg_sage;
int fdg_sage_create(fdg_ctx* ctx, const uint32_t* dims, uint32_t n_layers, const uint32_t* fanouts,
                    uint32_t max_seeds, fdg_sage** out);
int fdg_sage_destroy(fdg_sage* m);
/* Host fp32 weights of layer `layer`: w_neigh, w_self [dims[layer]][dims[layer+1]] row-major
 * (input-major: out = in . W), bias [dims[layer+1]] (NULL = 0). */
int fdg_sage_set_layer(fdg_sage* m, uint32_t layer, const float* w_neigh, const float* w_self, const float* bias);
/* Stream-ordered forward on one batch: x_dev = X [n_nodes][dims[0]] (table dtype), nodes /
 * edges / counts as written by fdg_sample_khop. *loss_dev (device float) = the loss;
 * logits_dev (nullable) = [D_0][dims[L]]. */
int fdg_sage_forward(fdg_sage* m, void* stream, const void* x_dev, const uint64_t* nodes_dev,
                     const uint32_t* edges_dev, const fdg_batch_counts* counts_dev, uint64_t label_seed,
                     float* loss_dev, float* logits_dev);
/* Host copies of layer `layer`'s current weights (grads = 0) or of its gradients from the
 * last fdg_sage_backward (grads = 1), in fdg_sage_set_layer's layout; NULL outputs skipped. */
int fdg_sage_get_layer(fdg_sage* m, uint32_t layer, int grads, float* w_neigh, float* w_self, float* bias);
/* The contiguous device parameter and gradient blocks (same layout: per layer W_neigh, W_self,
 * b): the gradient block is what a data-parallel all-reduce sums between backward and sgd. */
int fdg_sage_buffers(fdg_sage* m, float** params_dev, float** grads_dev, uint64_t* n_floats);
/* Backward of the last forward (same batch, same stream): d(loss)/d(W_neigh, W_self, b) of
 * every layer into the gradient block. ReLU masks, scatter-mean transposed with vector
 * atomics over the dst-sorted blocks, weight gradients as row-sliced A^T . dOut. */
int fdg_sage_backward(fdg_sage* m, void* stream, const uint64_t* nodes_dev, const uint32_t* edges_dev,
                      const fdg_batch_counts* counts_dev, uint64_t label_seed);
/* Test hook: out_dev [Kin x N] = A^T . B (+ the column sums of B appended, [N]) for device
 * A [R x Kin], B [R x N], through the backward's weight-gradient engine in Z row slices. */
int fdg_sage_wgrad_test(const float* A_dev, const float* B_dev, uint32_t R, uint32_t Kin, uint32_t N, uint32_t Z,
                        float* out_dev);
/* SGD step params -= lr * grads (stream-ordered), refreshing the kernels' weight layouts. */
int fdg_sage_sgd(fdg_sage* m, void* stream, float lr);
/* Run the model after each batch's extraction inside fdg_pipeline_run (NULL = off; the
 * pipeline must materialise X). Per-batch losses of the last run: fdg_pipeline_losses. */
int fdg_pipeline_set_model(fdg_pipeline* p, fdg_sage* m, uint64_t label_seed);
int fdg_pipeline_losses(fdg_pipeline* p, uint64_t first, uint64_t n, float* out);
/* Training mode of the train stage: lr != 0 adds backward + SGD after each batch's forward
 * (stream-ordered on the extraction stream; the loss recorded is the pre-update one). */
int fdg_pipeline_set_training(fdg_pipeline* p, float lr);

/* ---- tracing: per-launch CUDA-event timeline (DurationCounter analogue, common.hpp:240-260) */
int fdg_trace_enable(int on);          /* clears previous records when turning on */
int fdg_trace_dump(const char* path);  /* CSV: name,stream,start_ms,end_ms       */

/* ---- host helpers ------------------------------------------------------------------ */
/* partition_epoch (sampling.hpp:57-70) with the same libstdc++ std::shuffle. */
int fdg_partition_epoch(const uint64_t* train_ids, uint64_t n, uint64_t batch_size, uint64_t shuffle_seed,
                        uint64_t* out_ids);
uint64_t fdg_batch_seed(uint64_t seed, uint64_t epoch, uint64_t global_batch); /* pipeline.hpp:295-298 */

#ifdef __cplusplus
}
#endif
#endif /* FDG_H */
