// fdg_internal.cuh -- shared internals of libfdg (B200 / sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "fdg.h"

namespace fdg {

// ---- error plumbing -----------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define FDG_CUDA(call)                                                        \
    do {                                                                      \
        cudaError_t _e = (call);                                              \
        if (_e != cudaSuccess) return ::fdg::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

#define FDG_TRY(call)                      \
    do {                                   \
        int _rc = (call);                  \
        if (_rc != FDG_OK) return _rc;     \
    } while (0)

// ---- tracing (fdg_trace.cu) --------------------------------------------------------
extern bool g_trace;
class TraceScope {  // records events around the enclosed launches when tracing is on
public:
    TraceScope(const char* name, cudaStream_t st);
    ~TraceScope();

private:
    const char* name_;
    cudaStream_t st_;
    cudaEvent_t a_ = nullptr;
};
#define FDG_CAT2(a, b) a##b
#define FDG_CAT(a, b) FDG_CAT2(a, b)
#define FDG_TRACE(name, st) ::fdg::TraceScope FDG_CAT(_fdg_trace_, __LINE__)(name, st)


// Random loads with a 64-byte L2 fill. B200 fills a random load miss with a whole 128-byte
// line by default (scripts/probes/rand_gran.cu under ncu: 129.6 DRAM bytes per random 8-byte
// load under every cudaLimitMaxL2FetchGranularity setting); the .L2::64B prefetch-size hint
// halves that (66.8 B). Stores are sector-granular already (34 B read + 30 B written per
// random 8-byte store). FDG_RAND64=0 builds plain loads (A/B).
#ifndef FDG_RAND64
#define FDG_RAND64 1
#endif
__device__ __forceinline__ uint64_t ld_rand64(const void* p) {
    uint64_t v;
#if FDG_RAND64
    asm volatile("ld.global.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(p));
#else
    v = *static_cast<const uint64_t*>(p);
#endif
    return v;
}
__device__ __forceinline__ uint32_t ld_rand32(const void* p) {
    uint32_t v;
#if FDG_RAND64
    asm volatile("ld.global.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
#else
    v = *static_cast<const uint32_t*>(p);
#endif
    return v;
}

// ---- reference hashing on device (common.hpp:77-105) ------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t hash_combine(uint64_t a, uint64_t b) {
    return splitmix64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}
// k-th output (k >= 0) of a SplitMix stream seeded with `seed` (common.hpp:112-118):
// the state after k+1 calls is seed + (k+1)*gamma, so any draw is random-access.
__host__ __device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t k) {
    return splitmix64(seed + k * 0x9e3779b97f4a7c15ull);
}

// ---- once-per-device flags (function attributes are per device) --------------------
// first() is true the first time it is called with each current device.
struct PerDeviceOnce {
    unsigned long long mask = 0;
    bool first() {
        int d = 0;
        cudaGetDevice(&d);
        const unsigned long long bit = 1ull << (d & 63);
        return !(__atomic_fetch_or(&mask, bit, __ATOMIC_RELAXED) & bit);
    }
};

// ---- context ---------------------------------------------------------------------
struct Ctx {
    int device = 0;
    uint64_t num_nodes = 0;
    uint64_t num_edges = 0;
    uint32_t idx_bytes = 4;
    uint64_t* indptr = nullptr;   // u64[N+1]
    void* indices = nullptr;      // u32/u64[E]
    // features
    uint32_t row_bytes = 0;
    uint32_t dtype = 0;
    uint32_t n_shards = 0;
    uint64_t rows_per_shard = 0;
    uint64_t feat_nodes = 0;
    std::vector<void*> shard_bases;   // device pointers (may be peers)
    std::vector<void*> owned_shards;  // allocations owned by this ctx
    void* host_table = nullptr;       // out-of-core tier: pinned, mapped host copy (owned)
    uint64_t host_table_bytes = 0;    // > 0: an mmap'ed, registered mapping of this size (THP)
    const void** shard_table = nullptr;  // device copy of shard_bases
    cudaStream_t stream = nullptr;    // setup stream
    int sm_count = 148;
    // Work-claim counter pairs of the dynamically scheduled gathers: a ring on this
    // context's device (a launch takes the next pair; the kernel's last CTA resets it).
    uint32_t* dyn_ring = nullptr;
    mutable uint32_t dyn_next = 0;
};

}  // namespace fdg

struct fdg_ctx : fdg::Ctx {};

namespace fdg {
// generator entry points (fdg_generate.cu)
int generate_topology(Ctx& c, uint64_t seed, uint64_t num_nodes, uint32_t avg_degree);
int generate_features(Ctx& c, uint64_t seed, uint64_t num_nodes, uint32_t dim, uint32_t dtype, uint32_t n_shards);
int generate_feature_shard(Ctx& c, uint64_t seed, uint64_t n, uint32_t dim, uint32_t dtype, uint32_t shard,
                           uint32_t n_shards, void** base);
// MT19937-64 (fdg_mt.cu)
// rng_seeds: HOST array (passed by value to the kernel)
cudaError_t launch_mt_streams(cudaStream_t st, const uint64_t* rng_seeds, uint32_t n_streams,
                              uint64_t words_per_stream, uint64_t* out_dev, uint64_t out_stride);
// one CTA per stream, CTA i writing words [begin, end) (begin a multiple of 312, the last twist
// completed) of its stream to ring + slots[i] * stride; the 312-word engine state after the
// last twist is read from / written to state + slots[i] * 312 (state may be null if begin == 0)
cudaError_t launch_mt_streams_slots(cudaStream_t st, const uint64_t* rng_seeds, const uint32_t* slots,
                                    uint32_t n_streams, uint64_t begin, uint64_t end, uint64_t* ring, uint64_t stride,
                                    uint64_t* state);
// gather (fdg_gather.cu)
int launch_gather(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                  void* out, uint64_t* checksum);
// Tuning options (fdg_set_option; defaults are the measured best, profiles/README.md)
extern int g_gather_impl;             // standalone fdg_gather engine (FDG_GATHER_RB_DYN)
extern int64_t g_pipeline_gather_impl;  // gather engine of the pipeline runner (FDG_GATHER_LDG)
extern int64_t g_checksum_impl;       // engine of the fused-checksum gather (-1: same as g_gather_impl)
extern int g_gather_evict_first;      // L2 evict-first hints on the gather (0 off)
extern int64_t g_gather_pf64;         // 64-byte L2 fetch hint on table reads (0 off, 1 on, 2 rows % 128 != 0)
extern int g_gather_ctas_per_sm;      // chunk-striped gather: CTAs (512 threads) per SM
extern int64_t g_rb_ctas_per_sm;      // row-group gather: CTAs (8 warps) per SM
extern int64_t g_rb_chunk;            // row-group gather: 128- or 256-byte row chunks
extern int64_t g_hash_ctas;           // fused gather + checksum: absolute CTA count (0: per SM)
extern int64_t g_hash_ctas_per_sm;    // fused gather + checksum CTAs per SM (0 = min-blocks)
extern int64_t g_hash_dyn;            // fused gather + checksum: dynamic row-group claims
extern int64_t g_hash_chunk;          // k_gather_hash_rb staging chunk (0 = by row size)
extern int64_t g_hash_dyn;            // fused gather + checksum: row groups claimed dynamically (1) or static (0)
extern int64_t g_tma_cfg;             // TMA gather ring shape 0-3
int tc_write_hi(cudaStream_t st);       // 1: tcgen05 kind::tf32 GEMMs write A_hi (fdg_sage_tc.cu check)
extern int64_t g_sage_gemm;           // train-stage GEMMs: 1 tensor cores (3xTF32), 0 CUDA cores
extern int64_t g_bm_overlap;          // buffer-manager row move on its own stream (1) or after the metadata (0)
extern int64_t g_bm_eager;            // buffer managers created in eager-invalidation (debug) mode
extern int64_t g_bm_move_hash;        // buffer manager: row move + trainer checksum in one pass
extern int64_t g_bm_fuse_bind;        // buffer manager: select and bind in one kernel
extern int64_t g_bm_move_grid;        // buffer-manager LDG row move: 0 persistent grid, 1 a CTA per 64 rows
extern int64_t g_bm_split_move;       // pipeline: X rows moved after the acquire, slot fills after the bind
extern int64_t g_pipe_slots;          // pipeline: per-batch output slots (0: 2 x samplers x group)
extern int64_t g_records_stream;      // pipeline: batch records' D2H on their own stream
extern int64_t g_extract_prio;        // pipeline: extraction streams above the samplers' priority
extern int64_t g_bm_move_early;       // pipeline: batch j's row move starts after its bind, not after release j-1
extern int64_t g_bm_meta_prio;        // pipeline: the buffer manager's metadata stream at high priority
extern int64_t g_bm_move_impl;        // buffer-manager row move: 0 LDG (k_move), 1 TMA bulk copies (k_move_tma)
extern int64_t g_host_tier_pf;        // host-resident table: prefetch-size hint on the row reads (0, 1 = 128B, 2 = 256B)
extern int64_t g_bm_sorted_move;      // host-resident table: move the misses in node-id order
extern int64_t g_l2_persist_mb;       // L2 set-aside for the samplers' hash tables (0 off)
extern int64_t g_hash_load_pct;       // batch hash sizing (load factor, %)
extern int64_t g_force_idx64;         // test hook: u64 CSR indices (the N >= 2^32 kernels) for any N
extern int64_t g_early_bloom;         // sampler: Bloom filter over the early table for the last layer's lookups
extern int64_t g_intern_lean;         // sampler: lean next-frontier intern passes (0 never, 1 always, 2 pipelines without checksum)
extern int64_t g_early_fused;         // sampler: seeds + layer 0 in one shared-memory CTA (k_early)
extern int64_t g_hash_early_pct;      // early batch-hash table load factor (0: hash_load_pct)
extern int64_t g_sampler_ctas_per_sm; // sampler kernels: CTA cap per SM per launch
extern int64_t g_sampler_sms;         // > 0: pipeline samplers on their own green-context SM partition
extern int64_t g_extract_streams;     // 1 or 2 extraction streams in the pipeline runner
extern int64_t g_hash_clear;          // 1: clear batch hash tables with a fill kernel, 0: cudaMemsetAsync
extern int64_t g_hash_keep;           // evict_last L2 policy on the batch hash
extern int64_t g_mt_adaptive;         // prefetch the estimated MT draws (1), the draw bound (0), test (2)
extern int64_t g_replay;              // A/B only: 0 drops the in-stream replay launch
extern int64_t g_prefetch_upfront;
extern int64_t g_host_tier_thp;       // features_to_host on THP-backed registered memory    // A/B only: 1 requests every sampler's first MT chunk before sampling
extern int64_t g_debug_zero_word;     // pipeline test hook (option debug_zero_word)
extern int64_t g_debug_reject_batch;  // pipeline test hook (option debug_reject_batch)
int launch_gather_tma(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                      void* out, uint64_t* checksum, const uint32_t* status);
int launch_checksum_alias(const Ctx& c, cudaStream_t st, const void* region, const int64_t* alias,
                          const uint32_t* n_dev, uint64_t n_host, uint64_t* checksum,
                          const uint32_t* status = nullptr);
constexpr uint32_t kDynRing = 256;  // counter pairs per context
uint32_t* dyn_counter(const Ctx& c);
int launch_move_hash(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                     const uint32_t* status, const int64_t* alias, const uint8_t* is_load, const char* table,
                     char* region, char* out, uint64_t* checksum, int mode = 0);
int launch_gather_bound(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev,
                        uint64_t n_host, uint64_t n_bound, void* out, uint64_t* checksum, const uint32_t* status,
                        bool pipeline = false);
}  // namespace fdg
