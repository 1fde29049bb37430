/*
 * fd_oracle.h -- CPU restatement of GNNDrive/featdrive's sample -> extract path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the CUDA product
 * path (paper_2406_13984_b200/csrc). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product
 * never links or calls it.
 *
 * Every function restates one reference routine (file:line relative to
 * /root/reference/proj/include/featdrive). The restatement is pinned against
 * the reference itself, compiled from its own headers into oracle/_ref
 * (see oracle/Makefile and tests/test_oracle_vs_ref.py), and against the
 * committed golden vectors in tests/golden/ that were produced by that build.
 */
#ifndef FD_ORACLE_H
#define FD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    FDO_OK = 0,
    FDO_OUT_OF_RANGE = 1,  /* std::out_of_range  (sampling.hpp:90-91)   */
    FDO_INVALID_ARG = 2,   /* std::invalid_argument (sampling.hpp:24-28) */
    FDO_INVARIANT = 3,     /* InvariantViolation (common.hpp:36-65)     */
    FDO_CAPACITY = 4,      /* output / standby capacity exhausted       */
    FDO_STREAM_SHORT = 7,  /* explicit word stream ran out              */
};

/* common.hpp:77-82 / 84-86 / 88-105 */
uint64_t fdo_splitmix64(uint64_t x);
uint64_t fdo_hash_combine(uint64_t a, uint64_t b);
uint64_t fdo_hash_bytes64(const void* data, size_t n);
/* pipeline.hpp:295-298 */
uint64_t fdo_batch_seed(uint64_t seed, uint64_t epoch, uint64_t global_batch);

/* std::mt19937_64(splitmix64(rng_seed)) output words (sampling.hpp:78). */
void fdo_mt_stream(uint64_t rng_seed, uint64_t n, uint64_t* out);
/* libstdc++ uniform_int_distribution<u64>(0, j) applied to an explicit word
 * stream; returns the draw and advances *pos by the words consumed
 * (/usr/include/c++/13/bits/uniform_int_dist.h:257-281,313-320). */
uint64_t fdo_uniform_0_j(const uint64_t* words, uint64_t n_words, uint64_t* pos, uint64_t j);

/* generator.hpp:65-81, 85-96, 99-121 */
void fdo_synthetic_row(uint64_t seed, uint64_t node, uint32_t dim, float* out);
uint64_t fdo_synthetic_in_degree(uint64_t seed, uint64_t node, uint32_t avg_degree, uint64_t num_nodes);
uint64_t fdo_synthetic_in_neighbors(uint64_t seed, uint64_t node, uint32_t avg_degree,
                                    uint64_t num_nodes, uint64_t* out);
/* generator.hpp:575-596: indptr (N+1) then indices (E = indptr[N]). */
void fdo_generate_indptr(uint64_t seed, uint64_t num_nodes, uint32_t avg_degree, uint64_t* indptr);
void fdo_generate_indices(uint64_t seed, uint64_t num_nodes, uint32_t avg_degree,
                          const uint64_t* indptr, uint64_t* indices);

/*
 * sampling.hpp:72-134 sample_khop over an in-memory CSC (indptr u64[N+1],
 * indices u32 or u64 per idx_bytes). When `words` is NULL the MT19937-64
 * stream keyed by rng_seed is used (the reference behaviour); otherwise the
 * explicit word stream is consumed instead (used to exercise the Lemire
 * rejection path, which the MT stream essentially never hits).
 * layer_nodes[L+2]: node count before each layer's new nodes ([0]=0,[1]=seeds);
 * layer_edges[L+1]: edge count before each layer.
 */
int fdo_sample_khop(const uint64_t* indptr, const void* indices, int idx_bytes, uint64_t num_nodes,
                    const uint64_t* seeds, uint64_t n_seeds, const uint32_t* fanouts, uint32_t n_layers,
                    uint64_t rng_seed, const uint64_t* words, uint64_t n_words,
                    uint64_t* out_nodes, uint64_t nodes_cap, uint32_t* out_edges, uint64_t edges_cap,
                    uint64_t* n_nodes, uint64_t* n_edges, uint64_t* layer_nodes, uint64_t* layer_edges,
                    uint64_t* words_used, uint64_t* bad_seed);

/* sampling.hpp:32-40 Fanouts::max_batch_nodes */
uint64_t fdo_max_batch_nodes(const uint32_t* fanouts, uint32_t n_layers, uint64_t batch_size);

/*
 * featbuf/buffer_manager.hpp:222-527 BufferManager restated (dense mapping
 * table, LRU standby list, reverse map) and driven by the deterministic
 * single-extractor schedule: extract = acquire_for_batch (241-269) then, for
 * every to-load position in batch order, get_standby_slot (274-294) +
 * bind_slot (297-310), then publish_valid (313-324) for each; release =
 * release_batch (352-364).
 */
typedef struct fdo_bm fdo_bm;
fdo_bm* fdo_bm_create(uint64_t num_nodes, uint64_t slot_count, uint64_t min_reserved);
void fdo_bm_destroy(fdo_bm* bm);
/* alias[n]; load_pos (nullable, cap n) receives to-load positions; returns status. */
int fdo_bm_extract(fdo_bm* bm, const uint64_t* nodes, uint64_t n, int64_t* alias,
                   uint32_t* load_pos, uint64_t* n_load);
int fdo_bm_release(fdo_bm* bm, const uint64_t* nodes, uint64_t n);
/* out[7] = hits, loads, waits, evictions, takeovers, releases, standby_len (buffer_manager.hpp:192-200) */
void fdo_bm_stats(const fdo_bm* bm, uint64_t* out);
/* mapping entry (slot, ref, valid) for introspection (buffer_manager.hpp:420-424) */
void fdo_bm_entry(const fdo_bm* bm, uint64_t node, int64_t* slot, uint32_t* ref, uint32_t* valid);
int64_t fdo_bm_reverse(const fdo_bm* bm, uint64_t slot);
/* standby list LRU->MRU into out (cap); returns length (buffer_manager.hpp:100-109) */
uint64_t fdo_bm_standby(const fdo_bm* bm, int64_t* out, uint64_t cap);

/* Feature extraction restated as a row gather + pipeline.hpp:103-124 trainer_step checksum. */
uint64_t fdo_gather(const void* table, uint32_t row_bytes, const uint64_t* nodes, uint64_t n, void* out);
uint64_t fdo_checksum_rows(const void* rows, uint32_t row_bytes, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
