/*
 * fd_oracle.c -- CPU restatement of featdrive's sample -> extract path.
 *
 * TEST INFRASTRUCTURE ONLY (see fd_oracle.h). Plain C11 + unsigned __int128.
 * Each function cites the reference routine it restates; paths are relative
 * to /root/reference/proj/include/featdrive.
 *
 * Pinning: tests/test_oracle_vs_ref.py checks every function below against
 * the reference compiled from its own headers (oracle/_ref/libfdref.so) and
 * against tests/golden/ fixtures produced by that build (tests/golden/make_golden.py).
 */
#include "fd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- common -- */

/* common.hpp:77-82 */
uint64_t fdo_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* common.hpp:84-86 */
uint64_t fdo_hash_combine(uint64_t a, uint64_t b) {
    return fdo_splitmix64(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}

/* common.hpp:88-105: 8-byte little-endian lanes chained through splitmix64,
 * a length-tagged tail lane, then a final mix. */
uint64_t fdo_hash_bytes64(const void* data, size_t n) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0x27d4eb2f165667c5ull ^ ((uint64_t)n * 0x9e3779b97f4a7c15ull);
    while (n >= 8) {
        uint64_t lane;
        memcpy(&lane, p, 8);
        h = fdo_splitmix64(h ^ lane);
        p += 8;
        n -= 8;
    }
    if (n > 0) {
        uint64_t lane = 0;
        memcpy(&lane, p, n);
        h = fdo_splitmix64(h ^ lane ^ ((uint64_t)n << 56));
    }
    return fdo_splitmix64(h);
}

/* pipeline.hpp:295-298 */
uint64_t fdo_batch_seed(uint64_t seed, uint64_t epoch, uint64_t global_batch) {
    return fdo_hash_combine(fdo_hash_combine(seed, epoch), global_batch);
}

/* common.hpp:108-128 SplitMix (counter-mode) */
typedef struct { uint64_t state; } splitmix_t;
static uint64_t sm_next(splitmix_t* s) {
    s->state += 0x9e3779b97f4a7c15ull;
    uint64_t z = s->state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static double sm_next_unit(splitmix_t* s) { return (double)(sm_next(s) >> 11) * 0x1.0p-53; }
static uint64_t sm_next_below(splitmix_t* s, uint64_t n) { return n ? sm_next(s) % n : 0; }

/* ------------------------------------------------------------ mt19937_64 -- */
/* ISO C++ [rand.eng.mers] with the mt19937_64 parameters; seeded as
 * std::mt19937_64(splitmix64(rng_seed)) at sampling.hpp:78 and :61. */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ull
#define MT_UM 0xFFFFFFFF80000000ull
#define MT_LM 0x000000007FFFFFFFull

typedef struct { uint64_t x[MT_N]; int idx; } mt64_t;

static void mt_seed(mt64_t* g, uint64_t s) {
    g->x[0] = s;
    for (int i = 1; i < MT_N; ++i)
        g->x[i] = 6364136223846793005ull * (g->x[i - 1] ^ (g->x[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}

static void mt_twist(mt64_t* g) {
    for (int i = 0; i < MT_N; ++i) {
        uint64_t y = (g->x[i] & MT_UM) | (g->x[(i + 1) % MT_N] & MT_LM);
        g->x[i] = g->x[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1) ? MT_A : 0);
    }
    g->idx = 0;
}

static uint64_t mt_next(mt64_t* g) {
    if (g->idx >= MT_N) mt_twist(g);
    uint64_t z = g->x[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

void fdo_mt_stream(uint64_t rng_seed, uint64_t n, uint64_t* out) {
    mt64_t g;
    mt_seed(&g, fdo_splitmix64(rng_seed));
    for (uint64_t i = 0; i < n; ++i) out[i] = mt_next(&g);
}

/* Word source: the batch's MT stream, or an explicit caller-supplied stream. */
typedef struct {
    mt64_t mt;
    const uint64_t* words;
    uint64_t n_words;
    uint64_t pos;
    int short_stream;
} wordsrc_t;

static uint64_t ws_next(wordsrc_t* w) {
    if (w->words) {
        if (w->pos >= w->n_words) {
            w->short_stream = 1;
            return 0;
        }
        return w->words[w->pos++];
    }
    w->pos++;
    return mt_next(&w->mt);
}

/* libstdc++-13 uniform_int_distribution<u64>(0, j): __uerange = j + 1 and, as
 * the engine spans all 64 bits, _S_nd<unsigned __int128> (Lemire's nearly
 * divisionless method) -- uniform_int_dist.h:257-281 and 313-320. */
static uint64_t lemire(wordsrc_t* w, uint64_t j) {
    uint64_t range = j + 1;
    unsigned __int128 prod = (unsigned __int128)ws_next(w) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
        uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            prod = (unsigned __int128)ws_next(w) * range;
            low = (uint64_t)prod;
            if (w->short_stream) break;
        }
    }
    return (uint64_t)(prod >> 64);
}

uint64_t fdo_uniform_0_j(const uint64_t* words, uint64_t n_words, uint64_t* pos, uint64_t j) {
    wordsrc_t w;
    memset(&w, 0, sizeof(w));
    w.words = words + *pos;
    w.n_words = n_words - *pos;
    uint64_t r = lemire(&w, j);
    *pos += w.pos;
    return r;
}

/* ------------------------------------------------------------- generator -- */

/* generator.hpp:65-81: SplitMix keyed by hash_combine(hash_combine(seed,"row"),node);
 * each u64 yields two floats float(int32)*2^-31 (low half first). */
void fdo_synthetic_row(uint64_t seed, uint64_t node, uint32_t dim, float* out) {
    splitmix_t s = {fdo_hash_combine(fdo_hash_combine(seed, 0x726f77), node)};
    for (uint32_t i = 0; i < dim; i += 2) {
        uint64_t bits = sm_next(&s);
        float lo = (float)(int32_t)(uint32_t)(bits & 0xffffffffu) * 0x1.0p-31f;
        float hi = (float)(int32_t)(uint32_t)(bits >> 32) * 0x1.0p-31f;
        out[i] = lo;
        if (i + 1 < dim) out[i + 1] = hi;
    }
}

/* generator.hpp:85-96: capped Pareto(shape 2, scale avg/2). */
uint64_t fdo_synthetic_in_degree(uint64_t seed, uint64_t node, uint32_t avg_degree, uint64_t num_nodes) {
    if (avg_degree == 0 || num_nodes <= 1) return 0;
    splitmix_t s = {fdo_hash_combine(fdo_hash_combine(seed, 0x646567), node)};
    double u = sm_next_unit(&s);
    if (u < 1e-12) u = 1e-12;
    double scale = (double)avg_degree / 2.0;
    uint64_t d = (uint64_t)(scale / sqrt(u));
    uint64_t cap = (uint64_t)avg_degree * 4;
    if (d > cap) d = cap;
    if (d > num_nodes - 1) d = num_nodes - 1;
    return d;
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y);
}

/* generator.hpp:99-121: Floyd over [0, N-1) with self remapped to N-1, value
 * collision check, then ascending sort. Returns the degree. */
uint64_t fdo_synthetic_in_neighbors(uint64_t seed, uint64_t node, uint32_t avg_degree,
                                    uint64_t num_nodes, uint64_t* out) {
    uint64_t degree = fdo_synthetic_in_degree(seed, node, avg_degree, num_nodes);
    if (degree == 0) return 0;
    splitmix_t s = {fdo_hash_combine(fdo_hash_combine(seed, 0x6e6272), node)};
    uint64_t pool = num_nodes - 1;
    uint64_t n = 0;
    for (uint64_t j = pool - degree; j < pool; ++j) {
        uint64_t t = sm_next_below(&s, j + 1);
        if (t == node) t = num_nodes - 1;
        int found = 0;
        for (uint64_t k = 0; k < n; ++k)
            if (out[k] == t) { found = 1; break; }
        out[n++] = found ? (j == node ? num_nodes - 1 : j) : t;
    }
    qsort(out, n, sizeof(uint64_t), cmp_u64);
    return n;
}

void fdo_generate_indptr(uint64_t seed, uint64_t num_nodes, uint32_t avg_degree, uint64_t* indptr) {
    indptr[0] = 0;
    for (uint64_t n = 0; n < num_nodes; ++n)
        indptr[n + 1] = indptr[n] + fdo_synthetic_in_degree(seed, n, avg_degree, num_nodes);
}

void fdo_generate_indices(uint64_t seed, uint64_t num_nodes, uint32_t avg_degree,
                          const uint64_t* indptr, uint64_t* indices) {
    for (uint64_t n = 0; n < num_nodes; ++n)
        fdo_synthetic_in_neighbors(seed, n, avg_degree, num_nodes, indices + indptr[n]);
}

/* -------------------------------------------------------------- sampling -- */

uint64_t fdo_max_batch_nodes(const uint32_t* fanouts, uint32_t n_layers, uint64_t batch_size) {
    uint64_t total = 1, layer = 1;
    for (uint32_t l = 0; l < n_layers; ++l) {
        layer *= fanouts[l];
        total += layer;
    }
    return batch_size * total;
}

/* Open-addressing map NodeId -> local id standing in for the reference's
 * std::unordered_map (sampling.hpp:79-86); only lookup/insert semantics matter. */
typedef struct {
    uint64_t* keys;
    uint32_t* vals;
    uint64_t cap; /* power of two */
    uint64_t size;
} imap_t;

static const uint64_t kEmptyKey = ~0ull;

static uint64_t imap_hash(uint64_t k) { return fdo_splitmix64(k); }

static int imap_init(imap_t* m, uint64_t expect) {
    uint64_t cap = 1024;
    while (cap < expect * 2) cap <<= 1;
    m->keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
    m->vals = (uint32_t*)malloc(cap * sizeof(uint32_t));
    if (!m->keys || !m->vals) return -1;
    memset(m->keys, 0xff, cap * sizeof(uint64_t));
    m->cap = cap;
    m->size = 0;
    return 0;
}

static void imap_free(imap_t* m) {
    free(m->keys);
    free(m->vals);
}

static int imap_grow(imap_t* m);

/* Returns the existing value, or inserts `val` and returns UINT32_MAX... via *fresh. */
static uint32_t imap_find_or_insert(imap_t* m, uint64_t key, uint32_t val, int* fresh) {
    if ((m->size + 1) * 2 > m->cap) imap_grow(m);
    uint64_t mask = m->cap - 1, i = imap_hash(key) & mask;
    for (;;) {
        if (m->keys[i] == kEmptyKey) {
            m->keys[i] = key;
            m->vals[i] = val;
            m->size++;
            *fresh = 1;
            return val;
        }
        if (m->keys[i] == key) {
            *fresh = 0;
            return m->vals[i];
        }
        i = (i + 1) & mask;
    }
}

static int imap_grow(imap_t* m) {
    imap_t n;
    if (imap_init(&n, m->cap) != 0) return -1;
    for (uint64_t i = 0; i < m->cap; ++i)
        if (m->keys[i] != kEmptyKey) {
            int f;
            imap_find_or_insert(&n, m->keys[i], m->vals[i], &f);
        }
    imap_free(m);
    *m = n;
    return 0;
}

static inline uint64_t idx_at(const void* indices, int idx_bytes, uint64_t e) {
    return idx_bytes == 4 ? (uint64_t)((const uint32_t*)indices)[e] : ((const uint64_t*)indices)[e];
}

/* sampling.hpp:72-134 */
int fdo_sample_khop(const uint64_t* indptr, const void* indices, int idx_bytes, uint64_t num_nodes,
                    const uint64_t* seeds, uint64_t n_seeds, const uint32_t* fanouts, uint32_t n_layers,
                    uint64_t rng_seed, const uint64_t* words, uint64_t n_words,
                    uint64_t* out_nodes, uint64_t nodes_cap, uint32_t* out_edges, uint64_t edges_cap,
                    uint64_t* n_nodes, uint64_t* n_edges, uint64_t* layer_nodes, uint64_t* layer_edges,
                    uint64_t* words_used, uint64_t* bad_seed) {
    /* Fanouts::validate, sampling.hpp:23-29 */
    if (n_layers == 0) return FDO_INVALID_ARG;
    for (uint32_t l = 0; l < n_layers; ++l)
        if (fanouts[l] < 1) return FDO_INVALID_ARG;

    wordsrc_t ws;
    memset(&ws, 0, sizeof(ws));
    ws.words = words;
    ws.n_words = n_words;
    if (!words) mt_seed(&ws.mt, fdo_splitmix64(rng_seed)); /* sampling.hpp:78 */

    imap_t local;
    if (imap_init(&local, n_seeds * 4 + 16) != 0) return FDO_CAPACITY;
    uint64_t nn = 0, ne = 0;
    int rc = FDO_OK;
    uint64_t* frontier = NULL;
    uint64_t* next = NULL;
    uint64_t* picked = NULL;
    uint64_t picked_cap = 0;

    /* Seeds interned in chunk order; first out-of-range seed throws (89-93). */
    for (uint64_t i = 0; i < n_seeds; ++i) {
        if (seeds[i] >= num_nodes) {
            if (bad_seed) *bad_seed = seeds[i];
            rc = FDO_OUT_OF_RANGE;
            goto done;
        }
        int fresh;
        imap_find_or_insert(&local, seeds[i], (uint32_t)nn, &fresh);
        if (fresh) {
            if (nn >= nodes_cap) { rc = FDO_CAPACITY; goto done; }
            out_nodes[nn++] = seeds[i];
        }
    }
    /* frontier = sorted unique interned seeds = [0, nn) (95-96) */
    uint64_t f_lo = 0, f_hi = nn;
    layer_nodes[0] = 0;
    layer_nodes[1] = nn;
    for (uint32_t l = 0; l < n_layers; ++l) {
        layer_edges[l] = ne;
        uint32_t fanout = fanouts[l];
        if (picked_cap < fanout) {
            free(picked);
            picked_cap = fanout;
            picked = (uint64_t*)malloc(picked_cap * sizeof(uint64_t));
        }
        uint64_t next_lo = nn;
        for (uint64_t dst_local = f_lo; dst_local < f_hi; ++dst_local) {
            uint64_t dst = out_nodes[dst_local];
            uint64_t lo = indptr[dst], hi = indptr[dst + 1];
            uint64_t degree = hi - lo;
            uint64_t np = 0;
            const uint64_t* list = NULL;
            if (degree <= fanout) {
                np = degree; /* take all, list order (107-108) */
            } else {
                /* Floyd, value collision check (110-118) */
                for (uint64_t j = degree - fanout; j < degree; ++j) {
                    uint64_t t = lemire(&ws, j);
                    if (ws.short_stream) { rc = FDO_STREAM_SHORT; goto done; }
                    uint64_t cand = idx_at(indices, idx_bytes, lo + t);
                    for (uint64_t k = 0; k < np; ++k)
                        if (picked[k] == cand) { cand = idx_at(indices, idx_bytes, lo + j); break; }
                    picked[np++] = cand;
                }
                list = picked;
            }
            for (uint64_t k = 0; k < np; ++k) {
                uint64_t src = list ? list[k] : idx_at(indices, idx_bytes, lo + k);
                int fresh;
                uint32_t src_local = imap_find_or_insert(&local, src, (uint32_t)nn, &fresh);
                if (fresh) {
                    if (nn >= nodes_cap) { rc = FDO_CAPACITY; goto done; }
                    out_nodes[nn++] = src;
                }
                if (ne >= edges_cap) { rc = FDO_CAPACITY; goto done; }
                out_edges[2 * ne] = src_local;
                out_edges[2 * ne + 1] = (uint32_t)dst_local;
                ne++;
            }
        }
        /* next = fresh ids in increasing order = [next_lo, nn) (120-131) */
        f_lo = next_lo;
        f_hi = nn;
        layer_nodes[l + 2] = nn;
        if (f_lo == f_hi) {
            for (uint32_t r = l + 1; r < n_layers; ++r) {
                layer_edges[r] = ne;
                layer_nodes[r + 2] = nn;
            }
            break;
        }
    }
    layer_edges[n_layers] = ne;
done:
    *n_nodes = nn;
    *n_edges = ne;
    if (words_used) *words_used = ws.pos;
    free(frontier);
    free(next);
    free(picked);
    imap_free(&local);
    return rc;
}

/* -------------------------------------------------------- buffer manager -- */

struct fdo_bm {
    uint64_t num_nodes, slot_count;
    int64_t* map_slot;   /* MappingEntry.slot_index (buffer_manager.hpp:39-47) */
    uint32_t* map_ref;   /* MappingEntry.ref_count */
    uint8_t* map_valid;  /* MappingEntry.valid */
    int32_t* next;       /* StandbyList (54-119) */
    int32_t* prev;
    uint8_t* in_list;
    int32_t head, tail;
    uint64_t size;
    int64_t* reverse;    /* slot -> node, -1 = kNoNode (523) */
    uint64_t stats[7];
};

static void sb_push_mru(fdo_bm* b, int32_t s) {
    b->prev[s] = b->tail;
    b->next[s] = -1;
    if (b->tail != -1) b->next[b->tail] = s; else b->head = s;
    b->tail = s;
    b->in_list[s] = 1;
    b->size++;
}

static void sb_remove(fdo_bm* b, int32_t s) {
    if (b->prev[s] != -1) b->next[b->prev[s]] = b->next[s];
    if (b->next[s] != -1) b->prev[b->next[s]] = b->prev[s];
    if (b->head == s) b->head = b->next[s];
    if (b->tail == s) b->tail = b->prev[s];
    b->prev[s] = b->next[s] = -1;
    b->in_list[s] = 0;
    b->size--;
}

/* ctor: buffer_manager.hpp:224-233 (initial standby order 0..S-1) */
fdo_bm* fdo_bm_create(uint64_t num_nodes, uint64_t slot_count, uint64_t min_reserved) {
    if (slot_count == 0 || slot_count < min_reserved || slot_count >= (uint64_t)INT32_MAX) return NULL;
    fdo_bm* b = (fdo_bm*)calloc(1, sizeof(fdo_bm));
    b->num_nodes = num_nodes;
    b->slot_count = slot_count;
    b->map_slot = (int64_t*)malloc(num_nodes * sizeof(int64_t));
    b->map_ref = (uint32_t*)calloc(num_nodes, sizeof(uint32_t));
    b->map_valid = (uint8_t*)calloc(num_nodes, 1);
    b->next = (int32_t*)malloc(slot_count * sizeof(int32_t));
    b->prev = (int32_t*)malloc(slot_count * sizeof(int32_t));
    b->in_list = (uint8_t*)calloc(slot_count, 1);
    b->reverse = (int64_t*)malloc(slot_count * sizeof(int64_t));
    for (uint64_t n = 0; n < num_nodes; ++n) b->map_slot[n] = -1;
    b->head = b->tail = -1;
    for (uint64_t s = 0; s < slot_count; ++s) {
        b->reverse[s] = -1;
        sb_push_mru(b, (int32_t)s);
    }
    return b;
}

void fdo_bm_destroy(fdo_bm* b) {
    if (!b) return;
    free(b->map_slot); free(b->map_ref); free(b->map_valid);
    free(b->next); free(b->prev); free(b->in_list); free(b->reverse);
    free(b);
}

int fdo_bm_extract(fdo_bm* b, const uint64_t* nodes, uint64_t n, int64_t* alias,
                   uint32_t* load_pos, uint64_t* n_load) {
    uint32_t* to_load = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    uint64_t nl = 0;
    /* acquire_for_batch, buffer_manager.hpp:241-269 */
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t node = nodes[i];
        if (node >= b->num_nodes) { free(to_load); return FDO_INVARIANT; }
        alias[i] = -1;
        if (b->map_valid[node]) {
            if (b->map_ref[node] == 0) sb_remove(b, (int32_t)b->map_slot[node]);
            alias[i] = b->map_slot[node];
            b->stats[0]++;
        } else if (b->map_ref[node] > 0) {
            /* in flight elsewhere: impossible under the sequential schedule */
            free(to_load);
            return FDO_INVARIANT;
        } else {
            to_load[nl++] = (uint32_t)i;
            b->stats[1]++;
        }
        b->map_ref[node]++;
    }
    /* run_ticket binding loop, extractor.hpp:146-151: get_standby_slot + bind_slot */
    for (uint64_t k = 0; k < nl; ++k) {
        uint64_t node = nodes[to_load[k]];
        if (b->head == -1) { free(to_load); return FDO_CAPACITY; } /* StandbyTimeout */
        int32_t slot = b->head;
        sb_remove(b, slot);
        int64_t prev = b->reverse[slot];
        if (prev != -1) { /* evict previous owner (280-291) */
            b->map_valid[prev] = 0;
            b->map_slot[prev] = -1;
            b->reverse[slot] = -1;
            b->stats[3]++;
        }
        b->map_slot[node] = slot; /* bind_slot (297-310) */
        b->reverse[slot] = (int64_t)node;
        alias[to_load[k]] = slot;
    }
    /* publish_valid (313-324) once each row is in its slot */
    for (uint64_t k = 0; k < nl; ++k) b->map_valid[nodes[to_load[k]]] = 1;
    if (load_pos)
        for (uint64_t k = 0; k < nl; ++k) load_pos[k] = to_load[k];
    if (n_load) *n_load = nl;
    free(to_load);
    return FDO_OK;
}

/* release_batch + release_ref_locked, buffer_manager.hpp:352-364, 461-476 */
int fdo_bm_release(fdo_bm* b, const uint64_t* nodes, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t node = nodes[i];
        if (node >= b->num_nodes || !b->map_valid[node] || b->map_ref[node] == 0) return FDO_INVARIANT;
        if (--b->map_ref[node] == 0) sb_push_mru(b, (int32_t)b->map_slot[node]);
    }
    b->stats[5]++;
    return FDO_OK;
}

void fdo_bm_stats(const fdo_bm* b, uint64_t* out) {
    for (int i = 0; i < 6; ++i) out[i] = b->stats[i];
    out[6] = b->size;
}

void fdo_bm_entry(const fdo_bm* b, uint64_t node, int64_t* slot, uint32_t* ref, uint32_t* valid) {
    *slot = b->map_slot[node];
    *ref = b->map_ref[node];
    *valid = b->map_valid[node];
}

int64_t fdo_bm_reverse(const fdo_bm* b, uint64_t slot) { return b->reverse[slot]; }

uint64_t fdo_bm_standby(const fdo_bm* b, int64_t* out, uint64_t cap) {
    uint64_t k = 0;
    for (int32_t s = b->head; s != -1 && k < cap; s = b->next[s]) out[k++] = s;
    return k;
}

/* ------------------------------------------------------- gather/checksum -- */

/* Extraction's net effect on the mini-batch: row(nodes[i]) lands at position i
 * (extractor.hpp:374-386 copy into region.slot(alias[pos])); returns the
 * trainer_step checksum (pipeline.hpp:103-124). */
uint64_t fdo_gather(const void* table, uint32_t row_bytes, const uint64_t* nodes, uint64_t n, void* out) {
    const unsigned char* t = (const unsigned char*)table;
    unsigned char* o = (unsigned char*)out;
    uint64_t sum = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const unsigned char* row = t + nodes[i] * (uint64_t)row_bytes;
        if (o) memcpy(o + i * (uint64_t)row_bytes, row, row_bytes);
        sum += fdo_hash_bytes64(row, row_bytes);
    }
    return sum;
}

uint64_t fdo_checksum_rows(const void* rows, uint32_t row_bytes, uint64_t n) {
    const unsigned char* r = (const unsigned char*)rows;
    uint64_t sum = 0;
    for (uint64_t i = 0; i < n; ++i) sum += fdo_hash_bytes64(r + i * (uint64_t)row_bytes, row_bytes);
    return sum;
}
