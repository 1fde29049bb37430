// fdg_sample.cu -- k-hop uniform in-neighbor sampling with first-occurrence
// dedup/reindex, bit-exact with graph::sample_khop (sampling.hpp:72-134).
//
// Reference semantics (sequential): one std::mt19937_64(splitmix64(rng_seed))
// stream is consumed in (layer, frontier node, Floyd step) order, one
// uniform_int_distribution<u64>(0, j) draw (libstdc++ Lemire: 1 word unless a
// ~2^-57-probability rejection) per Floyd step; picks are interned into `nodes`
// in first-occurrence order; frontier l+1 = the fresh ids of layer l, which is
// the contiguous slice nodes[layer_nodes[l+1], layer_nodes[l+2]).
//
// Parallel restatement (stream-ordered, sizes stay on the device). Every kernel
// takes a Group of up to kGMax batches (blockIdx.y = batch): latency chains and
// kernel tails are paid once per group, not once per batch.
//   k_seeds    : init the batch record, range-check seeds, insert them into the
//                batch hash (key -> min pick position).
//   k_intern_s : one pass per pick list (seeds, then each layer). A pick is the
//                first occurrence iff its hash entry still holds its own pending
//                position; a striped single-pass decoupled look-back scan of
//                (first, min(deg,f), deg>f ? f : 0) assigns local ids in pick
//                order, writes `nodes` and every edge's src id, finalises the
//                entry and emits the next frontier's CSR start/degree and pick /
//                MT-draw offsets.
//   k_expand   : fanouts <= 16: a half-warp per frontier node, one pick per lane:
//                Floyd's draws from the pre-generated MT stream at the node's
//                prefix-summed offset (Lemire via __umul64hi), the value-compare
//                collision chain resolved by shuffles + ballots, hash insert, dst.
//   k_sample + k_insert : the thread-per-node path for fanouts > 16 and for the
//                exact mode.
// A Lemire rejection would consume an extra word and shift every later offset;
// it is detected, the batch is flagged FDG_REJECTION, and the host re-runs that
// batch in exact mode (offsets re-derived from per-node consumption).
#include <algorithm>
#include <cstring>
#include <string>

#include "fdg_internal.cuh"
#include "fdg_mt.cuh"

namespace fdg {
namespace {

constexpr uint32_t kPend = 0x80000000u;
// An edge's src field between the last expansion and the last intern pass holds either the
// pick's slot in tab_last or, with this bit, the final local id of an earlier layer's node.
constexpr uint32_t kFinalSrc = 0x80000000u;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kTile = kScanThreads * kScanItems;
constexpr int kMaxF = 16;  // half-warp / register-resident Floyd; larger fanouts use the global path
constexpr int kGMax = 8;   // batches per group launch

struct Tri {
    uint32_t c, p, d;
};
__device__ __forceinline__ Tri operator+(Tri a, Tri b) { return {a.c + b.c, a.p + b.p, a.d + b.d}; }

struct FrontierBuf {
    uint64_t* start;     // CSR start (indptr[v])
    uint32_t* deg;
    uint32_t* pick_off;  // exclusive scan of min(deg, f) within the layer
    uint32_t* draw_off;  // exclusive scan of (deg > f ? f : 0) within the layer
};

// Home slot of `key` in a table of `size` entries (any size: Fibonacci hash, then
// a multiply-shift range reduction instead of a power-of-two mask, so the table
// can be sized to the batch's node bound and stay small enough for L2).
__device__ __forceinline__ uint32_t hslot(uint64_t key, uint32_t size) {
    return __umulhi(uint32_t((key * 0x9E3779B97F4A7C15ull) >> 32), size);
}
__device__ __forceinline__ uint32_t hnext(uint32_t h, uint32_t size) { return h + 1 == size ? 0 : h + 1; }

// L2 residency of the batch hash: the clear and the intern pass's loads/stores carry
// an evict_last policy so the table (one per sampler lane, reused every batch) stays
// in L2 while the extraction streams ~1 GB per batch past it (atomics take no hint).
__device__ __forceinline__ uint64_t keep_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long ld_keep(const unsigned long long* p, uint64_t pol) {
    unsigned long long v;
    asm volatile("ld.global.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_keep(unsigned long long* p, unsigned long long v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// ---- batch hash: node id -> {pending min position | final local id} ----------------
// u32 ids: one packed 64-bit word per entry (key << 32 | value), so a new key
// costs one CAS and a lookup one load. u64 ids: separate key / value arrays.
template <typename IdT> struct HashTab;

// Early-table Bloom filter (2 bits per key, 32 bits per bounded key, right after the early
// table so the same all-ones fill clears it; a clear bit = present). Every last-layer pick
// looks its node up in the early table, and almost all are absent (Papers: ~0.1 % of picks
// are earlier layers' nodes), so the lookup probed to the next empty entry -- 8.4 probe
// iterations per warp, the longest of 30 lanes' chains. The filter answers "absent" for all
// but ~0.4 % of them with two loads from a ~0.4 MB L2-resident bitmap.
__device__ __forceinline__ void bloom_hash(uint32_t key, uint32_t nbits, uint32_t& b0, uint32_t& b1) {
    uint32_t h = key * 0x9E3779B1u;
    h ^= h >> 15;
    h *= 0x85EBCA77u;
    h ^= h >> 13;
    b0 = __umulhi(h, nbits);
    b1 = __umulhi(h * 0xC2B2AE3Du + 0x27D4EB2Fu, nbits);
}

template <> struct HashTab<uint32_t> {
    unsigned long long* e;
    uint32_t size;
    uint32_t keep;  // evict_last policy on loads / stores
    uint32_t* bloom;      // early table only (null: no filter)
    uint32_t bloom_bits;
    static constexpr unsigned long long kEmpty = ~0ull;
    __device__ __forceinline__ void* base() const { return e; }
    __device__ __forceinline__ void mark(uint32_t key) const {
        if (!bloom) return;
        uint32_t b0, b1;
        bloom_hash(key, bloom_bits, b0, b1);
        atomicAnd(bloom + (b0 >> 5), ~(1u << (b0 & 31)));
        atomicAnd(bloom + (b1 >> 5), ~(1u << (b1 & 31)));
    }
    __device__ __forceinline__ bool maybe_present(uint32_t key) const {
        if (!bloom) return true;
        uint32_t b0, b1;
        bloom_hash(key, bloom_bits, b0, b1);
        const uint32_t w0 = bloom[b0 >> 5], w1 = bloom[b1 >> 5];
        return !(((w0 >> (b0 & 31)) | (w1 >> (b1 & 31))) & 1u);
    }
    __device__ __forceinline__ uint32_t insert(uint32_t key, uint32_t pos) const {
        const unsigned long long want = (uint64_t(key) << 32) | (kPend | pos);
        uint32_t h = hslot(key, size);
        for (;;) {
            // CAS straight away: one scattered L2 operation per new key
            unsigned long long cur = atomicCAS(e + h, kEmpty, want);
            if (cur == kEmpty) return h;
            if (uint32_t(cur >> 32) == key) {
                // lower the pending minimum; a final id (< kPend) is never replaced
                while (uint32_t(cur) > uint32_t(want)) {
                    unsigned long long prev = atomicCAS(e + h, cur, want);
                    if (prev == cur) break;
                    cur = prev;
                }
                return h;
            }
            h = hnext(h, size);
        }
    }
    __device__ __forceinline__ void load(uint32_t h, uint32_t& key, uint32_t& val) const {
        unsigned long long v = keep ? ld_keep(e + h, keep_policy()) : e[h];
        key = uint32_t(v >> 32);
        val = uint32_t(v);
    }
    // Value of `key` (~0u when absent). Used on a table no thread is inserting final ids into.
    __device__ __forceinline__ uint32_t lookup(uint32_t key) const {
        uint32_t h = hslot(key, size);
        for (;;) {
            const unsigned long long v = keep ? ld_keep(e + h, keep_policy()) : e[h];
            if (v == kEmpty) return ~0u;
            if (uint32_t(v >> 32) == key) return uint32_t(v);
            h = hnext(h, size);
        }
    }
    __device__ __forceinline__ void finalize(uint32_t h, uint32_t key, uint32_t local) const {
        const unsigned long long v = (uint64_t(key) << 32) | local;
        if (keep) st_keep(e + h, v, keep_policy());
        else e[h] = v;
    }
};

template <> struct HashTab<uint64_t> {
    unsigned long long* keys;
    uint32_t* vals;
    uint32_t size;
    static constexpr unsigned long long kEmpty = ~0ull;
    __device__ __forceinline__ void* base() const { return keys; }  // keys, then vals, contiguous
    __device__ __forceinline__ uint32_t insert(uint64_t key, uint32_t pos) const {
        uint32_t h = hslot(key, size);
        for (;;) {
            unsigned long long cur = atomicCAS(keys + h, kEmpty, (unsigned long long)key);
            if (cur == kEmpty || cur == key) {
                atomicMin(vals + h, kPend | pos);
                return h;
            }
            h = hnext(h, size);
        }
    }
    __device__ __forceinline__ void load(uint32_t h, uint64_t& key, uint32_t& val) const {
        key = keys[h];
        val = vals[h];
    }
    __device__ __forceinline__ uint32_t lookup(uint64_t key) const {
        uint32_t h = hslot(key, size);
        for (;;) {
            const unsigned long long k = keys[h];
            if (k == kEmpty) return ~0u;
            if (k == key) return vals[h];
            h = hnext(h, size);
        }
    }
    __device__ __forceinline__ void finalize(uint32_t h, uint64_t, uint32_t local) const { vals[h] = local; }
    __device__ __forceinline__ void mark(uint64_t) const {}
    __device__ __forceinline__ bool maybe_present(uint64_t) const { return true; }
};

// Everything one batch needs (passed by value, kGMax per launch, in kernel params).
template <typename IdT>
struct Work {
    const uint64_t* indptr;
    const IdT* indices;
    uint64_t num_nodes;
    HashTab<IdT> tab;       // nodes of the passes before the last (seeds, layers < L-1)
    HashTab<IdT> tab_last;  // the last layer's new nodes (the exact replay: one table for all)
    const uint64_t* seeds;
    uint32_t n_seeds;
    uint32_t n_layers;
    uint32_t* seed_slot;  // [max_seeds]
    uint16_t* rank;       // [max_edges], tile-relative rank of first occurrences (< kTile)
    IdT* picks;           // [max_edges], picked neighbor ids (thread-per-node path)
    FrontierBuf fr[2];
    uint32_t* consumed;   // exact mode: words consumed per frontier node
    uint32_t* tile_flag;  // decoupled look-back state
    uint4* tile_agg;
    uint4* tile_incl;
    uint32_t* tile_ctr;   // per-pass dynamic tile counters
    const uint64_t* words;
    uint64_t words_cap;   // capacity of the word buffer
    uint64_t words_a;     // words generated before the chain starts (layers < L-1 may use them)
    uint64_t words_ready; // words generated before the last layer's expansion
    uint64_t* mt_state;   // engine state after words_ready (null: the stream is complete)
    uint64_t* nodes;      // output
    uint32_t* edges;      // output, {src, dst} pairs
    fdg_batch_counts* cnt;
    uint32_t fan[FDG_MAX_LAYERS];
};

template <typename IdT>
struct Group {
    Work<IdT> w[kGMax];
};

// Random CSR reads (a pick's neighbour entry, a frontier node's indptr pair) with a 64-byte L2
// fill instead of the default 128-byte line (ld_rand64, fdg_internal.cuh).
template <typename IdT>
__device__ __forceinline__ IdT ld_idx(const IdT* p) {
    if constexpr (sizeof(IdT) == 4) return ld_rand32(p);
    else return ld_rand64(p);
}

// libstdc++ uniform_int_distribution<u64>(0, j) on the word stream (uniform_int_dist.h:257-281).
__device__ __forceinline__ uint64_t lemire(const uint64_t* words, uint64_t cap, uint64_t& pos, uint64_t j,
                                           uint32_t& extra, bool& overflow) {
    const uint64_t r = j + 1;
    uint64_t w = pos < cap ? __ldg(words + pos) : 0;
    overflow |= pos >= cap;
    ++pos;
    uint64_t lo = w * r;
    uint64_t hi = __umul64hi(w, r);
    if (lo < r) {
        const uint64_t thr = (0 - r) % r;
        while (lo < thr) {
            w = pos < cap ? words[pos] : 0;
            overflow |= pos >= cap;
            ++pos;
            ++extra;
            lo = w * r;
            hi = __umul64hi(w, r);
            if (overflow) break;
        }
    }
    return hi;
}

// ---------------------------------------------------------------- k_seeds ----
// Initialises the batch record and inserts the seeds (one CTA per batch).
template <typename IdT>
__device__ __forceinline__ void seeds_body(const Work<IdT>& W) {
    fdg_batch_counts* cnt = W.cnt;
    if (threadIdx.x == 0) {
        cnt->status = 0;
        cnt->n_nodes = 0;
        cnt->n_edges = 0;
        cnt->rejections = 0;
        cnt->bad_seed = 0;
        cnt->checksum = 0;
        cnt->bad_seed_pos = 0xFFFFFFFFu;
        cnt->n_layers = W.n_layers;
        cnt->words_used = 0;
        cnt->replays = 0;
    }
    for (int i = threadIdx.x; i < FDG_MAX_LAYERS + 2; i += blockDim.x) {
        cnt->layer_nodes[i] = 0;
        if (i < FDG_MAX_LAYERS + 1) {
            cnt->layer_edges[i] = 0;
            cnt->layer_draws[i] = 0;
            W.tile_ctr[i] = 0;
        }
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < W.n_seeds; p += blockDim.x) {
        uint64_t s = W.seeds[p];
        if (s >= W.num_nodes) {  // sampling.hpp:89-93
            atomicMin(&cnt->bad_seed_pos, p);
            cnt->status = FDG_OUT_OF_RANGE;
            continue;
        }
        W.seed_slot[p] = W.tab.insert(IdT(s), p);
    }
    __syncthreads();
    if (threadIdx.x == 0 && cnt->status == FDG_OUT_OF_RANGE) cnt->bad_seed = W.seeds[cnt->bad_seed_pos];
}

template <typename IdT>
__global__ void __launch_bounds__(256) k_seeds(const __grid_constant__ Group<IdT> G) {
    seeds_body(G.w[blockIdx.y]);
}

// ----------------------------------------------------------- block scan ----
__device__ __forceinline__ Tri warp_incl_scan(Tri v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t c = __shfl_up_sync(0xffffffffu, v.c, o);
        uint32_t p = __shfl_up_sync(0xffffffffu, v.p, o);
        uint32_t d = __shfl_up_sync(0xffffffffu, v.d, o);
        if (lane >= o) v = v + Tri{c, p, d};
    }
    return v;
}

__device__ __forceinline__ uint32_t ld_volatile_u16(const uint16_t* p) {
    uint16_t v;
    asm volatile("ld.volatile.global.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_volatile4(const uint4* p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// CTA-wide look-back (all kScanThreads threads): thread t inspects tile (j - t), so a
// window of 256 predecessors is examined per step. Waits are for predecessors'
// AGGREGATES only (published as soon as each tile's local scan is done), so the
// wait is one tile's local work, not a serial chain of inclusive prefixes; the
// nearest inclusive predecessor in the window cuts the sum short. The caller has
// already published this tile's aggregate (flag E|1); this publishes the inclusive
// (E|2) unless publish_incl is false (the caller must then do it).
__device__ Tri tri_lookback_cta(uint32_t* flags, uint4* aggs, uint4* incls, uint32_t tile, uint32_t epoch) {
    __shared__ int s_stop[kScanThreads / 32];
    __shared__ Tri s_part[kScanThreads / 32];
    const uint32_t E = (epoch & 0x3FFFFFFFu) << 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Tri excl{0, 0, 0};
    for (int64_t j = int64_t(tile) - 1; j >= 0; j -= kScanThreads) {
        const int64_t jj = j - tid;
        uint32_t st = 2;  // before tile 0: an inclusive boundary of value 0
        if (jj >= 0) {
            for (;;) {
                const uint32_t fl = ld_volatile(flags + jj);
                st = (fl & ~3u) == E ? (fl & 3u) : 0u;
                if (st) break;
                __nanosleep(32);
            }
        }
        // nearest inclusive predecessor: the smallest tid with st == 2
        const uint32_t m = __ballot_sync(0xffffffffu, st == 2);
        if (lane == 0) s_stop[warp] = m ? warp * 32 + __ffs(m) - 1 : kScanThreads;
        __syncthreads();
        int stop = kScanThreads;
#pragma unroll
        for (int w = 0; w < kScanThreads / 32; ++w) stop = min(stop, s_stop[w]);
        __threadfence();
        Tri v{0, 0, 0};
        if (tid < stop) {
            const uint4 a = ld_volatile4(aggs + jj);
            v = Tri{a.x, a.y, a.z};
        } else if (tid == stop && jj >= 0) {
            const uint4 a = ld_volatile4(incls + jj);
            v = Tri{a.x, a.y, a.z};
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            v.c += __shfl_xor_sync(0xffffffffu, v.c, o);
            v.p += __shfl_xor_sync(0xffffffffu, v.p, o);
            v.d += __shfl_xor_sync(0xffffffffu, v.d, o);
        }
        if (lane == 0) s_part[warp] = v;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kScanThreads / 32; ++w) excl = excl + s_part[w];
        __syncthreads();  // s_stop / s_part reused by the next step
        if (stop < kScanThreads) break;
    }
    return excl;
}

// ------------------------------------------------------------- k_intern_s ----
// Pass q interns pick list q (q = 0: seeds; q = l+1: picks of layer l), writes the
// layer's edge src ids and sets up the frontier of layer q (when q < n_layers).
// Striped tiles: item k of thread t is position tile*kTile + k*256 + t, so every
// per-item global access of a warp is coalesced (L1TEX wavefronts, not DRAM bytes,
// bound the sampler); the scan runs as 8 row scans (one per k) -- one warp per
// row for the cross-warp step -- then one decoupled look-back per tile.
template <typename IdT, bool SEEDS, bool HAS_NEXT, bool PACK>
__device__ __forceinline__ void intern_tile(const Work<IdT>& W, uint32_t q, uint32_t epoch, uint32_t tile,
                                            uint32_t P, uint32_t ntiles);
template <typename IdT>
__device__ __forceinline__ void intern_tile_last(const Work<IdT>& W, uint32_t q, uint32_t epoch, uint32_t tile,
                                                 uint32_t P, uint32_t ntiles);
template <typename IdT, bool SEEDS>
__device__ __forceinline__ void intern_tile_next(const Work<IdT>& W, uint32_t q, uint32_t epoch, uint32_t tile,
                                                 uint32_t P, uint32_t ntiles);

// Persistent: a capped number of CTAs claim tiles in order (keeps SM slots free
// for the concurrently running gather; look-back needs only claim order).
// PACK (fanout of the next frontier <= 63): the warp scans carry (first, picks, draws)
// packed in one u32 (6 + 11 + 11 bits); the last pass (no next frontier) counts first
// occurrences with ballots alone.
template <typename IdT, bool SEEDS, bool HAS_NEXT, bool PACK = false, bool LEAN = false>
__device__ __forceinline__ void intern_pass(const Work<IdT>& W, uint32_t q, uint32_t epoch) {
    __shared__ uint32_t s_tile;
    fdg_batch_counts* cnt = W.cnt;
    if (cnt->status) return;
    const uint32_t P = SEEDS ? W.n_seeds : cnt->layer_edges[q] - cnt->layer_edges[q - 1];
    const uint32_t ntiles = P ? (P + kTile - 1) / kTile : 1;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(W.tile_ctr + q, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        __syncthreads();
        if (tile >= ntiles) return;
        if constexpr (!HAS_NEXT && !SEEDS) intern_tile_last<IdT>(W, q, epoch, tile, P, ntiles);
        else if constexpr (HAS_NEXT && PACK && LEAN) intern_tile_next<IdT, SEEDS>(W, q, epoch, tile, P, ntiles);
        else intern_tile<IdT, SEEDS, HAS_NEXT, PACK>(W, q, epoch, tile, P, ntiles);
        __syncthreads();
    }
}

#ifndef FDG_INTERN_MINB
#define FDG_INTERN_MINB 2
#endif
#ifndef FDG_INTERN_LAST_MINB
#define FDG_INTERN_LAST_MINB 6  // 40 registers with the one-register-per-item last pass (intern_tile_last)
#endif
template <typename IdT, bool SEEDS, bool HAS_NEXT, bool PACK, bool LEAN = false>
__global__ void __launch_bounds__(kScanThreads, HAS_NEXT ? (LEAN ? 3 : FDG_INTERN_MINB) : FDG_INTERN_LAST_MINB) k_intern_s(const __grid_constant__ Group<IdT> G, uint32_t q,
                                                           uint32_t epoch) {
    intern_pass<IdT, SEEDS, HAS_NEXT, PACK, LEAN>(G.w[blockIdx.y], q, epoch);
}

// Per-item scan values. Count-only (no next frontier): the first-occurrence bit, counted
// with ballots. Packed (fanout <= 63): (first, picks, draws) in one u32, 6 + 11 + 11 bits
// (a warp's sums fit). Otherwise a Tri. Items keep their warp-exclusive value in this
// compact form until the outputs, so the per-thread item arrays stay small.
template <bool HAS_NEXT, bool PACK>
struct ScanVal {
    using T = Tri;
    __device__ __forceinline__ static T make(uint32_t c, uint32_t p, uint32_t d) { return Tri{c, p, d}; }
    __device__ __forceinline__ static T incl(T v, int lane) { return warp_incl_scan(v, lane); }
    __device__ __forceinline__ static Tri tri(T v) { return v; }
    __device__ __forceinline__ static T sub(T a, T b) { return Tri{a.c - b.c, a.p - b.p, a.d - b.d}; }
};
template <bool PACK>
struct ScanVal<false, PACK> {
    using T = uint32_t;
    __device__ __forceinline__ static T make(uint32_t c, uint32_t, uint32_t) { return c; }
    __device__ __forceinline__ static T incl(T v, int lane) {
        return uint32_t(__popc(__ballot_sync(0xffffffffu, v != 0) & (0xffffffffu >> (31 - lane))));
    }
    __device__ __forceinline__ static Tri tri(T v) { return Tri{v, 0, 0}; }
    __device__ __forceinline__ static T sub(T a, T b) { return a - b; }
};
template <>
struct ScanVal<true, true> {
    using T = uint32_t;
    __device__ __forceinline__ static T make(uint32_t c, uint32_t p, uint32_t d) { return c | (p << 6) | (d << 17); }
    __device__ __forceinline__ static T incl(T x, int lane) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        return x;
    }
    __device__ __forceinline__ static Tri tri(T x) { return Tri{x & 63u, (x >> 6) & 2047u, x >> 17}; }
    __device__ __forceinline__ static T sub(T a, T b) { return a - b; }
};

template <typename IdT, bool SEEDS, bool HAS_NEXT, bool PACK>
__device__ __forceinline__ void intern_tile(const Work<IdT>& W, uint32_t q, uint32_t epoch, uint32_t tile,
                                            uint32_t P, uint32_t ntiles) {
    static_assert(kScanItems == kScanThreads / 32, "one warp per row scan");
    using SV = ScanVal<HAS_NEXT, PACK>;
    __shared__ Tri s_row[kScanItems][kScanThreads / 32];  // per row: warp inclusive -> exclusive
    __shared__ Tri s_rowx[kScanItems];                    // per row: exclusive offset within the tile
    __shared__ Tri s_excl, s_agg;
    fdg_batch_counts* cnt = W.cnt;
    const uint32_t ebase = SEEDS ? 0 : cnt->layer_edges[q - 1];
    const uint32_t node_base = cnt->layer_nodes[q];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t f = HAS_NEXT ? W.fan[q] : 0;
    const uint32_t p0 = tile * kTile + tid;  // item k: p0 + k * kScanThreads

    uint32_t slot[kScanItems], val[kScanItems];
    IdT key[kScanItems];
    uint32_t first_mask = 0, valid_mask = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t p = p0 + k * kScanThreads;
        if (p < P) {
            valid_mask |= 1u << k;
            slot[k] = SEEDS ? W.seed_slot[p] : W.edges[2 * (ebase + p)];  // the expansion parks the slot in src
        }
    }
    const HashTab<IdT>& T = HAS_NEXT ? W.tab : W.tab_last;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (valid_mask & (1u << k)) {
            if (!HAS_NEXT && (slot[k] & kFinalSrc)) {  // an earlier layer's node: its final id
                val[k] = slot[k] & ~kFinalSrc;
                continue;
            }
            T.load(slot[k], key[k], val[k]);
            if (val[k] == (kPend | (p0 + k * kScanThreads))) first_mask |= 1u << k;
        }
    uint64_t lo[HAS_NEXT ? kScanItems : 1];
    uint32_t dg[HAS_NEXT ? kScanItems : 1];
    if constexpr (HAS_NEXT) {
        uint64_t hi[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (first_mask & (1u << k)) {
                lo[k] = ld_rand64(W.indptr + uint64_t(key[k]));
                hi[k] = ld_rand64(W.indptr + uint64_t(key[k]) + 1);
            }
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) dg[k] = (first_mask & (1u << k)) ? uint32_t(hi[k] - lo[k]) : 0u;
    }
    // row scans: warp-inclusive per row; warp r turns row r's warp totals into exclusive
    // warp offsets; thread 0 turns the row totals into row offsets. xe[k] keeps item k's
    // warp-exclusive value.
    typename SV::T xe[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t c = (first_mask >> k) & 1u;
        const uint32_t d = HAS_NEXT ? dg[k] : 0u;
        const typename SV::T v = SV::make(c, HAS_NEXT ? (d < f ? d : f) : 0u, HAS_NEXT ? (d > f ? f : 0u) : 0u);
        const typename SV::T in = SV::incl(v, lane);
        xe[k] = SV::sub(in, v);
        if (lane == 31) s_row[k][warp] = SV::tri(in);
    }
    __syncthreads();
    {
        const int r = warp;
        Tri w = lane < kScanThreads / 32 ? s_row[r][lane] : Tri{0, 0, 0};
        Tri wi = w;
        if constexpr (HAS_NEXT) {
            wi = warp_incl_scan(w, lane);
        } else {
#pragma unroll
            for (int o = 1; o < kScanThreads / 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi.c, o);
                if (lane >= o) wi.c += y;
            }
        }
        if (lane < kScanThreads / 32) s_row[r][lane] = Tri{wi.c - w.c, wi.p - w.p, wi.d - w.d};
        if (lane == kScanThreads / 32 - 1) s_rowx[r] = wi;  // row total for now
    }
    __syncthreads();
    const uint32_t E = (epoch & 0x3FFFFFFFu) << 2;
    if (tid == 0) {
        Tri run{0, 0, 0};
        for (int r = 0; r < kScanItems; ++r) {
            Tri t = s_rowx[r];
            s_rowx[r] = run;
            run = run + t;
        }
        s_agg = run;
        // publish the aggregate at once: successors' look-backs wait only for this
        W.tile_agg[tile] = make_uint4(run.c, run.p, run.d, 0);
        __threadfence();
        atomicExch(W.tile_flag + tile, E | 1u);
    }
    __syncthreads();
    if (!SEEDS) {
        // tile-relative rank of every first occurrence, published (fenced) before this
        // tile's look-back flag so later tiles can resolve their repeated picks
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (first_mask & (1u << k))
                W.rank[ebase + p0 + k * kScanThreads] = uint16_t(s_rowx[k].c + s_row[k][warp].c + SV::tri(xe[k]).c);
        __threadfence();
        __syncthreads();
    }
    {
        const Tri agg = s_agg;
        const Tri excl = tri_lookback_cta(W.tile_flag, W.tile_agg, W.tile_incl, tile, epoch);
        if (tid == 0) {
            // ranks (above) and the aggregate are visible before the inclusive flag
            const Tri tot = excl + agg;
            W.tile_incl[tile] = make_uint4(tot.c, tot.p, tot.d, 0);
            __threadfence();
            atomicExch(W.tile_flag + tile, E | 2u);
            s_excl = excl;
            if (tile == ntiles - 1) {  // totals of this pass -> the batch record
                Tri tot = excl + agg;
                cnt->layer_nodes[q + 1] = node_base + tot.c;
                cnt->n_nodes = node_base + tot.c;
                if (HAS_NEXT) {
                    cnt->layer_edges[q + 1] = cnt->layer_edges[q] + tot.p;
                    cnt->layer_draws[q + 1] = cnt->layer_draws[q] + tot.d;
                } else {
                    cnt->n_edges = cnt->layer_edges[q];
                    cnt->words_used = cnt->layer_draws[q];
                }
            }
        }
    }
    __syncthreads();
    const Tri base = s_excl;
    const FrontierBuf fr = W.fr[q & 1];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (!(valid_mask & (1u << k))) continue;
        const uint32_t p = p0 + k * kScanThreads;
        if (first_mask & (1u << k)) {
            const Tri ex = s_rowx[k] + s_row[k][warp] + SV::tri(xe[k]);  // tile-relative exclusive prefix
            const uint32_t r = base.c + ex.c;
            const uint32_t local = node_base + r;
            W.nodes[local] = uint64_t(key[k]);
            if (HAS_NEXT) {  // no later pass reads the last layer's entries
                T.finalize(slot[k], key[k], local);
                T.mark(key[k]);
            }
            if (!SEEDS) W.edges[2 * (ebase + p)] = local;
            if constexpr (HAS_NEXT) {
                fr.start[r] = lo[k];
                fr.deg[r] = dg[k];
                fr.pick_off[r] = base.p + ex.p;
                fr.draw_off[r] = base.d + ex.d;
            }
        } else if (!SEEDS) {
            // src id of a repeated pick (LocalEdge.src, sampling.hpp:124): a final id is used
            // as is; a pending entry names its first occurrence, whose tile has published its
            // rank and (once inclusive) its exclusive prefix.
            uint32_t src = val[k];
            if (src & kPend) {
                const uint32_t pf = src & ~kPend;
                const uint32_t tf = pf / kTile;
                uint32_t bc;
                if (tf == tile) {
                    bc = base.c;
                } else {
                    while (ld_volatile(W.tile_flag + tf) != (E | 2u)) {
                    }
                    __threadfence();
                    const uint4 in = ld_volatile4(W.tile_incl + tf);
                    bc = tf == 0 ? 0u : in.x - ld_volatile4(W.tile_agg + tf).x;
                }
                src = node_base + bc + ld_volatile_u16(W.rank + ebase + pf);
            }
            W.edges[2 * (ebase + p)] = src;
        }
    }
}

// The last pass (no next frontier) with one register per item: an item keeps its key if it is
// a first occurrence and its entry's value otherwise (the hash slot is not needed after the
// load: the last layer's entries are never finalised), and its warp-relative rank is recounted
// from a ballot where it is used instead of being kept -- the general tile's four per-item
// arrays spilled 56-144 bytes at 64-40 registers.
template <typename IdT>
__device__ __forceinline__ void intern_tile_last(const Work<IdT>& W, uint32_t q, uint32_t epoch, uint32_t tile,
                                                 uint32_t P, uint32_t ntiles) {
    __shared__ uint32_t s_rowc[kScanItems][kScanThreads / 32];  // per row: warp counts -> exclusive offsets
    __shared__ uint32_t s_rowx[kScanItems];                     // per row: offset within the tile
    __shared__ uint32_t s_excl;
    fdg_batch_counts* cnt = W.cnt;
    const uint32_t ebase = cnt->layer_edges[q - 1];
    const uint32_t node_base = cnt->layer_nodes[q];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t p0 = tile * kTile + tid;  // item k: p0 + k * kScanThreads
    IdT kv[kScanItems];
    uint32_t first_mask = 0, valid_mask = 0;
    {
        uint32_t slot[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t p = p0 + k * kScanThreads;
            if (p < P) {
                valid_mask |= 1u << k;
                slot[k] = W.edges[2 * (ebase + p)];  // the expansion parks the slot in src
            }
        }
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (valid_mask & (1u << k)) {
                if (slot[k] & kFinalSrc) {  // an earlier layer's node: its final id
                    kv[k] = IdT(slot[k] & ~kFinalSrc);
                    continue;
                }
                IdT key;
                uint32_t val;
                W.tab_last.load(slot[k], key, val);
                if (val == (kPend | (p0 + k * kScanThreads))) {
                    first_mask |= 1u << k;
                    kv[k] = key;
                } else {
                    kv[k] = IdT(val);
                }
            }
    }
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t m = __ballot_sync(0xffffffffu, (first_mask >> k) & 1u);
        if (lane == 0) s_rowc[k][warp] = uint32_t(__popc(m));
    }
    __syncthreads();
    {  // warp r: exclusive offsets of row r's warps and the row total
        const int r = warp;
        const uint32_t c = lane < kScanThreads / 32 ? s_rowc[r][lane] : 0u;
        uint32_t in = c;
#pragma unroll
        for (int o = 1; o < kScanThreads / 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, in, o);
            if (lane >= o) in += y;
        }
        if (lane < kScanThreads / 32) s_rowc[r][lane] = in - c;
        if (lane == kScanThreads / 32 - 1) s_rowx[r] = in;
    }
    __syncthreads();
    const uint32_t E = (epoch & 0x3FFFFFFFu) << 2;
    __shared__ uint32_t s_agg;
    if (tid == 0) {
        uint32_t run = 0;
        for (int r = 0; r < kScanItems; ++r) {
            const uint32_t t = s_rowx[r];
            s_rowx[r] = run;
            run += t;
        }
        s_agg = run;
        W.tile_agg[tile] = make_uint4(run, 0, 0, 0);  // successors' look-backs wait only for this
        __threadfence();
        atomicExch(W.tile_flag + tile, E | 1u);
    }
    __syncthreads();
    // tile-relative ranks of the first occurrences, fenced before this tile's inclusive flag
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t m = __ballot_sync(0xffffffffu, (first_mask >> k) & 1u);
        if (first_mask & (1u << k))
            W.rank[ebase + p0 + k * kScanThreads] = uint16_t(s_rowx[k] + s_rowc[k][warp] + __popc(m & lt));
    }
    __threadfence();
    __syncthreads();
    {
        const uint32_t agg = s_agg;
        const Tri excl = tri_lookback_cta(W.tile_flag, W.tile_agg, W.tile_incl, tile, epoch);
        if (tid == 0) {
            const uint32_t tot = excl.c + agg;
            W.tile_incl[tile] = make_uint4(tot, 0, 0, 0);
            __threadfence();
            atomicExch(W.tile_flag + tile, E | 2u);
            s_excl = excl.c;
            if (tile == ntiles - 1) {  // totals of this pass -> the batch record
                cnt->layer_nodes[q + 1] = node_base + tot;
                cnt->n_nodes = node_base + tot;
                cnt->n_edges = cnt->layer_edges[q];
                cnt->words_used = cnt->layer_draws[q];
            }
        }
    }
    __syncthreads();
    const uint32_t base = s_excl;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t m = __ballot_sync(0xffffffffu, (first_mask >> k) & 1u);
        if (!(valid_mask & (1u << k))) continue;
        const uint32_t p = p0 + k * kScanThreads;
        if (first_mask & (1u << k)) {
            const uint32_t local = node_base + base + s_rowx[k] + s_rowc[k][warp] + uint32_t(__popc(m & lt));
            W.nodes[local] = uint64_t(kv[k]);
            W.edges[2 * (ebase + p)] = local;
        } else {
            // src id of a repeated pick (LocalEdge.src, sampling.hpp:124): a final id as is; a
            // pending entry names its first occurrence, whose tile published its rank first
            uint32_t src = uint32_t(kv[k]);
            if (src & kPend) {
                const uint32_t pf = src & ~kPend;
                const uint32_t tf = pf / kTile;
                uint32_t bc;
                if (tf == tile) {
                    bc = base;
                } else {
                    while (ld_volatile(W.tile_flag + tf) != (E | 2u)) {
                    }
                    __threadfence();
                    const uint4 in = ld_volatile4(W.tile_incl + tf);
                    bc = tf == 0 ? 0u : in.x - ld_volatile4(W.tile_agg + tf).x;
                }
                src = node_base + bc + ld_volatile_u16(W.rank + ebase + pf);
            }
            W.edges[2 * (ebase + p)] = src;
        }
    }
}

// The passes with a next frontier with the packed scan values in shared memory and the hash
// slot re-read for the outputs (three per-item register arrays instead of six: 80 registers
// instead of 128). Faster for the device-resident step (Papers 182.4 -> 178.4 us per batch)
// but not next to the fused checksum gather (190.2 -> 191.3), so the runner picks it for
// pipelines without the checksum (option intern_lean).
template <typename IdT, bool SEEDS>
__device__ __forceinline__ void intern_tile_next(const Work<IdT>& W, uint32_t q, uint32_t epoch, uint32_t tile,
                                                 uint32_t P, uint32_t ntiles) {
    using SV = ScanVal<true, true>;
    __shared__ Tri s_row[kScanItems][kScanThreads / 32];
    __shared__ Tri s_rowx[kScanItems];
    __shared__ Tri s_excl, s_agg;
    __shared__ uint32_t s_xe[kScanItems][kScanThreads];
    fdg_batch_counts* cnt = W.cnt;
    const uint32_t ebase = SEEDS ? 0 : cnt->layer_edges[q - 1];
    const uint32_t node_base = cnt->layer_nodes[q];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t f = W.fan[q];
    const uint32_t p0 = tile * kTile + tid;
    IdT kv[kScanItems];
    uint32_t dg[kScanItems];
    uint64_t lo[kScanItems];
    uint32_t first_mask = 0, valid_mask = 0;
    {
        uint32_t slot[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t p = p0 + k * kScanThreads;
            if (p < P) {
                valid_mask |= 1u << k;
                slot[k] = SEEDS ? W.seed_slot[p] : W.edges[2 * (ebase + p)];
            }
        }
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (valid_mask & (1u << k)) {
                IdT key;
                uint32_t val;
                W.tab.load(slot[k], key, val);
                if (val == (kPend | (p0 + k * kScanThreads))) {
                    first_mask |= 1u << k;
                    kv[k] = key;
                } else {
                    kv[k] = IdT(val);
                }
            }
    }
    {
        uint64_t hi[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (first_mask & (1u << k)) {
                lo[k] = ld_rand64(W.indptr + uint64_t(kv[k]));
                hi[k] = ld_rand64(W.indptr + uint64_t(kv[k]) + 1);
            }
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) dg[k] = (first_mask & (1u << k)) ? uint32_t(hi[k] - lo[k]) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t c = (first_mask >> k) & 1u, d = dg[k];
        const uint32_t v = SV::make(c, d < f ? d : f, d > f ? f : 0u);
        const uint32_t in = SV::incl(v, lane);
        s_xe[k][tid] = in - v;
        if (lane == 31) s_row[k][warp] = SV::tri(in);
    }
    __syncthreads();
    {
        const int r = warp;
        const Tri w = lane < kScanThreads / 32 ? s_row[r][lane] : Tri{0, 0, 0};
        const Tri wi = warp_incl_scan(w, lane);
        if (lane < kScanThreads / 32) s_row[r][lane] = Tri{wi.c - w.c, wi.p - w.p, wi.d - w.d};
        if (lane == kScanThreads / 32 - 1) s_rowx[r] = wi;
    }
    __syncthreads();
    const uint32_t E = (epoch & 0x3FFFFFFFu) << 2;
    if (tid == 0) {
        Tri run{0, 0, 0};
        for (int r = 0; r < kScanItems; ++r) {
            const Tri t = s_rowx[r];
            s_rowx[r] = run;
            run = run + t;
        }
        s_agg = run;
        W.tile_agg[tile] = make_uint4(run.c, run.p, run.d, 0);
        __threadfence();
        atomicExch(W.tile_flag + tile, E | 1u);
    }
    __syncthreads();
    if (!SEEDS) {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (first_mask & (1u << k))
                W.rank[ebase + p0 + k * kScanThreads] =
                    uint16_t(s_rowx[k].c + s_row[k][warp].c + SV::tri(s_xe[k][tid]).c);
        __threadfence();
        __syncthreads();
    }
    {
        const Tri agg = s_agg;
        const Tri excl = tri_lookback_cta(W.tile_flag, W.tile_agg, W.tile_incl, tile, epoch);
        if (tid == 0) {
            const Tri tot = excl + agg;
            W.tile_incl[tile] = make_uint4(tot.c, tot.p, tot.d, 0);
            __threadfence();
            atomicExch(W.tile_flag + tile, E | 2u);
            s_excl = excl;
            if (tile == ntiles - 1) {
                cnt->layer_nodes[q + 1] = node_base + tot.c;
                cnt->n_nodes = node_base + tot.c;
                cnt->layer_edges[q + 1] = cnt->layer_edges[q] + tot.p;
                cnt->layer_draws[q + 1] = cnt->layer_draws[q] + tot.d;
            }
        }
    }
    __syncthreads();
    const Tri base = s_excl;
    const FrontierBuf fr = W.fr[q & 1];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (!(valid_mask & (1u << k))) continue;
        const uint32_t p = p0 + k * kScanThreads;
        if (first_mask & (1u << k)) {
            const Tri ex = s_rowx[k] + s_row[k][warp] + SV::tri(s_xe[k][tid]);
            const uint32_t r = base.c + ex.c;
            const uint32_t local = node_base + r;
            const IdT key = kv[k];
            const uint32_t slot = SEEDS ? W.seed_slot[p] : W.edges[2 * (ebase + p)];
            W.nodes[local] = uint64_t(key);
            W.tab.finalize(slot, key, local);
            W.tab.mark(key);
            if (!SEEDS) W.edges[2 * (ebase + p)] = local;
            fr.start[r] = lo[k];
            fr.deg[r] = dg[k];
            fr.pick_off[r] = base.p + ex.p;
            fr.draw_off[r] = base.d + ex.d;
        } else if (!SEEDS) {
            uint32_t src = uint32_t(kv[k]);
            if (src & kPend) {
                const uint32_t pf = src & ~kPend;
                const uint32_t tf = pf / kTile;
                uint32_t bc;
                if (tf == tile) {
                    bc = base.c;
                } else {
                    while (ld_volatile(W.tile_flag + tf) != (E | 2u)) {
                    }
                    __threadfence();
                    const uint4 in = ld_volatile4(W.tile_incl + tf);
                    bc = tf == 0 ? 0u : in.x - ld_volatile4(W.tile_agg + tf).x;
                }
                src = node_base + bc + ld_volatile_u16(W.rank + ebase + pf);
            }
            W.edges[2 * (ebase + p)] = src;
        }
    }
}

// ---------------------------------------------------------------- k_sample ----
// Thread per frontier node (fanouts > 16 and exact mode). MODE 0: sample.
// MODE 1: exact-mode probe (count words consumed per node, no outputs). MODE 2:
// exact-mode final (offsets re-derived). Writes picks + edge dst; k_insert hashes.
template <typename IdT, bool SMALLF, int MODE>
__device__ __forceinline__ void sample_nodes(const Work<IdT>& W, uint32_t l, uint32_t first, uint32_t stride) {
    fdg_batch_counts* cnt = W.cnt;
    if (cnt->status) return;
    if (MODE == 0 && cnt->layer_draws[l + 1] > (l + 1 < W.n_layers ? W.words_a : W.words_ready)) {
        if (first == 0) atomicCAS(&cnt->status, 0u, uint32_t(FDG_REJECTION));  // words beyond the estimate
        return;
    }
    const uint32_t fs = cnt->layer_nodes[l];
    const uint32_t F = cnt->layer_nodes[l + 1] - fs;
    const uint32_t eb = cnt->layer_edges[l];
    const uint64_t db = cnt->layer_draws[l];
    const uint32_t f = W.fan[l];
    const FrontierBuf fr = W.fr[l & 1];
    for (uint32_t i = first; i < F; i += stride) {
        const uint64_t start = fr.start[i];
        const uint32_t deg = fr.deg[i];
        const uint32_t e0 = eb + fr.pick_off[i];
        const uint32_t dst = fs + i;
        if (deg <= f) {  // take all, in list order (sampling.hpp:107-108)
            if (MODE == 1) {
                W.consumed[i] = 0;
                continue;
            }
            for (uint32_t k = 0; k < deg; ++k) {
                W.picks[e0 + k] = W.indices[start + k];
                W.edges[2 * (e0 + k) + 1] = dst;
            }
            continue;
        }
        // Floyd's sampling with value-compare collisions (sampling.hpp:110-118)
        uint64_t pos = db + fr.draw_off[i];
        uint32_t extra = 0;
        bool overflow = false;
        const uint32_t jlo = deg - f;
        if (SMALLF) {
            uint32_t t[kMaxF];
#pragma unroll
            for (int k = 0; k < kMaxF; ++k)
                if (k < int(f)) t[k] = uint32_t(lemire(W.words, W.words_cap, pos, jlo + k, extra, overflow));
            if (MODE == 1) {
                W.consumed[i] = f + extra;
                continue;
            }
            IdT cand[kMaxF], alt[kMaxF];
#pragma unroll
            for (int k = 0; k < kMaxF; ++k)
                if (k < int(f)) {
                    cand[k] = ld_idx(W.indices + start + t[k]);
                    alt[k] = ld_idx(W.indices + start + jlo + k);
                }
            IdT picked[kMaxF];
#pragma unroll
            for (int k = 0; k < kMaxF; ++k) {
                if (k < int(f)) {
                    bool hit = false;
#pragma unroll
                    for (int m = 0; m < k; ++m) hit |= picked[m] == cand[k];
                    picked[k] = hit ? alt[k] : cand[k];
                }
            }
#pragma unroll
            for (int k = 0; k < kMaxF; ++k)
                if (k < int(f)) {
                    W.picks[e0 + k] = picked[k];
                    W.edges[2 * (e0 + k) + 1] = dst;
                }
        } else {
            IdT* picked = W.picks + e0;
            for (uint32_t k = 0; k < f; ++k) {
                uint64_t tk = lemire(W.words, W.words_cap, pos, jlo + k, extra, overflow);
                if (MODE == 1) continue;
                IdT c = W.indices[start + tk];
                for (uint32_t m = 0; m < k; ++m)
                    if (picked[m] == c) {
                        c = W.indices[start + jlo + k];
                        break;
                    }
                picked[k] = c;
                W.edges[2 * (e0 + k) + 1] = dst;
            }
            if (MODE == 1) {
                W.consumed[i] = f + extra;
                continue;
            }
        }
        if (overflow) atomicExch(&cnt->status, uint32_t(FDG_CAPACITY));
        if (MODE == 0 && extra) {
            atomicAdd(&cnt->rejections, extra);
            atomicCAS(&cnt->status, 0u, uint32_t(FDG_REJECTION));
        }
    }
}

template <typename IdT, bool SMALLF, int MODE>
__global__ void __launch_bounds__(256) k_sample(const __grid_constant__ Group<IdT> G, uint32_t l) {
    sample_nodes<IdT, SMALLF, MODE>(G.w[blockIdx.y], l, blockIdx.x * blockDim.x + threadIdx.x,
                                    gridDim.x * blockDim.x);
}

// ---------------------------------------------------------------- k_insert ----
// A pick's src-field value: its slot in the batch hash, or -- in the last layer, for a node
// an earlier pass already interned (a final id in W.tab) -- kFinalSrc | that id, with no
// insert. The last layer's new nodes go to tab_last (cleared right before the last
// expansion, so its lines are still in L2 for the expansion and the last intern pass).
template <typename IdT>
__device__ __forceinline__ uint32_t place_pick(const Work<IdT>& W, bool last, IdT key, uint32_t pos) {
    if (!last) return W.tab.insert(key, pos);
    if (W.tab.maybe_present(key)) {
        const uint32_t v = W.tab.lookup(key);
        if (v < kPend) return kFinalSrc | v;
    }
    return W.tab_last.insert(key, pos);
}

// Thread per pick of layer l (position = pick index within the layer).
template <typename IdT>
__device__ __forceinline__ void insert_picks(const Work<IdT>& W, uint32_t l, uint32_t first, uint32_t stride) {
    fdg_batch_counts* cnt = W.cnt;
    if (cnt->status) return;
    const uint32_t eb = cnt->layer_edges[l];
    const uint32_t P = cnt->layer_edges[l + 1] - eb;
    const bool last = l + 1 == W.n_layers;
    for (uint32_t p = first; p < P; p += stride) W.edges[2 * (eb + p)] = place_pick(W, last, W.picks[eb + p], p);
}

template <typename IdT>
__global__ void __launch_bounds__(256) k_insert(const __grid_constant__ Group<IdT> G, uint32_t l) {
    insert_picks(G.w[blockIdx.y], l, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// ---------------------------------------------------------------- k_expand ----
// Fast path for fanouts <= 16: floor(32 / f) frontier nodes per warp, f lanes per node,
// one pick per lane (f = 10: three nodes in 30 lanes). Lane k draws t_k from MT word
// db + draw_off + k (a Lemire rejection -- p ~ 2^-57 per draw -- flags the batch for the
// exact replay), loads cand_k = nb[t_k] and alt_k = nb[j_k]; Floyd's value-compare
// collision chain is resolved in k order with one shuffle + ballot per step; then every
// lane inserts its pick into the batch hash and writes its edge's dst
// (sampling.hpp:104-126).
#ifndef FDG_EXPAND_MINB
#define FDG_EXPAND_MINB 8  // <= 32 registers: the expansion is latency-bound (56 registers: 186 -> 203 us per Papers batch)
#endif
// FC: the fanout at compile time (0: read from the batch), so the Floyd chain's steps unroll
// with constant masks and bounds.
template <typename IdT, int FC = 0>
__global__ void __launch_bounds__(256, FDG_EXPAND_MINB) k_expand(const __grid_constant__ Group<IdT> G, uint32_t l) {
    const Work<IdT>& W = G.w[blockIdx.y];
    fdg_batch_counts* cnt = W.cnt;
    if (cnt->status) return;
    const uint32_t fs = cnt->layer_nodes[l];
    const uint32_t F = cnt->layer_nodes[l + 1] - fs;
    const uint32_t eb = cnt->layer_edges[l];
    const uint64_t db = cnt->layer_draws[l];
    const uint32_t f = FC ? uint32_t(FC) : W.fan[l];
    const FrontierBuf fr = W.fr[l & 1];
    // The prefetched stream holds an estimate of the words a batch draws (two pieces: the
    // early layers', then the rest); a batch drawing more goes to the exact replay, which
    // extends the stream from the saved engine state.
    if (cnt->layer_draws[l + 1] > (l + 1 < W.n_layers ? W.words_a : W.words_ready)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(&cnt->status, 0u, uint32_t(FDG_REJECTION));
        return;
    }
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t npw = 32 / f;                 // nodes per warp
    const uint32_t g = lane / f, k = lane - g * f;  // node slot in the warp, pick index
    const bool in_group = g < npw;
    const uint32_t gbase = in_group ? g * f : 0;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const bool last = l + 1 == W.n_layers;
    bool rejected = false;
    for (uint32_t wt = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wt * npw < F; wt += nwarps) {
        const uint32_t i = wt * npw + g;
        const bool live = in_group && i < F;
        uint64_t start = 0;
        uint32_t deg = 0, po = 0, dro = 0;
        if (live) {
            start = fr.start[i];
            deg = fr.deg[i];
            po = fr.pick_off[i];
            dro = fr.draw_off[i];
        }
        const bool floyd = deg > f;
        const uint32_t npick = floyd ? f : deg;
        IdT picked = 0, alt = 0;
        if (live && k < npick) {
            if (floyd) {
                const uint64_t j = uint64_t(deg - f) + k;
                const uint64_t r = j + 1;
                const uint64_t w = __ldg(W.words + db + dro + k);
                const uint64_t lo = w * r;
                if (lo < r && lo < (0 - r) % r) rejected = true;
                picked = ld_idx(W.indices + start + __umul64hi(w, r));
                alt = ld_idx(W.indices + start + j);
            } else {
                picked = W.indices[start + k];
            }
        }
        // Floyd collision chain: step s finalises pick s of every node in the warp
        if (__any_sync(0xffffffffu, live && floyd)) {
#pragma unroll
            for (uint32_t s = 1; s < (FC ? uint32_t(FC) : f); ++s) {
                const IdT c = __shfl_sync(0xffffffffu, picked, int(gbase + s));
                const uint32_t hits = __ballot_sync(0xffffffffu, in_group && k < s && picked == c);
                if (k == s && floyd && ((hits >> gbase) & ((1u << s) - 1u))) picked = alt;
            }
        }
        if (live && k < npick) {
            const uint32_t e = eb + po + k;
            // {hash slot, dst}: the intern pass reads the slot and overwrites it with the src id
            const uint32_t slot = place_pick(W, last, picked, po + k);
            *reinterpret_cast<uint2*>(W.edges + 2 * e) = make_uint2(slot, fs + i);
        }
    }
    if (rejected) {
        atomicAdd(&cnt->rejections, 1u);
        atomicCAS(&cnt->status, 0u, uint32_t(FDG_REJECTION));
    }
}

// ----------------------------------------------------------------- k_early ----
// The seeds and the first layer of a batch on one 1024-thread CTA, with the dedup hash in
// shared memory: what k_seeds, k_intern_s (seeds), k_expand (layer 0) and k_intern_s (layer-0
// picks) do in four launches and global hash round trips, for batches whose seeds and layer-0
// picks fit the shared table (<= kEarlyMaxKeys keys; Papers / products: 1,000 + 10,000). The
// interned nodes are then exported, with their final local ids, into the global early table
// that the next layers probe. Same outputs, bit for bit: nodes[0, layer_nodes[2]), the layer-0
// edges, the layer-1 frontier (fr[1]) and the batch record's layer counts.
constexpr int kEarlyThreads = 1024;
constexpr uint32_t kEarlyH = 16384;         // shared hash entries (128 KB), load factor <= 0.7
constexpr uint32_t kEarlyMaxKeys = 11468;   // seeds + layer-0 picks
constexpr uint32_t kEarlyMaxSeeds = kEarlyThreads;
constexpr size_t kEarlySmem = size_t(kEarlyH) * 8 + size_t(kEarlyMaxKeys) * 4 + size_t(kEarlyMaxSeeds) * 20;

__device__ __forceinline__ uint32_t sh_insert(unsigned long long* h, uint32_t key, uint32_t pos) {
    const unsigned long long want = (uint64_t(key) << 32) | (kPend | pos);
    uint32_t i = hslot(key, kEarlyH);
    for (;;) {
        unsigned long long cur = atomicCAS(h + i, ~0ull, want);
        if (cur == ~0ull) return i;
        if (uint32_t(cur >> 32) == key) {
            while (uint32_t(cur) > uint32_t(want)) {
                const unsigned long long prev = atomicCAS(h + i, cur, want);
                if (prev == cur) break;
                cur = prev;
            }
            return i;
        }
        i = (i + 1) & (kEarlyH - 1);
    }
}

// CTA-wide exclusive scan of (c, p, d) over kEarlyThreads threads; *tot = the totals.
__device__ __forceinline__ Tri early_scan(Tri v, Tri* s_warp, Tri* tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Tri in = warp_incl_scan(v, lane);
    if (lane == 31) s_warp[warp] = in;
    __syncthreads();
    if (warp == 0) {
        const Tri w = s_warp[lane];
        const Tri wi = warp_incl_scan(w, lane);
        s_warp[lane] = Tri{wi.c - w.c, wi.p - w.p, wi.d - w.d};
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    const Tri ex = s_warp[warp];
    *tot = s_warp[32];
    __syncthreads();  // s_warp is reused by the next scan
    return Tri{ex.c + in.c - v.c, ex.p + in.p - v.p, ex.d + in.d - v.d};
}

__global__ void __launch_bounds__(kEarlyThreads, 1) k_early(const __grid_constant__ Group<uint32_t> G) {
    extern __shared__ __align__(16) unsigned char early_smem[];
    __shared__ Tri s_warp[33];
    __shared__ uint32_t s_flag;
    const Work<uint32_t>& W = G.w[blockIdx.y];
    fdg_batch_counts* cnt = W.cnt;
    unsigned long long* h = reinterpret_cast<unsigned long long*>(early_smem);
    uint32_t* pslot = reinterpret_cast<uint32_t*>(h + kEarlyH);           // layer-0 pick -> hash slot
    uint64_t* f_start = reinterpret_cast<uint64_t*>(pslot + kEarlyMaxKeys);  // layer-0 frontier
    uint32_t* f_deg = reinterpret_cast<uint32_t*>(f_start + kEarlyMaxSeeds);
    uint32_t* f_po = f_deg + kEarlyMaxSeeds;
    uint32_t* f_do = f_po + kEarlyMaxSeeds;
    const int tid = threadIdx.x;
    // ---- the batch record (k_seeds) and the shared table
    if (tid == 0) {
        cnt->status = 0;
        cnt->n_nodes = 0;
        cnt->n_edges = 0;
        cnt->rejections = 0;
        cnt->bad_seed = 0;
        cnt->checksum = 0;
        cnt->bad_seed_pos = 0xFFFFFFFFu;
        cnt->n_layers = W.n_layers;
        cnt->words_used = 0;
        cnt->replays = 0;
        s_flag = 0;
    }
    for (int i = tid; i < FDG_MAX_LAYERS + 2; i += kEarlyThreads) {
        cnt->layer_nodes[i] = 0;
        if (i < FDG_MAX_LAYERS + 1) {
            cnt->layer_edges[i] = 0;
            cnt->layer_draws[i] = 0;
            W.tile_ctr[i] = 0;
        }
    }
    for (uint32_t i = tid; i < kEarlyH; i += kEarlyThreads) h[i] = ~0ull;
    __syncthreads();
    // ---- seeds: range check (sampling.hpp:89-93) and insert (key -> min position)
    const uint32_t S = W.n_seeds;  // <= kEarlyThreads (checked on the host)
    uint32_t key = 0, slot = 0;
    if (uint32_t(tid) < S) {
        const uint64_t sd = W.seeds[tid];
        if (sd >= W.num_nodes) {
            atomicMin(&cnt->bad_seed_pos, uint32_t(tid));
            s_flag = FDG_OUT_OF_RANGE;
        } else {
            key = uint32_t(sd);
            slot = sh_insert(h, key, uint32_t(tid));
        }
    }
    __syncthreads();
    if (s_flag) {
        if (tid == 0) {
            cnt->status = FDG_OUT_OF_RANGE;
            cnt->bad_seed = W.seeds[cnt->bad_seed_pos];
        }
        return;
    }
    // ---- intern the seeds (first occurrences in seed order) and set up frontier 0
    const uint32_t f0 = W.fan[0], f1 = W.fan[1];
    bool first = uint32_t(tid) < S && uint32_t(h[slot]) == (kPend | uint32_t(tid));
    uint64_t lo = 0, hi = 0;
    if (first) {
        lo = ld_rand64(W.indptr + key);
        hi = ld_rand64(W.indptr + uint64_t(key) + 1);
    }
    uint32_t dg = first ? uint32_t(hi - lo) : 0u;
    Tri tot0;
    Tri ex = early_scan(Tri{first ? 1u : 0u, min(dg, f0), dg > f0 ? f0 : 0u}, s_warp, &tot0);
    const uint32_t U0 = tot0.c, P0 = tot0.p, D0 = tot0.d;
    if (first) {
        W.nodes[ex.c] = uint64_t(key);
        h[slot] = (uint64_t(key) << 32) | ex.c;
        f_start[ex.c] = lo;
        f_deg[ex.c] = dg;
        f_po[ex.c] = ex.p;
        f_do[ex.c] = ex.d;
    }
    if (D0 > W.words_a) {  // words beyond the prefetched estimate: the exact replay re-runs the batch
        if (tid == 0) {
            cnt->layer_nodes[1] = U0;
            cnt->n_nodes = U0;
            cnt->layer_edges[1] = P0;
            cnt->layer_draws[1] = D0;
            atomicCAS(&cnt->status, 0u, uint32_t(FDG_REJECTION));
        }
        return;
    }
    __syncthreads();
    // ---- expand layer 0 (k_expand's warp layout: floor(32 / f0) nodes per warp, a lane per pick)
    {
        const uint32_t lane = tid & 31;
        const uint32_t npw = 32 / f0;
        const uint32_t g = lane / f0, k = lane - g * f0;
        const bool in_group = g < npw;
        const uint32_t gbase = in_group ? g * f0 : 0;
        bool rejected = false;
        for (uint32_t wt = uint32_t(tid) >> 5; wt * npw < U0; wt += kEarlyThreads / 32) {
            const uint32_t i = wt * npw + g;
            const bool live = in_group && i < U0;
            uint64_t start = 0;
            uint32_t deg = 0, po = 0, dro = 0;
            if (live) {
                start = f_start[i];
                deg = f_deg[i];
                po = f_po[i];
                dro = f_do[i];
            }
            const bool floyd = deg > f0;
            const uint32_t npick = floyd ? f0 : deg;
            uint32_t picked = 0, alt = 0;
            if (live && k < npick) {
                if (floyd) {
                    const uint64_t j = uint64_t(deg - f0) + k;
                    const uint64_t r = j + 1;
                    const uint64_t w = __ldg(W.words + dro + k);
                    const uint64_t lw = w * r;
                    if (lw < r && lw < (0 - r) % r) rejected = true;
                    picked = ld_idx(W.indices + start + __umul64hi(w, r));
                    alt = ld_idx(W.indices + start + j);
                } else {
                    picked = W.indices[start + k];
                }
            }
            if (__any_sync(0xffffffffu, live && floyd)) {
                for (uint32_t st = 1; st < f0; ++st) {
                    const uint32_t c = __shfl_sync(0xffffffffu, picked, int(gbase + st));
                    const uint32_t hits = __ballot_sync(0xffffffffu, in_group && k < st && picked == c);
                    if (k == st && floyd && ((hits >> gbase) & ((1u << st) - 1u))) picked = alt;
                }
            }
            if (live && k < npick) {
                pslot[po + k] = sh_insert(h, picked, po + k);
                W.edges[2 * (po + k) + 1] = i;  // dst: frontier node i is local id i
            }
        }
        if (rejected) {
            atomicAdd(&cnt->rejections, 1u);
            atomicCAS(&cnt->status, 0u, uint32_t(FDG_REJECTION));
            s_flag = 1;
        }
    }
    __syncthreads();
    if (s_flag) {  // a Lemire rejection: the exact replay re-runs the batch
        if (tid == 0) {
            cnt->layer_nodes[1] = U0;
            cnt->n_nodes = U0;
            cnt->layer_edges[1] = P0;
            cnt->layer_draws[1] = D0;
        }
        return;
    }
    // ---- intern the layer-0 picks in pick order; frontier 1 -> fr[1]
    Tri run{0, 0, 0};
    const FrontierBuf fr = W.fr[1];
    for (uint32_t b = 0; b < P0; b += kEarlyThreads) {
        const uint32_t pp = b + uint32_t(tid);
        uint32_t ps = 0;
        unsigned long long v = 0;
        bool fst = false;
        if (pp < P0) {
            ps = pslot[pp];
            v = h[ps];
            fst = uint32_t(v) == (kPend | pp);
        }
        uint64_t l1 = 0, h1 = 0;
        if (fst) {
            l1 = ld_rand64(W.indptr + (v >> 32));
            h1 = ld_rand64(W.indptr + (v >> 32) + 1);
        }
        const uint32_t d1 = fst ? uint32_t(h1 - l1) : 0u;
        Tri t;
        const Tri e = early_scan(Tri{fst ? 1u : 0u, min(d1, f1), d1 > f1 ? f1 : 0u}, s_warp, &t);
        uint32_t local = 0;
        if (fst) {
            const uint32_t r = run.c + e.c;
            local = U0 + r;
            W.nodes[local] = v >> 32;
            h[ps] = (v & 0xFFFFFFFF00000000ull) | local;
            fr.start[r] = l1;
            fr.deg[r] = d1;
            fr.pick_off[r] = run.p + e.p;
            fr.draw_off[r] = run.d + e.d;
        }
        run = run + t;
        __syncthreads();  // this round's first occurrences are final
        if (pp < P0) W.edges[2 * pp] = fst ? local : uint32_t(h[ps]);  // LocalEdge.src (sampling.hpp:124)
    }
    __syncthreads();
    // ---- export the interned nodes (final ids) to the global early table
    for (uint32_t i = tid; i < kEarlyH; i += kEarlyThreads) {
        const unsigned long long v = h[i];
        if (v == ~0ull) continue;
        uint32_t j = hslot(uint32_t(v >> 32), W.tab.size);
        while (atomicCAS(W.tab.e + j, ~0ull, v) != ~0ull) j = j + 1 == W.tab.size ? 0 : j + 1;
        W.tab.mark(uint32_t(v >> 32));
    }
    if (tid == 0) {
        cnt->layer_nodes[1] = U0;
        cnt->layer_edges[1] = P0;
        cnt->layer_draws[1] = D0;
        cnt->layer_nodes[2] = U0 + run.c;
        cnt->n_nodes = U0 + run.c;
        cnt->layer_edges[2] = P0 + run.p;
        cnt->layer_draws[2] = D0 + run.d;
    }
}

// ---------------------------------------------------------------- k_replay ----
// In-stream exact re-run of a batch whose fast path saw a Lemire rejection (an extra
// word consumed by some draw, p ~ 2^-57 per draw, shifting every later word offset;
// uniform_int_dist.h:257-281, sampling.hpp:113). Launched after every group chain
// with one 256-thread CTA per batch; it returns at once unless the batch's status is
// FDG_REJECTION, so nothing downstream (gather, buffer manager, train stage) ever
// sees a rejected batch and no host synchronisation is needed. When it fires it
// re-samples the batch from scratch on its CTA: hash cleared, seeds, then per layer
// the exact word offsets (iterated to a fixed point: probe each node's consumption at
// its current offset, rescan, repeat until no offset moves -- one extra round per
// rejection), the thread-per-node sampling at those offsets, hash inserts and the
// intern pass. Slow (~ms) but exact; the fast path never pays for it.

// Exact draw offsets of layer l on one CTA; sets layer_draws[l+1].
template <typename IdT, bool SMALLF>
__device__ void exact_offsets(const Work<IdT>& W, uint32_t l) {
    __shared__ uint32_t s_warp[8], s_carry, s_changed;
    fdg_batch_counts* cnt = W.cnt;
    const uint32_t F = cnt->layer_nodes[l + 1] - cnt->layer_nodes[l];
    const FrontierBuf fr = W.fr[l & 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int round = 0;; ++round) {
        sample_nodes<IdT, SMALLF, 1>(W, l, threadIdx.x, blockDim.x);  // consumed[i] at draw_off[i]
        __syncthreads();
        if (threadIdx.x == 0) {
            s_carry = 0;
            s_changed = 0;
        }
        __syncthreads();
        for (uint32_t base = 0; base < F; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            const uint32_t v = i < F ? W.consumed[i] : 0;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_warp[warp] = x;
            __syncthreads();
            if (warp == 0) {
                const uint32_t w = lane < int(blockDim.x / 32) ? s_warp[lane] : 0;
                uint32_t wx = w;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, wx, o);
                    if (lane >= o) wx += y;
                }
                if (lane < int(blockDim.x / 32)) s_warp[lane] = wx - w;
            }
            __syncthreads();
            const uint32_t excl = s_carry + s_warp[warp] + x - v;
            if (i < F && fr.draw_off[i] != excl) {
                fr.draw_off[i] = excl;
                s_changed = 1;
            }
            __syncthreads();
            if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
            __syncthreads();
        }
        if (!s_changed || cnt->status) break;
        __syncthreads();
    }
    if (threadIdx.x == 0) cnt->layer_draws[l + 1] = cnt->layer_draws[l] + s_carry;
    __syncthreads();
}

// Launched after every group chain, so its footprint must stay that of an ordinary sampler
// CTA (<= 64 registers: 4 CTAs per SM) -- a 255-register CTA would wait for an empty SM on
// every batch. The replay therefore samples through the global-picks path (no 16-wide
// register arrays), whatever the fanout.
template <typename IdT, bool SMALLF>
__global__ void __launch_bounds__(kScanThreads, 4) k_replay(const __grid_constant__ Group<IdT> G, uint32_t epoch0,
                                                            uint64_t hash_bytes) {
    __shared__ uint64_t s_mt[2][mt::kN];
    const Work<IdT>& W = G.w[blockIdx.y];
    fdg_batch_counts* cnt = W.cnt;
    if (*reinterpret_cast<volatile uint32_t*>(&cnt->status) != FDG_REJECTION) return;
    const uint32_t rejections = cnt->rejections, replays = cnt->replays;
    uint64_t gen = W.words_ready;  // words valid in the stream so far
    __syncthreads();
    // the batch hash back to all-empty (0xFF bytes: key ~0, pending values at their maximum)
    uint4* h = reinterpret_cast<uint4*>(W.tab.base());
    for (uint64_t k = threadIdx.x; k < hash_bytes / 16; k += blockDim.x) h[k] = make_uint4(~0u, ~0u, ~0u, ~0u);
    __threadfence_block();
    __syncthreads();
    seeds_body(W);
    if (W.n_layers) intern_pass<IdT, true, true>(W, 0, epoch0);
    else intern_pass<IdT, true, false>(W, 0, epoch0);
    __syncthreads();
    for (uint32_t l = 0; l < W.n_layers; ++l) {
        // the words layer l can touch: f draws per frontier node plus one per rejection (slack)
        const uint64_t F = cnt->layer_nodes[l + 1] - cnt->layer_nodes[l];
        const uint64_t bound = std::min<uint64_t>(W.words_cap, uint64_t(cnt->layer_draws[l]) + F * W.fan[l] + 1024);
        if (bound > gen) {
            if (!W.mt_state) {  // a complete stream: nothing to extend (an overflow is FDG_CAPACITY below)
                gen = W.words_cap;
            } else {
                const uint64_t end = std::min<uint64_t>((bound + mt::kN - 1) / mt::kN * mt::kN, W.words_cap);
                mt::generate(s_mt, 0, gen, end, W.words_cap, const_cast<uint64_t*>(W.words), W.mt_state);
                gen = end;
            }
        }
        exact_offsets<IdT, false>(W, l);
        sample_nodes<IdT, false, 2>(W, l, threadIdx.x, blockDim.x);
        __syncthreads();
        insert_picks(W, l, threadIdx.x, blockDim.x);
        __threadfence_block();
        __syncthreads();
        if (l + 1 < W.n_layers) intern_pass<IdT, false, true>(W, l + 1, epoch0 + 1 + l);
        else intern_pass<IdT, false, false>(W, l + 1, epoch0 + 1 + l);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cnt->rejections = rejections;
        cnt->replays = replays + 1;
    }
}

// Debug hook (option "debug_zero_word"): one word of a prefetched MT stream set to 0, which
// forces a genuine Lemire rejection for any range that is not a power of two.
__global__ void k_poke_zero(uint64_t* p) { *p = 0; }
// Test hook: a batch flagged as rejected without one (the replay must reproduce it).
__global__ void k_force_reject(fdg_batch_counts* cnt) {
    if (cnt->status == 0) {
        cnt->status = FDG_REJECTION;
        cnt->rejections += 1;
    }
}

// Degree statistics behind the prefetch-size estimate: for each layer's fanout f, over
// `samples` hashed picks of (a) uniform node ids (the seeds' distribution) and (b) uniform
// edge slots (a frontier node is an in-neighbour: its law is the edge-weighted one),
// count deg > f and sum min(deg, f). out[(kind * 8 + l) * 2 + {0: gt, 1: sum_min}].
struct Fans {
    uint32_t f[FDG_MAX_LAYERS];
    uint32_t n;
};
template <typename IdT>
__global__ void __launch_bounds__(256) k_degree_stats(const uint64_t* indptr, const IdT* indices, uint64_t N,
                                                      uint64_t E, Fans fans, uint64_t samples,
                                                      unsigned long long* out) {
    uint64_t acc[2][FDG_MAX_LAYERS][2] = {};
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < samples;
         t += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t v = __umul64hi(splitmix64(t), N);
        const uint64_t dv = indptr[v + 1] - indptr[v];
        uint64_t du = dv;
        if (E) {
            const uint64_t u = uint64_t(indices[__umul64hi(splitmix64(t ^ 0x5bd1e9955bd1e995ull), E)]);
            du = indptr[u + 1] - indptr[u];
        }
#pragma unroll
        for (int l = 0; l < FDG_MAX_LAYERS; ++l) {
            if (l >= int(fans.n)) break;
            const uint64_t f = fans.f[l];
            acc[0][l][0] += dv > f;
            acc[0][l][1] += dv < f ? dv : f;
            acc[1][l][0] += du > f;
            acc[1][l][1] += du < f ? du : f;
        }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int l = 0; l < FDG_MAX_LAYERS; ++l)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (l >= int(fans.n)) continue;
                uint64_t x = acc[k][l][j];
#pragma unroll
                for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                if ((threadIdx.x & 31) == 0 && x) atomicAdd(out + (k * FDG_MAX_LAYERS + l) * 2 + j, (unsigned long long)x);
            }
}

}  // namespace

int64_t g_l2_persist_mb = 0;
int64_t g_hash_load_pct = 50;
// Load factor (at the bound) of the early table alone (0: hash_load_pct). Every last-layer pick
// looks its node up there first, and an absent key probes to the next empty entry: the warp
// waits for the longest of its 30 lanes' chains (8.4 probes per warp at 0.5, ncu).
int64_t g_hash_early_pct = 0;
// Seeds + layer 0 fused into one shared-memory CTA per batch (k_early) when they fit. Measured
// neutral on the pipelined step (Papers 184.7 / 186.1 vs 186.7 / 184.5 us per batch, sample-only
// 68.0 / 71.6 vs 69.9 / 72.0; products 181.9 vs 176.8): the early layers are latency, not
// throughput, and 8 samplers in flight hide it. Off by default; parity-tested both ways.
int64_t g_early_fused = 0;
// Next-frontier intern passes in the lean form: 0 never, 1 always, 2 (default) in pipelines
// without the fused checksum (the runner decides; host-API samplers use the general form).
int64_t g_intern_lean = 2;
// Bloom filter over the early table's keys for the last layer's lookups (see bloom_hash).
int64_t g_early_bloom = 1;
int64_t g_sampler_ctas_per_sm = 16;
int64_t g_hash_clear = 1;
int64_t g_extract_streams = 2;
int64_t g_hash_keep = 1;
int64_t g_mt_adaptive = 1;
int64_t g_replay = 1;  // A/B only: 0 drops the replay launch (rejections then stay visible)  // prefetch the estimated draws (two pieces) instead of the draw bound

namespace {
// Fill `n16` 16-byte words with all-ones (the empty hash entry), grid-stride.
__global__ void __launch_bounds__(512) k_fill_ones(uint4* p, uint64_t n16, int keep) {
    const uint64_t pol = keep_policy();
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n16; i += uint64_t(gridDim.x) * blockDim.x) {
        if (keep)
            asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %1, %1, %1}, %2;" ::"l"(p + i), "r"(~0u), "l"(pol)
                         : "memory");
        else
            p[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
}
}  // namespace

cudaError_t clear_hash(void* base, uint64_t bytes, int sm_count, cudaStream_t st) {
    if (!g_hash_clear || (bytes & 15) || (uintptr_t(base) & 15)) return cudaMemsetAsync(base, 0xFF, bytes, st);
    const uint64_t n16 = bytes / 16;
    const uint64_t want = (n16 + 511) / 512;
    const int grid = int(std::min<uint64_t>(want, uint64_t(sm_count) * 4));
    k_fill_ones<<<std::max(grid, 1), 512, 0, st>>>((uint4*)base, n16, int(g_hash_keep));
    return cudaGetLastError();
}

// ------------------------------------------------------------------ Sampler ----
struct Lane {  // per-batch workspace of one group slot
    void* hash = nullptr;       // last-layer table: packed entries (u32 ids) or keys then vals (u64 ids)
    void* hash_a = nullptr;     // table of the earlier passes
    uint32_t* seed_slot = nullptr;
    uint16_t* rank = nullptr;
    void* picks = nullptr;
    FrontierBuf fr[2];
    uint32_t* consumed = nullptr;
    uint32_t* tile_flag = nullptr;
    uint4* tile_agg = nullptr;
    uint4* tile_incl = nullptr;
    uint32_t* tile_ctr = nullptr;
    uint32_t epoch = 1;
};

struct Sampler {
    Ctx* ctx = nullptr;
    uint32_t max_seeds = 0;
    uint32_t n_layers = 0;
    uint32_t gmax = 1;
    uint32_t fan[FDG_MAX_LAYERS] = {};
    uint64_t max_nodes = 0, max_edges = 0, max_draws = 0;
    uint64_t F_bound[FDG_MAX_LAYERS + 1] = {}, P_bound[FDG_MAX_LAYERS + 1] = {};
    uint32_t hsize = 0;    // last-layer table (sized for every node of a batch: the replay's one table)
    uint32_t hsize_a = 0;  // table of the passes before the last
    uint32_t bloom_bits = 0;  // early-table Bloom filter bits (0: none)
    bool small_f = true;
    bool early_fused = false;  // seeds + layer 0 in one shared-memory CTA per batch (k_early)
    bool lean_next = false;    // next-frontier intern passes in the lean form (intern_tile_next)
    void* arena = nullptr;
    void* hash_all = nullptr;  // the lanes' last-layer tables, contiguous (one fill per group)
    void* hash_all_a = nullptr;  // the lanes' early tables, contiguous, right before hash_all
    uint64_t hash_bytes_a = 0;
    std::vector<Lane> lanes;
    uint64_t hash_bytes = 0;   // per lane
    uint32_t* exact_flags = nullptr;  // [changed, total]
    uint64_t* words = nullptr;        // inline MT stream
    uint64_t words_cap = 0;           // draw bound + 4096 (the inline stream's length)
    uint64_t ring_stride = 0;         // ring slot capacity: words_cap rounded up to whole twists
    uint64_t words_a = 0, words_fast = 0;  // prefetch pieces: [0, words_a), [words_a, words_fast)
    uint64_t* ring_state = nullptr;   // per ring slot: the 312-word engine state after words_fast
    uint64_t* seeds_buf = nullptr;    // host-API staging
    // prefetch ring
    uint32_t ring_n = 0;
    uint64_t* ring_words = nullptr;
    std::vector<uint64_t> ring_seed;
    std::vector<bool> ring_valid;
    std::vector<uint32_t> ring_evt;   // slot -> the slot holding its prefetch chunk's events
    std::vector<cudaEvent_t> ring_ready_a, ring_ready, ring_done;  // first piece, whole prefetch, consumed
    uint32_t ring_next = 0;
    cudaStream_t host_stream = nullptr;
    fdg_batch_counts* cnt_buf = nullptr;  // host-API counts
    uint64_t* out_nodes = nullptr;        // host-API outputs
    uint32_t* out_edges = nullptr;
    int debug_reject = -1;                // test hook: lane of the next group flagged as rejected
};

}  // namespace fdg

struct fdg_sampler : fdg::Sampler {};

namespace fdg {

struct BatchArgs {  // one batch of a group launch
    const uint64_t* seeds;
    uint32_t n_seeds;
    const uint64_t* words;
    uint64_t words_cap;
    uint64_t* nodes;
    uint32_t* edges;
    fdg_batch_counts* cnt;
    uint64_t words_a = ~0ull, words_ready = ~0ull;  // complete stream unless set
    uint64_t* mt_state = nullptr;
    cudaEvent_t ready = nullptr;  // the stream's second piece (waited before the last layer)
};

namespace {

template <typename IdT>
Work<IdT> make_work(Sampler& s, const Lane& ln, const BatchArgs& a) {
    Work<IdT> w;
    w.indptr = s.ctx->indptr;
    w.indices = static_cast<const IdT*>(s.ctx->indices);
    w.num_nodes = s.ctx->num_nodes;
    auto set_tab = [&](HashTab<IdT>& t, void* base, uint32_t size) {
        if constexpr (sizeof(IdT) == 4) {
            t.e = static_cast<unsigned long long*>(base);
            t.keep = uint32_t(g_hash_keep);
            t.bloom = nullptr;
            t.bloom_bits = 0;
        } else {
            t.keys = static_cast<unsigned long long*>(base);
            t.vals = reinterpret_cast<uint32_t*>(static_cast<char*>(base) + uint64_t(size) * 8);
        }
        t.size = size;
    };
    set_tab(w.tab, ln.hash_a, s.hsize_a);
    set_tab(w.tab_last, ln.hash, s.hsize);
    if constexpr (sizeof(IdT) == 4) {
        if (s.bloom_bits) {  // right after the early table, inside the region the early fill clears
            w.tab.bloom = reinterpret_cast<uint32_t*>(static_cast<char*>(ln.hash_a) + uint64_t(s.hsize_a) * 8);
            w.tab.bloom_bits = s.bloom_bits;
        }
    }
    w.seeds = a.seeds;
    w.n_seeds = a.n_seeds;
    w.n_layers = s.n_layers;
    w.seed_slot = ln.seed_slot;
    w.rank = ln.rank;
    w.picks = static_cast<IdT*>(ln.picks);
    w.fr[0] = ln.fr[0];
    w.fr[1] = ln.fr[1];
    w.consumed = ln.consumed;
    w.tile_flag = ln.tile_flag;
    w.tile_agg = ln.tile_agg;
    w.tile_incl = ln.tile_incl;
    w.tile_ctr = ln.tile_ctr;
    w.words = a.words;
    w.words_cap = a.words_cap;
    w.words_a = std::min(a.words_a, a.words_cap);
    w.words_ready = std::min(a.words_ready, a.words_cap);
    w.mt_state = a.mt_state;
    w.nodes = a.nodes;
    w.edges = a.edges;
    w.cnt = a.cnt;
    for (uint32_t l = 0; l < FDG_MAX_LAYERS; ++l) w.fan[l] = l < s.n_layers ? s.fan[l] : 0;
    return w;
}

uint32_t grid_for(uint64_t items, int threads, int max_blocks) {
    uint64_t b = (items + threads - 1) / threads;
    return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(b, uint64_t(std::max(max_blocks, 1)))));
}

// All lanes of a group share one look-back epoch per pass (their flag arrays differ).
template <typename IdT>
void launch_intern(Sampler& s, cudaStream_t st, const Group<IdT>& G, uint32_t n, uint32_t q, uint32_t max_seeds,
                   uint32_t epoch) {
    const bool seeds = q == 0;
    const bool has_next = q < s.n_layers;
    const uint64_t P = seeds ? max_seeds : s.P_bound[q - 1];
    const uint64_t tiles = std::max<uint64_t>(1, (P + kTile - 1) / kTile);
    const uint64_t cap = std::max<uint64_t>(1, uint64_t(s.ctx->sm_count) * g_sampler_ctas_per_sm / n);
    const dim3 grid(uint32_t(std::min(tiles, cap)), n);
    const bool pack = has_next && s.fan[q] <= 63;
    if (seeds) {
        if (pack && s.lean_next) k_intern_s<IdT, true, true, true, true><<<grid, kScanThreads, 0, st>>>(G, q, epoch);
        else if (pack) k_intern_s<IdT, true, true, true><<<grid, kScanThreads, 0, st>>>(G, q, epoch);
        else if (has_next) k_intern_s<IdT, true, true, false><<<grid, kScanThreads, 0, st>>>(G, q, epoch);
        else k_intern_s<IdT, true, false, false><<<grid, kScanThreads, 0, st>>>(G, q, epoch);
    } else {
        if (pack && s.lean_next) k_intern_s<IdT, false, true, true, true><<<grid, kScanThreads, 0, st>>>(G, q, epoch);
        else if (pack) k_intern_s<IdT, false, true, true><<<grid, kScanThreads, 0, st>>>(G, q, epoch);
        else if (has_next) k_intern_s<IdT, false, true, false><<<grid, kScanThreads, 0, st>>>(G, q, epoch);
        else k_intern_s<IdT, false, false, false><<<grid, kScanThreads, 0, st>>>(G, q, epoch);
    }
}

template <typename IdT, int MODE>
void launch_sample(Sampler& s, cudaStream_t st, const Group<IdT>& G, uint32_t n, uint32_t l) {
    const dim3 grid(grid_for(s.F_bound[l], 256, s.ctx->sm_count * 16 / int(n)), n);
    if (s.small_f) k_sample<IdT, true, MODE><<<grid, 256, 0, st>>>(G, l);
    else k_sample<IdT, false, MODE><<<grid, 256, 0, st>>>(G, l);
}

template <typename IdT>
void launch_insert(Sampler& s, cudaStream_t st, const Group<IdT>& G, uint32_t n, uint32_t l) {
    const dim3 grid(grid_for(s.P_bound[l], 256, s.ctx->sm_count * 16 / int(n)), n);
    k_insert<IdT><<<grid, 256, 0, st>>>(G, l);
}

uint32_t next_epoch(Sampler& s, uint32_t n) {
    uint32_t e = 0;
    for (uint32_t i = 0; i < n; ++i) e = std::max(e, s.lanes[i].epoch);
    for (uint32_t i = 0; i < n; ++i) s.lanes[i].epoch = e + 1;
    return e;
}

// Fast path: a group of n batches, stream-ordered, no host synchronisation.
template <typename IdT>
int run_group(Sampler& s, cudaStream_t st, uint32_t n, const BatchArgs* a) {
    Group<IdT> G;
    uint32_t max_seeds = 1;
    for (uint32_t i = 0; i < n; ++i) {
        G.w[i] = make_work<IdT>(s, s.lanes[i], a[i]);
        max_seeds = std::max(max_seeds, a[i].n_seeds);
    }
    {
        FDG_TRACE("memset", st);
        FDG_CUDA(clear_hash(s.hash_all_a, s.hash_bytes_a * n, s.ctx->sm_count, st));
    }
    uint32_t l0 = 0;  // first layer expanded by the loop below
    if constexpr (sizeof(IdT) == 4) {
        if (s.early_fused) {  // seeds + layer 0 on one CTA per batch, shared-memory hash
            FDG_TRACE("early", st);
            static PerDeviceOnce attr;
            if (attr.first())
                FDG_CUDA(cudaFuncSetAttribute(k_early, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kEarlySmem)));
            k_early<<<dim3(1, n), kEarlyThreads, kEarlySmem, st>>>(G);
            next_epoch(s, n);
            next_epoch(s, n);
            l0 = 1;
        }
    }
    if (l0 == 0) {
        {
            FDG_TRACE("seeds", st);
            k_seeds<IdT><<<dim3(1, n), 256, 0, st>>>(G);
        }
        {
            FDG_TRACE("intern0", st);
            launch_intern<IdT>(s, st, G, n, 0, max_seeds, next_epoch(s, n));
        }
    }
    static const char* names[2][FDG_MAX_LAYERS] = {
        {"expand0", "expand1", "expand2", "expand3", "expand4", "expand5", "expand6", "expand7"},
        {"intern1", "intern2", "intern3", "intern4", "intern5", "intern6", "intern7", "intern8"}};
    for (uint32_t l = l0; l < s.n_layers; ++l) {
        if (l + 1 == s.n_layers) {  // the last layer draws from the prefetch's second piece
            for (uint32_t i = 0; i < n; ++i)
                if (a[i].ready) FDG_CUDA(cudaStreamWaitEvent(st, a[i].ready, 0));
            FDG_TRACE("memset_last", st);  // the last layer's table, filled right before its use
            FDG_CUDA(clear_hash(s.hash_all, s.hash_bytes * n, s.ctx->sm_count, st));
        }
        {
            FDG_TRACE(names[0][l], st);
            if (s.small_f) {
                const uint64_t npw = 32 / s.fan[l];  // nodes per warp
                const dim3 grid(grid_for((s.F_bound[l] + npw - 1) / npw * 32, 256,
                                         int(s.ctx->sm_count * g_sampler_ctas_per_sm / n)), n);
                switch (s.fan[l]) {  // compile-time fanouts of the benchmarked configurations
                    case 5: k_expand<IdT, 5><<<grid, 256, 0, st>>>(G, l); break;
                    case 10: k_expand<IdT, 10><<<grid, 256, 0, st>>>(G, l); break;
                    case 15: k_expand<IdT, 15><<<grid, 256, 0, st>>>(G, l); break;
                    default: k_expand<IdT><<<grid, 256, 0, st>>>(G, l); break;
                }
            } else {
                launch_sample<IdT, 0>(s, st, G, n, l);
                launch_insert<IdT>(s, st, G, n, l);
            }
        }
        {
            FDG_TRACE(names[1][l], st);
            launch_intern<IdT>(s, st, G, n, l + 1, max_seeds, next_epoch(s, n));  // also writes edge src ids
        }
    }
    if (s.debug_reject >= 0 && uint32_t(s.debug_reject) < n) {  // test hook: flag one lane as rejected
        k_force_reject<<<1, 1, 0, st>>>(a[s.debug_reject].cnt);
        s.debug_reject = -1;
    }
    if (g_replay) {
        FDG_TRACE("replay", st);  // exact re-run of rejected batches (no-op otherwise)
        const uint32_t e0 = next_epoch(s, n);
        for (uint32_t l = 0; l < s.n_layers; ++l) next_epoch(s, n);
        Group<IdT> R = G;  // the replay samples the whole batch through the last-layer table
        for (uint32_t i = 0; i < n; ++i) R.w[i].tab = R.w[i].tab_last;  // (no filter on the last table)
        k_replay<IdT, false><<<dim3(1, n), kScanThreads, 0, st>>>(R, e0, s.hash_bytes);
    }
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int dispatch_group(Sampler& s, cudaStream_t st, uint32_t n, const BatchArgs* a) {
    return s.ctx->idx_bytes == 4 ? run_group<uint32_t>(s, st, n, a) : run_group<uint64_t>(s, st, n, a);
}


}  // namespace

void sampler_destroy(Sampler* s);

namespace {
// How many MT words to prefetch per batch: the expected draws with a 20 % margin (the
// prefetch is split into the words of the layers before the last one and the rest, so a
// pipeline's first batch starts sampling after the first piece). Expected draws of layer l
// = F_l * f_l * P(deg > f_l), F_{l+1} = F_l * E[min(deg, f_l)] (dedup ignored: an upper
// estimate), with the seeds' degrees uniform over nodes and a frontier node's degree
// edge-weighted (an in-neighbour), measured on 2^20 hashed samples of the CSR. A batch drawing
// more than the estimate is re-run exactly in-stream, extending its stream (k_replay).
int estimate_words(Sampler& s, uint32_t max_seeds) {
    constexpr uint64_t kN312 = mt::kN;
    auto round312 = [&](uint64_t w) { return (w + kN312 - 1) / kN312 * kN312; };
    s.ring_stride = round312(s.words_cap);
    s.words_a = s.words_fast = s.ring_stride;
    const Ctx& c = *s.ctx;
    if (!g_mt_adaptive || (s.words_cap < (1u << 16) && g_mt_adaptive != 2) || c.num_nodes == 0) return FDG_OK;
    Fans fans{};
    fans.n = s.n_layers;
    for (uint32_t l = 0; l < s.n_layers; ++l) fans.f[l] = s.fan[l];
    unsigned long long* d = nullptr;
    const size_t bytes = 2 * FDG_MAX_LAYERS * 2 * sizeof(unsigned long long);
    FDG_CUDA(cudaMalloc(&d, bytes));
    FDG_CUDA(cudaMemset(d, 0, bytes));
    const uint64_t samples = 1u << 20;
    if (c.idx_bytes == 4)
        k_degree_stats<uint32_t><<<c.sm_count * 4, 256>>>(c.indptr, static_cast<const uint32_t*>(c.indices),
                                                          c.num_nodes, c.num_edges, fans, samples, d);
    else
        k_degree_stats<uint64_t><<<c.sm_count * 4, 256>>>(c.indptr, static_cast<const uint64_t*>(c.indices),
                                                          c.num_nodes, c.num_edges, fans, samples, d);
    unsigned long long h[2 * FDG_MAX_LAYERS * 2];
    cudaError_t e = cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "degree statistics", __FILE__, __LINE__);
    double F = double(std::min<uint64_t>(max_seeds, c.num_nodes)), before_last = 0, total = 0;
    for (uint32_t l = 0; l < s.n_layers; ++l) {
        const int k = l == 0 ? 0 : 1;
        const double p_gt = double(h[(k * FDG_MAX_LAYERS + l) * 2]) / double(samples);
        const double e_min = double(h[(k * FDG_MAX_LAYERS + l) * 2 + 1]) / double(samples);
        const double w = F * double(s.fan[l]) * p_gt;
        total += w;
        if (l + 1 < s.n_layers) before_last += w;
        F = std::min(F * e_min, double(c.num_nodes));
    }
    uint64_t fast = round312(uint64_t(1.2 * total) + 4096);
    uint64_t a = round312(uint64_t(1.25 * before_last) + 2048);
    if (g_mt_adaptive == 2) {  // test mode: a deliberately short prefetch, every batch replays
        fast = round312(fast / 8);
        a = round312(a / 8);
    } else if (fast >= s.ring_stride * 9 / 10) {
        return FDG_OK;  // the bound is nearly reached anyway
    }
    s.words_fast = std::min(fast, s.ring_stride);
    s.words_a = std::min(a, s.words_fast);
    return FDG_OK;
}
}  // namespace

int sampler_create(Ctx* ctx, uint32_t max_seeds, const uint32_t* fanouts, uint32_t n_layers, Sampler** out,
                   uint32_t group) {
    if (!ctx->indptr) return fail(FDG_NOT_LOADED, "sampler: no topology loaded");
    if (n_layers == 0) return fail(FDG_INVALID_ARG, "fanouts: need at least one layer");
    if (n_layers > FDG_MAX_LAYERS) return fail(FDG_INVALID_ARG, "fanouts: more than FDG_MAX_LAYERS layers");
    for (uint32_t l = 0; l < n_layers; ++l)
        if (fanouts[l] < 1) return fail(FDG_INVALID_ARG, "fanouts: every entry must be >= 1");
    if (max_seeds == 0) max_seeds = 1;
    group = std::max<uint32_t>(1, std::min<uint32_t>(group, kGMax));
    auto s = new Sampler();
    s->ctx = ctx;
    s->max_seeds = max_seeds;
    s->n_layers = n_layers;
    s->gmax = group;
    const uint64_t N = ctx->num_nodes;
    uint64_t F = std::min<uint64_t>(max_seeds, N), nodes = F, edges = 0;
    uint32_t fmax = 0;
    for (uint32_t l = 0; l < n_layers; ++l) {
        s->fan[l] = fanouts[l];
        fmax = std::max(fmax, fanouts[l]);
        s->F_bound[l] = F;
        s->P_bound[l] = F * fanouts[l];
        edges += s->P_bound[l];
        F = std::min<uint64_t>(s->P_bound[l], N);
        nodes += F;
    }
    s->max_nodes = std::min<uint64_t>(nodes, N);
    s->max_edges = edges;
    s->max_draws = edges;
    if (s->max_edges >= (1ull << 31) || s->max_nodes >= (1ull << 31)) {
        delete s;
        return fail(FDG_INVALID_ARG, "sampler: batch bound exceeds 2^31 picks");
    }
    s->small_f = fmax <= uint32_t(kMaxF);
    s->early_fused = g_early_fused && ctx->idx_bytes == 4 && n_layers >= 2 && fanouts[0] <= uint32_t(kMaxF) &&
                     max_seeds <= kEarlyMaxSeeds && uint64_t(max_seeds) + s->P_bound[0] <= kEarlyMaxKeys;
    // exact sizing (load factor g_hash_load_pct at the batch's node bound); any size works (hslot)
    s->hsize = uint32_t((std::max<uint64_t>(s->max_nodes * 100 / uint64_t(g_hash_load_pct), 1024) + 31) & ~uint64_t(31));
    const uint32_t ib = ctx->idx_bytes;
    auto al = [](uint64_t b) { return (b + 255) & ~uint64_t(255); };
    s->hash_bytes = al(uint64_t(s->hsize) * (ib == 4 ? 8 : 12));
    // the early table holds the nodes interned before the last pass (seeds, layers < L-1)
    const uint64_t early = std::min<uint64_t>(N, nodes - std::min<uint64_t>(s->P_bound[n_layers - 1], N));
    const uint64_t early_pct = g_hash_early_pct > 0 ? uint64_t(g_hash_early_pct) : uint64_t(g_hash_load_pct);
    s->hsize_a = uint32_t((std::max<uint64_t>(early * 100 / early_pct, 1024) + 31) & ~uint64_t(31));
    s->bloom_bits = (ib == 4 && g_early_bloom && n_layers >= 2)
                        ? uint32_t(std::min<uint64_t>(std::max<uint64_t>(early * 32, 1024), 1ull << 31) & ~uint64_t(31))
                        : 0u;
    s->hash_bytes_a = al(uint64_t(s->hsize_a) * (ib == 4 ? 8 : 12) + uint64_t(s->bloom_bits) / 8);
    uint64_t fmaxF = 1;
    for (uint32_t l = 0; l < n_layers; ++l) fmaxF = std::max(fmaxF, s->F_bound[l]);
    const uint64_t tiles = (std::max<uint64_t>(s->max_edges, max_seeds) + kTile - 1) / kTile + 1;
    s->words_cap = s->max_draws + 4096;
    // per-lane layout
    uint64_t lz = 0;
    const uint64_t o_seed = lz; lz += al(uint64_t(max_seeds) * 4);
    const uint64_t o_rank = lz; lz += al(std::max<uint64_t>(s->max_edges, 1) * 2);
    const uint64_t o_picks = lz; lz += al(std::max<uint64_t>(s->max_edges, 1) * ib);  // exact replay (any lane)
    uint64_t o_fr[2];
    for (int b = 0; b < 2; ++b) { o_fr[b] = lz; lz += al(fmaxF * 8) + 3 * al(fmaxF * 4); }
    const uint64_t o_cons = lz; lz += al(fmaxF * 4);
    const uint64_t o_flag = lz; lz += al(tiles * 4);
    const uint64_t o_agg = lz; lz += al(tiles * 16);
    const uint64_t o_inc = lz; lz += al(tiles * 16);
    const uint64_t o_ctr = lz; lz += al((FDG_MAX_LAYERS + 2) * 4);
    // sampler-wide layout: hashes of all lanes first (contiguous), then lanes, then shared
    uint64_t sz = 0;
    const uint64_t o_hash_a = sz; sz += s->hash_bytes_a * group;
    const uint64_t o_hash = sz; sz += s->hash_bytes * group;
    const uint64_t o_lanes = sz; sz += lz * group;
    const uint64_t o_ex = sz; sz += al(16);
    const uint64_t o_words = sz; sz += al(s->words_cap * 8);
    const uint64_t o_seeds = sz; sz += al(uint64_t(max_seeds) * 8);
    const uint64_t o_cnt = sz; sz += al(sizeof(fdg_batch_counts));
    cudaError_t e = cudaMalloc(&s->arena, sz);
    if (e != cudaSuccess) {
        delete s;
        return cuda_fail(e, "cudaMalloc(sampler arena)", __FILE__, __LINE__);
    }
    char* A = static_cast<char*>(s->arena);
    s->hash_all = A + o_hash;
    s->hash_all_a = A + o_hash_a;
    s->lanes.resize(group);
    for (uint32_t g = 0; g < group; ++g) {
        Lane& ln = s->lanes[g];
        char* a = A + o_lanes + g * lz;
        ln.hash = A + o_hash + g * s->hash_bytes;
        ln.hash_a = A + o_hash_a + g * s->hash_bytes_a;
        ln.seed_slot = reinterpret_cast<uint32_t*>(a + o_seed);
        ln.rank = reinterpret_cast<uint16_t*>(a + o_rank);
        ln.picks = a + o_picks;
        for (int b = 0; b < 2; ++b) {
            char* p = a + o_fr[b];
            ln.fr[b].start = reinterpret_cast<uint64_t*>(p);
            p += al(fmaxF * 8);
            ln.fr[b].deg = reinterpret_cast<uint32_t*>(p);
            p += al(fmaxF * 4);
            ln.fr[b].pick_off = reinterpret_cast<uint32_t*>(p);
            p += al(fmaxF * 4);
            ln.fr[b].draw_off = reinterpret_cast<uint32_t*>(p);
        }
        ln.consumed = reinterpret_cast<uint32_t*>(a + o_cons);
        ln.tile_flag = reinterpret_cast<uint32_t*>(a + o_flag);
        ln.tile_agg = reinterpret_cast<uint4*>(a + o_agg);
        ln.tile_incl = reinterpret_cast<uint4*>(a + o_inc);
        ln.tile_ctr = reinterpret_cast<uint32_t*>(a + o_ctr);
        cudaMemset(ln.tile_flag, 0, tiles * 4);
    }
    s->exact_flags = reinterpret_cast<uint32_t*>(A + o_ex);
    s->words = reinterpret_cast<uint64_t*>(A + o_words);
    s->seeds_buf = reinterpret_cast<uint64_t*>(A + o_seeds);
    s->cnt_buf = reinterpret_cast<fdg_batch_counts*>(A + o_cnt);
    e = cudaStreamCreateWithFlags(&s->host_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate", __FILE__, __LINE__);
    {
        const int rc = estimate_words(*s, max_seeds);
        if (rc != FDG_OK) {
            sampler_destroy(s);
            return rc;
        }
    }
    *out = s;
    return FDG_OK;
}

int sampler_create(Ctx* ctx, uint32_t max_seeds, const uint32_t* fanouts, uint32_t n_layers, Sampler** out) {
    return sampler_create(ctx, max_seeds, fanouts, n_layers, out, 1);
}

void sampler_destroy(Sampler* s) {
    if (!s) return;
    for (auto ev : s->ring_ready_a) cudaEventDestroy(ev);
    for (auto ev : s->ring_ready) cudaEventDestroy(ev);
    for (auto ev : s->ring_done) cudaEventDestroy(ev);
    if (s->ring_words) cudaFree(s->ring_words);
    if (s->ring_state) cudaFree(s->ring_state);
    if (s->out_nodes) cudaFree(s->out_nodes);
    if (s->out_edges) cudaFree(s->out_edges);
    if (s->arena) cudaFree(s->arena);
    if (s->host_stream) cudaStreamDestroy(s->host_stream);
    delete s;
}

// (Re)allocates the prefetch ring for n streams (synchronises the device: callers size it
// once, e.g. the pipeline runner at creation, so runs never allocate).
int sampler_reserve_ring(Sampler* s, uint32_t n) {
    if (s->ring_n >= n) return FDG_OK;
    FDG_CUDA(cudaDeviceSynchronize());
    for (auto ev : s->ring_ready_a) cudaEventDestroy(ev);
    for (auto ev : s->ring_ready) cudaEventDestroy(ev);
    for (auto ev : s->ring_done) cudaEventDestroy(ev);
    if (s->ring_words) cudaFree(s->ring_words);
    if (s->ring_state) cudaFree(s->ring_state);
    s->ring_words = nullptr;
    s->ring_state = nullptr;
    s->ring_n = 0;
    FDG_CUDA(cudaMalloc(&s->ring_words, uint64_t(n) * s->ring_stride * 8));
    FDG_CUDA(cudaMalloc(&s->ring_state, uint64_t(n) * mt::kN * 8));
    s->ring_n = n;
    s->ring_seed.assign(n, 0);
    s->ring_valid.assign(n, false);
    s->ring_evt.assign(n, 0);
    for (uint32_t i = 0; i < n; ++i) s->ring_evt[i] = i;
    s->ring_ready_a.resize(n);
    s->ring_ready.resize(n);
    s->ring_done.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        FDG_CUDA(cudaEventCreateWithFlags(&s->ring_ready_a[i], cudaEventDisableTiming));
        FDG_CUDA(cudaEventRecord(s->ring_ready_a[i], s->host_stream));
        FDG_CUDA(cudaEventCreateWithFlags(&s->ring_ready[i], cudaEventDisableTiming));
        FDG_CUDA(cudaEventCreateWithFlags(&s->ring_done[i], cudaEventDisableTiming));
        FDG_CUDA(cudaEventRecord(s->ring_done[i], s->host_stream));
    }
    s->ring_next = 0;
    return FDG_OK;
}

// MT streams of upcoming batches, generated concurrently (one CTA each) in a
// single launch on `st`; the ring holds 2x the largest prefetch group.
int sampler_prefetch(Sampler* s, cudaStream_t st, const uint64_t* rng_seeds, uint32_t n) {
    if (n == 0) return FDG_OK;
    if (n > 32) {
        for (uint32_t at = 0; at < n; at += 32) FDG_TRY(sampler_prefetch(s, st, rng_seeds + at, std::min(32u, n - at)));
        return FDG_OK;
    }
    if (s->ring_n < 2 * n) FDG_TRY(sampler_reserve_ring(s, 2 * n));
    uint32_t slots[32];
    for (uint32_t k = 0; k < n; ++k) {
        uint32_t slot = (s->ring_next + k) % s->ring_n;
        slots[k] = slot;
        s->ring_seed[slot] = rng_seeds[k];
        s->ring_valid[slot] = true;
        s->ring_evt[slot] = (s->ring_next) % s->ring_n;  // the chunk's events live at its first slot
    }
    // Slots are consumed in ring order on the sampler's one stream, so the previous occupant of
    // the chunk's last slot is the last of them to be released: one wait covers the chunk, and
    // one pair of events announces it (the host enqueue at a run's start is a few calls per
    // sampler, not a few per batch).
    FDG_CUDA(cudaStreamWaitEvent(st, s->ring_done[slots[n - 1]], 0));
    {
        FDG_TRACE("mt", st);  // piece 1: the words the layers before the last one draw (estimate)
        FDG_CUDA(launch_mt_streams_slots(st, rng_seeds, slots, n, 0, s->words_a, s->ring_words, s->ring_stride,
                                         s->ring_state));
    }
    FDG_CUDA(cudaEventRecord(s->ring_ready_a[slots[0]], st));
    if (s->words_fast > s->words_a) {
        FDG_TRACE("mt", st);  // piece 2: up to the estimate of the whole batch, from the saved state
        FDG_CUDA(launch_mt_streams_slots(st, rng_seeds, slots, n, s->words_a, s->words_fast, s->ring_words,
                                         s->ring_stride, s->ring_state));
    }
    FDG_CUDA(cudaEventRecord(s->ring_ready[slots[0]], st));
    s->ring_next = (s->ring_next + n) % s->ring_n;
    return FDG_OK;
}

// Test hooks (pipeline options "debug_zero_word" / "debug_reject_batch"): zero word `pos` of
// the prefetched stream of `rng_seed` (a genuine Lemire rejection), or flag lane `lane` of the
// next group as rejected. Both are exercised through the in-stream exact replay.
int sampler_debug_zero_word(Sampler* s, cudaStream_t st, uint64_t rng_seed, uint64_t pos) {
    if (pos >= s->words_a) return fail(FDG_INVALID_ARG, "debug_zero_word: position beyond the stream's first piece");
    for (uint32_t r = 0; r < s->ring_n; ++r)
        if (s->ring_valid[r] && s->ring_seed[r] == rng_seed) {
            k_poke_zero<<<1, 1, 0, st>>>(s->ring_words + uint64_t(r) * s->ring_stride + pos);
            FDG_CUDA(cudaGetLastError());
            FDG_CUDA(cudaEventRecord(s->ring_ready_a[s->ring_evt[r]], st));
            FDG_CUDA(cudaEventRecord(s->ring_ready[s->ring_evt[r]], st));
            return FDG_OK;
        }
    return fail(FDG_INVALID_ARG, "debug_zero_word: stream not prefetched");
}

void sampler_debug_reject(Sampler* s, int lane) { s->debug_reject = lane; }
void sampler_set_lean(Sampler* s, bool lean) { s->lean_next = lean; }

// A group of n <= gmax batches in one launch chain on `st`. MT words come from the
// prefetch ring when present, else they are generated inline (one CTA per batch).
int sampler_sample_group(Sampler* s, cudaStream_t st, uint32_t n, const uint64_t* const* seeds, const uint32_t* n_seeds,
                         const uint64_t* rng_seeds, uint64_t* const* nodes, uint32_t* const* edges, uint64_t cap,
                         fdg_batch_counts* const* cnt) {
    if (n == 0) return FDG_OK;
    if (n > s->gmax) return fail(FDG_INVALID_ARG, "sample_group: more batches than the sampler's group size");
    if (cap < s->max_nodes || cap < s->max_edges) return fail(FDG_INVALID_ARG, "sample_khop: output capacity below bound");
    BatchArgs a[kGMax];
    int ring_slot[kGMax];
    uint64_t inline_seeds[kGMax];
    uint32_t n_inline = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (n_seeds[i] > s->max_seeds) return fail(FDG_INVALID_ARG, "sample_khop: more seeds than the sampler was sized for");
        ring_slot[i] = -1;
        for (uint32_t r = 0; r < s->ring_n; ++r)
            if (s->ring_valid[r] && s->ring_seed[r] == rng_seeds[i]) {
                ring_slot[i] = int(r);
                break;
            }
        a[i] = BatchArgs{seeds[i], n_seeds[i], nullptr, s->words_cap, nodes[i], edges[i], cnt[i]};
        if (ring_slot[i] >= 0) {
            const uint32_t r = uint32_t(ring_slot[i]);
            if (i == 0 || s->ring_evt[r] != s->ring_evt[uint32_t(ring_slot[i - 1])])
                FDG_CUDA(cudaStreamWaitEvent(st, s->ring_ready_a[s->ring_evt[r]], 0));
            a[i].words = s->ring_words + uint64_t(r) * s->ring_stride;
            a[i].words_cap = s->ring_stride;
            a[i].words_a = s->words_a;
            a[i].words_ready = s->words_fast;
            a[i].mt_state = s->ring_state + uint64_t(r) * mt::kN;
            a[i].ready = s->ring_ready[s->ring_evt[r]];
            s->ring_valid[ring_slot[i]] = false;
        } else {
            if (n_inline > 0) return fail(FDG_INVALID_ARG, "sample_group: at most one batch without a prefetched stream");
            inline_seeds[n_inline++] = rng_seeds[i];
            a[i].words = s->words;
        }
    }
    if (n_inline) FDG_CUDA(launch_mt_streams(st, inline_seeds, 1, s->words_cap, s->words, s->words_cap));
    FDG_TRY(dispatch_group(*s, st, n, a));
    for (uint32_t i = 0; i < n; ++i)
        if (ring_slot[i] >= 0) FDG_CUDA(cudaEventRecord(s->ring_done[ring_slot[i]], st));
    return FDG_OK;
}

int sampler_sample(Sampler* s, cudaStream_t st, const uint64_t* seeds, uint32_t n_seeds, uint64_t rng_seed,
                   uint64_t* nodes, uint32_t* edges, uint64_t cap, fdg_batch_counts* cnt) {
    return sampler_sample_group(s, st, 1, &seeds, &n_seeds, &rng_seed, &nodes, &edges, cap, &cnt);
}

int sampler_sample_host(Sampler* s, const uint64_t* seeds, uint32_t n_seeds, uint64_t rng_seed,
                        const uint64_t* ext_words, uint64_t n_ext_words, uint64_t* nodes, uint32_t* edges,
                        uint64_t cap, uint64_t* n_nodes, uint64_t* n_edges, uint64_t* layer_nodes,
                        uint64_t* layer_edges, uint64_t* words_used) {
    if (n_seeds > s->max_seeds) return fail(FDG_INVALID_ARG, "sample_khop: more seeds than the sampler was sized for");
    // Reference error order: the first out-of-range seed in chunk order throws.
    for (uint32_t i = 0; i < n_seeds; ++i)
        if (seeds[i] >= s->ctx->num_nodes)
            return fail(FDG_OUT_OF_RANGE, "sample_khop: seed " + std::to_string(seeds[i]) + " out of range");
    cudaStream_t st = s->host_stream;
    if (!s->out_nodes) {
        FDG_CUDA(cudaMalloc(&s->out_nodes, std::max<uint64_t>(s->max_nodes, 1) * 8));
        FDG_CUDA(cudaMalloc(&s->out_edges, std::max<uint64_t>(s->max_edges, 1) * 8));
    }
    FDG_CUDA(cudaMemcpyAsync(s->seeds_buf, seeds, uint64_t(n_seeds) * 8, cudaMemcpyHostToDevice, st));
    uint64_t* ext = nullptr;
    BatchArgs a{s->seeds_buf, n_seeds, s->words, s->words_cap, s->out_nodes, s->out_edges, s->cnt_buf};
    if (ext_words) {
        FDG_CUDA(cudaMalloc(&ext, std::max<uint64_t>(n_ext_words, 1) * 8));
        FDG_CUDA(cudaMemcpyAsync(ext, ext_words, n_ext_words * 8, cudaMemcpyHostToDevice, st));
        a.words = ext;
        a.words_cap = n_ext_words;
    } else {
        FDG_CUDA(launch_mt_streams(st, &rng_seed, 1, s->words_cap, s->words, s->words_cap));
    }
    int rc = dispatch_group(*s, st, 1, &a);
    if (rc) {
        if (ext) cudaFree(ext);
        return rc;
    }
    fdg_batch_counts h;  // a rejected batch was already re-run exactly in-stream (k_replay)
    FDG_CUDA(cudaMemcpyAsync(&h, s->cnt_buf, sizeof(h), cudaMemcpyDeviceToHost, st));
    FDG_CUDA(cudaStreamSynchronize(st));
    if (ext) cudaFree(ext);
    if (h.status == FDG_CAPACITY) return fail(FDG_CAPACITY, "sample_khop: random word stream exhausted");
    if (h.status == FDG_OUT_OF_RANGE)
        return fail(FDG_OUT_OF_RANGE, "sample_khop: seed " + std::to_string(h.bad_seed) + " out of range");
    if (h.status) return fail(int(h.status), "sample_khop: device status " + std::to_string(h.status));
    *n_nodes = h.n_nodes;
    *n_edges = h.n_edges;
    if (h.n_nodes > cap || h.n_edges > cap) return fail(FDG_CAPACITY, "sample_khop: output buffer too small");
    if (nodes) FDG_CUDA(cudaMemcpy(nodes, s->out_nodes, uint64_t(h.n_nodes) * 8, cudaMemcpyDeviceToHost));
    if (edges) FDG_CUDA(cudaMemcpy(edges, s->out_edges, uint64_t(h.n_edges) * 8, cudaMemcpyDeviceToHost));
    if (layer_nodes)
        for (uint32_t i = 0; i < s->n_layers + 2; ++i) layer_nodes[i] = h.layer_nodes[i];
    if (layer_edges)
        for (uint32_t i = 0; i < s->n_layers + 1; ++i) layer_edges[i] = h.layer_edges[i];
    if (words_used) *words_used = h.words_used;
    return FDG_OK;
}

void sampler_hash_region(const Sampler* s, void** base, uint64_t* bytes) {
    *base = s->hash_all_a;  // both tables of every lane (contiguous)
    *bytes = (s->hash_bytes_a + s->hash_bytes) * s->gmax;
}

void sampler_capacity(const Sampler* s, uint64_t* max_nodes, uint64_t* max_edges) {
    *max_nodes = s->max_nodes;
    *max_edges = s->max_edges;
}

}  // namespace fdg
