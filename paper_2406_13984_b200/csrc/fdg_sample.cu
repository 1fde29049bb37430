// fdg_sample.cu -- k-hop uniform in-neighbor sampling with first-occurrence
// dedup/reindex, bit-exact with graph::sample_khop (sampling.hpp:72-134).
//
// Reference semantics (sequential): one std::mt19937_64(splitmix64(rng_seed))
// stream is consumed in (layer, frontier node, Floyd step) order, one
// uniform_int_distribution<u64>(0, j) draw (libstdc++ Lemire, 1 word unless a
// ~2^-57-probability rejection) per Floyd step; picks are interned into
// `nodes` in first-occurrence order; frontier l+1 = fresh ids of layer l, which
// is the contiguous slice nodes[layer_nodes[l+1], layer_nodes[l+2]).
//
// Parallel restatement per batch (all stream-ordered, sizes stay on device):
//   k_seeds    : init the batch record; insert seeds into the batch hash
//                (key -> min position, atomicMin), range-check seeds.
//   k_intern   : one pass per pick list (seeds, then each layer): an entry is a
//                first occurrence iff its pending min position equals the pick's
//                position; a single-pass decoupled look-back scan of
//                (first, min(deg,f), deg>f ? f : 0) assigns local ids in pick
//                order, writes `nodes`, finalises the hash entry, and emits the
//                next frontier's CSR start/degree and pick / MT-draw offsets.
//   k_sample   : one thread per frontier node: Floyd's draws from the
//                pre-generated MT stream at the node's prefix-summed offset
//                (Lemire via __umul64hi), value-compare collisions, insert picks
//                into the hash, write edge dst; also fixes edge src ids of the
//                previous layer (fused with the next layer's launch).
//   k_fix_src  : edge src ids of the last layer.
// A Lemire rejection would consume an extra word and shift every later offset;
// it is detected, the batch is flagged FDG_REJECTION, and the host runs the
// batch again in exact mode (offsets re-derived from per-node consumption).
#include <algorithm>
#include <cstring>
#include <unordered_map>

#include "fdg_internal.cuh"

namespace fdg {
namespace {

constexpr uint32_t kPend = 0x80000000u;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kTile = kScanThreads * kScanItems;
constexpr int kMaxF = 16;  // register-resident Floyd; larger fanouts use the scratch path

template <typename IdT> struct Empty;
template <> struct Empty<uint32_t> { static constexpr uint32_t v = 0xFFFFFFFFu; };
template <> struct Empty<uint64_t> { static constexpr uint64_t v = ~0ull; };

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

template <typename IdT>
struct Work {
    const uint64_t* indptr;
    const IdT* indices;
    uint64_t num_nodes;
    IdT* keys;           // hash keys
    uint32_t* vals;      // hash values: final local id, or kPend | min position
    uint32_t hmask;
    uint32_t* seed_slot; // [max_seeds]
    uint32_t* pick_slot; // [max_edges], indexed by global edge position
    IdT* scratch;        // [max_edges] picks for the large-fanout path
    FrontierBuf fr[2];
    uint32_t* consumed;  // exact mode: words consumed per frontier node
    uint32_t* tile_flag; // decoupled look-back state
    uint4* tile_agg;
    uint4* tile_incl;
    uint32_t* tile_ctr;  // per-pass dynamic tile counters
    const uint64_t* words;
    uint64_t words_cap;
    uint64_t* nodes;     // output
    uint32_t* edges;     // output, {src, dst} pairs
    fdg_batch_counts* cnt;
    uint32_t fan[FDG_MAX_LAYERS];
    uint32_t n_layers;
};

__device__ __forceinline__ uint32_t hslot(uint64_t key, uint32_t mask) {
    return uint32_t((key * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}

__device__ __forceinline__ uint32_t atomic_cas_key(uint32_t* p, uint32_t cmp, uint32_t v) { return atomicCAS(p, cmp, v); }
__device__ __forceinline__ uint64_t atomic_cas_key(uint64_t* p, uint64_t cmp, uint64_t v) {
    return atomicCAS(reinterpret_cast<unsigned long long*>(p), (unsigned long long)cmp, (unsigned long long)v);
}

// Insert `key` (or find it) and lower its pending position to `pos`. Entries
// finalised by an earlier pass hold a local id < kPend and are left unchanged.
template <typename IdT>
__device__ __forceinline__ uint32_t hash_insert(IdT* keys, uint32_t* vals, uint32_t mask, IdT key, uint32_t pos) {
    uint32_t h = hslot(key, mask);
    for (;;) {
        IdT cur = keys[h];
        if (cur == Empty<IdT>::v) cur = atomic_cas_key(keys + h, Empty<IdT>::v, key);
        if (cur == Empty<IdT>::v || cur == key) {
            atomicMin(vals + h, kPend | pos);
            return h;
        }
        h = (h + 1) & mask;
    }
}

// libstdc++ uniform_int_distribution<u64>(0, j) on word stream w (uniform_int_dist.h:257-281).
__device__ __forceinline__ uint64_t lemire(const uint64_t* words, uint64_t cap, uint64_t& pos, uint64_t j,
                                           uint32_t& extra, bool& overflow) {
    const uint64_t r = j + 1;
    uint64_t w = pos < cap ? words[pos] : 0;
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
template <typename IdT>
__global__ void __launch_bounds__(1024) k_seeds(Work<IdT> W, const uint64_t* seeds, uint32_t n_seeds) {
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
        cnt->pad = 0;
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
    for (uint32_t p = threadIdx.x; p < n_seeds; p += blockDim.x) {
        uint64_t s = seeds[p];
        if (s >= W.num_nodes) {  // sampling.hpp:89-93
            atomicMin(&cnt->bad_seed_pos, p);
            cnt->status = FDG_OUT_OF_RANGE;
            continue;
        }
        W.seed_slot[p] = hash_insert<IdT>(W.keys, W.vals, W.hmask, IdT(s), p);
    }
    __syncthreads();
    if (threadIdx.x == 0 && cnt->status == FDG_OUT_OF_RANGE) cnt->bad_seed = seeds[cnt->bad_seed_pos];
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

// ---------------------------------------------------------------- k_intern ----
// Pass q interns pick list q (q = 0: seeds; q = l+1: picks of layer l) and sets
// up the frontier of layer q (when q < n_layers).
template <typename IdT, bool SEEDS, bool HAS_NEXT>
__global__ void __launch_bounds__(kScanThreads) k_intern(Work<IdT> W, uint32_t q, uint32_t n_seeds, uint32_t epoch) {
    __shared__ Tri s_warp[kScanThreads / 32];
    __shared__ Tri s_excl;
    __shared__ uint32_t s_tile;
    fdg_batch_counts* cnt = W.cnt;
    if (cnt->status) return;
    const uint32_t P = SEEDS ? n_seeds : cnt->layer_edges[q] - cnt->layer_edges[q - 1];
    const uint32_t ebase = SEEDS ? 0 : cnt->layer_edges[q - 1];
    const uint32_t node_base = cnt->layer_nodes[q];
    const uint32_t ntiles = P ? (P + kTile - 1) / kTile : 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(W.tile_ctr + q, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint32_t f = HAS_NEXT ? W.fan[q] : 0;
    const uint32_t p0 = tile * kTile + tid * kScanItems;

    uint32_t slot[kScanItems];
    uint32_t first_mask = 0;
    uint32_t degs[kScanItems];
    IdT key[kScanItems];
    Tri mine{0, 0, 0};
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        uint32_t p = p0 + k;
        degs[k] = 0;
        if (p < P) {
            slot[k] = SEEDS ? W.seed_slot[p] : W.pick_slot[ebase + p];
            if (W.vals[slot[k]] == (kPend | p)) {
                first_mask |= 1u << k;
                key[k] = W.keys[slot[k]];
                mine.c += 1;
                if (HAS_NEXT) {
                    uint64_t v = uint64_t(key[k]);
                    uint32_t d = uint32_t(W.indptr[v + 1] - W.indptr[v]);
                    degs[k] = d;
                    mine.p += d < f ? d : f;
                    mine.d += d > f ? f : 0;
                }
            }
        }
    }
    // block exclusive scan of `mine`
    Tri incl = warp_incl_scan(mine, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        Tri w = lane < kScanThreads / 32 ? s_warp[lane] : Tri{0, 0, 0};
        Tri wi = warp_incl_scan(w, lane);
        if (lane < kScanThreads / 32) s_warp[lane] = Tri{wi.c - w.c, wi.p - w.p, wi.d - w.d};
        Tri agg{__shfl_sync(0xffffffffu, wi.c, 31), __shfl_sync(0xffffffffu, wi.p, 31),
                __shfl_sync(0xffffffffu, wi.d, 31)};
        // decoupled look-back
        const uint32_t E = (epoch & 0x3FFFFFFFu) << 2;
        Tri excl{0, 0, 0};
        if (tile == 0) {
            if (lane == 0) {
                W.tile_incl[0] = make_uint4(agg.c, agg.p, agg.d, 0);
                __threadfence();
                atomicExch(W.tile_flag + 0, E | 2u);
            }
        } else {
            if (lane == 0) {
                W.tile_agg[tile] = make_uint4(agg.c, agg.p, agg.d, 0);
                __threadfence();
                atomicExch(W.tile_flag + tile, E | 1u);
            }
            int j = int(tile) - 1;
            for (;;) {
                int jj = j - lane;
                uint32_t st = 2;
                if (jj >= 0) {
                    uint32_t fl = ld_volatile(W.tile_flag + jj);
                    st = (fl & ~3u) == E ? (fl & 3u) : 0u;
                }
                if (__any_sync(0xffffffffu, st == 0)) continue;
                uint32_t im = __ballot_sync(0xffffffffu, st == 2);
                int stop = im ? __ffs(im) - 1 : 32;  // nearest inclusive predecessor in this window
                __threadfence();
                Tri v{0, 0, 0};
                if (lane < stop) {
                    uint4 a = ld_volatile4(W.tile_agg + jj);
                    v = Tri{a.x, a.y, a.z};
                } else if (lane == stop && jj >= 0) {
                    uint4 a = ld_volatile4(W.tile_incl + jj);
                    v = Tri{a.x, a.y, a.z};
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    v.c += __shfl_xor_sync(0xffffffffu, v.c, o);
                    v.p += __shfl_xor_sync(0xffffffffu, v.p, o);
                    v.d += __shfl_xor_sync(0xffffffffu, v.d, o);
                }
                excl = excl + v;
                if (stop < 32) break;
                j -= 32;
            }
            if (lane == 0) {
                Tri tot = excl + agg;
                W.tile_incl[tile] = make_uint4(tot.c, tot.p, tot.d, 0);
                __threadfence();
                atomicExch(W.tile_flag + tile, E | 2u);
            }
        }
        if (lane == 0) {
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
                if (SEEDS && !HAS_NEXT) cnt->n_edges = 0;
            }
        }
    }
    __syncthreads();
    Tri run = s_excl + s_warp[warp] + Tri{incl.c - mine.c, incl.p - mine.p, incl.d - mine.d};
    if (first_mask) {
        const FrontierBuf fr = W.fr[q & 1];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (first_mask & (1u << k)) {
                const uint32_t local = node_base + run.c;
                W.nodes[local] = uint64_t(key[k]);
                W.vals[slot[k]] = local;
                if (HAS_NEXT) {
                    uint32_t d = degs[k];
                    fr.start[run.c] = W.indptr[uint64_t(key[k])];
                    fr.deg[run.c] = d;
                    fr.pick_off[run.c] = run.p;
                    fr.draw_off[run.c] = run.d;
                    run.p += d < f ? d : f;
                    run.d += d > f ? f : 0;
                }
                run.c += 1;
            }
        }
    }
}

// ---------------------------------------------------------------- k_sample ----
// MODE 0: sample + insert (fast path). MODE 1: exact-mode probe (count words
// consumed per node, no inserts). MODE 2: exact-mode final (inserts, offsets
// from W.consumed-derived draw_off).
template <typename IdT, bool SMALLF, int MODE>
__global__ void __launch_bounds__(256) k_sample(Work<IdT> W, uint32_t l) {
    fdg_batch_counts* cnt = W.cnt;
    if (cnt->status) return;
    const uint32_t fs = cnt->layer_nodes[l];
    const uint32_t F = cnt->layer_nodes[l + 1] - fs;
    const uint32_t eb = cnt->layer_edges[l];
    const uint64_t db = cnt->layer_draws[l];
    const uint32_t f = W.fan[l];
    // edge src fix-up of the previous layer (its ids are final now)
    const uint32_t fix_lo = l > 0 ? cnt->layer_edges[l - 1] : 0;
    const uint32_t fix_hi = l > 0 ? eb : 0;
    const FrontierBuf fr = W.fr[l & 1];
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t span = max(F, fix_hi - fix_lo);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < span; i += stride) {
        if (MODE != 1 && i < fix_hi - fix_lo) {
            uint32_t e = fix_lo + i;
            W.edges[2 * e] = W.vals[W.pick_slot[e]];
        }
        if (i >= F) continue;
        const uint64_t start = fr.start[i];
        const uint32_t deg = fr.deg[i];
        const uint32_t po = fr.pick_off[i];
        const uint32_t dst = fs + i;
        const uint32_t e0 = eb + po;
        if (deg <= f) {  // take all, in list order (sampling.hpp:107-108)
            if (MODE == 1) {
                W.consumed[i] = 0;
                continue;
            }
            for (uint32_t k = 0; k < deg; ++k) {
                IdT v = W.indices[start + k];
                W.pick_slot[e0 + k] = hash_insert<IdT>(W.keys, W.vals, W.hmask, v, po + k);
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
                    cand[k] = W.indices[start + t[k]];
                    alt[k] = W.indices[start + jlo + k];
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
                    W.pick_slot[e0 + k] = hash_insert<IdT>(W.keys, W.vals, W.hmask, picked[k], po + k);
                    W.edges[2 * (e0 + k) + 1] = dst;
                }
        } else {
            IdT* picked = W.scratch + e0;
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
            }
            if (MODE == 1) {
                W.consumed[i] = f + extra;
                continue;
            }
            for (uint32_t k = 0; k < f; ++k) {
                W.pick_slot[e0 + k] = hash_insert<IdT>(W.keys, W.vals, W.hmask, picked[k], po + k);
                W.edges[2 * (e0 + k) + 1] = dst;
            }
        }
        if (overflow) atomicExch(&cnt->status, uint32_t(FDG_CAPACITY));
        if (MODE == 0 && extra) {
            atomicAdd(&cnt->rejections, extra);
            atomicCAS(&cnt->status, 0u, uint32_t(FDG_REJECTION));
        }
    }
}

template <typename IdT>
__global__ void k_fix_src(Work<IdT> W, uint32_t l) {
    fdg_batch_counts* cnt = W.cnt;
    if (cnt->status) return;
    const uint32_t lo = cnt->layer_edges[l], hi = cnt->layer_edges[l + 1];
    for (uint32_t e = lo + blockIdx.x * blockDim.x + threadIdx.x; e < hi; e += gridDim.x * blockDim.x)
        W.edges[2 * e] = W.vals[W.pick_slot[e]];
}

// exact mode helper: draw_off = exclusive scan(consumed) over the frontier (single block)
__global__ void k_rescan_draws(uint32_t* consumed, uint32_t* draw_off, const fdg_batch_counts* cnt, uint32_t l,
                               uint32_t* changed, uint32_t* total) {
    __shared__ uint32_t s_carry;
    __shared__ uint32_t s_warp[32];
    const uint32_t F = cnt->layer_nodes[l + 1] - cnt->layer_nodes[l];
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t base = 0; base < F; base += blockDim.x) {
        uint32_t i = base + threadIdx.x;
        uint32_t v = i < F ? consumed[i] : 0;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = lane < int(blockDim.x / 32) ? s_warp[lane] : 0;
            uint32_t wx = w;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, wx, o);
                if (lane >= o) wx += y;
            }
            if (lane < int(blockDim.x / 32)) s_warp[lane] = wx - w;
        }
        __syncthreads();
        uint32_t excl = s_carry + s_warp[warp] + x - v;
        if (i < F) {
            if (draw_off[i] != excl) *changed = 1;
            draw_off[i] = excl;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

}  // namespace

// ------------------------------------------------------------------ Sampler ----
struct Sampler {
    Ctx* ctx = nullptr;
    uint32_t max_seeds = 0;
    uint32_t n_layers = 0;
    uint32_t fan[FDG_MAX_LAYERS] = {};
    uint64_t max_nodes = 0, max_edges = 0, max_draws = 0;
    uint64_t F_bound[FDG_MAX_LAYERS + 1] = {}, P_bound[FDG_MAX_LAYERS + 1] = {};
    uint32_t hsize = 0;
    bool small_f = true;
    void* arena = nullptr;
    // carved pointers
    void* keys = nullptr;
    uint32_t* vals = nullptr;
    uint32_t* seed_slot = nullptr;
    uint32_t* pick_slot = nullptr;
    void* scratch = nullptr;
    FrontierBuf fr[2];
    uint32_t* consumed = nullptr;
    uint32_t* tile_flag = nullptr;
    uint4* tile_agg = nullptr;
    uint4* tile_incl = nullptr;
    uint32_t* tile_ctr = nullptr;
    uint32_t* exact_flags = nullptr;  // [changed, total]
    uint64_t* words = nullptr;         // inline MT stream
    uint64_t words_cap = 0;
    uint64_t* seeds_buf = nullptr;     // host-API staging
    uint64_t hash_bytes = 0;
    uint32_t epoch = 1;
    // prefetch ring
    uint32_t ring_n = 0;
    uint64_t* ring_words = nullptr;
    std::vector<uint64_t> ring_seed;
    std::vector<bool> ring_valid;
    std::vector<cudaEvent_t> ring_ready, ring_done;
    uint32_t ring_next = 0;
    cudaStream_t host_stream = nullptr;
    fdg_batch_counts* cnt_buf = nullptr;  // host-API counts
    uint64_t* out_nodes = nullptr;        // host-API outputs
    uint32_t* out_edges = nullptr;
};

}  // namespace fdg

struct fdg_sampler : fdg::Sampler {};

namespace fdg {
namespace {

uint64_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

template <typename IdT>
Work<IdT> make_work(Sampler& s, const uint64_t* words, uint64_t words_cap, uint64_t* nodes, uint32_t* edges,
                    fdg_batch_counts* cnt) {
    Work<IdT> w;
    w.indptr = s.ctx->indptr;
    w.indices = static_cast<const IdT*>(s.ctx->indices);
    w.num_nodes = s.ctx->num_nodes;
    w.keys = static_cast<IdT*>(s.keys);
    w.vals = s.vals;
    w.hmask = s.hsize - 1;
    w.seed_slot = s.seed_slot;
    w.pick_slot = s.pick_slot;
    w.scratch = static_cast<IdT*>(s.scratch);
    w.fr[0] = s.fr[0];
    w.fr[1] = s.fr[1];
    w.consumed = s.consumed;
    w.tile_flag = s.tile_flag;
    w.tile_agg = s.tile_agg;
    w.tile_incl = s.tile_incl;
    w.tile_ctr = s.tile_ctr;
    w.words = words;
    w.words_cap = words_cap;
    w.nodes = nodes;
    w.edges = edges;
    w.cnt = cnt;
    for (uint32_t l = 0; l < FDG_MAX_LAYERS; ++l) w.fan[l] = l < s.n_layers ? s.fan[l] : 0;
    w.n_layers = s.n_layers;
    return w;
}

uint32_t grid_for(uint64_t items, int threads, int max_blocks) {
    uint64_t b = (items + threads - 1) / threads;
    return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(b, uint64_t(max_blocks))));
}

template <typename IdT>
void launch_intern(Sampler& s, cudaStream_t st, const Work<IdT>& W, uint32_t q, uint32_t n_seeds) {
    const bool seeds = q == 0;
    const bool has_next = q < s.n_layers;
    const uint64_t P = seeds ? n_seeds : s.P_bound[q - 1];
    const uint32_t tiles = uint32_t(std::max<uint64_t>(1, (P + kTile - 1) / kTile));
    const uint32_t ep = s.epoch++;
    if (seeds) {
        if (has_next) k_intern<IdT, true, true><<<tiles, kScanThreads, 0, st>>>(W, q, n_seeds, ep);
        else k_intern<IdT, true, false><<<tiles, kScanThreads, 0, st>>>(W, q, n_seeds, ep);
    } else {
        if (has_next) k_intern<IdT, false, true><<<tiles, kScanThreads, 0, st>>>(W, q, n_seeds, ep);
        else k_intern<IdT, false, false><<<tiles, kScanThreads, 0, st>>>(W, q, n_seeds, ep);
    }
}

template <typename IdT, int MODE>
void launch_sample(Sampler& s, cudaStream_t st, const Work<IdT>& W, uint32_t l) {
    uint64_t span = std::max<uint64_t>(s.F_bound[l], l > 0 ? s.P_bound[l - 1] : 0);
    uint32_t blocks = grid_for(span, 256, s.ctx->sm_count * 8);
    if (s.small_f) k_sample<IdT, true, MODE><<<blocks, 256, 0, st>>>(W, l);
    else k_sample<IdT, false, MODE><<<blocks, 256, 0, st>>>(W, l);
}

// Fast path: everything stream-ordered, no host synchronisation.
template <typename IdT>
int run_batch(Sampler& s, cudaStream_t st, const uint64_t* seeds, uint32_t n_seeds, const uint64_t* words,
              uint64_t words_cap, uint64_t* nodes, uint32_t* edges, fdg_batch_counts* cnt) {
    Work<IdT> W = make_work<IdT>(s, words, words_cap, nodes, edges, cnt);
    FDG_CUDA(cudaMemsetAsync(s.keys, 0xFF, s.hash_bytes, st));
    k_seeds<IdT><<<1, 1024, 0, st>>>(W, seeds, n_seeds);
    launch_intern<IdT>(s, st, W, 0, n_seeds);
    for (uint32_t l = 0; l < s.n_layers; ++l) {
        launch_sample<IdT, 0>(s, st, W, l);
        launch_intern<IdT>(s, st, W, l + 1, n_seeds);
    }
    uint32_t lastl = s.n_layers - 1;
    k_fix_src<IdT><<<grid_for(s.P_bound[lastl], 256, s.ctx->sm_count * 8), 256, 0, st>>>(W, lastl);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

// Exact mode (after a Lemire rejection): per layer, iterate probe -> rescan of
// the per-node word consumption until the draw offsets are self-consistent,
// then run the inserting pass. Host-synchronising; never taken in practice.
template <typename IdT>
int run_batch_exact(Sampler& s, cudaStream_t st, const uint64_t* seeds, uint32_t n_seeds, const uint64_t* words,
                    uint64_t words_cap, uint64_t* nodes, uint32_t* edges, fdg_batch_counts* cnt) {
    Work<IdT> W = make_work<IdT>(s, words, words_cap, nodes, edges, cnt);
    FDG_CUDA(cudaMemsetAsync(s.keys, 0xFF, s.hash_bytes, st));
    k_seeds<IdT><<<1, 1024, 0, st>>>(W, seeds, n_seeds);
    launch_intern<IdT>(s, st, W, 0, n_seeds);
    for (uint32_t l = 0; l < s.n_layers; ++l) {
        for (int it = 0;; ++it) {
            launch_sample<IdT, 1>(s, st, W, l);
            FDG_CUDA(cudaMemsetAsync(s.exact_flags, 0, 8, st));
            k_rescan_draws<<<1, 1024, 0, st>>>(s.consumed, s.fr[l & 1].draw_off, cnt, l, s.exact_flags,
                                               s.exact_flags + 1);
            uint32_t h[2];
            FDG_CUDA(cudaMemcpyAsync(h, s.exact_flags, 8, cudaMemcpyDeviceToHost, st));
            FDG_CUDA(cudaStreamSynchronize(st));
            if (!h[0]) {
                // fix the next layer's draw base: layer_draws[l+1] = layer_draws[l] + total
                uint32_t base = 0;
                FDG_CUDA(cudaMemcpy(&base, &cnt->layer_draws[l], 4, cudaMemcpyDeviceToHost));
                uint32_t nb = base + h[1];
                FDG_CUDA(cudaMemcpy(&cnt->layer_draws[l + 1], &nb, 4, cudaMemcpyHostToDevice));
                break;
            }
            if (it > 1 << 20) return fail(FDG_INVARIANT, "exact mode did not converge");
        }
        launch_sample<IdT, 2>(s, st, W, l);
        launch_intern<IdT>(s, st, W, l + 1, n_seeds);  // bases layer_draws[l+2] on the corrected [l+1]
    }
    uint32_t lastl = s.n_layers - 1;
    k_fix_src<IdT><<<grid_for(s.P_bound[lastl], 256, s.ctx->sm_count * 8), 256, 0, st>>>(W, lastl);
    FDG_CUDA(cudaGetLastError());
    FDG_CUDA(cudaStreamSynchronize(st));
    return FDG_OK;
}

int dispatch_batch(Sampler& s, cudaStream_t st, const uint64_t* seeds, uint32_t n_seeds, const uint64_t* words,
                   uint64_t words_cap, uint64_t* nodes, uint32_t* edges, fdg_batch_counts* cnt, bool exact) {
    if (s.ctx->idx_bytes == 4)
        return exact ? run_batch_exact<uint32_t>(s, st, seeds, n_seeds, words, words_cap, nodes, edges, cnt)
                     : run_batch<uint32_t>(s, st, seeds, n_seeds, words, words_cap, nodes, edges, cnt);
    return exact ? run_batch_exact<uint64_t>(s, st, seeds, n_seeds, words, words_cap, nodes, edges, cnt)
                 : run_batch<uint64_t>(s, st, seeds, n_seeds, words, words_cap, nodes, edges, cnt);
}

}  // namespace

int sampler_create(Ctx* ctx, uint32_t max_seeds, const uint32_t* fanouts, uint32_t n_layers, Sampler** out) {
    if (!ctx->indptr) return fail(FDG_NOT_LOADED, "sampler: no topology loaded");
    if (n_layers == 0) return fail(FDG_INVALID_ARG, "fanouts: need at least one layer");
    if (n_layers > FDG_MAX_LAYERS) return fail(FDG_INVALID_ARG, "fanouts: more than FDG_MAX_LAYERS layers");
    for (uint32_t l = 0; l < n_layers; ++l)
        if (fanouts[l] < 1) return fail(FDG_INVALID_ARG, "fanouts: every entry must be >= 1");
    if (max_seeds == 0) max_seeds = 1;
    auto s = new Sampler();
    s->ctx = ctx;
    s->max_seeds = max_seeds;
    s->n_layers = n_layers;
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
    s->hsize = uint32_t(next_pow2(std::max<uint64_t>(2 * s->max_nodes, 1024)));
    const uint32_t ib = ctx->idx_bytes;
    s->hash_bytes = uint64_t(s->hsize) * (ib + 4);
    uint64_t fmaxF = 1;
    for (uint32_t l = 0; l < n_layers; ++l) fmaxF = std::max(fmaxF, s->F_bound[l]);
    const uint64_t tiles = (std::max<uint64_t>(s->max_edges, max_seeds) + kTile - 1) / kTile + 1;
    s->words_cap = s->max_draws + 4096;
    auto al = [](uint64_t b) { return (b + 255) & ~uint64_t(255); };
    uint64_t sz = 0;
    const uint64_t o_keys = sz; sz += al(s->hash_bytes);  // keys then vals: one memset
    const uint64_t o_seed = sz; sz += al(uint64_t(max_seeds) * 4);
    const uint64_t o_pick = sz; sz += al(std::max<uint64_t>(s->max_edges, 1) * 4);
    const uint64_t o_scr = sz; sz += s->small_f ? 0 : al(std::max<uint64_t>(s->max_edges, 1) * ib);
    uint64_t o_fr[2];
    for (int b = 0; b < 2; ++b) { o_fr[b] = sz; sz += al(fmaxF * 8) + 3 * al(fmaxF * 4); }
    const uint64_t o_cons = sz; sz += al(fmaxF * 4);
    const uint64_t o_flag = sz; sz += al(tiles * 4);
    const uint64_t o_agg = sz; sz += al(tiles * 16);
    const uint64_t o_inc = sz; sz += al(tiles * 16);
    const uint64_t o_ctr = sz; sz += al((FDG_MAX_LAYERS + 2) * 4);
    const uint64_t o_ex = sz; sz += al(16);
    const uint64_t o_words = sz; sz += al(s->words_cap * 8);
    const uint64_t o_seeds = sz; sz += al(uint64_t(max_seeds) * 8);
    const uint64_t o_cnt = sz; sz += al(sizeof(fdg_batch_counts));
    cudaError_t e = cudaMalloc(&s->arena, sz);
    if (e != cudaSuccess) {
        delete s;
        return cuda_fail(e, "cudaMalloc(sampler arena)", __FILE__, __LINE__);
    }
    char* a = static_cast<char*>(s->arena);
    s->keys = a + o_keys;
    s->vals = reinterpret_cast<uint32_t*>(a + o_keys + uint64_t(s->hsize) * ib);
    s->seed_slot = reinterpret_cast<uint32_t*>(a + o_seed);
    s->pick_slot = reinterpret_cast<uint32_t*>(a + o_pick);
    s->scratch = s->small_f ? nullptr : a + o_scr;
    for (int b = 0; b < 2; ++b) {
        char* p = a + o_fr[b];
        s->fr[b].start = reinterpret_cast<uint64_t*>(p);
        p += al(fmaxF * 8);
        s->fr[b].deg = reinterpret_cast<uint32_t*>(p);
        p += al(fmaxF * 4);
        s->fr[b].pick_off = reinterpret_cast<uint32_t*>(p);
        p += al(fmaxF * 4);
        s->fr[b].draw_off = reinterpret_cast<uint32_t*>(p);
    }
    s->consumed = reinterpret_cast<uint32_t*>(a + o_cons);
    s->tile_flag = reinterpret_cast<uint32_t*>(a + o_flag);
    s->tile_agg = reinterpret_cast<uint4*>(a + o_agg);
    s->tile_incl = reinterpret_cast<uint4*>(a + o_inc);
    s->tile_ctr = reinterpret_cast<uint32_t*>(a + o_ctr);
    s->exact_flags = reinterpret_cast<uint32_t*>(a + o_ex);
    s->words = reinterpret_cast<uint64_t*>(a + o_words);
    s->seeds_buf = reinterpret_cast<uint64_t*>(a + o_seeds);
    s->cnt_buf = reinterpret_cast<fdg_batch_counts*>(a + o_cnt);
    cudaMemset(s->tile_flag, 0, tiles * 4);
    e = cudaStreamCreateWithFlags(&s->host_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate", __FILE__, __LINE__);
    *out = s;
    return FDG_OK;
}

void sampler_destroy(Sampler* s) {
    if (!s) return;
    for (auto ev : s->ring_ready) cudaEventDestroy(ev);
    for (auto ev : s->ring_done) cudaEventDestroy(ev);
    if (s->ring_words) cudaFree(s->ring_words);
    if (s->out_nodes) cudaFree(s->out_nodes);
    if (s->out_edges) cudaFree(s->out_edges);
    if (s->arena) cudaFree(s->arena);
    if (s->host_stream) cudaStreamDestroy(s->host_stream);
    delete s;
}

int sampler_prefetch(Sampler* s, cudaStream_t st, const uint64_t* rng_seeds, uint32_t n) {
    if (n == 0) return FDG_OK;
    if (s->ring_n < n) {
        // (re)build a ring of n stream slots
        FDG_CUDA(cudaDeviceSynchronize());
        for (auto ev : s->ring_ready) cudaEventDestroy(ev);
        for (auto ev : s->ring_done) cudaEventDestroy(ev);
        if (s->ring_words) cudaFree(s->ring_words);
        s->ring_n = n;
        FDG_CUDA(cudaMalloc(&s->ring_words, uint64_t(n) * s->words_cap * 8));
        s->ring_seed.assign(n, 0);
        s->ring_valid.assign(n, false);
        s->ring_ready.resize(n);
        s->ring_done.resize(n);
        for (uint32_t i = 0; i < n; ++i) {
            FDG_CUDA(cudaEventCreateWithFlags(&s->ring_ready[i], cudaEventDisableTiming));
            FDG_CUDA(cudaEventCreateWithFlags(&s->ring_done[i], cudaEventDisableTiming));
            FDG_CUDA(cudaEventRecord(s->ring_done[i], st));
        }
        s->ring_next = 0;
    }
    // claim n consecutive ring slots (wrapping), one MT CTA per stream
    for (uint32_t k = 0; k < n; ++k) {
        uint32_t slot = (s->ring_next + k) % s->ring_n;
        FDG_CUDA(cudaStreamWaitEvent(st, s->ring_done[slot], 0));
        s->ring_seed[slot] = rng_seeds[k];
        s->ring_valid[slot] = true;
        FDG_CUDA(launch_mt_streams(st, &rng_seeds[k], 1, s->words_cap, s->ring_words + uint64_t(slot) * s->words_cap,
                                   s->words_cap));
        FDG_CUDA(cudaEventRecord(s->ring_ready[slot], st));
    }
    s->ring_next = (s->ring_next + n) % s->ring_n;
    return FDG_OK;
}

int sampler_sample(Sampler* s, cudaStream_t st, const uint64_t* seeds, uint32_t n_seeds, uint64_t rng_seed,
                   uint64_t* nodes, uint32_t* edges, uint64_t cap, fdg_batch_counts* cnt) {
    if (n_seeds > s->max_seeds) return fail(FDG_INVALID_ARG, "sample_khop: more seeds than the sampler was sized for");
    if (cap < s->max_nodes || cap < s->max_edges) return fail(FDG_INVALID_ARG, "sample_khop: output capacity below bound");
    const uint64_t* words = nullptr;
    int ring_slot = -1;
    for (uint32_t i = 0; i < s->ring_n; ++i)
        if (s->ring_valid[i] && s->ring_seed[i] == rng_seed) {
            ring_slot = int(i);
            break;
        }
    if (ring_slot >= 0) {
        FDG_CUDA(cudaStreamWaitEvent(st, s->ring_ready[ring_slot], 0));
        words = s->ring_words + uint64_t(ring_slot) * s->words_cap;
        s->ring_valid[ring_slot] = false;
    } else {
        FDG_CUDA(launch_mt_streams(st, &rng_seed, 1, s->words_cap, s->words, s->words_cap));
        words = s->words;
    }
    FDG_TRY(dispatch_batch(*s, st, seeds, n_seeds, words, s->words_cap, nodes, edges, cnt, false));
    if (ring_slot >= 0) FDG_CUDA(cudaEventRecord(s->ring_done[ring_slot], st));
    return FDG_OK;
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
    const uint64_t* words;
    uint64_t wcap;
    uint64_t* ext = nullptr;
    if (ext_words) {
        FDG_CUDA(cudaMalloc(&ext, std::max<uint64_t>(n_ext_words, 1) * 8));
        FDG_CUDA(cudaMemcpyAsync(ext, ext_words, n_ext_words * 8, cudaMemcpyHostToDevice, st));
        words = ext;
        wcap = n_ext_words;
    } else {
        FDG_CUDA(launch_mt_streams(st, &rng_seed, 1, s->words_cap, s->words, s->words_cap));
        words = s->words;
        wcap = s->words_cap;
    }
    int rc = dispatch_batch(*s, st, s->seeds_buf, n_seeds, words, wcap, s->out_nodes, s->out_edges, s->cnt_buf, false);
    if (rc) {
        if (ext) cudaFree(ext);
        return rc;
    }
    fdg_batch_counts h;
    FDG_CUDA(cudaMemcpyAsync(&h, s->cnt_buf, sizeof(h), cudaMemcpyDeviceToHost, st));
    FDG_CUDA(cudaStreamSynchronize(st));
    if (h.status == FDG_REJECTION) {
        rc = dispatch_batch(*s, st, s->seeds_buf, n_seeds, words, wcap, s->out_nodes, s->out_edges, s->cnt_buf, true);
        if (rc == FDG_OK) {
            FDG_CUDA(cudaMemcpyAsync(&h, s->cnt_buf, sizeof(h), cudaMemcpyDeviceToHost, st));
            FDG_CUDA(cudaStreamSynchronize(st));
        }
    }
    if (ext) cudaFree(ext);
    if (rc) return rc;
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

}  // namespace fdg

namespace fdg {
void sampler_capacity(const Sampler* s, uint64_t* max_nodes, uint64_t* max_edges) {
    *max_nodes = s->max_nodes;
    *max_edges = s->max_edges;
}
}  // namespace fdg
