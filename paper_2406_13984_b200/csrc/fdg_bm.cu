// fdg_bm.cu -- the holistic feature-buffer manager on the GPU.
//
// Replaces featbuf::BufferManager (buffer_manager.hpp:222-527) + FeatureRegion
// (device_region.hpp:24-50) + the extractor's metadata protocol
// (extractor.hpp:142-151, 391-394) for stream-ordered batches. Exactly the
// reference's state transitions and LRU order, computed batch-parallel:
//
//   mapping table  node -> packed {i32 slot, u32 valid<<31}  (8 B/node), invalidated
//                  lazily: an entry is live only while slot[entry.slot]'s owner still
//                  names the node, so an eviction rebinds the slot without touching the
//                  previous owner's entry (two random DRAM accesses per miss saved; the
//                  acquire's owner check reads the slot record, which mostly hits L2)
//   slot table     slot -> {u64 owner node (40 bits; all ones = free) | reference count
//                  << 40, u64 ring position of its live standby entry (~0 = not in the
//                  standby list)}: one 16-byte record, so the reverse map, the bound node's
//                  reference count (the reference keeps it in the mapping entry) and list
//                  membership share a sector -- an acquire hit, a bind and a release each
//                  touch one random record instead of a record plus a separate count
//   standby list   the reference's intrusive LRU list becomes a FIFO ring of
//                  slot ids with tombstones: push_mru = append at `tail`
//                  (recording the slot's ring position), remove(slot) on a hit
//                  = clear the slot's position (the stale ring entry is skipped
//                  later), pop_lru = the next live entry from `head`. An entry
//                  at position p is live iff slot[s].pos == p.
//
// The metadata kernels are bound by random DRAM sector accesses (~23 G sectors/s
// on B200, measured: long-scoreboard stalls at <1 TB/s): every kernel issues all
// of a thread's independent random loads before its first store (items of one
// batch are distinct nodes / slots, so there are no hazards between them), and the
// row traffic of k_move is marked L2 evict-first so the batch's metadata sectors
// stay L2-resident between acquire, bind and the lag-1 release.
//
// extract(nodes):                                   reference
//   k_acquire  classify + ref++ + standby remove;   acquire_for_batch 241-269
//              ordered rank of to-load positions (decoupled look-back)
//   k_select   first L live ring entries from head  get_standby_slot 274-294 (xL, batch order)
//   k_bind     evict previous owner, bind, publish  bind_slot 297-310, publish_valid 313-324
//   k_move     misses: table -> slot (and -> X); hits: slot -> X (mini-batch tensor)
// release(nodes):
//   k_release  ref--; slots reaching 0 appended in batch order   release_batch 352-364, 461-476
//   k_compact  drops tombstones when the ring nears capacity (persistent grid, no-op otherwise)
//
// Parity: alias lists, hits/loads/evictions and mapping entries equal the
// reference BufferManager driven by the same sequential schedule (tests/).
#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "fdg_internal.cuh"
#include "fdg_tma.cuh"

namespace fdg {
namespace {

constexpr uint32_t kValid = 0x80000000u;
constexpr uint64_t kNoNode = ~0ull;
#ifndef FDG_BM_THREADS
#define FDG_BM_THREADS 256
#endif
constexpr int kT = FDG_BM_THREADS;  // threads per tile
constexpr int kI = 8;          // items per thread
constexpr int kTileN = kT * kI;

struct Entry {
    int32_t slot;
    uint32_t refv;
};

constexpr uint64_t kUnlisted = ~0ull;
constexpr int kRefShift = 40;
constexpr uint64_t kFree = (1ull << kRefShift) - 1;  // owner field of a free slot (node ids < 2^40 - 1)
constexpr uint64_t kRef1 = 1ull << kRefShift;
struct __align__(16) SlotMeta {
    uint64_t nr;   // owner node (low 40 bits, kFree = free) | reference count << 40
    uint64_t pos;  // ring position of the live standby entry (kUnlisted = none)
};
__host__ __device__ __forceinline__ uint64_t m_node(uint64_t nr) { return nr & kFree; }
__host__ __device__ __forceinline__ uint32_t m_ref(uint64_t nr) { return uint32_t(nr >> kRefShift); }
// Random metadata reads. FDG_BM_RAND64=1: with a 64-byte L2 fill (ld_rand64, fdg_internal.cuh);
// measured 540 vs 536 us per Papers batch with plain loads (the metadata chain is bound by the
// random-access rate, not bytes), so plain loads by default.
#ifndef FDG_BM_RAND64
#define FDG_BM_RAND64 0
#endif
__device__ __forceinline__ uint64_t ld_meta(const void* p) {
#if FDG_BM_RAND64
    return ld_rand64(p);
#else
    return *static_cast<const uint64_t*>(p);
#endif
}
__device__ __forceinline__ Entry ld_entry(const Entry* p) {
    const uint64_t v = ld_meta(p);
    return Entry{int32_t(uint32_t(v)), uint32_t(v >> 32)};
}
__device__ __forceinline__ uint64_t ld_nr(const SlotMeta* p) { return ld_meta(&p->nr); }
__device__ __forceinline__ uint64_t ld_pos(const SlotMeta* p) { return ld_meta(&p->pos); }

struct BmState {
    uint64_t head, tail;   // ring positions (monotonic)
    uint64_t live;         // standby size
    uint64_t hits, loads, waits, evictions, takeovers, releases;
    uint32_t status;
    uint32_t n_load;       // to-load count of the current batch
    uint32_t done;         // select finished
    uint32_t ring_sel;     // which ring buffer is current
    uint32_t tile_ctr[4];
    uint64_t new_head;
    uint64_t compactions;  // k_compact_finish swaps (test introspection)
};

struct BmDev {
    Entry* map;
    SlotMeta* slot;       // slot -> {owner node | reference count, live ring position}
    int32_t* ring[2];
    uint64_t R;           // ring capacity
    uint64_t S;           // slots
    uint64_t N;           // nodes
    BmState* st;
    unsigned long long* tiles;  // packed look-back words
    uint32_t* load_pos;   // [max_batch] to-load rank -> batch position
    uint32_t* sel;        // [max_batch] to-load rank -> slot
    uint8_t* is_load[2];  // [max_batch] per batch parity: acquire of batch j+1 may run under the move of j
    uint64_t max_batch;
    uint32_t eager;       // debug: evictions also clear the previous owner's entry (no stale entries)
};

// 64-bit packed look-back word: [63:62] state (1 aggregate, 2 inclusive),
// [61:32] epoch, [31:0] value. One atomic store publishes value + state.
__device__ __forceinline__ unsigned long long lb_pack(uint32_t state, uint32_t epoch, uint32_t v) {
    return (uint64_t(state) << 62) | (uint64_t(epoch & 0x3FFFFFFFu) << 32) | v;
}
__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// Warp 0 of a block: exclusive prefix of this tile's aggregate `agg`.
__device__ uint32_t lookback(unsigned long long* tiles, uint32_t tile, uint32_t agg, uint32_t epoch, int lane) {
    if (tile == 0) {
        if (lane == 0) atomicExch(tiles, lb_pack(2, epoch, agg));
        return 0;
    }
    if (lane == 0) atomicExch(tiles + tile, lb_pack(1, epoch, agg));
    uint32_t excl = 0;
    int j = int(tile) - 1;
    for (;;) {
        int jj = j - lane;
        uint32_t st = 2, v = 0;
        if (jj >= 0) {
            unsigned long long w = lb_load(tiles + jj);
            st = ((w >> 32) & 0x3FFFFFFFu) == (epoch & 0x3FFFFFFFu) ? uint32_t(w >> 62) : 0u;
            v = uint32_t(w);
        }
        if (__any_sync(0xffffffffu, st == 0)) continue;
        uint32_t im = __ballot_sync(0xffffffffu, st == 2);
        int stop = im ? __ffs(im) - 1 : 32;  // nearest inclusive predecessor in this window
        uint32_t c = lane <= stop ? v : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        excl += c;
        if (stop < 32) break;
        j -= 32;
    }
    if (lane == 0) atomicExch(tiles + tile, lb_pack(2, epoch, excl + agg));
    return excl;
}

// Block-wide: exclusive scan of per-thread counts + decoupled look-back.
// Returns this thread's exclusive global prefix; *total_out (smem) = tile incl total.
__device__ uint32_t block_rank(unsigned long long* tiles, uint32_t tile, uint32_t mine, uint32_t epoch,
                               uint32_t* s_warp, uint32_t* s_misc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kT / 32 ? s_warp[lane] : 0, wx = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, wx, o);
            if (lane >= o) wx += y;
        }
        if (lane < kT / 32) s_warp[lane] = wx - w;
        uint32_t agg = __shfl_sync(0xffffffffu, wx, 31);
        uint32_t ex = lookback(tiles, tile, agg, epoch, lane);
        if (lane == 0) {
            s_misc[0] = ex;
            s_misc[1] = ex + agg;
        }
    }
    __syncthreads();
    return s_misc[0] + s_warp[warp] + x - mine;
}

__device__ __forceinline__ uint64_t load_n(const uint32_t* n_dev, uint64_t n_host) { return n_dev ? *n_dev : n_host; }

// ------------------------------------------------------------- k_acquire ----
__global__ void __launch_bounds__(kT) k_acquire(BmDev B, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                                                int64_t* alias, uint8_t* is_load, uint32_t epoch) {
    __shared__ uint32_t s_warp[kT / 32], s_misc[2], s_tile;
    __shared__ unsigned long long s_hits, s_removed;
    BmState* S = B.st;
    if (S->status) return;
    const uint64_t n = load_n(n_dev, n_host);
    const uint32_t ntiles = n ? uint32_t((n + kTileN - 1) / kTileN) : 1;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(&S->tile_ctr[0], 1u);
        s_hits = 0;
        s_removed = 0;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint64_t i0 = uint64_t(tile) * kTileN + threadIdx.x * kI;
    uint32_t load_mask = 0, mine = 0, hits = 0, removed = 0;
    bool bad = false;
    uint64_t nd[kI], nr[kI];
    Entry en[kI];
#pragma unroll
    for (int k = 0; k < kI; ++k) nd[k] = i0 + k < n ? nodes[i0 + k] : kNoNode;
#pragma unroll
    for (int k = 0; k < kI; ++k) en[k] = nd[k] < B.N ? ld_entry(B.map + nd[k]) : Entry{-1, 0u};  // all loads in flight
#pragma unroll
    for (int k = 0; k < kI; ++k) nr[k] = (en[k].refv & kValid) ? ld_nr(B.slot + en[k].slot) : kFree;
#pragma unroll
    for (int k = 0; k < kI; ++k)  // lazy invalidation: an entry is live only while its slot still names the node
        if ((en[k].refv & kValid) && m_node(nr[k]) != nd[k]) en[k] = Entry{-1, 0u};
#pragma unroll
    for (int k = 0; k < kI; ++k) {
        const uint64_t i = i0 + k;
        if (i >= n) break;
        const uint64_t node = nd[k];
        if (node >= B.N) {
            bad = true;
            continue;
        }
        const Entry e = en[k];
        if (e.refv & kValid) {  // hit: ref++ (a batch's nodes, hence slots, are distinct)
            if (m_ref(nr[k]) == 0) {  // StandbyList::remove (buffer_manager.hpp:250)
                B.slot[e.slot] = SlotMeta{nr[k] + kRef1, kUnlisted};
                ++removed;
            } else {
                B.slot[e.slot].nr = nr[k] + kRef1;
            }
            alias[i] = e.slot;
            is_load[i] = 0;
            ++hits;
        } else {  // miss: its ref starts at 1 when k_bind gives it a slot
            alias[i] = -1;
            is_load[i] = 1;
            load_mask |= 1u << k;
            ++mine;
        }
    }
    if (bad) atomicExch(&S->status, uint32_t(FDG_INVARIANT));
    if (hits) atomicAdd(&s_hits, (unsigned long long)hits);
    if (removed) atomicAdd(&s_removed, (unsigned long long)removed);
    uint32_t r = block_rank(B.tiles, tile, mine, epoch, s_warp, s_misc);
#pragma unroll
    for (int k = 0; k < kI; ++k)
        if (load_mask & (1u << k)) B.load_pos[r++] = uint32_t(i0 + k);
    if (threadIdx.x == 0) {
        if (s_hits) atomicAdd((unsigned long long*)&S->hits, s_hits);
        if (s_removed) atomicAdd((unsigned long long*)&S->live, (unsigned long long)(-(long long)s_removed));
        if (tile == ntiles - 1) {
            S->n_load = s_misc[1];
            S->loads += s_misc[1];
            S->done = 0;
            S->new_head = S->head;
        }
    }
}

// ------------------------------------------------------------- k_select ----
// Persistent CTAs claim ring tiles from `head` in order and rank live entries;
// the first L live slots are the reference's L successive pop_lru() results.
// BIND: the thread that ranks a popped slot also binds it (what k_bind does for miss r):
// the liveness check already brings the slot's record in, so the eviction check and the
// rebind cost no second random read and no extra launch; k_bind_finish moves head.
template <bool BIND>
__global__ void __launch_bounds__(kT) k_select(BmDev B, uint32_t epoch, const uint64_t* nodes, int64_t* alias) {
    __shared__ uint32_t s_warp[kT / 32], s_misc[2], s_tile;
    __shared__ unsigned long long s_ev;
    BmState* S = B.st;
    if (S->status) return;
    const uint32_t L = S->n_load;
    if (L == 0) return;
    const uint64_t head = S->head, tail = S->tail;
    const int32_t* ring = B.ring[S->ring_sel];
    if (BIND && threadIdx.x == 0) s_ev = 0;
    for (;;) {
        if (threadIdx.x == 0) s_tile = *(volatile uint32_t*)&S->done ? 0xFFFFFFFFu : atomicAdd(&S->tile_ctr[1], 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        __syncthreads();
        if (tile == 0xFFFFFFFFu) break;
        const uint64_t p0 = head + uint64_t(tile) * kTileN;
        // Past the ring end: nothing to rank (the tile holding tail-1 -- or tile 0 of
        // an empty ring -- reports a short standby list). No look-back slot is used,
        // so tile ids stay within the tiles array.
        if (p0 >= tail && tile > 0) break;
        uint32_t live_mask = 0, mine = 0;
        int32_t slots[kI];
        uint64_t nr[BIND ? kI : 1];
#pragma unroll
        for (int k = 0; k < kI; ++k) {
            uint64_t p = p0 + threadIdx.x * kI + k;
            slots[k] = -1;
            if (p < tail) {
                slots[k] = ring[p % B.R];
            }
        }
#pragma unroll
        for (int k = 0; k < kI; ++k) {  // list membership: one random record load per entry, all in flight
            const uint64_t p = p0 + threadIdx.x * kI + k;
            bool live = false;
            if (slots[k] >= 0) {
                if constexpr (BIND) {
                    const ulonglong2 m = *reinterpret_cast<const ulonglong2*>(B.slot + slots[k]);
                    nr[k] = m.x;
                    live = m.y == p;
                } else {
                    live = ld_pos(B.slot + slots[k]) == p;
                }
            }
            if (live) {
                live_mask |= 1u << k;
                ++mine;
            } else {
                slots[k] = -1;
            }
        }
        uint32_t r = block_rank(B.tiles, tile, mine, epoch, s_warp, s_misc);
        uint32_t ev = 0;
#pragma unroll
        for (int k = 0; k < kI; ++k)
            if (live_mask & (1u << k)) {
                if (r < L) {
                    if constexpr (BIND) {  // k_bind for miss r (buffer_manager.hpp:281-310)
                        const int32_t slot = slots[k];
                        const uint32_t i = B.load_pos[r];
                        const uint64_t node = nodes[i];
                        const uint64_t prev = m_node(nr[k]);
                        if (prev != kFree) {  // evict the previous owner: rebinding the slot invalidates its entry
                            if (m_ref(nr[k]) != 0) atomicExch(&S->status, uint32_t(FDG_INVARIANT));
                            if (B.eager) B.map[prev] = Entry{-1, 0u};
                            ++ev;
                        }
                        B.map[node] = Entry{slot, kValid};  // bind + publish
                        B.slot[slot] = SlotMeta{node | kRef1, kUnlisted};
                        alias[i] = slot;
                    } else {
                        B.sel[r] = slots[k];
                    }
                }
                if (r == L - 1) {
                    S->new_head = p0 + threadIdx.x * kI + k + 1;
                    atomicExch(&S->done, 1u);
                }
                ++r;
            }
        if (BIND && ev) atomicAdd(&s_ev, (unsigned long long)ev);
        if (threadIdx.x == 0 && s_misc[1] < L && p0 + kTileN >= tail) atomicExch(&S->status, uint32_t(FDG_CAPACITY));
        __syncthreads();
    }
    if (BIND) {
        __syncthreads();
        if (threadIdx.x == 0 && s_ev) atomicAdd((unsigned long long*)&S->evictions, s_ev);
    }
}

// After the fused select + bind: the L popped slots left the standby list.
__global__ void k_bind_finish(BmDev B) {
    BmState* S = B.st;
    if (S->status) return;
    S->live -= S->n_load;
    S->head = S->new_head;
}

// --------------------------------------------------------------- k_bind ----
// One miss per thread (grid covers the batch bound): the chain sel -> slot record ->
// previous owner's entry is three dependent random loads, so parallelism comes
// from threads, not from a per-thread loop (whose stores would serialise it).
__global__ void k_bind(BmDev B, const uint64_t* nodes, int64_t* alias) {
    BmState* S = B.st;
    if (S->status) return;
    const uint32_t L = S->n_load;
    uint32_t ev = 0;
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < L) {
        const int32_t slot = B.sel[k];
        const uint32_t i = B.load_pos[k];
        const uint64_t node = nodes[i];
        const uint64_t pnr = ld_nr(B.slot + slot);
        const uint64_t prev = m_node(pnr);
        if (prev != kFree) {  // evict the previous owner (buffer_manager.hpp:281-291): rebinding the
            // slot below is the invalidation -- its mapping entry goes stale
            if (m_ref(pnr) != 0) atomicExch(&S->status, uint32_t(FDG_INVARIANT));
            // eager (debug) mode: the reference's invalidation (buffer_manager.hpp:284-287). prev
            // cannot be a miss of this batch: its entry is live, so it would have been a hit.
            if (B.eager) B.map[prev] = Entry{-1, 0u};
            ++ev;
        }
        B.map[node] = Entry{slot, kValid};  // bind + publish
        B.slot[slot] = SlotMeta{node | kRef1, kUnlisted};  // its reference from acquire_for_batch
        alias[i] = slot;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
    if ((threadIdx.x & 31) == 0 && ev) atomicAdd((unsigned long long*)&S->evictions, (unsigned long long)ev);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd((unsigned long long*)&S->live, (unsigned long long)(-(long long)L));
        S->head = S->new_head;
    }
}

// --------------------------------------------------------------- k_move ----
// Misses read the table row and fill their slot (and X); hits read their slot (into
// X). Without X only misses move. Reads only per-batch state (alias, is_load[parity]),
// so it runs on its own stream while the next batch's acquire / select / bind proceed
// -- which is why it is launched on half the SM's thread slots (2 x 512 per SM): a
// full-occupancy grid keeps the latency-bound metadata kernels off the SMs (release
// 332 us in the pipeline at 4 x 512 per SM vs 32 us alone). A warp moves kMoveRows rows
// at a time: their metadata (one lane per row, shuffled) resolves first, then every
// lane has kMoveRows 16-byte loads in flight.
#ifndef FDG_MOVE_ROWS
#define FDG_MOVE_ROWS 4
#endif
#ifndef FDG_MOVE_MINB
#define FDG_MOVE_MINB 2
#endif
#ifndef FDG_MOVE_CTAS
#define FDG_MOVE_CTAS 2
#endif
constexpr int kMoveRows = FDG_MOVE_ROWS;
__global__ void __launch_bounds__(512, FDG_MOVE_MINB) k_move(BmDev B, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                                              const int64_t* alias, const uint8_t* is_load, const char* table,
                                              char* region, uint32_t rb, char* X, uint32_t host_table) {
    BmState* S = B.st;
    if (S->status) return;
    const uint32_t cpr = rb / 16;
    const uint64_t n = load_n(n_dev, n_host);
    uint64_t pol;  // row traffic must not flush the batch's metadata sectors out of L2
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t r0 = warp * kMoveRows; r0 < n; r0 += nwarps * kMoveRows) {
        // lane q < kMoveRows resolves row r0 + q: source row, slot row, miss flag
        const char* my_src = nullptr;
        char* my_slot = nullptr;
        uint32_t my_miss = 0;
        if (lane < kMoveRows && r0 + lane < n) {
            const uint64_t i = r0 + lane;
            my_miss = is_load[i];
            my_slot = region + uint64_t(alias[i]) * rb;
            my_src = my_miss ? table + nodes[i] * rb : my_slot;
        }
        const char* src[kMoveRows];
        char* slot[kMoveRows];
        uint32_t miss[kMoveRows];
#pragma unroll
        for (int q = 0; q < kMoveRows; ++q) {
            src[q] = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_src), q));
            slot[q] = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_slot), q));
            miss[q] = __shfl_sync(0xffffffffu, my_miss, q);
        }
        for (uint32_t c = lane; c < cpr; c += 32) {
            uint4 v[kMoveRows];
#pragma unroll
            for (int q = 0; q < kMoveRows; ++q)
                if (src[q] && (miss[q] || X)) {
                    if (host_table && miss[q])  // mapped host memory: no L2 policy on PCIe reads
                        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(v[q].x), "=r"(v[q].y), "=r"(v[q].z), "=r"(v[q].w)
                                     : "l"(reinterpret_cast<const uint4*>(src[q]) + c));
                    else
                        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                                     : "=r"(v[q].x), "=r"(v[q].y), "=r"(v[q].z), "=r"(v[q].w)
                                     : "l"(reinterpret_cast<const uint4*>(src[q]) + c), "l"(pol));
                }
#pragma unroll
            for (int q = 0; q < kMoveRows; ++q) {
                if (!src[q] || !(miss[q] || X)) continue;
                if (miss[q])
                    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(
                                     reinterpret_cast<uint4*>(slot[q]) + c),
                                 "r"(v[q].x), "r"(v[q].y), "r"(v[q].z), "r"(v[q].w), "l"(pol)
                                 : "memory");
                if (X)
                    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(
                                     reinterpret_cast<uint4*>(X + (r0 + q) * rb) + c),
                                 "r"(v[q].x), "r"(v[q].y), "r"(v[q].z), "r"(v[q].w), "l"(pol)
                                 : "memory");
            }
        }
    }
}

// ------------------------------------------------------------ TMA move ----
// The row move on the TMA: each row lands in shared memory by one cp.async.bulk (completing on
// its stage's mbarrier) and leaves by bulk stores to X and, for a miss, to its slot. The bytes
// in flight sit in shared memory, not registers: one 4-warp CTA per SM keeps ~96 KB of rows in
// flight with a few thousand registers, so the rest of the SM stays free for the next batch's
// metadata kernels, the samplers and the MT prefetch (the LDG k_move's 2 x 512 threads at 60
// registers hold the whole register file for its ~290 us). Warp w of CTA c takes row chunks
// w + 4c, w + 4c + 4 * grid, ... (RS rows each, one row per lane); each warp runs a D-stage
// ring with A chunks of loads in flight.
constexpr int kMoveTmaWarps = 4;
template <int D, int A>
__global__ void __launch_bounds__(kMoveTmaWarps * 32, 1)
    k_move_tma(BmDev B, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host, const int64_t* alias,
               const uint8_t* is_load, const char* table, char* region, uint32_t rb, uint32_t RS, char* X) {
    static_assert(A < D, "lookahead must leave a stage for the stores in flight");
    using namespace tma;
    extern __shared__ __align__(128) char mv_smem[];
    __shared__ __align__(8) uint64_t bars[kMoveTmaWarps][D];
    if (B.st->status) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t stage_bytes = RS * rb;
    uint64_t pol;  // row traffic must not flush the batch's metadata sectors out of L2
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    char* wbase = mv_smem + size_t(warp) * D * stage_bytes;
    const uint64_t n = load_n(n_dev, n_host);
    const uint64_t nchunks = (n + RS - 1) / RS;
    const uint64_t gw = uint64_t(blockIdx.x) * kMoveTmaWarps + warp, nw = uint64_t(gridDim.x) * kMoveTmaWarps;
    const uint64_t my_n = gw < nchunks ? (nchunks - gw + nw - 1) / nw : 0;
    if (lane == 0)
        for (int d = 0; d < D; ++d) mbar_init(smem_u32(&bars[warp][d]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    struct Src {
        const char* p;  // null: nothing to load for this lane
    };
    auto src_of = [&](uint64_t i) -> Src {  // this lane's row of chunk i
        const uint64_t r = (gw + i * nw) * RS + lane;
        if (i >= my_n || lane >= int(RS) || r >= n) return Src{nullptr};
        const uint32_t miss = is_load[r];
        if (!miss && !X) return Src{nullptr};  // a hit without X: nothing moves
        return Src{miss ? table + nodes[r] * rb : region + uint64_t(alias[r]) * rb};
    };
    auto issue = [&](uint64_t i, Src sr) {
        const int s = int(i % D);
        const uint32_t bar = smem_u32(&bars[warp][s]);
        const uint32_t loading = __ballot_sync(0xffffffffu, sr.p != nullptr);
        if (lane == 0) mbar_arrive_expect_tx(bar, uint32_t(__popc(loading)) * rb);
        __syncwarp();
        if (sr.p) bulk_load(smem_u32(wbase + s * stage_bytes + lane * rb), sr.p, rb, bar, pol);
    };
    for (int i = 0; i < A; ++i)
        if (uint64_t(i) < my_n) issue(i, src_of(i));
    Src pa = src_of(A), pb = src_of(A + 1);  // sources two chunks ahead of issue
    for (uint64_t i = 0; i < my_n; ++i) {
        const int s = int(i % D);
        const uint64_t r = (gw + i * nw) * RS + lane;
        mbar_wait(smem_u32(&bars[warp][s]), uint32_t((i / D) & 1));
        if (lane < int(RS) && r < n) {
            const uint32_t srow = smem_u32(wbase + s * stage_bytes + lane * rb);
            const uint32_t miss = is_load[r];
            if (X) bulk_store(X + r * rb, srow, rb, pol);  // with X every row was loaded
            if (miss) bulk_store(region + uint64_t(alias[r]) * rb, srow, rb, pol);
        }
        bulk_commit();
        const uint64_t j = i + A;
        if (j < my_n) {
            bulk_wait_read<D - A>();  // the stores that last read stage j % D have drained
            issue(j, pa);
            pa = pb;
            pb = src_of(j + 2);
        }
    }
    bulk_wait_all();
}

// ----------------------------------------------------------- sorted move ----
// Host-resident table (out-of-core tier): misses are moved in node-id order. Random 512-B
// rows over a 57 GB mapped host table reach 26 GB/s over PCIe in batch order but 47 GB/s in
// address order (0.84 of the measured copy peak; scripts/host_tier_gather.py): the host
// side's address translation is the limit, not the link. Keys: the node id of a miss, ~0 for
// a hit (sorted to the end, moved slot -> X); values: batch positions.
__global__ void __launch_bounds__(256) k_move_keys(const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                                                   const uint8_t* is_load, uint32_t* keys, uint32_t* pos,
                                                   uint64_t bound) {
    const uint64_t n = load_n(n_dev, n_host);
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < bound;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const bool live = i < n;
        keys[i] = live && is_load[i] ? uint32_t(nodes[i]) : (live ? 0xFFFFFFFEu : 0xFFFFFFFFu);
        pos[i] = uint32_t(i);
    }
}

// Chunk-striped over the sorted (position) list: 16-byte chunks, 4 loads in flight per thread.
__global__ void __launch_bounds__(512) k_move_sorted(BmDev B, const uint32_t* keys, const uint32_t* pos,
                                                     uint64_t bound, const int64_t* alias, const char* table,
                                                     char* region, uint32_t rb, char* X, int pf) {
    if (B.st->status) return;
    const uint32_t cpr = rb / 16;
    const uint64_t total = bound * cpr;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t c0 = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c0 < total; c0 += 4 * stride) {
        uint4 v[4];
        uint32_t k[4], p[4], col[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t c = c0 + u * stride;
            k[u] = 0xFFFFFFFFu;
            if (c < total) {
                const uint64_t s = c / cpr;
                col[u] = uint32_t(c - s * cpr);
                k[u] = keys[s];
                p[u] = pos[s];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (k[u] == 0xFFFFFFFFu) continue;  // past the batch
            const char* src = k[u] != 0xFFFFFFFEu ? table + uint64_t(k[u]) * rb : region + uint64_t(alias[p[u]]) * rb;
            if (k[u] == 0xFFFFFFFEu && !X) continue;  // a hit without X: nothing to move
            const uint4* a = reinterpret_cast<const uint4*>(src) + col[u];
            if (pf == 2)  // larger read requests over PCIe (option host_tier_pf)
                asm volatile("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(a));
            else if (pf == 1)
                asm volatile("ld.global.nc.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(a));
            else
                asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(a));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (k[u] == 0xFFFFFFFFu || (k[u] == 0xFFFFFFFEu && !X)) continue;
            if (k[u] != 0xFFFFFFFEu) reinterpret_cast<uint4*>(region + uint64_t(alias[p[u]]) * rb)[col[u]] = v[u];
            if (X) reinterpret_cast<uint4*>(X + uint64_t(p[u]) * rb)[col[u]] = v[u];
        }
    }
}

// ------------------------------------------------------------ k_release ----
// Slots come from the batch's alias list (ALIAS) or from the mapping entries of its
// node ids (the public release_batch(nodes) form).
template <bool ALIAS>
__global__ void __launch_bounds__(kT) k_release(BmDev B, const uint64_t* nodes, const int64_t* alias,
                                                const uint32_t* n_dev, uint64_t n_host, uint32_t epoch) {
    __shared__ uint32_t s_warp[kT / 32], s_misc[2], s_tile;
    __shared__ uint64_t s_tail;
    BmState* S = B.st;
    if (S->status) return;
    const uint64_t n = load_n(n_dev, n_host);
    const uint32_t ntiles = n ? uint32_t((n + kTileN - 1) / kTileN) : 1;
    if (threadIdx.x == 0) {
        // The ring tail this launch appends at is read BEFORE the tile claim: the CTA of the last
        // tile advances S->tail once its look-back has seen every other tile's aggregate, i.e.
        // after every other claim -- a read after the look-back could see the advanced tail
        // (a race that shifted whole tiles of MRU pushes, found by the Papers-scale parity test).
        s_tail = *reinterpret_cast<volatile uint64_t*>(&S->tail);
        __threadfence();
        s_tile = atomicAdd(&S->tile_ctr[2], 1u);
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint64_t i0 = uint64_t(tile) * kTileN + threadIdx.x * kI;
    uint32_t mask = 0, mine = 0;
    int32_t slots[kI];
    bool bad = false;
    int32_t sl[kI];
    uint64_t nr[kI];
    if constexpr (ALIAS) {
#pragma unroll
        for (int k = 0; k < kI; ++k) {
            const int64_t a = i0 + k < n ? alias[i0 + k] : -1;
            sl[k] = (a >= 0 && uint64_t(a) < B.S) ? int32_t(a) : -1;
        }
#pragma unroll
        for (int k = 0; k < kI; ++k) nr[k] = sl[k] >= 0 ? ld_nr(B.slot + sl[k]) : kFree;  // all loads in flight
    } else {
        uint64_t nd[kI];
#pragma unroll
        for (int k = 0; k < kI; ++k) nd[k] = i0 + k < n ? nodes[i0 + k] : kNoNode;
#pragma unroll
        for (int k = 0; k < kI; ++k) {  // all loads in flight
            const Entry e = nd[k] < B.N ? ld_entry(B.map + nd[k]) : Entry{-1, 0u};
            sl[k] = (e.refv & kValid) ? e.slot : -1;
        }
#pragma unroll
        for (int k = 0; k < kI; ++k) {
            nr[k] = sl[k] >= 0 ? ld_nr(B.slot + sl[k]) : kFree;
            if (sl[k] >= 0 && m_node(nr[k]) != nd[k]) sl[k] = -1;  // stale entry: not resident
        }
    }
#pragma unroll
    for (int k = 0; k < kI; ++k) {
        if (i0 + k >= n) break;
        const uint32_t rf = sl[k] >= 0 ? m_ref(nr[k]) : 0u;
        if (sl[k] < 0 || rf == 0) {  // not resident / no reference (buffer_manager.hpp:357, 462)
            bad = true;
            continue;
        }
        nr[k] -= kRef1;
        if (rf == 1) {  // written with its ring position below
            slots[k] = sl[k];
            mask |= 1u << k;
            ++mine;
        } else {
            B.slot[sl[k]].nr = nr[k];
        }
    }
    if (bad) atomicExch(&S->status, uint32_t(FDG_INVARIANT));
    uint32_t r = block_rank(B.tiles, tile, mine, epoch, s_warp, s_misc);
    const uint64_t tail = s_tail;
    int32_t* ring = B.ring[S->ring_sel];
#pragma unroll
    for (int k = 0; k < kI; ++k)
        if (mask & (1u << k)) {  // push_mru in batch order (buffer_manager.hpp:467)
            uint64_t p = tail + r++;
            ring[p % B.R] = slots[k];
            B.slot[slots[k]] = SlotMeta{nr[k], p};
        }
    if (threadIdx.x == 0 && tile == ntiles - 1) {
        uint32_t tot = s_misc[1];
        if (tail + tot - S->head > B.R) atomicExch(&S->status, uint32_t(FDG_CAPACITY));
        S->tail = tail + tot;
        S->live += tot;
        S->releases += 1;
    }
}

// ------------------------------------------------------------ k_compact ----
// Persistent grid (all CTAs co-resident): when tombstones make the ring too
// long, copy the live entries of [head, tail) in order into the other ring.
__global__ void __launch_bounds__(kT) k_compact(BmDev B, uint64_t slack, uint32_t epoch) {
    __shared__ uint32_t s_warp[kT / 32], s_misc[2], s_tile;
    BmState* S = B.st;
    if (S->status) return;
    const uint64_t head = S->head, tail = S->tail;
    if ((tail - head) + slack <= B.R) return;
    const int32_t* src = B.ring[S->ring_sel];
    int32_t* dst = B.ring[S->ring_sel ^ 1];
    const uint64_t len = tail - head;
    const uint32_t ntiles = uint32_t((len + kTileN - 1) / kTileN);
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&S->tile_ctr[3], 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        __syncthreads();
        if (tile >= ntiles) break;
        const uint64_t p0 = head + uint64_t(tile) * kTileN + threadIdx.x * kI;
        uint32_t mask = 0, mine = 0;
        int32_t slots[kI];
#pragma unroll
        for (int k = 0; k < kI; ++k) {
            uint64_t p = p0 + k;
            if (p < tail) {
                int32_t s = src[p % B.R];
                if (B.slot[s].pos == p) {
                    slots[k] = s;
                    mask |= 1u << k;
                    ++mine;
                }
            }
        }
        uint32_t r = block_rank(B.tiles, tile, mine, epoch, s_warp, s_misc);
#pragma unroll
        for (int k = 0; k < kI; ++k)
            if (mask & (1u << k)) {
                dst[r] = slots[k];
                B.slot[slots[k]].pos = r;
                ++r;
            }
        if (threadIdx.x == 0 && tile == ntiles - 1) S->new_head = s_misc[1];  // live count
        __syncthreads();
    }
}

__global__ void k_compact_finish(BmDev B, uint64_t slack) {
    BmState* S = B.st;
    if (S->status) return;
    if ((S->tail - S->head) + slack <= B.R) return;
    S->ring_sel ^= 1;
    S->head = 0;
    S->tail = S->new_head;
    S->compactions += 1;
}

__global__ void k_status_to(const BmState* S, uint32_t* dst) {
    if (S->status && *dst == 0) *dst = S->status;
}

__global__ void k_reset_ctrs(BmState* S) {
    if (threadIdx.x < 4) S->tile_ctr[threadIdx.x] = 0;
}

__global__ void k_init(BmDev B) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < B.N; v += stride) B.map[v] = Entry{-1, 0u};
    for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < B.S; s += stride) {
        B.slot[s] = SlotMeta{kFree, s};
        B.ring[0][s] = int32_t(s);
    }
}


// ---------------------------------------------------------- per-node protocol ----
// The reference's fine-grained BufferManager calls (buffer_manager.hpp:274-324, 370-409)
// as batch kernels, for callers that drive the protocol themselves (the C++ drop-in's
// get_standby_slot / bind_slot / publish_valid / unwind_bound / release_ref). The fused
// extract path (k_acquire .. k_move) is what the extractor and the runner use.

__global__ void k_set_nload(BmState* S, uint32_t count) {
    S->n_load = count;
    S->done = 0;
    S->new_head = S->head;
    for (int i = 0; i < 4; ++i) S->tile_ctr[i] = 0;
}

// get_standby_slot x count: the popped slots (k_select ranked them) lose their previous
// owner (eviction) and become free, off the standby list.
__global__ void k_pop(BmDev B, int64_t* slots_out) {
    BmState* S = B.st;
    if (S->status) return;
    const uint32_t L = S->n_load;
    uint32_t ev = 0;
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < L) {
        const int32_t slot = B.sel[k];
        const uint64_t pnr = B.slot[slot].nr;
        const uint64_t prev = m_node(pnr);
        if (prev != kFree) {
            if (m_ref(pnr) != 0) atomicExch(&S->status, uint32_t(FDG_INVARIANT));
            if (B.eager) B.map[prev] = Entry{-1, 0u};
            ++ev;
        }
        B.slot[slot] = SlotMeta{kFree, kUnlisted};
        slots_out[k] = slot;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
    if ((threadIdx.x & 31) == 0 && ev) atomicAdd((unsigned long long*)&S->evictions, (unsigned long long)ev);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd((unsigned long long*)&S->live, (unsigned long long)(-(long long)L));
        S->head = S->new_head;
    }
}

__device__ __forceinline__ bool entry_live(const BmDev& B, uint64_t node, Entry* out) {
    const Entry e = B.map[node];
    *out = e;
    return e.slot >= 0 && uint64_t(e.slot) < B.S && m_node(B.slot[e.slot].nr) == node;
}

// bind_slot (297-310): the node takes a free slot, not yet valid; its reference from
// acquire_for_batch starts counting here.
__global__ void k_bind_explicit(BmDev B, const uint64_t* nodes, const int64_t* slots, uint32_t n) {
    BmState* S = B.st;
    if (S->status) return;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t node = nodes[i];
    const int64_t slot = slots[i];
    Entry e;
    if (node >= B.N || slot < 0 || uint64_t(slot) >= B.S || entry_live(B, node, &e) ||
        B.slot[slot].nr != kFree || B.slot[slot].pos != kUnlisted) {
        atomicExch(&S->status, uint32_t(FDG_INVARIANT));  // FD_CHECKs of bind_slot
        return;
    }
    B.map[node] = Entry{int32_t(slot), 0u};
    B.slot[slot].nr = node | kRef1;
}

// publish_valid (313-324)
__global__ void k_publish(BmDev B, const uint64_t* nodes, uint32_t n) {
    BmState* S = B.st;
    if (S->status) return;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Entry e;
    if (nodes[i] >= B.N || !entry_live(B, nodes[i], &e) || (e.refv & kValid)) {
        atomicExch(&S->status, uint32_t(FDG_INVARIANT));
        return;
    }
    B.map[nodes[i]].refv = e.refv | kValid;
}

// unwind_bound (372-388): an unpublished bind is reverted, its slot goes back to the MRU end
// as free space. release_ref (392-400): one reference dropped without the validity
// requirement (a published node at 0 goes to the MRU end). One node per launch (the
// reference's per-node calls), single thread.
__global__ void k_unwind_or_release(BmDev B, uint64_t node, int unwind) {
    BmState* S = B.st;
    if (S->status) return;
    Entry e;
    const bool live = node < B.N && entry_live(B, node, &e);
    int32_t push = -1;
    if (unwind) {
        if (!live || (e.refv & kValid)) {
            atomicExch(&S->status, uint32_t(FDG_INVARIANT));
            return;
        }
        B.slot[e.slot].nr = kFree;  // the node's reference goes with its entry
        B.map[node] = Entry{-1, 0u};
        push = e.slot;
    } else {
        if (!live) return;  // a miss never bound holds no slot-side reference here
        const uint64_t nr = B.slot[e.slot].nr;
        const uint32_t r = m_ref(nr);
        if (r == 0) {
            atomicExch(&S->status, uint32_t(FDG_INVARIANT));  // ref_count decrement below zero
            return;
        }
        if (r == 1 && !(e.refv & kValid)) {  // "unreferenced invalid node with a slot" (467-472)
            atomicExch(&S->status, uint32_t(FDG_INVARIANT));
            return;
        }
        B.slot[e.slot].nr = nr - kRef1;
        if (r == 1) push = e.slot;
    }
    if (push >= 0) {
        const uint64_t p = S->tail;
        B.ring[S->ring_sel][p % B.R] = push;
        B.slot[push].pos = p;
        S->tail = p + 1;
        S->live += 1;
        if (S->tail - S->head > B.R) atomicExch(&S->status, uint32_t(FDG_CAPACITY));
    }
}

// Explicit loads: table rows -> region slots (the extractor's load + transfer for a plan).
__global__ void __launch_bounds__(256) k_load_rows(const uint64_t* nodes, const int64_t* slots, uint32_t n,
                                                   const char* table, char* region, uint32_t rb) {
    const uint32_t cpr = rb / 16;
    for (uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c < uint64_t(n) * cpr;
         c += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = c / cpr, k = c % cpr;
        reinterpret_cast<uint4*>(region + uint64_t(slots[i]) * rb)[k] =
            reinterpret_cast<const uint4*>(table + nodes[i] * rb)[k];
    }
}

__global__ void k_copy_nload(const BmState* S, uint32_t* dst) { *dst = S->n_load; }

}  // namespace

struct Bm {
    Ctx* ctx = nullptr;
    fdg_ctx* own_ctx = nullptr;     // standalone buffer manager: a device-only context of its own
    BmDev d{};
    void* arena = nullptr;
    char* region = nullptr;
    bool own_region = true;         // false: the region is a caller's FeatureRegion allocation
    bool host_src = false;          // standalone: the bound table lives in mapped host memory
    // sorted-move scratch (host-resident tables): keys / positions in and out, CUB temp storage
    void* sort_arena = nullptr;
    uint64_t sort_cap = 0;
    size_t sort_tmp_bytes = 0;
    uint64_t slots = 0;
    uint32_t max_batch = 0;
    uint32_t epoch = 1;
    bool eager = false;             // option bm_eager_invalidate at creation
    cudaStream_t stream = nullptr;  // for stats/validate
};

}  // namespace fdg

struct fdg_bm : fdg::Bm {};

namespace fdg {
int bm_release(fdg_bm* b, cudaStream_t st, const uint64_t* nodes, const int64_t* alias, const uint32_t* n_dev,
               uint64_t n_host);
}  // namespace fdg

using namespace fdg;

int64_t fdg::g_bm_eager = 0;
int64_t fdg::g_bm_sorted_move = 1;
int64_t fdg::g_host_tier_pf = 0;
int64_t fdg::g_bm_move_impl = 2;  // row-group move (k_move_hash_rb without the hash): 524.7 -> 514.4 us per batch
int64_t fdg::g_bm_move_grid = 0;
int64_t fdg::g_bm_move_hash = 1;
int64_t fdg::g_bm_fuse_bind = 1;  // select + bind fused: 543 -> 527.5 us per Papers batch (config 3)

namespace {

uint32_t n_tiles_for(uint64_t n) { return uint32_t(std::max<uint64_t>(1, (n + kTileN - 1) / kTileN)); }

#ifndef FDG_BM_PERSIST
#define FDG_BM_PERSIST 2
#endif
int bm_persistent_grid(const Bm* b) { return b->ctx->sm_count * FDG_BM_PERSIST; }

}  // namespace

extern "C" {

}  // extern "C"

namespace {
// Buffer manager over `ctx` (the miss source when it holds a table); the region is
// allocated here unless `region` is given (then owned by the caller).
int bm_build(fdg_ctx* ctx, uint64_t slot_count, uint64_t min_reserved, uint32_t max_batch_nodes, char* region,
             bool alloc_region, fdg_bm** out) {
    if (slot_count == 0) return fail(FDG_INVARIANT, "slot_count must be positive");
    if (slot_count < min_reserved) return fail(FDG_INVARIANT, "feature buffer smaller than the N_e * M_b reservation");
    if (slot_count >= uint64_t(INT32_MAX)) return fail(FDG_INVALID_ARG, "slot_count must be < 2^31");
    if (ctx->row_bytes == 0) return fail(FDG_NOT_LOADED, "buffer manager needs a feature table");
    if (ctx->row_bytes % 16) return fail(FDG_INVALID_ARG, "buffer manager: row_bytes must be a multiple of 16");
    if (ctx->n_shards > 1) return fail(FDG_INVALID_ARG, "buffer manager: sharded tables not supported yet");
    if ((ctx->num_nodes ? ctx->num_nodes : ctx->feat_nodes) >= kFree)
        return fail(FDG_INVALID_ARG, "buffer manager: node ids must be < 2^40 - 1");
    cudaSetDevice(ctx->device);
    auto b = new fdg_bm();
    b->ctx = ctx;
    b->slots = slot_count;
    b->max_batch = std::max<uint32_t>(max_batch_nodes, 1);
    const uint64_t N = ctx->num_nodes ? ctx->num_nodes : ctx->feat_nodes;
    const uint64_t R = 2 * slot_count + 8 * uint64_t(b->max_batch) + kTileN;
    auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
    uint64_t sz = 0;
    const uint64_t o_map = sz; sz += al(N * 8);
    const uint64_t o_slot = sz; sz += al(slot_count * sizeof(SlotMeta));
    const uint64_t o_r0 = sz; sz += al(R * 4);
    const uint64_t o_r1 = sz; sz += al(R * 4);
    const uint64_t o_st = sz; sz += al(sizeof(BmState));
    const uint64_t tiles = R / kTileN + 2 + n_tiles_for(b->max_batch);
    const uint64_t o_tl = sz; sz += al(tiles * 8);
    const uint64_t o_lp = sz; sz += al(uint64_t(b->max_batch) * 4);
    const uint64_t o_sel = sz; sz += al(uint64_t(b->max_batch) * 4);
    const uint64_t o_isl = sz; sz += al(uint64_t(b->max_batch));
    const uint64_t o_isl1 = sz; sz += al(uint64_t(b->max_batch));
    cudaError_t e = cudaMalloc(&b->arena, sz);
    b->own_region = region == nullptr && alloc_region;
    b->region = region;
    if (e == cudaSuccess && b->own_region) e = cudaMalloc((void**)&b->region, slot_count * ctx->row_bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        if (b->arena) cudaFree(b->arena);
        delete b;
        return cuda_fail(e, "fdg_bm_create", __FILE__, __LINE__);
    }
    char* a = static_cast<char*>(b->arena);
    BmDev& d = b->d;
    d.map = reinterpret_cast<Entry*>(a + o_map);
    d.slot = reinterpret_cast<SlotMeta*>(a + o_slot);
    d.ring[0] = reinterpret_cast<int32_t*>(a + o_r0);
    d.ring[1] = reinterpret_cast<int32_t*>(a + o_r1);
    d.R = R;
    d.S = slot_count;
    d.N = N;
    d.st = reinterpret_cast<BmState*>(a + o_st);
    d.tiles = reinterpret_cast<unsigned long long*>(a + o_tl);
    d.load_pos = reinterpret_cast<uint32_t*>(a + o_lp);
    d.sel = reinterpret_cast<uint32_t*>(a + o_sel);
    d.is_load[0] = reinterpret_cast<uint8_t*>(a + o_isl);
    d.is_load[1] = reinterpret_cast<uint8_t*>(a + o_isl1);
    d.max_batch = b->max_batch;
    b->eager = g_bm_eager != 0;
    d.eager = b->eager ? 1u : 0u;
    FDG_CUDA(cudaMemset(d.st, 0, sizeof(BmState)));
    FDG_CUDA(cudaMemset(d.tiles, 0, tiles * 8));
    BmState h{};
    h.head = 0;
    h.tail = slot_count;
    h.live = slot_count;
    FDG_CUDA(cudaMemcpy(d.st, &h, sizeof(h), cudaMemcpyHostToDevice));
    k_init<<<ctx->sm_count * 8, 256>>>(d);
    FDG_CUDA(cudaGetLastError());
    FDG_CUDA(cudaDeviceSynchronize());
    *out = b;
    return FDG_OK;
}
}  // namespace

extern "C" {

int fdg_bm_create(fdg_ctx* ctx, uint64_t slot_count, uint64_t min_reserved, uint32_t max_batch_nodes, fdg_bm** out) {
    return bm_build(ctx, slot_count, min_reserved, max_batch_nodes, nullptr, true, out);
}

int fdg_bm_create_standalone(int device, uint64_t num_nodes, uint64_t slot_count, uint32_t row_bytes,
                             uint64_t min_reserved, uint32_t max_batch_nodes, void* region_dev, fdg_bm** out) {
    if (num_nodes == 0) return fail(FDG_INVALID_ARG, "buffer manager: num_nodes must be positive");
    fdg_ctx* c = nullptr;
    FDG_TRY(fdg_ctx_create(device, &c));
    c->num_nodes = num_nodes;
    c->feat_nodes = num_nodes;
    c->row_bytes = row_bytes;
    c->n_shards = 0;  // no miss source until fdg_bm_bind_table
    const int rc = bm_build(c, slot_count, min_reserved, max_batch_nodes, static_cast<char*>(region_dev), false, out);
    if (rc != FDG_OK) {
        fdg_ctx_destroy(c);
        return rc;
    }
    (*out)->own_ctx = c;
    return FDG_OK;
}

int fdg_bm_bind_table(fdg_bm* b, const fdg_ctx* table, void* region_dev) {
    if (!b->own_ctx) return fail(FDG_INVALID_ARG, "bm_bind_table: only a standalone buffer manager takes a table");
    if (table->shard_bases.empty() || table->n_shards != 1)
        return fail(FDG_NOT_LOADED, "bm_bind_table: the table context holds no single-shard feature table");
    if (table->row_bytes != b->own_ctx->row_bytes || table->feat_nodes != b->d.N)
        return fail(FDG_INVALID_ARG, "bm_bind_table: table shape differs from the buffer config (row_bytes / num_nodes)");
    if (table->device != b->own_ctx->device) return fail(FDG_INVALID_ARG, "bm_bind_table: table on another device");
    cudaSetDevice(b->own_ctx->device);
    if (region_dev && region_dev != b->region) {
        if (b->own_region && b->region) cudaFree(b->region);
        b->region = static_cast<char*>(region_dev);
        b->own_region = false;
    } else if (!b->region) {
        FDG_CUDA(cudaMalloc((void**)&b->region, b->slots * b->own_ctx->row_bytes));
        b->own_region = true;
    }
    fdg_ctx* c = b->own_ctx;
    c->shard_bases = table->shard_bases;
    c->n_shards = 1;
    c->rows_per_shard = table->rows_per_shard;
    c->dtype = table->dtype;
    b->host_src = table->host_table != nullptr;
    return FDG_OK;
}

int fdg_bm_destroy(fdg_bm* b) {
    if (!b) return FDG_OK;
    cudaSetDevice(b->ctx->device);
    cudaFree(b->arena);
    if (b->own_region) cudaFree(b->region);
    if (b->sort_arena) cudaFree(b->sort_arena);
    cudaStreamDestroy(b->stream);
    if (b->own_ctx) fdg_ctx_destroy(b->own_ctx);
    delete b;
    return FDG_OK;
}

}  // extern "C"

namespace fdg {
// Algorithm 1's metadata half for one batch (acquire, LRU pops, bind + publish):
// strictly stream-ordered with the releases, it fixes the alias list.
int bm_extract_meta(fdg_bm* b, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                    int64_t* alias, uint32_t parity, cudaEvent_t after_acquire) {
    const uint64_t bound = n_host;
    if (bound > b->max_batch) return fail(FDG_INVALID_ARG, "bm_extract: batch larger than max_batch_nodes");
    const BmDev& d = b->d;
    k_reset_ctrs<<<1, 32, 0, st>>>(d.st);
    {
        FDG_TRACE("bm_acquire", st);
        k_acquire<<<n_tiles_for(bound), kT, 0, st>>>(d, nodes, n_dev, n_host, alias, d.is_load[parity & 1],
                                                    b->epoch++);
    }
    if (after_acquire) FDG_CUDA(cudaEventRecord(after_acquire, st));
    if (g_bm_fuse_bind) {  // select + bind in one pass over the popped slots' records
        FDG_TRACE("bm_select", st);
        k_select<true><<<bm_persistent_grid(b), kT, 0, st>>>(d, b->epoch++, nodes, alias);
        k_bind_finish<<<1, 1, 0, st>>>(d);
    } else {
        {
            FDG_TRACE("bm_select", st);
            k_select<false><<<bm_persistent_grid(b), kT, 0, st>>>(d, b->epoch++, nullptr, nullptr);
        }
        {
            FDG_TRACE("bm_bind", st);
            k_bind<<<std::max<uint32_t>(1, uint32_t((bound + 255) / 256)), 256, 0, st>>>(d, nodes, alias);
        }
    }
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

// The row half: misses table -> slot (-> X), hits slot -> X, optional trainer
// checksum over the batch's slots. Reads only the batch's alias list and
// is_load[parity], so it can overlap the next batch's metadata half.
int bm_extract_move(fdg_bm* b, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                    const int64_t* alias, void* out, uint64_t* checksum, uint32_t parity, int mode) {
    const BmDev& d = b->d;
    const uint32_t rb = b->ctx->row_bytes;
    if (b->ctx->shard_bases.empty() || !b->region)
        return fail(FDG_NOT_LOADED, "bm_extract: no feature table / region bound (fdg_bm_bind_table)");
    const char* table = static_cast<const char*>(b->ctx->shard_bases[0]);
    const uint64_t chunks = n_host * (rb / 16);
    // g_bm_move_grid 0: persistent (FDG_MOVE_CTAS per SM, grid-stride); 1: one 4-row group per warp
    // over the batch bound, so CTAs retire during the move and the block scheduler can put the
    // next batch's metadata kernels and the samplers (higher-priority streams) in between.
    const int blocks = g_bm_move_grid
        ? int(std::max<uint64_t>(1, (n_host + 16 * kMoveRows - 1) / (16 * kMoveRows)))
        : int(std::max<uint64_t>(1, std::min<uint64_t>((chunks + 511) / 512, uint64_t(b->ctx->sm_count) * FDG_MOVE_CTAS)));
    const bool host = b->own_ctx ? b->host_src : b->ctx->host_table != nullptr;
    if (mode == 1 || mode == 2) {  // split move (the pipeline checks the row size and the tier)
        FDG_TRACE(mode == 1 ? "bm_move_x" : "bm_fill", st);
        const int rc = launch_move_hash(*b->ctx, st, nodes, n_dev, n_host, &d.st->status, alias,
                                        d.is_load[parity & 1], table, b->region, static_cast<char*>(out), nullptr, mode);
        return rc == -1 ? fail(FDG_INVALID_ARG, "bm split move: no instantiation for this row size") : rc;
    }
    if (!host && out && ((checksum && g_bm_move_hash) || (!checksum && g_bm_move_impl == 2))) {
        // move + trainer checksum in one pass over the rows (or the same row-group move alone)
        FDG_TRACE("bm_move", st);
        const int rc = launch_move_hash(*b->ctx, st, nodes, n_dev, n_host, &d.st->status, alias, d.is_load[parity & 1],
                                        table, b->region, static_cast<char*>(out), checksum);
        if (rc != -1) return rc;
    }
    if (host && g_bm_sorted_move && d.N < 0xFFFFFFFEull && n_host > 0) {
        // misses in node-id order (address locality for the host side's translation)
        if (b->sort_cap < n_host) {
            if (b->sort_arena) cudaFree(b->sort_arena);
            b->sort_arena = nullptr;
            b->sort_cap = 0;
            size_t tmp = 0;
            FDG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                                     (const uint32_t*)nullptr, (uint32_t*)nullptr, int64_t(n_host)));
            FDG_CUDA(cudaMalloc(&b->sort_arena, 16 * n_host + tmp + 256));
            b->sort_cap = n_host;
            b->sort_tmp_bytes = tmp;
        }
        uint32_t* kin = static_cast<uint32_t*>(b->sort_arena);
        uint32_t* kout = kin + b->sort_cap;
        uint32_t* pin = kout + b->sort_cap;
        uint32_t* pout = pin + b->sort_cap;
        void* tmp = pout + b->sort_cap;
        FDG_TRACE("bm_move", st);
        k_move_keys<<<std::max<int>(1, int(std::min<uint64_t>((n_host + 255) / 256, uint64_t(b->ctx->sm_count) * 8))),
                      256, 0, st>>>(nodes, n_dev, n_host, d.is_load[parity & 1], kin, pin, n_host);
        size_t tb = b->sort_tmp_bytes;
        FDG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, pin, pout, int64_t(n_host), 0, 32, st));
        k_move_sorted<<<blocks, 512, 0, st>>>(d, kout, pout, n_host, alias, table, b->region, rb,
                                              static_cast<char*>(out), int(g_host_tier_pf));
    } else if (!host && g_bm_move_impl == 1 && rb <= 4096) {
        FDG_TRACE("bm_move", st);
        constexpr int D = 8, A = 6;
        const uint32_t RS = std::max<uint32_t>(1, std::min<uint32_t>(
            32, uint32_t(std::min<uint64_t>(4096 / rb, (160u << 10) / (uint64_t(kMoveTmaWarps) * D * rb)))));
        const size_t smem = size_t(kMoveTmaWarps) * D * RS * rb;
        static PerDeviceOnce attr;
        if (attr.first())
            FDG_CUDA(cudaFuncSetAttribute(k_move_tma<D, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 << 10));
        k_move_tma<D, A><<<b->ctx->sm_count, kMoveTmaWarps * 32, smem, st>>>(
            d, nodes, n_dev, n_host, alias, d.is_load[parity & 1], table, b->region, rb, RS, static_cast<char*>(out));
    } else {
        FDG_TRACE("bm_move", st);
        k_move<<<blocks, 512, 0, st>>>(d, nodes, n_dev, n_host, alias, d.is_load[parity & 1], table, b->region, rb,
                                       static_cast<char*>(out), host ? 1u : 0u);
    }
    FDG_CUDA(cudaGetLastError());
    if (checksum) {
        FDG_TRACE("bm_checksum", st);
        FDG_TRY(launch_checksum_alias(*b->ctx, st, b->region, alias, n_dev, n_host, checksum, &d.st->status));
    }
    return FDG_OK;
}
}  // namespace fdg

extern "C" {

int fdg_bm_extract(fdg_bm* b, void* stv, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host, int64_t* alias,
                   void* out, uint64_t* checksum) {
    cudaStream_t st = (cudaStream_t)stv;
    FDG_TRY(bm_extract_meta(b, st, nodes, n_dev, n_host, alias, 0, nullptr));
    return bm_extract_move(b, st, nodes, n_dev, n_host, alias, out, checksum, 0, 0);
}

int fdg_bm_release(fdg_bm* b, void* stv, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host) {
    return bm_release(b, (cudaStream_t)stv, nodes, nullptr, n_dev, n_host);
}

}  // extern "C"

namespace fdg {
// release_batch (buffer_manager.hpp:352-364) from the batch's node ids or -- when the
// caller still holds it -- from its alias list (no mapping-table reads).
int bm_release(fdg_bm* b, cudaStream_t st, const uint64_t* nodes, const int64_t* alias, const uint32_t* n_dev,
               uint64_t n_host) {
    const BmDev& d = b->d;
    const uint64_t slack = 2 * uint64_t(b->max_batch) + kTileN;
    k_reset_ctrs<<<1, 32, 0, st>>>(d.st);
    {
        FDG_TRACE("bm_release", st);
        if (alias)
            k_release<true><<<n_tiles_for(n_host), kT, 0, st>>>(d, nodes, alias, n_dev, n_host, b->epoch++);
        else
            k_release<false><<<n_tiles_for(n_host), kT, 0, st>>>(d, nodes, alias, n_dev, n_host, b->epoch++);
    }
    {
        FDG_TRACE("bm_compact", st);
        k_compact<<<bm_persistent_grid(b), kT, 0, st>>>(d, slack, b->epoch++);
    }
    k_compact_finish<<<1, 1, 0, st>>>(d, slack);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

// Copies a device-detected buffer-manager error into a batch record's status (stream-ordered).
int bm_status_to(fdg_bm* b, cudaStream_t st, uint32_t* dst) {
    k_status_to<<<1, 1, 0, st>>>(b->d.st, dst);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}
}  // namespace fdg

extern "C" {

int fdg_bm_stats_get(fdg_bm* b, fdg_bm_stats* out) {
    FDG_CUDA(cudaDeviceSynchronize());
    BmState h;
    FDG_CUDA(cudaMemcpy(&h, b->d.st, sizeof(h), cudaMemcpyDeviceToHost));
    out->hits = h.hits;
    out->loads = h.loads;
    out->waits = h.waits;
    out->evictions = h.evictions;
    out->takeovers = h.takeovers;
    out->releases = h.releases;
    out->standby_len = h.live;
    return FDG_OK;
}

int fdg_bm_status(fdg_bm* b) {
    if (cudaDeviceSynchronize() != cudaSuccess) return FDG_CUDA_ERROR;
    BmState h;
    if (cudaMemcpy(&h, b->d.st, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return FDG_CUDA_ERROR;
    return int(h.status);
}

void* fdg_bm_region(fdg_bm* b) { return b->region; }

int fdg_bm_entry(fdg_bm* b, uint64_t node, int64_t* slot, uint32_t* ref, uint32_t* valid) {
    if (node >= b->d.N) return fail(FDG_OUT_OF_RANGE, "bm_entry: node out of range");
    FDG_CUDA(cudaDeviceSynchronize());
    Entry e;
    FDG_CUDA(cudaMemcpy(&e, b->d.map + node, sizeof(e), cudaMemcpyDeviceToHost));
    uint64_t nr = kFree;
    if (e.slot >= 0) {  // a stale entry (slot rebound since) reads as the reference's evicted state
        FDG_CUDA(cudaMemcpy(&nr, &b->d.slot[e.slot].nr, 8, cudaMemcpyDeviceToHost));
        if (m_node(nr) != node) e = Entry{-1, 0u};
    }
    *slot = e.slot;
    *ref = e.slot >= 0 ? m_ref(nr) : 0u;
    *valid = e.refv >> 31;
    return FDG_OK;
}

int fdg_bm_ring_info(fdg_bm* b, uint64_t* head, uint64_t* tail, uint64_t* capacity, uint64_t* compactions) {
    FDG_CUDA(cudaDeviceSynchronize());
    BmState h;
    FDG_CUDA(cudaMemcpy(&h, b->d.st, sizeof(h), cudaMemcpyDeviceToHost));
    if (head) *head = h.head;
    if (tail) *tail = h.tail;
    if (capacity) *capacity = b->d.R;
    if (compactions) *compactions = h.compactions;
    return FDG_OK;
}

int fdg_bm_reverse(fdg_bm* b, uint64_t slot, int64_t* node) {
    if (slot >= b->slots) return fail(FDG_OUT_OF_RANGE, "bm_reverse: slot out of range");
    FDG_CUDA(cudaDeviceSynchronize());
    uint64_t v;
    FDG_CUDA(cudaMemcpy(&v, &b->d.slot[slot].nr, 8, cudaMemcpyDeviceToHost));
    *node = m_node(v) == kFree ? -1 : int64_t(m_node(v));
    return FDG_OK;
}

// validate_locked (buffer_manager.hpp:488-515) on a host copy: bijection between
// mapping and reverse, no valid entry without a slot, standby soundness, and
// the live-ring count equals the standby size.
int fdg_bm_validate(fdg_bm* b) {
    FDG_CUDA(cudaDeviceSynchronize());
    const BmDev& d = b->d;
    std::vector<Entry> map(d.N);
    std::vector<SlotMeta> meta(d.S);
    std::vector<uint64_t> rev(d.S), pos(d.S);
    BmState h;
    FDG_CUDA(cudaMemcpy(&h, d.st, sizeof(h), cudaMemcpyDeviceToHost));
    if (h.status) return fail(int(h.status), "buffer manager in error state " + std::to_string(h.status));
    FDG_CUDA(cudaMemcpy(map.data(), d.map, d.N * 8, cudaMemcpyDeviceToHost));
    FDG_CUDA(cudaMemcpy(meta.data(), d.slot, d.S * sizeof(SlotMeta), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> ref(d.S);
    for (uint64_t s = 0; s < d.S; ++s) {
        rev[s] = m_node(meta[s].nr);
        ref[s] = m_ref(meta[s].nr);
        pos[s] = meta[s].pos;
    }
    // Lazy invalidation: stale entries (slot rebound since) are the reference's evicted
    // entries. In eager (debug) mode there are none, so any such entry is a corruption and
    // fails the bijection check below.
    if (!b->eager)
        for (uint64_t v = 0; v < d.N; ++v)
            if (map[v].slot >= 0 && uint64_t(map[v].slot) < d.S && rev[map[v].slot] != v) map[v] = Entry{-1, 0u};
    std::vector<int32_t> ring(d.R);
    FDG_CUDA(cudaMemcpy(ring.data(), d.ring[h.ring_sel], d.R * 4, cudaMemcpyDeviceToHost));
    std::vector<uint8_t> seen(d.S, 0);
    for (uint64_t v = 0; v < d.N; ++v) {
        const Entry& e = map[v];
        if (e.slot < 0 && (e.refv & kValid)) return fail(FDG_INVARIANT, "impossible state: valid without slot");
        if (e.slot >= 0) {
            if (uint64_t(e.slot) >= d.S) return fail(FDG_INVARIANT, "slot out of range");
            if (rev[e.slot] != v) return fail(FDG_INVARIANT, "mapping/reverse mismatch for node " + std::to_string(v));
            if (seen[e.slot]) return fail(FDG_INVARIANT, "slot mapped by two nodes");
            seen[e.slot] = 1;
        }
    }
    uint64_t live = 0;
    for (uint64_t p = h.head; p < h.tail; ++p) {
        int32_t s = ring[p % d.R];
        if (pos[s] != p) continue;
        ++live;
        if (ref[s] != 0) return fail(FDG_INVARIANT, "standby slot whose node still holds references");
    }
    if (live != h.live) return fail(FDG_INVARIANT, "standby size mismatch");
    for (uint64_t s = 0; s < d.S; ++s) {
        if (rev[s] == kFree) {
            if (ref[s] != 0) return fail(FDG_INVARIANT, "free slot with references");
            continue;
        }
        if (map[rev[s]].slot != int32_t(s)) return fail(FDG_INVARIANT, "reverse mapping points at node without matching slot");
    }
    return FDG_OK;
}

}  // extern "C"

// ---- the reference's per-node protocol (C++ drop-in), stream-ordered ---------------
extern "C" {

int fdg_bm_acquire(fdg_bm* b, void* stv, const uint64_t* nodes_dev, uint64_t n, int64_t* alias_dev,
                   uint32_t* to_load_dev, uint32_t* n_load_dev) {
    cudaStream_t st = (cudaStream_t)stv;
    if (n > b->max_batch) return fail(FDG_INVALID_ARG, "bm_acquire: batch larger than max_batch_nodes");
    const BmDev& d = b->d;
    k_reset_ctrs<<<1, 32, 0, st>>>(d.st);
    k_acquire<<<n_tiles_for(n), kT, 0, st>>>(d, nodes_dev, nullptr, n, alias_dev, d.is_load[0], b->epoch++);
    FDG_CUDA(cudaGetLastError());
    if (to_load_dev && n) FDG_CUDA(cudaMemcpyAsync(to_load_dev, d.load_pos, n * 4, cudaMemcpyDeviceToDevice, st));
    if (n_load_dev) {
        k_copy_nload<<<1, 1, 0, st>>>(d.st, n_load_dev);
        FDG_CUDA(cudaGetLastError());
    }
    return FDG_OK;
}

int fdg_bm_pop_standby(fdg_bm* b, void* stv, uint32_t count, int64_t* slots_dev) {
    cudaStream_t st = (cudaStream_t)stv;
    if (count == 0) return FDG_OK;
    if (count > b->max_batch) return fail(FDG_INVALID_ARG, "bm_pop_standby: more slots than max_batch_nodes");
    const BmDev& d = b->d;
    k_set_nload<<<1, 1, 0, st>>>(d.st, count);
    k_select<false><<<bm_persistent_grid(b), kT, 0, st>>>(d, b->epoch++, nullptr, nullptr);
    k_pop<<<(count + 255) / 256, 256, 0, st>>>(d, slots_dev);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int fdg_bm_bind(fdg_bm* b, void* stv, const uint64_t* nodes_dev, const int64_t* slots_dev, uint32_t n) {
    if (n == 0) return FDG_OK;
    k_bind_explicit<<<(n + 255) / 256, 256, 0, (cudaStream_t)stv>>>(b->d, nodes_dev, slots_dev, n);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int fdg_bm_publish(fdg_bm* b, void* stv, const uint64_t* nodes_dev, uint32_t n) {
    if (n == 0) return FDG_OK;
    k_publish<<<(n + 255) / 256, 256, 0, (cudaStream_t)stv>>>(b->d, nodes_dev, n);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int fdg_bm_unwind_bound(fdg_bm* b, void* stv, uint64_t node) {
    k_unwind_or_release<<<1, 1, 0, (cudaStream_t)stv>>>(b->d, node, 1);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int fdg_bm_release_ref(fdg_bm* b, void* stv, uint64_t node) {
    k_unwind_or_release<<<1, 1, 0, (cudaStream_t)stv>>>(b->d, node, 0);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int fdg_bm_load_rows(fdg_bm* b, void* stv, const uint64_t* nodes_dev, const int64_t* slots_dev, uint32_t n) {
    if (n == 0) return FDG_OK;
    if (b->ctx->shard_bases.empty() || !b->region) return fail(FDG_NOT_LOADED, "bm_load_rows: no feature table bound");
    const uint32_t rb = b->ctx->row_bytes;
    const uint64_t chunks = uint64_t(n) * (rb / 16);
    const int blocks = int(std::max<uint64_t>(1, std::min<uint64_t>((chunks + 255) / 256, uint64_t(b->ctx->sm_count) * 8)));
    k_load_rows<<<blocks, 256, 0, (cudaStream_t)stv>>>(nodes_dev, slots_dev, n,
                                                       static_cast<const char*>(b->ctx->shard_bases[0]), b->region, rb);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

}  // extern "C"
