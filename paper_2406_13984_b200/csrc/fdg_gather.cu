// fdg_gather.cu -- feature extraction as an HBM gather into the mini-batch
// tensor: X[i, :] = row(nodes[i]).
//
// Replaces the reference's extraction byte movement: per-row copies from the
// staging arena into FeatureRegion slots (extractor.hpp:374-386,
// device_region.hpp:60-64) that the trainer then reads by alias
// (pipeline.hpp:103-124). On B200 the whole table is HBM-resident, so a batch's
// rows move table -> X in one pass: 16-byte vector loads that bypass L1
// (ld.global.nc.L1::no_allocate) and 16-byte streaming stores, consecutive
// threads on consecutive 16 B chunks of the flattened [n, row_bytes] output
// (coalesced writes; each row read as whole 32 B sectors). HBM-bound:
// algorithmic bytes = 2 * n * row_bytes per launch.
//
// k_gather_hash additionally folds trainer_step's checksum
// sum_i hash_bytes64(row_i) (common.hpp:88-105): a warp stages 32 rows in
// shared memory and each lane then runs one row's sequential splitmix chain.
#include <algorithm>
#include <atomic>

#include "fdg_internal.cuh"

namespace fdg {
namespace {

struct FastDiv {  // Granlund-Montgomery round-up division by a runtime constant (n < 2^32)
    uint32_t m, l;
    __host__ void init(uint32_t d) {
        l = 0;
        while ((1ull << l) < d) ++l;
        m = uint32_t(((1ull << 32) * ((1ull << l) - d)) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return uint32_t((uint64_t(__umulhi(n, m)) + n) >> l);
    }
};

struct TableRef {
    const char* base;              // single shard
    const char* const* shards;     // sharded: device array of bases
    uint64_t rows_per_shard;
    uint32_t n_shards;
    uint32_t row_bytes;
    uint32_t evict_first;
    uint32_t pf64;  // 64-byte L2 fetch hint on table reads
    FastDiv sdiv;   // node -> shard for node ids < 2^32 (a 64-bit division per 16-byte chunk
    uint32_t sdiv_ok;  // made the sharded gather 1.75x slower than the single-shard one)
};

template <bool SHARDED>
__device__ __forceinline__ const char* row_ptr(const TableRef& t, uint64_t node) {
    if constexpr (!SHARDED) {
        return t.base + node * t.row_bytes;
    } else {
        const uint64_t s = (t.sdiv_ok && node < 0xFFFFFFFFull) ? t.sdiv.div(uint32_t(node)) : node / t.rows_per_shard;
        return t.shards[s] + (node - s * t.rows_per_shard) * t.row_bytes;
    }
}

// Optional L2 evict-first marking of the gather stream (option "gather_evict_first",
// off by default: the samplers' hash tables carry evict-last hints instead).
__device__ __forceinline__ uint64_t gather_policy(bool evict_first) {
    uint64_t pol;
    if (evict_first)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// "gather_evict_first": 0 off, 1 loads and stores, 2 table loads only, 3 X stores only.
__device__ __forceinline__ uint64_t gather_policy_ld(uint32_t ef) { return gather_policy(ef == 1 || ef == 2); }
__device__ __forceinline__ uint64_t gather_policy_st(uint32_t ef) { return gather_policy(ef == 1 || ef == 3); }
__device__ __forceinline__ uint4 ldg_stream(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
// 64-byte L2 fetches (LDG .LTC64B) instead of the default line fill, for rows whose length
// is not a multiple of 128 B (a 400-byte row otherwise costs 4 full lines). A compile-time
// choice: a runtime branch around the loads costs the fused-checksum kernel its MLP
// (products extraction + checksum 147 -> 212 us per batch).
template <bool PF64>
__device__ __forceinline__ uint4 ldg_row(const uint4* p, uint64_t pol) {
    if constexpr (!PF64) return ldg_stream(p, pol);
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void stg_stream(uint4* p, uint4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(pol)
                 : "memory");
}

constexpr int kUnroll = 4;
// 2 x 512 threads per SM (half the SM's warp slots): enough bytes in flight to
// saturate HBM while leaving room for the next batch's sampling kernels and the
// MT prefetch CTAs to co-reside (they run on other streams).

// Dynamically scheduled variant: CTAs claim units of kUnroll * 512 * kDynIters
// chunks (64 KB) from a per-launch counter, so CTAs that become resident late
// (the SMs are shared with the samplers' kernels) take less of the work instead
// of stretching the launch. The last CTA to finish resets the counter pair.
constexpr int kDynIters = 2;

template <bool SHARDED, bool PF64 = false>
__global__ void __launch_bounds__(512) k_gather16_dyn(const uint64_t* __restrict__ nodes, const uint32_t* n_dev,
                                                      uint64_t n_host, const uint32_t* status, TableRef t,
                                                      FastDiv cdiv, uint32_t cpr, uint4* __restrict__ out,
                                                      uint32_t* ctr) {
    __shared__ uint32_t s_unit;
    const bool skip = status && *status;
    const uint64_t n = skip ? 0 : (n_dev ? *n_dev : n_host);
    const uint32_t total = uint32_t(n * cpr);
    constexpr uint32_t kStep = kUnroll * 512;
    constexpr uint32_t kUnit = kStep * kDynIters;
    const uint64_t pol = gather_policy_ld(t.evict_first), pol_st = gather_policy_st(t.evict_first);
    for (;;) {
        if (threadIdx.x == 0) s_unit = atomicAdd(ctr, 1u);
        __syncthreads();
        const uint64_t u0l = uint64_t(s_unit) * kUnit;
        __syncthreads();
        if (u0l >= total) break;
        const uint32_t u0 = uint32_t(u0l), u1 = uint32_t(min(uint64_t(total), u0l + kUnit));
#pragma unroll 1
        for (uint32_t b = u0; b < u1; b += kStep) {
            if (b + kStep <= u1) {
                uint4 v[kUnroll];
                uint32_t cc[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    cc[u] = b + u * 512 + threadIdx.x;
                    uint32_t row = cdiv.div(cc[u]);
                    uint32_t col = cc[u] - row * cpr;
                    v[u] = ldg_row<PF64>(reinterpret_cast<const uint4*>(row_ptr<SHARDED>(t, __ldg(nodes + row))) + col,
                                      pol);
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) stg_stream(out + cc[u], v[u], pol_st);
            } else {
                for (uint32_t c = b + threadIdx.x; c < u1; c += 512) {
                    uint32_t row = cdiv.div(c);
                    uint32_t col = c - row * cpr;
                    stg_stream(out + c,
                               ldg_row<PF64>(reinterpret_cast<const uint4*>(row_ptr<SHARDED>(t, __ldg(nodes + row))) + col,
                                          pol),
                               pol_st);
                }
            }
        }
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // every CTA has claimed past the end
            ctr[0] = 0;
            ctr[1] = 0;
            __threadfence();
        }
    }
}

// 4-byte fallback for rows that are not a multiple of 16 bytes.
template <bool SHARDED>
__global__ void k_gather4(const uint64_t* __restrict__ nodes, const uint32_t* n_dev, uint64_t n_host,
                          const uint32_t* status, TableRef t, FastDiv cdiv, uint32_t cpr, uint32_t* __restrict__ out) {
    if (status && *status) return;
    const uint64_t n = n_dev ? *n_dev : n_host;
    const uint64_t total = n * cpr;
    for (uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c < total;
         c += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t row = c / cpr, col = c - row * cpr;
        out[c] = reinterpret_cast<const uint32_t*>(row_ptr<SHARDED>(t, nodes[row]))[col];
    }
}

// Software-pipelined gather + checksum for any row size that is a multiple of 16 bytes
// (k_gather_hash_rb below covers the benchmarked row sizes at compile time): a warp owns
// 32-row groups walked in 128-byte chunks and issues the loads of its NEXT item (the next
// chunk of the group, or chunk 0 of its next group) before it hashes the current one from
// shared memory, so loads stay in flight during the serial splitmix chains (a load-then-
// hash kernel measured 217 vs 160 us per Papers batch). Up to kHpMinBlocks x 8 warps per SM
// keep ~128 KB of rows in flight.
constexpr int kHpWarps = 8;
constexpr int kH16Stride = 144;  // staged 128-byte chunk row stride (conflict-free 16-byte lane reads)
constexpr int kHpMinBlocks = 3;

template <bool SHARDED, bool ALIAS>
__global__ void __launch_bounds__(kHpWarps * 32, kHpMinBlocks)
    k_gather_hash_pipe(const uint64_t* __restrict__ nodes, const uint32_t* n_dev, uint64_t n_host,
                       const uint32_t* status, TableRef t, char* __restrict__ out, uint64_t* checksum) {
    __shared__ __align__(16) char smem[kHpWarps][32 * kH16Stride];
    if (status && *status) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* wbuf = smem[warp];
    const uint32_t rb = t.row_bytes;
    const uint32_t nch = (rb + 127) >> 7;  // 128-byte chunks per row
    const uint64_t n = n_dev ? *n_dev : n_host;
    const uint64_t groups = (n + 31) / 32;
    const uint64_t gstride = uint64_t(gridDim.x) * kHpWarps;
    const uint64_t g0 = blockIdx.x * uint64_t(kHpWarps) + warp;
    if (g0 >= groups) return;
    const uint64_t my_groups = (groups - g0 + gstride - 1) / gstride;
    const uint64_t items = my_groups * nch;
    const uint64_t pol = gather_policy(t.evict_first);
    const uint32_t part = lane & 7;
    auto node_of = [&](uint64_t g) -> uint64_t {
        const uint64_t r = g * 32 + lane;
        return (g < groups && r < n) ? __ldg(nodes + r) : 0;
    };
    auto rows_of = [&](uint64_t g) -> uint32_t { return uint32_t(n - g * 32 < 32 ? n - g * 32 : 32); };
    uint4 v[8];
    auto issue = [&](uint64_t g, uint32_t c, uint64_t node_reg) {
        const uint32_t rows = rows_of(g);
        const uint32_t c0 = c << 7;
        const uint32_t parts = (rb - c0 < 128 ? rb - c0 : 128) >> 4;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t r = k * 4 + (lane >> 3);
            const uint64_t node = __shfl_sync(0xffffffffu, node_reg, int(r));
            if (r < rows && part < parts) {
                const char* src = ALIAS ? t.base + node * rb : row_ptr<SHARDED>(t, node);
                v[k] = ldg_stream(reinterpret_cast<const uint4*>(src + c0) + part, pol);
            }
        }
    };
    uint64_t cur_node = node_of(g0);
    uint64_t nxt_node = node_of(g0 + gstride);
    const uint64_t seed = 0x27d4eb2f165667c5ull ^ (uint64_t(rb) * 0x9e3779b97f4a7c15ull);
    uint64_t h = seed, sum = 0;
    issue(g0, 0, cur_node);
    uint64_t g = g0;
    uint32_t c = 0;
    for (uint64_t it = 0; it < items; ++it) {
        const uint32_t rows = rows_of(g);
        const uint32_t c0 = c << 7;
        const uint32_t parts = (rb - c0 < 128 ? rb - c0 : 128) >> 4;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t r = k * 4 + (lane >> 3);
            if (r < rows && part < parts) {
                if (!ALIAS && out) stg_stream(reinterpret_cast<uint4*>(out + (g * 32 + r) * rb + c0) + part, v[k], pol);
                *reinterpret_cast<uint4*>(wbuf + r * kH16Stride + part * 16) = v[k];
            }
        }
        __syncwarp();
        const bool last = c + 1 == nch;
        if (it + 1 < items) issue(last ? g + gstride : g, last ? 0 : c + 1, last ? nxt_node : cur_node);
        if (lane < int(rows)) {
            const uint4* p = reinterpret_cast<const uint4*>(wbuf + lane * kH16Stride);
            for (uint32_t s = 0; s < parts; ++s) {
                const uint4 w = p[s];
                h = splitmix64(h ^ (uint64_t(w.y) << 32 | w.x));
                h = splitmix64(h ^ (uint64_t(w.w) << 32 | w.z));
            }
        }
        __syncwarp();
        if (last) {
            if (lane < int(rows)) sum += splitmix64(h);
            h = seed;
            g += gstride;
            c = 0;
            cur_node = nxt_node;
            nxt_node = node_of(g + gstride);
        } else {
            ++c;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0 && sum) atomicAdd(reinterpret_cast<unsigned long long*>(checksum), (unsigned long long)sum);
}

// Lean variant of k_gather_hash_pipe for a compile-time row size RB, staging
// CH-byte chunks of 32 rows. ncu of the runtime-rb kernel (Friendster, 1 KB rows)
// showed 744 warp-instructions per 32-row x 128-byte item against 320 for the
// splitmix chains themselves: per-chunk shuffles of node ids, 64-bit address
// arithmetic and predicated loads. Here a full 32-row group resolves its per-lane
// source pointers once (reused by every chunk), destination offsets are
// immediates, and only the one ragged last group takes the predicated path.
// CH = 256 (rows >= 256 B): a row's bytes are requested in 256-byte runs instead
// of 128-byte ones spaced a whole hash phase apart. Measured per batch with the
// checksum, extraction alone: Papers 155 us (128-byte chunks: 176 us; plain
// gather without checksum: 159 us), Friendster 312 us (361 us).
template <int CH>
struct HashRbShape {
    static constexpr int LPR = CH / 16;    // lanes per row in one load instruction
    static constexpr int RPI = 32 / LPR;   // rows per load instruction
    static constexpr int NI = 32 / RPI;    // load instructions per chunk (= 16-byte parts per row chunk)
    static constexpr int STRIDE = CH + 16; // staged row stride: conflict-free 16-byte lane reads
    static constexpr int MINB = CH == 128 ? 3 : 2;
};

// DYN: warps claim 32-row groups from a per-launch counter (one group ahead) instead of a
// static stride, so CTAs that become resident late next to the samplers take less work.
template <int RB, int CH, bool SHARDED, bool ALIAS, bool HASH = true, bool DYN = false>
__global__ void __launch_bounds__(kHpWarps * 32, HashRbShape<CH>::MINB)
    k_gather_hash_rb(const uint64_t* __restrict__ nodes, const uint32_t* n_dev, uint64_t n_host,
                     const uint32_t* status, TableRef t, char* __restrict__ out, uint64_t* checksum,
                     uint32_t* ctr = nullptr) {
    using S = HashRbShape<CH>;
    static_assert(RB % 16 == 0, "16-byte rows");
    constexpr int NCH = (RB + CH - 1) / CH;
    constexpr int LASTP = (RB - (NCH - 1) * CH) / 16;  // 16-byte parts in the last chunk
    constexpr bool EVEN = RB % CH == 0;
    extern __shared__ __align__(16) char rb_smem[];  // kHpWarps x 32 rows x STRIDE
    const bool skip = status && *status;
    if (!DYN && skip) return;  // (DYN: every CTA still takes part in the counter reset)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* wbuf = rb_smem + warp * 32 * S::STRIDE;
    const uint64_t n = skip ? 0 : (n_dev ? *n_dev : n_host);
    const uint64_t full = n / 32;
    const uint64_t gstride = uint64_t(gridDim.x) * kHpWarps;
    const uint64_t pol = gather_policy_ld(t.evict_first), pol_st = gather_policy_st(t.evict_first);
    const uint32_t part = lane % S::LPR, rsub = lane / S::LPR;
    const uint64_t seed = 0x27d4eb2f165667c5ull ^ (uint64_t(RB) * 0x9e3779b97f4a7c15ull);
    // this warp's group sequence: g0, g0 + gstride, ... (static) or its claims (DYN); the first
    // value >= full ends it, and the warp whose sequence ends exactly at `full` owns the ragged
    // last group
    auto next = [&](uint64_t g) -> uint64_t {
        if constexpr (DYN) {
            uint32_t c = 0;
            if (lane == 0) c = atomicAdd(ctr, 1u);
            return __shfl_sync(0xffffffffu, c, 0);
        } else {
            return g + gstride;
        }
    };
    uint64_t sum = 0;
    uint64_t g = DYN ? next(0) : blockIdx.x * uint64_t(kHpWarps) + warp;
    if (g < full) {
        const char* src[S::NI];
        uint4 v[S::NI];
        auto setup = [&](uint64_t node_reg) {
#pragma unroll
            for (int k = 0; k < S::NI; ++k) {
                const uint64_t node = __shfl_sync(0xffffffffu, node_reg, k * S::RPI + int(rsub));
                src[k] = (ALIAS ? t.base + node * RB : row_ptr<SHARDED>(t, node)) + part * 16;
            }
        };
        auto issue = [&](int c) {
#pragma unroll
            for (int k = 0; k < S::NI; ++k)
                if (EVEN || c + 1 < NCH || int(part) < LASTP)
                    v[k] = ldg_row<RB % 128 != 0>(reinterpret_cast<const uint4*>(src[k] + c * CH), pol);
        };
        uint64_t gn = next(g);
        uint64_t nxt_node = gn < full ? __ldg(nodes + gn * 32 + lane) : 0;
        setup(__ldg(nodes + g * 32 + lane));
        issue(0);
        while (g < full) {
            char* dst = ALIAS ? nullptr : out + (g * 32 + rsub) * RB + part * 16;
            uint64_t h = seed;
            uint64_t g2 = gn;
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) {
                const bool lastc = c + 1 == NCH;
#pragma unroll
                for (int k = 0; k < S::NI; ++k) {
                    if (EVEN || !lastc || int(part) < LASTP) {
                        if (!ALIAS && out)
                            stg_stream(reinterpret_cast<uint4*>(dst + k * S::RPI * RB + c * CH), v[k], pol_st);
                        if (HASH) *reinterpret_cast<uint4*>(wbuf + (k * S::RPI + rsub) * S::STRIDE + part * 16) = v[k];
                    }
                }
                if (HASH) __syncwarp();
                if (!lastc) {
                    issue(c + 1);
                } else if (gn < full) {  // chunk 0 of this warp's next group
                    setup(nxt_node);
                    issue(0);
                    g2 = next(gn);
                    nxt_node = g2 < full ? __ldg(nodes + g2 * 32 + lane) : 0;
                }
                if (HASH) {
                    const uint4* p = reinterpret_cast<const uint4*>(wbuf + lane * S::STRIDE);
                    const int parts = (EVEN || !lastc) ? S::NI : LASTP;
#pragma unroll
                    for (int s = 0; s < S::NI; ++s) {
                        if (s < parts) {
                            const uint4 w = p[s];
                            h = splitmix64(h ^ (uint64_t(w.y) << 32 | w.x));
                            h = splitmix64(h ^ (uint64_t(w.w) << 32 | w.z));
                        }
                    }
                    __syncwarp();
                }
            }
            if (HASH) sum += splitmix64(h);
            g = gn;
            gn = g2;
        }
    }
    // the ragged last group (n % 32 rows), if this warp's sequence ends at it
    const uint64_t tail = full;
    if (n % 32 && g == tail) {
        const uint32_t rows = uint32_t(n - tail * 32);
        const uint64_t my_node = lane < int(rows) ? __ldg(nodes + tail * 32 + lane) : 0;
        uint64_t h = seed;
        for (int c = 0; c < NCH; ++c) {
            const int parts = c + 1 < NCH ? S::NI : LASTP;
#pragma unroll
            for (int k = 0; k < S::NI; ++k) {
                const uint32_t r = k * S::RPI + rsub;
                const uint64_t node = __shfl_sync(0xffffffffu, my_node, int(r));
                if (r < rows && int(part) < parts) {
                    const char* src = ALIAS ? t.base + node * RB : row_ptr<SHARDED>(t, node);
                    const uint4 w = ldg_row<RB % 128 != 0>(reinterpret_cast<const uint4*>(src + c * CH) + part, pol);
                    if (!ALIAS && out)
                        stg_stream(reinterpret_cast<uint4*>(out + (tail * 32 + r) * RB + c * CH) + part, w, pol_st);
                    if (HASH) *reinterpret_cast<uint4*>(wbuf + r * S::STRIDE + part * 16) = w;
                }
            }
            if (!HASH) continue;
            __syncwarp();
            if (lane < int(rows)) {
                const uint4* p = reinterpret_cast<const uint4*>(wbuf + lane * S::STRIDE);
                for (int s = 0; s < parts; ++s) {
                    const uint4 w = p[s];
                    h = splitmix64(h ^ (uint64_t(w.y) << 32 | w.x));
                    h = splitmix64(h ^ (uint64_t(w.w) << 32 | w.z));
                }
            }
            __syncwarp();
        }
        if (HASH && lane < int(rows)) sum += splitmix64(h);
    }
    if (HASH) {
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0 && sum) atomicAdd(reinterpret_cast<unsigned long long*>(checksum), (unsigned long long)sum);
    }
    if constexpr (DYN) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // every CTA has claimed past the end
                ctr[0] = 0;
                ctr[1] = 0;
                __threadfence();
            }
        }
    }
}


// The buffer manager's row move with the trainer checksum folded in (config 3's e2e path):
// per row, a miss reads the table and writes its slot and X, a hit reads its slot and writes X
// (k_move's semantics), and every row is staged in shared memory and hashed by one lane, as in
// k_gather_hash_rb. Replaces k_move + a second pass over the batch's slots for the checksum
// (another n x row_bytes of reads). Lane l's row of a group: is_load / alias / node resolve
// once into a source pointer and a slot pointer (null for a hit), shuffled per load.
// MODE 0: the whole move; 1: X rows only (before the bind: misses read the table, hits their
// pinned slots); 2: the misses' slot fills only (after the bind). Split moves are never hashed.
template <int RB, int CH, bool HASH = true, int MODE = 0>
__global__ void __launch_bounds__(kHpWarps * 32, 1)  // one CTA per SM (g_hash_ctas_per_sm): no register cap
    k_move_hash_rb(const uint64_t* __restrict__ nodes, const uint32_t* n_dev, uint64_t n_host,
                   const uint32_t* status, const int64_t* __restrict__ alias, const uint8_t* __restrict__ is_load,
                   const char* __restrict__ table, char* __restrict__ region, char* __restrict__ out,
                   uint64_t* checksum) {
    using S = HashRbShape<CH>;
    static_assert(RB % 16 == 0, "16-byte rows");
    constexpr int NCH = (RB + CH - 1) / CH;
    constexpr int LASTP = (RB - (NCH - 1) * CH) / 16;
    constexpr bool EVEN = RB % CH == 0;
    extern __shared__ __align__(16) char rb_smem[];
    if (status && *status) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* wbuf = rb_smem + warp * 32 * S::STRIDE;
    const uint64_t n = n_dev ? *n_dev : n_host;
    const uint64_t groups = (n + 31) / 32;
    const uint64_t gstride = uint64_t(gridDim.x) * kHpWarps;
    uint64_t pol;  // row traffic must not flush the batch's metadata sectors out of L2
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const uint32_t part = lane % S::LPR, rsub = lane / S::LPR;
    const uint64_t seed = 0x27d4eb2f165667c5ull ^ (uint64_t(RB) * 0x9e3779b97f4a7c15ull);
    uint64_t sum = 0;
    auto resolve = [&](uint64_t g, uintptr_t& src, uintptr_t& slot) {  // this lane's row of group g
        const uint64_t r = g * 32 + lane;
        src = 0;
        slot = 0;
        if (g < groups && r < n) {
            if (is_load[r]) {
                src = reinterpret_cast<uintptr_t>(table + nodes[r] * RB);
                if (MODE != 1) slot = reinterpret_cast<uintptr_t>(region + uint64_t(alias[r]) * RB);  // bound
            } else if (MODE != 2) {
                src = reinterpret_cast<uintptr_t>(region + uint64_t(alias[r]) * RB);
            }
        }
    };
    uint64_t g = blockIdx.x * uint64_t(kHpWarps) + warp;
    if (g >= groups) return;
    uintptr_t my_src, my_slot, nx_src, nx_slot;
    resolve(g, my_src, my_slot);
    resolve(g + gstride, nx_src, nx_slot);
    const char* src[S::NI];
    uint4 v[S::NI];
    uint32_t live = 0;  // MODE 2: rows of this lane's loads that move (misses)
    auto setup = [&](uintptr_t s_reg) {
        live = 0;
#pragma unroll
        for (int k = 0; k < S::NI; ++k) {
            const uintptr_t sp = __shfl_sync(0xffffffffu, s_reg, k * S::RPI + int(rsub));
            src[k] = reinterpret_cast<const char*>(sp) + part * 16;
            if (sp) live |= 1u << k;
        }
    };
    auto issue = [&](int c, uint32_t rows) {
#pragma unroll
        for (int k = 0; k < S::NI; ++k)
            if ((EVEN || c + 1 < NCH || int(part) < LASTP) && uint32_t(k * S::RPI) + rsub < rows &&
                (MODE != 2 || (live & (1u << k))))
                v[k] = ldg_row<RB % 128 != 0>(reinterpret_cast<const uint4*>(src[k] + c * CH), pol);
    };
    auto rows_of = [&](uint64_t gg) -> uint32_t { return uint32_t(n - gg * 32 < 32 ? n - gg * 32 : 32); };
    setup(my_src);
    issue(0, rows_of(g));
    while (g < groups) {
        const uint32_t rows = rows_of(g);
        uint64_t h = seed;
        const uint64_t gn = g + gstride;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
            const bool lastc = c + 1 == NCH;
#pragma unroll
            for (int k = 0; k < S::NI; ++k) {
                const uint32_t r = k * S::RPI + rsub;
                const uintptr_t sl = __shfl_sync(0xffffffffu, my_slot, int(r));
                if ((EVEN || !lastc || int(part) < LASTP) && r < rows && (MODE != 2 || (live & (1u << k)))) {
                    const uint32_t off = c * CH + part * 16;
                    if (MODE != 2 && out) stg_stream(reinterpret_cast<uint4*>(out + (g * 32 + r) * RB + off), v[k], pol);
                    if (sl) stg_stream(reinterpret_cast<uint4*>(reinterpret_cast<char*>(sl) + off), v[k], pol);
                    if (HASH) *reinterpret_cast<uint4*>(wbuf + r * S::STRIDE + part * 16) = v[k];
                }
            }
            if (HASH) __syncwarp();
            if (!lastc) {
                issue(c + 1, rows);
            } else if (gn < groups) {  // chunk 0 of this warp's next group
                setup(nx_src);
                issue(0, rows_of(gn));
            }
            if (HASH && lane < int(rows)) {
                const uint4* p = reinterpret_cast<const uint4*>(wbuf + lane * S::STRIDE);
                const int parts = (EVEN || !lastc) ? S::NI : LASTP;
#pragma unroll
                for (int s2 = 0; s2 < S::NI; ++s2) {
                    if (s2 < parts) {
                        const uint4 w = p[s2];
                        h = splitmix64(h ^ (uint64_t(w.y) << 32 | w.x));
                        h = splitmix64(h ^ (uint64_t(w.w) << 32 | w.z));
                    }
                }
            }
            if (HASH) __syncwarp();
        }
        if (HASH && lane < int(rows)) sum += splitmix64(h);
        g = gn;
        my_src = nx_src;
        my_slot = nx_slot;
        resolve(g + gstride, nx_src, nx_slot);
    }
    if (!HASH) return;
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0 && sum) atomicAdd(reinterpret_cast<unsigned long long*>(checksum), (unsigned long long)sum);
}

template <int RB, int CH>
int launch_move_hash_one(const Ctx& c, cudaStream_t st, uint64_t groups, const uint64_t* nodes, const uint32_t* n_dev,
                         uint64_t n_host, const uint32_t* status, const int64_t* alias, const uint8_t* is_load,
                         const char* table, char* region, char* out, uint64_t* checksum, int mode) {
    constexpr int smem = kHpWarps * 32 * HashRbShape<CH>::STRIDE;
    static PerDeviceOnce attr;
    if (attr.first()) {
        FDG_CUDA(cudaFuncSetAttribute(k_move_hash_rb<RB, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        FDG_CUDA(
            cudaFuncSetAttribute(k_move_hash_rb<RB, CH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    if (mode == 1 || mode == 2) {  // split move (no hash, no shared memory)
        if (mode == 1)
            k_move_hash_rb<RB, CH, false, 1><<<std::max<int>(1, int(std::min<uint64_t>((groups + kHpWarps - 1) / kHpWarps,
                                                                              uint64_t(c.sm_count)))),
                                               kHpWarps * 32, 0, st>>>(nodes, n_dev, n_host, status, alias, is_load,
                                                                       table, region, out, nullptr);
        else
            k_move_hash_rb<RB, CH, false, 2><<<std::max<int>(1, int(std::min<uint64_t>((groups + kHpWarps - 1) / kHpWarps,
                                                                              uint64_t(c.sm_count)))),
                                               kHpWarps * 32, 0, st>>>(nodes, n_dev, n_host, status, alias, is_load,
                                                                       table, region, nullptr, nullptr);
        FDG_CUDA(cudaGetLastError());
        return FDG_OK;
    }
    const int per_sm = g_hash_ctas_per_sm > 0 ? int(g_hash_ctas_per_sm) : HashRbShape<CH>::MINB;
    const int blocks = int(std::max<uint64_t>(1, std::min<uint64_t>((groups + kHpWarps - 1) / kHpWarps,
                                                                   uint64_t(c.sm_count) * per_sm)));
    if (checksum)
        k_move_hash_rb<RB, CH><<<blocks, kHpWarps * 32, smem, st>>>(nodes, n_dev, n_host, status, alias, is_load,
                                                                   table, region, out, checksum);
    else  // the same row-group move without the hash (option bm_move_impl 2)
        k_move_hash_rb<RB, CH, false><<<blocks, kHpWarps * 32, 0, st>>>(nodes, n_dev, n_host, status, alias,
                                                                       is_load, table, region, out, nullptr);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

template <int RB, int CH, bool SHARDED, bool ALIAS>
int launch_hash_rb_one(int blocks, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                       const uint32_t* status, const TableRef& t, char* out, uint64_t* checksum, uint32_t* ctr) {
    constexpr int smem = kHpWarps * 32 * HashRbShape<CH>::STRIDE;
    static PerDeviceOnce attr;
    if (attr.first()) {
        FDG_CUDA(cudaFuncSetAttribute(k_gather_hash_rb<RB, CH, SHARDED, ALIAS>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        FDG_CUDA(cudaFuncSetAttribute(k_gather_hash_rb<RB, CH, SHARDED, ALIAS, true, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    if (ctr)
        k_gather_hash_rb<RB, CH, SHARDED, ALIAS, true, true><<<blocks, kHpWarps * 32, smem, st>>>(
            nodes, n_dev, n_host, status, t, out, checksum, ctr);
    else
        k_gather_hash_rb<RB, CH, SHARDED, ALIAS><<<blocks, kHpWarps * 32, smem, st>>>(nodes, n_dev, n_host, status, t,
                                                                                       out, checksum);
    return FDG_OK;
}

// Row sizes with a compile-time instantiation of k_gather_hash_rb (the bench and
// BASELINE shapes: 100/128/256 x f32, 768 x f16, 768 x f32, plus 64 x f32).
// Returns -1 when the row size has no instantiation (the caller falls back).
template <bool SHARDED, bool ALIAS>
int launch_hash_rb(const Ctx& c, cudaStream_t st, uint64_t groups, const uint64_t* nodes, const uint32_t* n_dev,
                    uint64_t n_host, const uint32_t* status, const TableRef& t, char* out, uint64_t* checksum) {
    const int ch = g_hash_chunk ? int(g_hash_chunk) : (c.row_bytes >= 256 ? 256 : 128);
    const int minb = ch == 128 ? HashRbShape<128>::MINB : HashRbShape<256>::MINB;
    // rows that are not a multiple of 128 bytes (products: 400) leave lanes idle in the last
    // chunk: two CTAs per SM there (products with checksum 191.5 -> 189.6 us per batch)
    const int per_sm = g_hash_ctas_per_sm > 0 ? int(g_hash_ctas_per_sm) + (c.row_bytes % 128 ? 1 : 0) : minb;
    const uint64_t cap = g_hash_ctas > 0 ? uint64_t(g_hash_ctas) : uint64_t(c.sm_count) * per_sm;
    const int blocks = int(std::min<uint64_t>((groups + kHpWarps - 1) / kHpWarps, cap));
    uint32_t* ctr = g_hash_dyn ? dyn_counter(c) : nullptr;
#define FDG_HRB(R)                                                                                      \
    case R:                                                                                             \
        if (ch == 256)                                                                                  \
            FDG_TRY((launch_hash_rb_one<R, 256, SHARDED, ALIAS>(blocks, st, nodes, n_dev, n_host, status, t, out, \
                                                               checksum, ctr)));                             \
        else                                                                                            \
            FDG_TRY((launch_hash_rb_one<R, 128, SHARDED, ALIAS>(blocks, st, nodes, n_dev, n_host, status, t, out, \
                                                               checksum, ctr)));                             \
        return FDG_OK;
    switch (c.row_bytes) {
        FDG_HRB(256)
        FDG_HRB(400)
        FDG_HRB(512)
        FDG_HRB(1024)
        FDG_HRB(1536)
        FDG_HRB(3072)
        default:
            return -1;
    }
#undef FDG_HRB
}

// Dynamically scheduled row-group gather (FDG_GATHER_RB_DYN): warps claim 32-row groups
// from a per-launch counter (claimed one group ahead, so the next group's node ids and first
// loads are in flight while the current group drains), 256-byte row chunks, 16 loads in
// flight per lane. The row-group layout reads each row's chunks back to back (166 vs 203 us
// for the chunk-striped gather in isolation); dynamic claiming lets CTAs that become resident
// late take less work next to the samplers' kernels.
template <int RB, bool SHARDED, bool PF64, int CH = 256>
__global__ void __launch_bounds__(256) k_gather_rb_dyn(const uint64_t* __restrict__ nodes, const uint32_t* n_dev,
                                                       uint64_t n_host, const uint32_t* status, TableRef t,
                                                       char* __restrict__ out, uint32_t* ctr) {
    using S = HashRbShape<CH>;
    constexpr int NCH = (RB + CH - 1) / CH;
    constexpr int LASTP = (RB - (NCH - 1) * CH) / 16;
    constexpr bool EVEN = RB % CH == 0;
    const bool skip = status && *status;
    const uint64_t n = skip ? 0 : (n_dev ? *n_dev : n_host);
    const uint32_t full = uint32_t(n / 32), total = full + (n % 32 ? 1u : 0u);
    const int lane = threadIdx.x & 31;
    const uint32_t part = lane % S::LPR, rsub = lane / S::LPR;
    const uint64_t pol = gather_policy_ld(t.evict_first), pol_st = gather_policy_st(t.evict_first);
    auto claim = [&]() -> uint32_t {
        uint32_t g = 0;
        if (lane == 0) g = atomicAdd(ctr, 1u);
        return __shfl_sync(0xffffffffu, g, 0);
    };
    auto node_of = [&](uint32_t g) -> uint64_t {
        const uint64_t r = uint64_t(g) * 32 + lane;
        return (g < total && r < n) ? __ldg(nodes + r) : 0;
    };
    const char* src[S::NI];
    uint4 v[S::NI];
    auto setup = [&](uint64_t node_reg) {
#pragma unroll
        for (int k = 0; k < S::NI; ++k) {
            const uint64_t node = __shfl_sync(0xffffffffu, node_reg, k * S::RPI + int(rsub));
            src[k] = row_ptr<SHARDED>(t, node) + part * 16;
        }
    };
    auto issue = [&](int c) {
#pragma unroll
        for (int k = 0; k < S::NI; ++k)
            if (EVEN || c + 1 < NCH || int(part) < LASTP)
                v[k] = ldg_row<PF64>(reinterpret_cast<const uint4*>(src[k] + c * CH), pol);
    };
    uint32_t g = claim();
    uint64_t cur_node = node_of(g);
    uint32_t gn = g < total ? claim() : total;
    uint64_t nxt_node = node_of(gn);
    if (g < full) {
        setup(cur_node);
        issue(0);
    }
    while (g < total) {
        if (g < full) {
            char* dst = out + (uint64_t(g) * 32 + rsub) * RB + part * 16;
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) {
                const bool lastc = c + 1 == NCH;
#pragma unroll
                for (int k = 0; k < S::NI; ++k)
                    if (EVEN || !lastc || int(part) < LASTP)
                        stg_stream(reinterpret_cast<uint4*>(dst + k * S::RPI * RB + c * CH), v[k], pol_st);
                if (!lastc) {
                    issue(c + 1);
                } else if (gn < full) {  // the next (already claimed) group's first chunk
                    setup(nxt_node);
                    issue(0);
                }
            }
        } else {  // the ragged last group (n % 32 rows)
            const uint32_t rows = uint32_t(n - uint64_t(g) * 32);
            for (int c = 0; c < NCH; ++c) {
                const int parts = c + 1 < NCH ? S::NI : LASTP;
#pragma unroll
                for (int k = 0; k < S::NI; ++k) {
                    const uint32_t r = k * S::RPI + rsub;
                    const uint64_t node = __shfl_sync(0xffffffffu, cur_node, int(r));
                    if (r < rows && int(part) < parts) {
                        const uint4 w = ldg_row<PF64>(
                            reinterpret_cast<const uint4*>(row_ptr<SHARDED>(t, node) + c * CH) + part, pol);
                        stg_stream(reinterpret_cast<uint4*>(out + (uint64_t(g) * 32 + r) * RB + c * CH) + part, w,
                                   pol_st);
                    }
                }
            }
            if (gn < full) {
                setup(nxt_node);
                issue(0);
            }
        }
        g = gn;
        cur_node = nxt_node;
        gn = g < total ? claim() : total;
        nxt_node = node_of(gn);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // every CTA has claimed past the end
            ctr[0] = 0;
            ctr[1] = 0;
            __threadfence();
        }
    }
}

template <bool SHARDED, bool PF64>
int launch_gather_rb_dyn(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                         const uint32_t* status, const TableRef& t, char* out, uint32_t* ctr, int blocks) {
#define FDG_GRD(R)                                                                                            \
    case R:                                                                                                   \
        if (g_rb_chunk == 128)                                                                                \
            k_gather_rb_dyn<R, SHARDED, PF64, 128><<<blocks, 256, 0, st>>>(nodes, n_dev, n_host, status, t, out, \
                                                                           ctr);                              \
        else                                                                                                  \
            k_gather_rb_dyn<R, SHARDED, PF64><<<blocks, 256, 0, st>>>(nodes, n_dev, n_host, status, t, out, ctr); \
        return FDG_OK;
    switch (c.row_bytes) {
        FDG_GRD(400)
        FDG_GRD(512)
        FDG_GRD(1024)
        FDG_GRD(1536)
        FDG_GRD(3072)
        default:
            return -1;
    }
#undef FDG_GRD
}

constexpr int kHashWarps = 4;

__host__ __device__ __forceinline__ uint32_t hash_stride(uint32_t rb) {
    uint32_t s = (rb + 7) & ~7u;
    return ((s >> 3) & 1) ? s : s + 8;
}

__device__ __forceinline__ uint64_t hash_row_smem(const char* row, uint32_t n) {
    uint64_t h = 0x27d4eb2f165667c5ull ^ (uint64_t(n) * 0x9e3779b97f4a7c15ull);
    uint32_t full = n >> 3;
    const uint2* p = reinterpret_cast<const uint2*>(row);
    for (uint32_t s = 0; s < full; ++s) {
        uint2 w = p[s];
        h = splitmix64(h ^ (uint64_t(w.y) << 32 | w.x));
    }
    uint32_t rem = n & 7;
    if (rem) {  // rows are 4-byte multiples: a 4-byte tail lane
        uint64_t lane = reinterpret_cast<const uint32_t*>(row + (full << 3))[0];
        h = splitmix64(h ^ lane ^ (uint64_t(rem) << 56));
    }
    return splitmix64(h);
}

// Gather + trainer checksum. Rows are staged per warp in shared memory with a
// stride (hash_stride) that is 8-byte aligned and an odd number of 8-byte words, so
// the per-lane 8-byte hash reads of 16 lanes hit 16 distinct bank pairs.
// ALIAS: rows are FeatureRegion slots addressed by the alias list (t.base = region,
// `nodes` holds the i64 aliases) -- trainer_step's region.slot(alias[i]) read.
template <bool SHARDED, bool ALIAS = false>
__global__ void __launch_bounds__(kHashWarps * 32) k_gather_hash(const uint64_t* __restrict__ nodes,
                                                                 const uint32_t* n_dev, uint64_t n_host,
                                                                 const uint32_t* status, TableRef t,
                                                                 char* __restrict__ out, uint64_t* checksum) {
    extern __shared__ __align__(16) char smem[];
    if (status && *status) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rb = t.row_bytes;
    const uint32_t stride = hash_stride(rb);
    char* wbuf = smem + size_t(warp) * 32 * stride;
    const uint64_t n = n_dev ? *n_dev : n_host;
    const uint64_t groups = (n + 31) / 32;
    const uint32_t words = rb >> 2;  // 4-byte words per row
    uint64_t sum = 0;
    for (uint64_t g = blockIdx.x * uint64_t(kHashWarps) + warp; g < groups; g += uint64_t(gridDim.x) * kHashWarps) {
        const uint64_t r0 = g * 32;
        const uint32_t rows = uint32_t(n - r0 < 32 ? n - r0 : 32);
        uint64_t my_node = lane < rows ? nodes[r0 + lane] : 0;
        for (uint32_t r = 0; r < rows; ++r) {
            uint64_t node = __shfl_sync(0xffffffffu, my_node, r);
            const uint32_t* src = reinterpret_cast<const uint32_t*>(ALIAS ? t.base + node * rb : row_ptr<SHARDED>(t, node));
            uint32_t* sm = reinterpret_cast<uint32_t*>(wbuf + r * stride);
            if (out) {
                uint32_t* dst = reinterpret_cast<uint32_t*>(out + (r0 + r) * rb);
                for (uint32_t w = lane; w < words; w += 32) {
                    uint32_t v = __ldg(src + w);
                    dst[w] = v;
                    sm[w] = v;
                }
            } else {
                for (uint32_t w = lane; w < words; w += 32) sm[w] = __ldg(src + w);
            }
        }
        __syncwarp();
        if (lane < rows) sum += hash_row_smem(wbuf + lane * stride, rb);
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0 && sum) atomicAdd(reinterpret_cast<unsigned long long*>(checksum), (unsigned long long)sum);
}

TableRef table_ref(const Ctx& c) {
    TableRef t;
    t.base = c.shard_bases.empty() ? nullptr : static_cast<const char*>(c.shard_bases[0]);
    t.shards = reinterpret_cast<const char* const*>(c.shard_table);
    t.rows_per_shard = c.rows_per_shard;
    t.n_shards = c.n_shards;
    t.row_bytes = c.row_bytes;
    t.evict_first = g_gather_evict_first;
    t.pf64 = g_gather_pf64 == 1 || (g_gather_pf64 == 2 && c.row_bytes % 128 != 0);
    t.sdiv_ok = c.rows_per_shard > 0 && c.rows_per_shard < 0x80000000ull;
    if (t.sdiv_ok) t.sdiv.init(uint32_t(c.rows_per_shard));
    return t;
}

}  // namespace

// Standalone gathers (fdg_gather) default to the dynamically scheduled row-group kernel:
// 155 us per Papers batch vs 166 (static row groups), 206 (chunk-striped LDG) and 203 (TMA
// bulk); it also resolves shards once per row group (2 local shards: 157 vs 329 us).
// Inside the pipeline the chunk-striped dynamic LDG kernel is faster next to the samplers
// (199 vs 222 us per batch), so the runner has its own choice.
int g_gather_impl = FDG_GATHER_RB_DYN;
int64_t g_pipeline_gather_impl = FDG_GATHER_LDG;
// L2 evict-first on the gather stream: helped the gather in isolation in an earlier version
// (177 vs 186 us), but with the current samplers (evict-last hash tables) the pipeline is
// faster without it: Papers 199 vs 206 us per batch, Friendster 330 vs 338, extraction
// alone 154 vs 159 (scripts/sweep_overlap.sh). Off by default.
int g_gather_evict_first = 0;
// 64-byte L2 fetches on table reads: 0 off, 1 on, 2 (default) rows not a multiple of 128 B.
// products (400-byte rows): extraction 133 -> 128 us, pipeline 192 -> 188 us per batch.
int64_t g_gather_pf64 = 2;
int g_gather_ctas_per_sm = 1;
int64_t g_rb_ctas_per_sm = 2;  // row-group plain gather: CTAs (8 warps) per SM per launch
int64_t g_rb_chunk = 256;      // row-group plain gather: 128- or 256-byte row chunks
// Fused gather + trainer checksum on the LDG engine: k_gather_hash_rb (compile-time row size,
// 256-byte chunks) for the benchmarked row sizes, k_gather_hash_pipe for other 16-byte
// multiples, k_gather_hash for the rest. Papers batch extraction with checksum 155 us vs
// 242 us for TMA + per-warp hashing (the round-1 default), Friendster 312 vs 636 us
// (scripts/ab_checksum.sh). Round 2 removed the striped and warp-specialised variants that
// never won an A/B (profiles/README.md, decisions).
// Fused gather + checksum: row groups claimed from a per-launch counter (1) or a static stride (0).
int64_t g_hash_dyn = 0;
// Fused gather + checksum CTAs per SM (0: the kernel's min-blocks, 2). At 124 registers x 256
// threads, two CTAs hold 97 % of an SM's register file, so nothing else (the samplers, the MT
// prefetch) fits beside them. One per SM: Papers pipeline with checksum 201.3 vs 204.0 us per
// batch (products and Friendster unchanged; alone 156 vs 152 us).
int64_t g_hash_ctas_per_sm = 1;
int64_t g_hash_ctas = 0;  // option: an absolute CTA count for the fused gather + checksum (0: per SM)
int64_t g_hash_chunk = 0;  // 0: 256-byte chunks for rows >= 256 B, else 128; or force 128 / 256
int64_t g_checksum_impl = FDG_GATHER_LDG;

namespace {
// Gather + checksum: the compile-time row-size kernel, else the pipelined one, else generic.
int launch_checksum(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                    uint64_t n_bound, const uint32_t* status, const TableRef& t, char* out, uint64_t* checksum,
                    bool sharded, bool alias) {
    const uint64_t groups = (std::max<uint64_t>(n_bound, 1) + 31) / 32;
    if (c.row_bytes % 16 == 0) {
        const int rc = alias ? launch_hash_rb<false, true>(c, st, groups, nodes, n_dev, n_host, status, t, out, checksum)
                       : sharded ? launch_hash_rb<true, false>(c, st, groups, nodes, n_dev, n_host, status, t, out,
                                                               checksum)
                                 : launch_hash_rb<false, false>(c, st, groups, nodes, n_dev, n_host, status, t, out,
                                                                checksum);
        if (rc > 0) return rc;
        if (rc < 0) {  // no compile-time instantiation for this row size
            const int pb =
                int(std::min<uint64_t>((groups + kHpWarps - 1) / kHpWarps, uint64_t(c.sm_count) * kHpMinBlocks));
            if (alias)
                k_gather_hash_pipe<false, true><<<pb, kHpWarps * 32, 0, st>>>(nodes, n_dev, n_host, status, t, nullptr,
                                                                             checksum);
            else if (sharded)
                k_gather_hash_pipe<true, false><<<pb, kHpWarps * 32, 0, st>>>(nodes, n_dev, n_host, status, t, out,
                                                                             checksum);
            else
                k_gather_hash_pipe<false, false><<<pb, kHpWarps * 32, 0, st>>>(nodes, n_dev, n_host, status, t, out,
                                                                              checksum);
        }
        FDG_CUDA(cudaGetLastError());
        return FDG_OK;
    }
    const size_t smem = size_t(kHashWarps) * 32 * hash_stride(c.row_bytes);
    if (smem > 200 * 1024) return fail(FDG_INVALID_ARG, "gather: row too large for the fused checksum");
    static PerDeviceOnce attr_set[3];
    auto kfn = alias ? k_gather_hash<false, true> : sharded ? k_gather_hash<true> : k_gather_hash<false>;
    const int which = alias ? 2 : int(sharded);
    if (attr_set[which].first())
        FDG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    const int blocks = int(std::min<uint64_t>((groups + kHashWarps - 1) / kHashWarps, uint64_t(c.sm_count) * 8));
    kfn<<<blocks, kHashWarps * 32, smem, st>>>(nodes, n_dev, n_host, status, t, out, checksum);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}
}  // namespace

// Buffer-manager row move + trainer checksum in one pass (k_move_hash_rb) for the compiled row
// sizes; returns -1 when the row size has none (the caller moves and hashes separately).
int launch_move_hash(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                     const uint32_t* status, const int64_t* alias, const uint8_t* is_load, const char* table,
                     char* region, char* out, uint64_t* checksum, int mode) {
    const uint64_t groups = (std::max<uint64_t>(n_host, 1) + 31) / 32;
    switch (c.row_bytes) {
        case 512:
            return launch_move_hash_one<512, 256>(c, st, groups, nodes, n_dev, n_host, status, alias, is_load, table,
                                                  region, out, checksum, mode);
        case 400:
            return launch_move_hash_one<400, 256>(c, st, groups, nodes, n_dev, n_host, status, alias, is_load, table,
                                                  region, out, checksum, mode);
        case 1024:
            return launch_move_hash_one<1024, 256>(c, st, groups, nodes, n_dev, n_host, status, alias, is_load, table,
                                                   region, out, checksum, mode);
        default:
            return -1;
    }
}

int launch_gather_bound(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev,
                        uint64_t n_host, uint64_t n_bound, void* out, uint64_t* checksum, const uint32_t* status,
                        bool pipeline) {
    if (c.row_bytes == 0 || c.shard_bases.empty()) return fail(FDG_NOT_LOADED, "gather: no feature table loaded");
    TableRef t = table_ref(c);
    const bool sharded = c.n_shards > 1;
    if (n_bound == 0) return FDG_OK;
    int impl = (checksum && g_checksum_impl >= 0) ? int(g_checksum_impl)
               : pipeline                             ? int(g_pipeline_gather_impl)
                                                      : g_gather_impl;
    if (sharded && impl == FDG_GATHER_LDG && !checksum) impl = FDG_GATHER_RB_DYN;  // shard once per row group
    if (impl == FDG_GATHER_TMA && out &&
        launch_gather_tma(c, st, nodes, n_dev, n_host, out, checksum, status) == FDG_OK)
        return FDG_OK;  // rows that do not suit the TMA path fall through to the LDG kernels
    if (checksum)
        return launch_checksum(c, st, nodes, n_dev, n_host, n_bound, status, t, static_cast<char*>(out), checksum,
                               sharded, false);
    if (impl == FDG_GATHER_RB_DYN && out) {
        uint32_t* ctr = dyn_counter(c);
        if (!ctr) return fail(FDG_NOT_LOADED, "gather: context has no work-claim counters");
        const uint64_t groups = (n_bound + 31) / 32;
        const int blocks = int(std::max<uint64_t>(1, std::min<uint64_t>((groups + 7) / 8,
                                                                      uint64_t(c.sm_count) * g_rb_ctas_per_sm)));
        int rc;
        if (sharded)
            rc = launch_gather_rb_dyn<true, false>(c, st, nodes, n_dev, n_host, status, t, static_cast<char*>(out),
                                                   ctr, blocks);
        else if (t.pf64)
            rc = launch_gather_rb_dyn<false, true>(c, st, nodes, n_dev, n_host, status, t, static_cast<char*>(out),
                                                   ctr, blocks);
        else
            rc = launch_gather_rb_dyn<false, false>(c, st, nodes, n_dev, n_host, status, t, static_cast<char*>(out),
                                                    ctr, blocks);
        if (rc == FDG_OK) {
            FDG_CUDA(cudaGetLastError());
            return FDG_OK;
        }
    }
    if (c.row_bytes % 16 == 0) {  // chunk-striped 16-byte gather, work claimed dynamically
        uint32_t cpr = c.row_bytes / 16;
        if (n_bound * cpr >= (1ull << 32)) return fail(FDG_INVALID_ARG, "gather: batch too large");
        FastDiv d;
        d.init(cpr);
        uint64_t total = n_bound * cpr;
        int blocks = int(std::min<uint64_t>((total + 511) / 512, uint64_t(c.sm_count) * g_gather_ctas_per_sm));
        uint32_t* ctr = dyn_counter(c);
        if (!ctr) return fail(FDG_NOT_LOADED, "gather: context has no work-claim counters");
        if (sharded)
            k_gather16_dyn<true><<<blocks, 512, 0, st>>>(nodes, n_dev, n_host, status, t, d, cpr,
                                                         static_cast<uint4*>(out), ctr);
        else if (t.pf64)
            k_gather16_dyn<false, true><<<blocks, 512, 0, st>>>(nodes, n_dev, n_host, status, t, d, cpr,
                                                                static_cast<uint4*>(out), ctr);
        else
            k_gather16_dyn<false><<<blocks, 512, 0, st>>>(nodes, n_dev, n_host, status, t, d, cpr,
                                                          static_cast<uint4*>(out), ctr);
    } else {
        uint32_t cpr = c.row_bytes / 4;
        FastDiv d;
        d.init(cpr);
        uint64_t total = n_bound * cpr;
        int blocks = int(std::min<uint64_t>((total + 255) / 256, uint64_t(c.sm_count) * 8));
        if (sharded)
            k_gather4<true><<<blocks, 256, 0, st>>>(nodes, n_dev, n_host, status, t, d, cpr, static_cast<uint32_t*>(out));
        else
            k_gather4<false><<<blocks, 256, 0, st>>>(nodes, n_dev, n_host, status, t, d, cpr, static_cast<uint32_t*>(out));
    }
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int launch_gather(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                  void* out, uint64_t* checksum) {
    uint64_t bound = n_dev ? std::max<uint64_t>(n_host, 1) : n_host;
    return launch_gather_bound(c, st, nodes, n_dev, n_host, bound, out, checksum, nullptr, false);
}

int launch_checksum_alias(const Ctx& c, cudaStream_t st, const void* region, const int64_t* alias,
                          const uint32_t* n_dev, uint64_t n_host, uint64_t* checksum, const uint32_t* status) {
    if (c.row_bytes == 0) return fail(FDG_NOT_LOADED, "checksum: no feature table loaded");
    if (!checksum) return fail(FDG_INVALID_ARG, "checksum: null output");
    TableRef t = table_ref(c);
    t.base = static_cast<const char*>(region);
    return launch_checksum(c, st, reinterpret_cast<const uint64_t*>(alias), n_dev, n_host, n_host, status, t, nullptr,
                           checksum, false, true);
}

}  // namespace fdg

namespace {
// Byte compare of region[alias[i]] with table[nodes[i]] (trainer_step's verify against the
// synchronous read oracle, pipeline.hpp:110-121): the smallest mismatching i -> *first_bad.
__global__ void __launch_bounds__(256) k_verify_rows(const char* region, const int64_t* alias, const uint64_t* nodes,
                                                     uint64_t n, const char* table, uint32_t rb,
                                                     unsigned long long* first_bad) {
    const uint32_t cpr = rb / 4;
    for (uint64_t c = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; c < n * cpr;
         c += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = c / cpr, k = c % cpr;
        if (reinterpret_cast<const uint32_t*>(region + uint64_t(alias[i]) * rb)[k] !=
            reinterpret_cast<const uint32_t*>(table + nodes[i] * rb)[k])
            atomicMin(first_bad, (unsigned long long)i);
    }
}
}  // namespace

extern "C" {

int fdg_region_checksum(void* stream, const void* region_dev, uint32_t row_bytes, const int64_t* alias_dev, uint64_t n,
                        uint64_t* checksum_dev) {
    fdg::Ctx c;
    int dev = 0;
    FDG_CUDA(cudaGetDevice(&dev));
    c.device = dev;
    FDG_CUDA(cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, dev));
    c.row_bytes = row_bytes;
    c.n_shards = 1;
    return fdg::launch_checksum_alias(c, (cudaStream_t)stream, region_dev, alias_dev, nullptr, n, checksum_dev);
}

int fdg_region_verify(const fdg_ctx* table, void* stream, const void* region_dev, const int64_t* alias_dev,
                      const uint64_t* nodes_dev, uint64_t n, uint64_t* first_bad_dev) {
    if (table->shard_bases.empty() || table->n_shards != 1)
        return fdg::fail(FDG_NOT_LOADED, "region_verify: no single-shard feature table");
    if (table->row_bytes % 4) return fdg::fail(FDG_INVALID_ARG, "region_verify: row_bytes must be a multiple of 4");
    FDG_CUDA(cudaMemsetAsync(first_bad_dev, 0xFF, 8, (cudaStream_t)stream));
    if (n == 0) return FDG_OK;
    const uint64_t chunks = n * (table->row_bytes / 4);
    const int blocks = int(std::max<uint64_t>(1, std::min<uint64_t>((chunks + 255) / 256, uint64_t(table->sm_count) * 8)));
    k_verify_rows<<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<const char*>(region_dev), alias_dev, nodes_dev,
                                                            n, static_cast<const char*>(table->shard_bases[0]),
                                                            table->row_bytes,
                                                            reinterpret_cast<unsigned long long*>(first_bad_dev));
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

}  // extern "C"
