// fdg_gather_tma.cu -- the mini-batch gather on the Tensor Memory Accelerator.
//
// X[i, :] = row(nodes[i]) (extraction's byte movement, extractor.hpp:374-386 ->
// the trainer's region reads, pipeline.hpp:103-124) moved by cp.async.bulk:
// each row is one 1-D bulk copy global -> shared (completing on an mbarrier
// with its byte count), then one bulk copy shared -> global into X. One CTA of
// 4 warps per SM; each warp runs its own D-stage ring with A chunks of loads in
// flight, so an SM keeps ~100 KB of rows in flight with 128 threads and a few
// dozen registers -- the rest of the SM stays free for the next batch's
// sampling kernels, which run concurrently on other streams.
//
// With HASH the warp also folds trainer_step's checksum (sum of hash_bytes64
// over rows, common.hpp:88-105) from the staged rows: one lane per row, 16-byte
// shared loads over a row stride of row_bytes + 16 (conflict-free).
#include <algorithm>

#include "fdg_internal.cuh"
#include "fdg_tma.cuh"

namespace fdg {
namespace {

constexpr int kTmaWarps = 4;
using namespace tma;

// L2 evict-first on both directions: the gather stream must not flush the
// samplers' hash tables / CSR lines out of L2.
__device__ __forceinline__ uint64_t gather_policy(bool evict_first) {
    uint64_t pol;
    if (evict_first)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_stream(uint4* p, uint4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t hash_row16(const char* row, uint32_t n) {
    uint64_t h = 0x27d4eb2f165667c5ull ^ (uint64_t(n) * 0x9e3779b97f4a7c15ull);
    const uint4* p = reinterpret_cast<const uint4*>(row);
    for (uint32_t s = 0; s < (n >> 4); ++s) {
        uint4 v = p[s];
        h = splitmix64(h ^ (uint64_t(v.y) << 32 | v.x));
        h = splitmix64(h ^ (uint64_t(v.w) << 32 | v.z));
    }
    return splitmix64(h);
}

template <bool HASH, int D, int A>
__global__ void __launch_bounds__(kTmaWarps * 32, 1)
    k_gather_tma(const uint64_t* __restrict__ nodes, const uint32_t* n_dev, uint64_t n_host, const uint32_t* status,
                 const char* __restrict__ table, uint32_t rb, uint32_t RS, char* __restrict__ out, uint64_t* checksum,
                 int evict_first) {
    static_assert(A < D, "lookahead must leave a stage for the store in flight");
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t bars[kTmaWarps][D];
    if (status && *status) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rstride = rb + 16;
    const uint32_t stage_bytes = RS * rstride;
    const uint64_t pol = gather_policy(evict_first);
    char* wbase = smem + size_t(warp) * D * stage_bytes;
    const uint64_t n = n_dev ? *n_dev : n_host;
    const uint64_t nchunks = (n + RS - 1) / RS;
    const uint64_t gw = uint64_t(blockIdx.x) * kTmaWarps + warp, nw = uint64_t(gridDim.x) * kTmaWarps;
    const uint64_t my_n = gw < nchunks ? (nchunks - gw + nw - 1) / nw : 0;
    if (lane == 0)
        for (int d = 0; d < D; ++d) mbar_init(smem_u32(&bars[warp][d]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    auto row_of = [&](uint64_t i) { return (gw + i * nw) * RS + lane; };
    auto load_id = [&](uint64_t i) -> uint64_t {
        uint64_t r = row_of(i);
        return (i < my_n && lane < int(RS) && r < n) ? __ldg(nodes + r) : 0;
    };
    auto issue = [&](uint64_t i, uint64_t node) {
        const uint64_t row0 = (gw + i * nw) * RS;
        const uint32_t rows = uint32_t(n - row0 < RS ? n - row0 : RS);
        const int s = int(i % D);
        const uint32_t bar = smem_u32(&bars[warp][s]);
        if (lane == 0) mbar_arrive_expect_tx(bar, rows * rb);
        __syncwarp();
        if (lane < int(rows))
            bulk_load(smem_u32(wbase + s * stage_bytes + lane * rstride), table + node * rb, rb, bar, pol);
    };

    for (int i = 0; i < A; ++i)
        if (uint64_t(i) < my_n) issue(i, load_id(i));
    uint64_t id_a = load_id(A), id_b = load_id(A + 1);  // node ids two chunks ahead of issue
    uint64_t sum = 0;
    for (uint64_t i = 0; i < my_n; ++i) {
        const int s = int(i % D);
        const uint64_t row0 = (gw + i * nw) * RS;
        const uint32_t rows = uint32_t(n - row0 < RS ? n - row0 : RS);
        mbar_wait(smem_u32(&bars[warp][s]), uint32_t((i / D) & 1));
        const char* srow = wbase + s * stage_bytes + lane * rstride;
        if (lane < int(rows)) {
            if (HASH) sum += hash_row16(srow, rb);
            bulk_store(out + (row0 + lane) * rb, smem_u32(srow), rb, pol);
        }
        bulk_commit();
        const uint64_t j = i + A;
        if (j < my_n) {
            bulk_wait_read<D - A>();  // the store that last read stage j % D has drained
            issue(j, id_a);
            id_a = id_b;
            id_b = load_id(j + 2);
        }
    }
    bulk_wait_all();
    if (HASH) {
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0 && sum) atomicAdd(reinterpret_cast<unsigned long long*>(checksum), (unsigned long long)sum);
    }
}

constexpr int kDh = 3, kAh = 2;   // fused checksum: 32-row stages for one-row-per-lane hashing
constexpr size_t kSmemBudget = 200 * 1024;
constexpr size_t kSmemMax = 227 * 1024;

}  // namespace

// Returns FDG_OK if launched, FDG_INVALID_ARG if the shape does not suit the TMA path.
int launch_gather_tma(const Ctx& c, cudaStream_t st, const uint64_t* nodes, const uint32_t* n_dev, uint64_t n_host,
                      void* out, uint64_t* checksum, const uint32_t* status) {
    const uint32_t rb = c.row_bytes;
    if (rb % 16 || c.n_shards != 1 || rb > 8192) return FDG_INVALID_ARG;
    // plain-gather ring shapes (option tma_cfg): {stages, chunks in flight, row cap per stage, smem}
    struct Cfg { int D, A; uint32_t rs_cap; size_t budget; };
    static const Cfg cfgs[4] = {{8, 6, 0, kSmemBudget}, {8, 7, 16, kSmemMax}, {12, 10, 16, kSmemMax},
                                {16, 14, 16, kSmemMax}};
    const Cfg cf = checksum ? Cfg{kDh, kAh, 32, kSmemBudget} : cfgs[std::min<int64_t>(std::max<int64_t>(g_tma_cfg, 0), 3)];
    const int D = cf.D;
    uint32_t rs_cap = cf.rs_cap ? cf.rs_cap : std::max<uint32_t>(1, 4096 / rb);
    uint32_t RS = uint32_t(std::min<size_t>(rs_cap, cf.budget / (size_t(kTmaWarps) * D * (rb + 16))));
    if (RS == 0) return FDG_INVALID_ARG;
    const size_t smem = size_t(kTmaWarps) * D * RS * (rb + 16);
    using KFn = void (*)(const uint64_t*, const uint32_t*, uint64_t, const uint32_t*, const char*, uint32_t, uint32_t,
                         char*, uint64_t*, int);
    KFn kfn = checksum          ? KFn(k_gather_tma<true, kDh, kAh>)
              : cf.D == 8 && cf.A == 6 ? KFn(k_gather_tma<false, 8, 6>)
              : cf.D == 8          ? KFn(k_gather_tma<false, 8, 7>)
              : cf.D == 12         ? KFn(k_gather_tma<false, 12, 10>)
                                   : KFn(k_gather_tma<false, 16, 14>);
    FDG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kfn<<<c.sm_count, kTmaWarps * 32, smem, st>>>(nodes, n_dev, n_host, status,
                                                   static_cast<const char*>(c.shard_bases[0]), rb, RS,
                                                   static_cast<char*>(out), checksum, g_gather_evict_first);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int64_t g_tma_cfg = 0;  // plain TMA gather ring shape (launch_gather_tma)
}  // namespace fdg
