// fdg_generate.cu -- bit-exact GPU port of the reference's synthetic dataset
// (storage/generator.hpp:65-121), so Papers100M / Friendster / MAG240M-shaped
// inputs are built directly in HBM instead of shipping 57-750 GB files.
//
// Every quantity is counter-based per node (SplitMix keyed by hash_combine), so
// rows and neighbor lists are generated independently. Floating point is IEEE
// round-to-nearest on both sides: double sqrt and divide (generator.hpp:92),
// double(x>>11)*2^-53 (common.hpp:121) and float(int32)*2^-31 (generator.hpp:72-73);
// no FMA-contractible expression appears.
#include <cub/device/device_scan.cuh>
#include <cuda_fp16.h>

#include "fdg_internal.cuh"

namespace fdg {
namespace {

constexpr uint64_t kRowTag = 0x726f77;  // "row"
constexpr uint64_t kDegTag = 0x646567;  // "deg"
constexpr uint64_t kNbrTag = 0x6e6272;  // "nbr"
constexpr uint32_t kMaxGenDegree = 512;  // 4 * avg_degree limit of the warp kernel
constexpr int kGenWarps = 4;

// generator.hpp:85-96
__device__ __forceinline__ uint64_t in_degree(uint64_t seed, uint64_t node, uint32_t avg, uint64_t n) {
    if (avg == 0 || n <= 1) return 0;
    uint64_t s = hash_combine(hash_combine(seed, kDegTag), node);
    double u = double(splitmix_at(s, 0) >> 11) * 0x1.0p-53;
    if (u < 1e-12) u = 1e-12;
    double scale = double(avg) / 2.0;
    uint64_t d = uint64_t(__ddiv_rn(scale, __dsqrt_rn(u)));
    uint64_t cap = uint64_t(avg) * 4;
    d = d < cap ? d : cap;
    return d < n - 1 ? d : n - 1;
}

__global__ void k_degrees(uint64_t seed, uint64_t n, uint32_t avg, uint64_t* indptr) {
    for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < n; v += uint64_t(gridDim.x) * blockDim.x)
        indptr[v + 1] = in_degree(seed, v, avg, n);
    if (blockIdx.x == 0 && threadIdx.x == 0) indptr[0] = 0;
}

// generator.hpp:99-121, one warp per node. Floyd's draws t_k = next_below(j_k+1)
// are independent (random-access SplitMix), so the only sequential part is the
// collision chain: with S_k the picks before step k,
//   t_k in S_k  <=>  (exists m<k: t_m == t_k) or (exists m<k: collided_m and j_m == t_k),
// and j_m == t_k pins m = t_k - j_0, so collisions resolve by a short fixpoint
// over a bitmask. remap (self -> N-1) is injective on [0, N-1), so comparing
// pre-remap values equals the reference's value compare. The ascending sort is
// a rank computation over distinct values.
template <typename IdT>
__global__ void __launch_bounds__(kGenWarps * 32) k_neighbors(uint64_t seed, uint64_t n, uint32_t avg,
                                                              const uint64_t* indptr, IdT* indices) {
    __shared__ uint64_t s_t[kGenWarps][kMaxGenDegree];
    __shared__ uint64_t s_p[kGenWarps][kMaxGenDegree];
    __shared__ uint32_t s_c[kGenWarps][kMaxGenDegree / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* T = s_t[warp];
    uint64_t* Pk = s_p[warp];
    uint32_t* Cm = s_c[warp];
    const uint64_t nwarps = uint64_t(gridDim.x) * kGenWarps;
    for (uint64_t v = blockIdx.x * uint64_t(kGenWarps) + warp; v < n; v += nwarps) {
        const uint64_t lo = indptr[v];
        const uint32_t d = uint32_t(indptr[v + 1] - lo);
        if (d == 0) continue;
        const uint64_t s = hash_combine(hash_combine(seed, kNbrTag), v);
        const uint64_t pool = n - 1;
        const uint64_t j0 = pool - d;
        for (uint32_t k = lane; k < d; k += 32) T[k] = splitmix_at(s, k) % (j0 + k + 1);
        __syncwarp();
        // A_k: an earlier draw hit the same index
        for (uint32_t w = 0; w < (d + 31) / 32; ++w) {
            uint32_t k = w * 32 + lane;
            bool a = false;
            if (k < d) {
                uint64_t tk = T[k];
                for (uint32_t m = 0; m < k; ++m) a |= (T[m] == tk);
            }
            uint32_t bits = __ballot_sync(0xffffffffu, a);
            if (lane == 0) Cm[w] = bits;
        }
        __syncwarp();
        // fixpoint: collided_k |= collided_{t_k - j0} for t_k - j0 in [0, k)
        for (;;) {
            bool changed = false;
            for (uint32_t w = 0; w < (d + 31) / 32; ++w) {
                uint32_t k = w * 32 + lane;
                bool c = false;
                if (k < d) {
                    c = (Cm[w] >> lane) & 1u;
                    uint64_t tk = T[k];
                    if (!c && tk >= j0 && tk - j0 < k) {
                        uint32_t m = uint32_t(tk - j0);
                        c = (Cm[m >> 5] >> (m & 31)) & 1u;
                    }
                }
                uint32_t bits = __ballot_sync(0xffffffffu, c);
                changed |= bits != Cm[w];
                __syncwarp();
                if (lane == 0) Cm[w] = bits;
                __syncwarp();
            }
            if (!changed) break;
        }
        for (uint32_t k = lane; k < d; k += 32) {
            uint64_t p = ((Cm[k >> 5] >> (k & 31)) & 1u) ? j0 + k : T[k];
            Pk[k] = (p == v) ? n - 1 : p;
        }
        __syncwarp();
        for (uint32_t k = lane; k < d; k += 32) {
            uint64_t pk = Pk[k];
            uint32_t r = 0;
            for (uint32_t m = 0; m < d; ++m) r += Pk[m] < pk;
            indices[lo + r] = IdT(pk);
        }
        __syncwarp();
    }
}

// generator.hpp:65-81, one warp per row, lanes over elements; element i is the
// low (i even) or high (i odd) int32 of SplitMix draw i/2, scaled by 2^-31.
template <typename OutT>
__global__ void k_rows(uint64_t seed, uint64_t first, uint64_t count, uint32_t dim, OutT* out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t base = hash_combine(seed, kRowTag);
    for (uint64_t r = warp; r < count; r += nwarps) {
        const uint64_t s = hash_combine(base, first + r);
        OutT* row = out + r * dim;
        for (uint32_t i = lane; i < dim; i += 32) {
            uint64_t bits = splitmix_at(s, i >> 1);
            int32_t x = int32_t(uint32_t((i & 1) ? (bits >> 32) : (bits & 0xffffffffu)));
            float f = __fmul_rn(__int2float_rn(x), 0x1.0p-31f);
            if constexpr (sizeof(OutT) == 4)
                row[i] = f;
            else
                row[i] = __float2half_rn(f);
        }
    }
}

}  // namespace

int generate_topology(Ctx& c, uint64_t seed, uint64_t n, uint32_t avg) {
    if (n == 0) return fail(FDG_INVALID_ARG, "generate_topology: num_nodes must be >= 1");
    if (uint64_t(avg) * 4 > kMaxGenDegree)
        return fail(FDG_INVALID_ARG, "generate_topology: avg_degree > 128 not supported by the GPU generator");
    cudaStream_t st = c.stream;
    if (c.indptr) cudaFree(c.indptr);
    if (c.indices) cudaFree(c.indices);
    c.indptr = nullptr;
    c.indices = nullptr;
    FDG_CUDA(cudaMalloc(&c.indptr, (n + 1) * sizeof(uint64_t)));
    const int threads = 256;
    int blocks = int(std::min<uint64_t>((n + threads - 1) / threads, uint64_t(c.sm_count) * 32));
    k_degrees<<<blocks, threads, 0, st>>>(seed, n, avg, c.indptr);
    FDG_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    FDG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, c.indptr + 1, c.indptr + 1, int64_t(n), st));
    void* tmp = nullptr;
    FDG_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    FDG_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, c.indptr + 1, c.indptr + 1, int64_t(n), st));
    FDG_CUDA(cudaFreeAsync(tmp, st));
    uint64_t e = 0;
    FDG_CUDA(cudaMemcpyAsync(&e, c.indptr + n, sizeof(e), cudaMemcpyDeviceToHost, st));
    FDG_CUDA(cudaStreamSynchronize(st));
    c.num_nodes = n;
    c.num_edges = e;
    c.idx_bytes = (n <= 0xFFFFFFFFull && !g_force_idx64) ? 4 : 8;
    FDG_CUDA(cudaMalloc(&c.indices, std::max<uint64_t>(e, 1) * c.idx_bytes));
    int gblocks = int(std::min<uint64_t>((n + kGenWarps - 1) / kGenWarps, uint64_t(c.sm_count) * 64));
    if (c.idx_bytes == 4)
        k_neighbors<uint32_t><<<gblocks, kGenWarps * 32, 0, st>>>(seed, n, avg, c.indptr, (uint32_t*)c.indices);
    else
        k_neighbors<uint64_t><<<gblocks, kGenWarps * 32, 0, st>>>(seed, n, avg, c.indptr, (uint64_t*)c.indices);
    FDG_CUDA(cudaGetLastError());
    FDG_CUDA(cudaStreamSynchronize(st));
    return FDG_OK;
}

int generate_feature_shard(Ctx& c, uint64_t seed, uint64_t n, uint32_t dim, uint32_t dtype, uint32_t shard,
                           uint32_t n_shards, void** base) {
    if (n == 0 || dim == 0 || n_shards == 0 || shard >= n_shards)
        return fail(FDG_INVALID_ARG, "generate_feature_shard: bad geometry");
    if (dtype > 1) return fail(FDG_INVALID_ARG, "generate_feature_shard: dtype must be 0 (f32) or 1 (f16)");
    const uint32_t row_bytes = dim * (dtype == 0 ? 4 : 2);
    const uint64_t rps = (n + n_shards - 1) / n_shards;
    const uint64_t first = uint64_t(shard) * rps;
    const uint64_t count = first < n ? std::min<uint64_t>(rps, n - first) : 0;
    void* p = nullptr;
    FDG_CUDA(cudaMalloc(&p, std::max<uint64_t>(count, 1) * row_bytes));
    c.owned_shards.push_back(p);
    if (count) {
        int blocks = int(std::min<uint64_t>((count + 7) / 8, uint64_t(c.sm_count) * 16));
        if (dtype == 0)
            k_rows<float><<<blocks, 256, 0, c.stream>>>(seed, first, count, dim, (float*)p);
        else
            k_rows<__half><<<blocks, 256, 0, c.stream>>>(seed, first, count, dim, (__half*)p);
        FDG_CUDA(cudaGetLastError());
    }
    FDG_CUDA(cudaStreamSynchronize(c.stream));
    *base = p;
    return FDG_OK;
}

int generate_features(Ctx& c, uint64_t seed, uint64_t n, uint32_t dim, uint32_t dtype, uint32_t n_shards) {
    if (n == 0 || dim == 0) return fail(FDG_INVALID_ARG, "generate_features: empty table");
    if (dtype > 1) return fail(FDG_INVALID_ARG, "generate_features: dtype must be 0 (f32) or 1 (f16)");
    if (n_shards == 0) n_shards = 1;
    const uint32_t esz = dtype == 0 ? 4 : 2;
    const uint32_t row_bytes = dim * esz;
    for (void* p : c.owned_shards) cudaFree(p);
    c.owned_shards.clear();
    c.shard_bases.clear();
    const uint64_t rps = (n + n_shards - 1) / n_shards;
    for (uint32_t s = 0; s < n_shards; ++s) {
        uint64_t first = uint64_t(s) * rps;
        uint64_t count = first < n ? std::min<uint64_t>(rps, n - first) : 0;
        void* p = nullptr;
        FDG_CUDA(cudaMalloc(&p, std::max<uint64_t>(count, 1) * row_bytes));
        c.owned_shards.push_back(p);
        c.shard_bases.push_back(p);
        if (count == 0) continue;
        int blocks = int(std::min<uint64_t>((count + 7) / 8, uint64_t(c.sm_count) * 16));
        if (dtype == 0)
            k_rows<float><<<blocks, 256, 0, c.stream>>>(seed, first, count, dim, (float*)p);
        else
            k_rows<__half><<<blocks, 256, 0, c.stream>>>(seed, first, count, dim, (__half*)p);
        FDG_CUDA(cudaGetLastError());
    }
    FDG_CUDA(cudaStreamSynchronize(c.stream));
    c.row_bytes = row_bytes;
    c.dtype = dtype;
    c.n_shards = n_shards;
    c.rows_per_shard = rps;
    c.feat_nodes = n;
    if (c.shard_table) cudaFree((void*)c.shard_table);
    FDG_CUDA(cudaMalloc((void**)&c.shard_table, n_shards * sizeof(void*)));
    FDG_CUDA(cudaMemcpy((void*)c.shard_table, c.shard_bases.data(), n_shards * sizeof(void*), cudaMemcpyHostToDevice));
    return FDG_OK;
}

}  // namespace fdg
