// fdg_mt.cu -- MT19937-64 output streams on device, bit-identical to
// std::mt19937_64(splitmix64(rng_seed)) as seeded by sample_khop
// (sampling.hpp:78) and consumed through uniform_int_distribution.
//
// The engine is sequential across twists, so one WARP generates one stream with
// the whole 312-word state in registers: lane l holds x[32k+l] (a[k]) and
// x[156+32k+l] (b[k]) for k < 5 (k = 4: lanes < 28). In the standard in-place
// twist, x'[i] (i < 156) = x[i+156] ^ tw(x[i], x[i+1]) and x'[i+156] = x'[i] ^
// tw(x[i+156], x[i+157]) with x[312] = x'[0]: every neighbour word comes from the
// next lane (a shuffle) or, at a row end, from lane 0 of the next row -- so a twist
// is ~20 independent shuffles and 10 twist evaluations, no shared memory and no
// barrier (the previous one-CTA-per-stream kernel paid a 156-thread barrier per
// twist: 4x the latency). Four streams per CTA. The latency of a Papers-shaped batch
// stream is still hidden by generating upcoming batches' streams ahead of time
// (fdg_sampler_prefetch), but the pipeline's first batch waits for it.
#include "fdg_internal.cuh"

namespace fdg {
namespace {

constexpr int kN = 312, kM = 156;
constexpr uint64_t kA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUM = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLM = 0x000000007FFFFFFFull;

__device__ __forceinline__ uint64_t twist(uint64_t hi, uint64_t lo) {
    uint64_t y = (hi & kUM) | (lo & kLM);
    return (y >> 1) ^ ((y & 1) ? kA : 0ull);
}

__device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

struct MtSeeds {
    uint64_t s[32];
    uint32_t slot[32];  // output block of stream i = out + slot[i] * stride
    uint32_t n;         // streams in this launch
};

constexpr int kMtWarps = 4;  // streams per CTA

__global__ void __launch_bounds__(kMtWarps * 32) k_mt_stream(MtSeeds seeds, uint64_t words, uint64_t* __restrict__ out,
                                                           uint64_t stride) {
    __shared__ uint64_t init[kMtWarps][kN];
    const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint32_t sid = blockIdx.x * kMtWarps + warp;
    if (sid >= seeds.n) return;  // whole warps only: no block-level synchronisation below
    uint64_t* dst = out + uint64_t(seeds.slot[sid]) * stride;
    uint64_t* x = init[warp];
    if (l == 0) {  // [rand.eng.mers] seeding: x_i = f*(x_{i-1} ^ (x_{i-1} >> (w-2))) + i
        uint64_t v = splitmix64(seeds.s[sid]);
        x[0] = v;
        for (int k = 1; k < kN; ++k) {
            v = 6364136223846793005ull * (v ^ (v >> 62)) + uint64_t(k);
            x[k] = v;
        }
    }
    __syncwarp();
    uint64_t a[5], b[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = 32 * k + l;
        a[k] = i < kM ? x[i] : 0;
        b[k] = i < kM ? x[i + kM] : 0;
    }
    const uint64_t twists = (words + kN - 1) / kN;
    for (uint64_t t = 0; t < twists; ++t) {
        // neighbours x[i+1] and x[i+157] of the OLD state
        uint64_t an[5], bn[5];
        const uint64_t b00 = __shfl_sync(0xffffffffu, b[0], 0);  // x[156] (a-row end)
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const uint64_t ua = __shfl_down_sync(0xffffffffu, a[k], 1);
            const uint64_t ub = __shfl_down_sync(0xffffffffu, b[k], 1);
            const uint64_t wa = k < 4 ? __shfl_sync(0xffffffffu, a[k < 4 ? k + 1 : 4], 0) : 0;
            const uint64_t wb = k < 4 ? __shfl_sync(0xffffffffu, b[k < 4 ? k + 1 : 4], 0) : 0;
            an[k] = l < 31 ? ua : wa;
            bn[k] = l < 31 ? ub : wb;
        }
        if (l == kM - 1 - 32 * 4) an[4] = b00;  // i = 155: x[156]
        uint64_t na[5], nb[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) na[k] = b[k] ^ twist(a[k], an[k]);
        const uint64_t x0 = __shfl_sync(0xffffffffu, na[0], 0);  // x'[0]
        if (l == kM - 1 - 32 * 4) bn[4] = x0;                   // i = 311: x[312] = x'[0]
#pragma unroll
        for (int k = 0; k < 5; ++k) nb[k] = na[k] ^ twist(b[k], bn[k]);
        const uint64_t base = t * kN;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            a[k] = na[k];
            b[k] = nb[k];
            const int i = 32 * k + l;
            if (i < kM) {
                if (base + i < words) dst[base + i] = temper(na[k]);
                if (base + i + kM < words) dst[base + i + kM] = temper(nb[k]);
            }
        }
    }
}

void launch_chunk(cudaStream_t st, const MtSeeds& p, uint64_t words, uint64_t* out, uint64_t stride) {
    k_mt_stream<<<(p.n + kMtWarps - 1) / kMtWarps, kMtWarps * 32, 0, st>>>(p, words, out, stride);
}

}  // namespace

cudaError_t launch_mt_streams(cudaStream_t st, const uint64_t* rng_seeds, uint32_t n_streams,
                              uint64_t words_per_stream, uint64_t* out_dev, uint64_t out_stride) {
    for (uint32_t base = 0; base < n_streams; base += 32) {
        MtSeeds p;
        uint32_t k = n_streams - base < 32 ? n_streams - base : 32;
        for (uint32_t i = 0; i < k; ++i) {
            p.s[i] = rng_seeds[base + i];
            p.slot[i] = base + i;
        }
        p.n = k;
        launch_chunk(st, p, words_per_stream, out_dev, out_stride);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_mt_streams_slots(cudaStream_t st, const uint64_t* rng_seeds, const uint32_t* slots,
                                    uint32_t n_streams, uint64_t words_per_stream, uint64_t* ring, uint64_t stride) {
    for (uint32_t base = 0; base < n_streams; base += 32) {
        MtSeeds p;
        uint32_t k = n_streams - base < 32 ? n_streams - base : 32;
        for (uint32_t i = 0; i < k; ++i) {
            p.s[i] = rng_seeds[base + i];
            p.slot[i] = slots[base + i];
        }
        p.n = k;
        launch_chunk(st, p, words_per_stream, ring, stride);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace fdg
