// fdg_mt.cu -- MT19937-64 output streams on device, bit-identical to
// std::mt19937_64(splitmix64(rng_seed)) as seeded by sample_khop
// (sampling.hpp:78) and consumed through uniform_int_distribution.
//
// The engine is inherently sequential across twists, so one CTA generates one
// stream: thread i (< 156) keeps x[i] and x[i+156] in registers. In the
// standard in-place twist, x'[i] (i < 156) needs old x[i], x[i+1], x[i+156];
// x'[i+156] needs old x[i+156], x[i+157] and NEW x'[i] (own register), except
// x'[311] which needs x'[0] -- recomputed locally by thread 155 from old
// x[0], x[1], x[156]. Hence one neighbour exchange and ONE barrier per 312
// words. Latency (~0.8 ms for a 1.11 M-word stream) is hidden by generating
// streams for upcoming batches ahead of time (fdg_sampler_prefetch), one CTA
// per stream.
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
    uint32_t slot[32];  // output block of CTA i = out + slot[i] * stride
};

__global__ void __launch_bounds__(160) k_mt_stream(MtSeeds seeds, uint64_t words, uint64_t* __restrict__ out,
                                                   uint64_t stride) {
    __shared__ uint64_t buf[2][kN];
    const int i = threadIdx.x;
    uint64_t* dst = out + uint64_t(seeds.slot[blockIdx.x]) * stride;
    if (i == 0) {  // [rand.eng.mers] seeding: x_i = f*(x_{i-1} ^ (x_{i-1} >> (w-2))) + i
        uint64_t x = splitmix64(seeds.s[blockIdx.x]);
        buf[0][0] = x;
        for (int k = 1; k < kN; ++k) {
            x = 6364136223846793005ull * (x ^ (x >> 62)) + uint64_t(k);
            buf[0][k] = x;
        }
    }
    __syncthreads();
    uint64_t a = 0, b = 0;
    if (i < kM) {
        a = buf[0][i];
        b = buf[0][i + kM];
    }
    __syncthreads();
    const uint64_t twists = (words + kN - 1) / kN;
    for (uint64_t t = 0; t < twists; ++t) {
        uint64_t* s = buf[t & 1];
        if (i < kM) {
            s[i] = a;
            s[i + kM] = b;
        }
        __syncthreads();
        if (i < kM) {
            uint64_t a_next, b_next;
            if (i < kM - 1) {
                a_next = s[i + 1];
                b_next = s[i + kM + 1];
            } else {
                a_next = s[kM];                               // old x[156]
                b_next = s[kM] ^ twist(s[0], s[1]);            // new x'[0]
            }
            uint64_t na = b ^ twist(a, a_next);                // x'[i]     = x[i+156] ^ tw(x[i], x[i+1])
            uint64_t nb = na ^ twist(b, b_next);               // x'[i+156] = x'[i]    ^ tw(x[i+156], x[i+157])
            a = na;
            b = nb;
            uint64_t w0 = t * kN + i, w1 = w0 + kM;
            if (w0 < words) dst[w0] = temper(na);
            if (w1 < words) dst[w1] = temper(nb);
        }
    }
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
        k_mt_stream<<<k, 160, 0, st>>>(p, words_per_stream, out_dev, out_stride);
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
        k_mt_stream<<<k, 160, 0, st>>>(p, words_per_stream, ring, stride);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace fdg
