// fdg_mt.cuh -- the MT19937-64 block generator shared by the prefetch kernel (fdg_mt.cu) and
// the sampler's in-stream exact replay (fdg_sample.cu), bit-identical to std::mt19937_64
// (seeded by sample_khop with splitmix64(rng_seed), sampling.hpp:78).
//
// The engine is sequential across twists, so one CTA generates one stream: thread i (< 156)
// keeps x[i] and x[i+156] in registers. In the standard in-place twist, x'[i] (i < 156)
// needs old x[i], x[i+1], x[i+156]; x'[i+156] needs old x[i+156], x[i+157] and NEW x'[i]
// (own register), except x'[311] which needs x'[0] -- recomputed locally by thread 155 from
// old x[0], x[1], x[156]. Hence one neighbour exchange and ONE barrier per 312 words. The
// 312-word state can be saved and resumed at any twist boundary, so a stream is generated in
// pieces (the words of the early layers first) and extended on demand.
#pragma once

#include "fdg_internal.cuh"

namespace fdg {
namespace mt {

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

// Block-level generation (blockDim.x >= 156; every thread must call it):
// words [begin, end) of the stream (begin a multiple of 312; the last twist is completed)
// into dst[w] for w < limit. begin == 0 seeds from splitmix64(rng_seed) ([rand.eng.mers]
// seeding x_i = f*(x_{i-1} ^ (x_{i-1} >> 62)) + i); otherwise the state after word `begin` is
// read from state[0..312). When state != nullptr the final state is written back there.
// buf: 2 x 312 words of shared memory.
__device__ __forceinline__ void generate(uint64_t (*buf)[kN], uint64_t rng_seed, uint64_t begin, uint64_t end,
                                         uint64_t limit, uint64_t* __restrict__ dst, uint64_t* state) {
    const int i = threadIdx.x;
    if (begin == 0) {
        if (i == 0) {
            uint64_t x = splitmix64(rng_seed);
            buf[0][0] = x;
            for (int k = 1; k < kN; ++k) {
                x = 6364136223846793005ull * (x ^ (x >> 62)) + uint64_t(k);
                buf[0][k] = x;
            }
        }
    } else {
        for (int k = i; k < kN; k += blockDim.x) buf[0][k] = state[k];
    }
    __syncthreads();
    uint64_t a = 0, b = 0;
    if (i < kM) {
        a = buf[0][i];
        b = buf[0][i + kM];
    }
    __syncthreads();
    const uint64_t t0 = begin / kN, t1 = (end + kN - 1) / kN;
    // With >= 312 threads, threads 156..311 temper and store twist t-1's words (they sit in
    // the shared buffer the recurrence threads fill at the start of twist t). Measured slower
    // (1.09 vs 0.81 ms per 1.11 M words: the 10-warp barrier costs more than the stores), so
    // the prefetch kernel runs 160 threads; the split only engages for larger blocks.
    const bool split = blockDim.x >= 2 * kM;
    for (uint64_t t = t0; t < t1; ++t) {
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
                a_next = s[kM];                     // old x[156]
                b_next = s[kM] ^ twist(s[0], s[1]);  // new x'[0]
            }
            const uint64_t na = b ^ twist(a, a_next);   // x'[i]     = x[i+156] ^ tw(x[i], x[i+1])
            const uint64_t nb = na ^ twist(b, b_next);  // x'[i+156] = x'[i]    ^ tw(x[i+156], x[i+157])
            a = na;
            b = nb;
            if (!split) {
                const uint64_t w0 = t * kN + i, w1 = w0 + kM;
                if (w0 < limit) dst[w0] = temper(na);
                if (w1 < limit) dst[w1] = temper(nb);
            }
        } else if (split && i < 2 * kM && t > t0) {  // the words of twist t-1
            const int k = i - kM;
            const uint64_t w0 = (t - 1) * kN + k, w1 = w0 + kM;
            if (w0 < limit) dst[w0] = temper(s[k]);
            if (w1 < limit) dst[w1] = temper(s[k + kM]);
        }
    }
    if (split && t1 > t0) {  // the last twist's words
        uint64_t* s = buf[t1 & 1];
        if (i < kM) {
            s[i] = a;
            s[i + kM] = b;
        }
        __syncthreads();
        if (i >= kM && i < 2 * kM) {
            const int k = i - kM;
            const uint64_t w0 = (t1 - 1) * kN + k, w1 = w0 + kM;
            if (w0 < limit) dst[w0] = temper(s[k]);
            if (w1 < limit) dst[w1] = temper(s[k + kM]);
        }
    }
    if (state && i < kM) {
        state[i] = a;
        state[i + kM] = b;
    }
    __syncthreads();
}

}  // namespace mt
}  // namespace fdg
