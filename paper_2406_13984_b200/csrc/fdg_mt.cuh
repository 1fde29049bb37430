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

// Barrier-free variant for a CTA of exactly 5 warps (160 threads). Warp w holds
// x[32w + l] and x[156 + 32w + l]; within a twist every neighbour word comes from the next
// lane (a shuffle) except at a warp's last lane, which needs lane 0 of the next warp (and
// warp 4's last row, x[155], needs x[156] and x'[0] = x[156] ^ tw(x[0], x[1]) from warp 0).
// So a warp waits only for its successor to publish those words for the twist (a flag in
// shared memory), never for the whole CTA: the warps form a ring and run at most 4 twists
// apart (8 publish slots). Same words, same state, same arguments as generate().
struct alignas(16) MtPub {
    uint64_t a0, b0, a1, pad;
};
__device__ __forceinline__ void generate_ring(uint64_t (*buf)[kN], MtPub (*pub)[5], volatile int64_t* flag,
                                              uint64_t rng_seed, uint64_t begin, uint64_t end, uint64_t limit,
                                              uint64_t* __restrict__ dst, uint64_t* state) {
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    const int i = 32 * w + l;
    const bool valid = i < kM;
    if (begin == 0) {
        if (tid == 0) {
            uint64_t x = splitmix64(rng_seed);
            buf[0][0] = x;
            for (int k = 1; k < kN; ++k) {
                x = 6364136223846793005ull * (x ^ (x >> 62)) + uint64_t(k);
                buf[0][k] = x;
            }
        }
    } else {
        for (int k = tid; k < kN; k += blockDim.x) buf[0][k] = state[k];
    }
    if (tid < 5) flag[tid] = -1;
    __syncthreads();
    uint64_t a = valid ? buf[0][i] : 0, b = valid ? buf[0][i + kM] : 0;
    const uint64_t t0 = begin / kN, t1 = (end + kN - 1) / kN;
    const int succ = w == 4 ? 0 : w + 1;
    const int last = w == 4 ? kM - 1 - 128 : 31;  // the lane whose neighbours live in the next warp
    auto publish = [&](uint64_t t) {
        const uint64_t a1 = __shfl_sync(0xffffffffu, a, 1);
        if (l == 0) {
            MtPub& p = pub[t & 7][w];
            p.a0 = a;
            p.b0 = b;
            p.a1 = a1;
            __threadfence_block();
            flag[w] = int64_t(t);
        }
        __syncwarp();
    };
    publish(t0);
    for (uint64_t t = t0; t < t1; ++t) {
        // old neighbours: the next lane's words; at the warp's last lane, the successor's
        const uint64_t ua = __shfl_down_sync(0xffffffffu, a, 1), ub = __shfl_down_sync(0xffffffffu, b, 1);
        uint64_t an = ua, bn = ub;
        if (l == last) {
            while (flag[succ] < int64_t(t)) {
            }
            __threadfence_block();
            const volatile MtPub& p = pub[t & 7][succ];
            const uint64_t pa0 = p.a0, pb0 = p.b0;
            if (w < 4) {
                an = pa0;  // x[32(w+1)]
                bn = pb0;  // x[156 + 32(w+1)]
            } else {
                an = pb0;                      // x[156]
                bn = pb0 ^ twist(pa0, p.a1);   // x'[0]
            }
        }
        const uint64_t na = b ^ twist(a, an);   // x'[i]     = x[i+156] ^ tw(x[i], x[i+1])
        const uint64_t nb = na ^ twist(b, bn);  // x'[i+156] = x'[i]    ^ tw(x[i+156], x[i+157])
        a = na;
        b = nb;
        publish(t + 1);
        if (valid) {
            const uint64_t w0 = t * kN + i, w1 = w0 + kM;
            if (w0 < limit) dst[w0] = temper(na);
            if (w1 < limit) dst[w1] = temper(nb);
        }
    }
    if (state && valid) {
        state[i] = a;
        state[i + kM] = b;
    }
    __syncthreads();
}

}  // namespace mt
}  // namespace fdg
