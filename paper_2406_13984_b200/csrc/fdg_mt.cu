// fdg_mt.cu -- MT19937-64 output streams on device, bit-identical to
// std::mt19937_64(splitmix64(rng_seed)) as seeded by sample_khop (sampling.hpp:78) and
// consumed through uniform_int_distribution: one CTA per stream (fdg_mt.cuh). Latency
// (~0.8 ms for a 1.11 M-word stream) is hidden by generating the streams of upcoming
// batches ahead of time (fdg_sampler_prefetch), in two pieces: the words the early layers
// consume first, the rest after (the state is saved in between).
#include "fdg_internal.cuh"

#include "fdg_mt.cuh"

namespace fdg {
namespace {

struct MtSeeds {
    uint64_t s[32];
    uint32_t slot[32];  // output block of CTA i = out + slot[i] * stride, state at state + slot[i] * 312
};

__global__ void __launch_bounds__(160) k_mt_stream(MtSeeds seeds, uint64_t begin, uint64_t end, uint64_t limit,
                                                   uint64_t* __restrict__ out, uint64_t stride, uint64_t* state) {
    // One CTA of 160 threads per stream with one barrier per twist (fdg_mt.cuh). Measured
    // alternatives, per 568 k words under ncu: a warp-per-stream kernel 2.5x slower (one SMSP
    // does all 312 words of a twist), a 5-warp ring synchronised by shared-memory flags
    // instead of the barrier 760 vs 549 us, 320 threads with the tempering on the second
    // half 1.09 vs 0.81 ms per 1.11 M words.
    __shared__ uint64_t buf[2][mt::kN];
    const uint64_t slot = seeds.slot[blockIdx.x];
    mt::generate(buf, seeds.s[blockIdx.x], begin, end, limit, out + slot * stride,
                 state ? state + slot * mt::kN : nullptr);
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
        k_mt_stream<<<k, 160, 0, st>>>(p, 0, words_per_stream, words_per_stream, out_dev, out_stride, nullptr);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_mt_streams_slots(cudaStream_t st, const uint64_t* rng_seeds, const uint32_t* slots,
                                    uint32_t n_streams, uint64_t begin, uint64_t end, uint64_t* ring, uint64_t stride,
                                    uint64_t* state) {
    for (uint32_t base = 0; base < n_streams; base += 32) {
        MtSeeds p;
        uint32_t k = n_streams - base < 32 ? n_streams - base : 32;
        for (uint32_t i = 0; i < k; ++i) {
            p.s[i] = rng_seeds[base + i];
            p.slot[i] = slots[base + i];
        }
        k_mt_stream<<<k, 160, 0, st>>>(p, begin, end, stride, ring, stride, state);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace fdg
