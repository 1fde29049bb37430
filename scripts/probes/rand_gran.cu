// DRAM bytes per random access on B200: 4M random 8-byte loads (or read-modify-write
// stores) over a 4 GB buffer, under each cudaLimitMaxL2FetchGranularity setting and with the
// PTX prefetch-size hints. Run under ncu for dram__bytes_read/write per launch; prints CUDA-event
// times. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rand_gran rand_gran.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_rand(const unsigned long long* __restrict__ buf, const uint32_t* __restrict__ idx, uint64_t n,
                       unsigned long long* out) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const unsigned long long* p = buf + uint64_t(idx[i]) * 16;  // 128-byte-aligned entries
        unsigned long long v;
        if (MODE == 0) v = *p;
        else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
        else if (MODE == 2) asm volatile("ld.global.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(p));
        else if (MODE == 3) asm volatile("ld.global.L2::128B.b64 %0, [%1];" : "=l"(v) : "l"(p));
        else {  // MODE 4: 8-byte store (partial sector)
            *const_cast<unsigned long long*>(p) = i;
            v = 0;
        }
        acc += v;
    }
    if (acc == 0x123456789ull) *out = acc;
}

int main() {
    const uint64_t bytes = 4ull << 30, entries = bytes / 128, n = 4u << 20;
    unsigned long long* buf;
    uint32_t* idx;
    unsigned long long* out;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 8);
    cudaMemset(buf, 1, bytes);
    std::vector<uint32_t> h(n);
    uint64_t x = 88172645463325252ull;
    for (auto& v : h) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        v = uint32_t(x % entries);
    }
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[5] = {"ld", "ld.nc.no_allocate", "ld.L2::64B", "ld.L2::128B", "st.8B"};
    for (size_t gran : {size_t(0), size_t(32), size_t(64), size_t(128)}) {
        if (gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t g = 0;
        cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
        for (int m = 0; m < 5; ++m) {
            cudaMemset(buf, 1, 256 << 20);  // push the previous kernel's lines out of L2
            cudaEventRecord(a);
            switch (m) {
                case 0: k_rand<0><<<sms * 8, 256>>>(buf, idx, n, out); break;
                case 1: k_rand<1><<<sms * 8, 256>>>(buf, idx, n, out); break;
                case 2: k_rand<2><<<sms * 8, 256>>>(buf, idx, n, out); break;
                case 3: k_rand<3><<<sms * 8, 256>>>(buf, idx, n, out); break;
                default: k_rand<4><<<sms * 8, 256>>>(buf, idx, n, out); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("granularity_limit %zu mode %-18s %8.1f us  %6.2f G accesses/s\n", g, names[m], ms * 1e3,
                   n / (ms * 1e-3) / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
