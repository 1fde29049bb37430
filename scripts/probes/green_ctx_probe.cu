// Probe: do runtime-API launches on a green-context stream (a) run, (b) see primary-context
// allocations, (c) stay on the partition's SMs? nvcc -arch=sm_100a green_ctx_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

__global__ void k_smid(const int* in, int* out, int n) {
    int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i] + 1;
    if (threadIdx.x == 0) out[n + blockIdx.x] = smid;
}

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

int main() {
    RK(cudaFree(0));
    const int n = 1 << 20, blocks = n / 256;
    int *in, *out;
    RK(cudaMalloc(&in, n * 4));
    RK(cudaMalloc(&out, (n + blocks) * 4));
    RK(cudaMemset(in, 0, n * 4));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all, parts[1], rest;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    unsigned int ng = 1;
    CK(cuDevSmResourceSplitByCount(parts, &ng, &all, &rest, 0, 32));
    printf("group SMs: %u, remaining SMs: %u\n", parts[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc d1, d2;
    CK(cuDevResourceGenerateDesc(&d1, parts, 1));
    CK(cuDevResourceGenerateDesc(&d2, &rest, 1));
    CUgreenCtx g1, g2;
    CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s1, s2;
    CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, 0));
    for (int pass = 0; pass < 2; ++pass) {
        CUstream s = pass ? s2 : s1;
        k_smid<<<blocks, 256, 0, (cudaStream_t)s>>>(in, out, n);
        RK(cudaGetLastError());
        RK(cudaStreamSynchronize((cudaStream_t)s));
        std::vector<int> h(n + blocks);
        RK(cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost));
        bool ok = true;
        for (int i = 0; i < n; ++i) ok &= h[i] == 1;
        std::set<int> sms(h.begin() + n, h.end());
        printf("stream %d: data %s, distinct SMs used %zu (min %d max %d)\n", pass, ok ? "ok" : "BAD", sms.size(),
               *sms.begin(), *sms.rbegin());
    }
    // an event recorded on a green stream, waited on by a primary-context stream
    cudaStream_t ps;
    RK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
    cudaEvent_t ev;
    RK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    k_smid<<<blocks, 256, 0, (cudaStream_t)s1>>>(in, out, n);
    RK(cudaEventRecord(ev, (cudaStream_t)s1));
    RK(cudaStreamWaitEvent(ps, ev, 0));
    k_smid<<<blocks, 256, 0, ps>>>(in, out, n);
    RK(cudaStreamSynchronize(ps));
    printf("cross-context event ok\n");
    return 0;
}
