// fdg_sage.cu -- the train stage: GraphSAGE forward + loss on a sampled batch.
//
// The reference's trainer is a checksum over the extracted rows
// (pipeline.hpp:103-124); the paper trains a 3-layer GraphSAGE with hidden size
// 256 on exactly these blocks. This is that consumer,
// fed straight from the mini-batch tensor X the extraction wrote:
//
//   layer k = 1..L computes h^k for the nodes within L-k hops of the seeds,
//   D_{L-k} = layer_nodes[L-k+1] of the batch record (local ids [0, D)), as
//     h^k_v = W_neigh^k . mean_{(u -> v) in edges} h^{k-1}_u + W_self^k . h^{k-1}_v + b^k
//   (PyG SAGEConv, mean aggregator; ReLU between layers; a node without sampled
//   in-edges aggregates 0), with h^0 = X. Every node is expanded at most once and
//   sample_khop emits a frontier's edges in ascending dst order
//   (sampling.hpp:97-131), so `edges` is a dst-sorted COO: node v's in-edges are
//   one contiguous run, and for v < D_{L-k} all sources lie in [0, D_{L-k+1}).
//   loss = mean over the unique seeds of softmax cross-entropy against
//   label(v) = splitmix64(node_id ^ label_seed) % C.
//
// Kernels (fp32 on the CUDA cores: the loss is checked at 1e-5 relative against
// an fp64 restatement, which TF32/BF16 tensor-core products would not meet):
//   k_seg_clear / k_seg   per-dst [begin, end) of its edge run
//   k_aggregate           warp per dst row: A[v] = [mean of in-neighbour rows | own row]
//                         (f32 or f16 input), 16-byte loads
//   k_sgemm               C = act(A . [W_neigh; W_self] + b), 128x128x8 tiles, 8x8
//                         outputs per thread, register-prefetched double-buffered smem
//   k_splitk_sum          split-K slices added in order (+ bias, ReLU) for the small layers
//   k_loss_rows/_mean     warp per seed row: log-softmax CE; one CTA: fixed-order mean
// Row counts live on the device (the batch record), so a forward is enqueued
// without a host round trip; grids are sized from the fanout bounds.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "fdg_internal.cuh"

namespace fdg {
// tensor-core GEMM (fdg_sage_tc.cu)
int tc_make_map(CUtensorMap* map, const float* base, uint64_t rows, uint32_t K);
int tc_gemm(cudaStream_t st, const CUtensorMap& tA, const CUtensorMap& tBhi, const CUtensorMap& tBlo,
            const float* bias, float* C, const fdg_batch_counts* cnt, int j, uint64_t rows_bound, int N, int npad,
            int K, bool relu);
int tc_make_map_mn(CUtensorMap* map, const float* base, uint64_t rows, uint32_t cols);
int tc_wgrad(cudaStream_t st, const CUtensorMap& tA, const CUtensorMap& tB, float* P, const fdg_batch_counts* cnt,
             int j, int Kin, int N, int Z);
int tc_write_hi(cudaStream_t st);  // 1: the split warps write A_hi (kind::tf32 does not truncate)
// 1: layer GEMMs on the tensor cores (tcgen05 kind::tf32, 3xTF32 fp32-accurate); 0: CUDA-core fp32
int64_t g_sage_gemm = 1;

namespace {

constexpr int kBM = 128, kBN = 128, kBK = 8;
constexpr int kMaxSplit = 16;

// K slices for a GEMM whose row bound gives fewer than ~2 waves of 128x128 tiles
// (2 CTAs per SM): the layers nearer the seeds (D_1 ~ 10 k rows, D_0 = 1 k rows).
int splitk_for(uint64_t rows, uint32_t K, uint32_t col_tiles, int sms) {
    const uint64_t tiles = (rows + kBM - 1) / kBM * col_tiles;
    int z = 1;
    while (z < kMaxSplit && tiles * uint64_t(z) < uint64_t(sms) * 4 && K % (uint32_t(2 * z) * kBK) == 0) z *= 2;
    return z;
}

// D_j: nodes within j hops (running max, so hops that sampling never reached --
// an empty frontier -- count every node).
__device__ __forceinline__ uint32_t d_rows(const fdg_batch_counts* c, int j) {
    uint32_t d = 0;
    for (int i = 0; i <= j + 1 && i < FDG_MAX_LAYERS + 2; ++i) d = max(d, c->layer_nodes[i]);
    return min(d, c->n_nodes);
}

__global__ void k_seg_clear(uint2* seg, const fdg_batch_counts* cnt, int j) {
    const uint32_t n = d_rows(cnt, j);
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) seg[v] = make_uint2(0, 0);
}

__global__ void k_seg(const uint2* __restrict__ edges, const fdg_batch_counts* cnt, uint2* seg) {
    const uint32_t E = cnt->n_edges;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const uint32_t d = edges[e].y;
        if (e == 0 || edges[e - 1].y != d) seg[d].x = e;
        if (e + 1 == E || edges[e + 1].y != d) seg[d].y = e + 1;
    }
}

__device__ __forceinline__ float4 load4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 load4(const __half* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
}

// A[v] = [mean_{e in seg(v)} h[src(e)] | h[v]] for v < D_j.
template <typename T>
__global__ void __launch_bounds__(256) k_aggregate(const T* __restrict__ h, uint32_t d, const uint2* __restrict__ seg,
                                                   const uint2* __restrict__ edges, const fdg_batch_counts* cnt,
                                                   int j, float* __restrict__ A) {
    const uint32_t rows = d_rows(cnt, j);
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t v = warp; v < rows; v += nwarps) {
        const uint2 sg = seg[v];
        const uint32_t deg = sg.y - sg.x;
        const float inv = deg ? 1.0f / float(deg) : 0.0f;
        float* out = A + size_t(v) * 2 * d;
        for (uint32_t c = lane * 4; c < d; c += 128) {
            float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
            uint32_t e = sg.x;
            for (; e + 1 < sg.y; e += 2) {  // two rows in flight
                const float4 x0 = load4(h + size_t(edges[e].x) * d + c);
                const float4 x1 = load4(h + size_t(edges[e + 1].x) * d + c);
                s.x += x0.x; s.y += x0.y; s.z += x0.z; s.w += x0.w;
                s.x += x1.x; s.y += x1.y; s.z += x1.z; s.w += x1.w;
            }
            if (e < sg.y) {
                const float4 x0 = load4(h + size_t(edges[e].x) * d + c);
                s.x += x0.x; s.y += x0.y; s.z += x0.z; s.w += x0.w;
            }
            *reinterpret_cast<float4*>(out + c) = make_float4(s.x * inv, s.y * inv, s.z * inv, s.w * inv);
            *reinterpret_cast<float4*>(out + d + c) = load4(h + size_t(v) * d + c);
        }
    }
}

// C[M x N] = act(A[M x K] . W[K x Npad] + bias), M = D_j from the batch record.
// Split-K (gridDim.z > 1, for GEMMs with too few row tiles to fill the SMs): slice z
// covers K range [z Kc, (z+1) Kc) and writes its raw partial sums to
// C + z * M_bound * N; k_splitk_sum adds the slices in order (deterministic).
template <bool RELU>
__global__ void __launch_bounds__(256) k_sgemm(const float* __restrict__ A, const float* __restrict__ W,
                                               const float* __restrict__ bias, float* __restrict__ C,
                                               const fdg_batch_counts* cnt, int j, int N, int K, int Npad,
                                               uint64_t slice_stride) {
    const int M = int(d_rows(cnt, j));
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
    if (m0 >= M) return;
    const bool split = gridDim.z > 1;
    const int Kc = K / int(gridDim.z);
    A += size_t(blockIdx.z) * Kc;
    W += size_t(blockIdx.z) * Kc * Npad;
    C += size_t(blockIdx.z) * slice_stride;
    K = Kc;
    __shared__ __align__(16) float As[2][kBK][kBM + 4];
    __shared__ __align__(16) float Bs[2][kBK][kBN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int ar = tid >> 1, ak = (tid & 1) * 4;
    const int lda = split ? Kc * int(gridDim.z) : K;
    const float* Ap = A + size_t(min(m0 + ar, M - 1)) * lda + ak;
    const int bk = tid >> 5, bn = (tid & 31) * 4;
    const float* Wp = W + size_t(bk) * Npad + n0 + bn;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[i][q] = 0.f;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 ra = ak < K ? *reinterpret_cast<const float4*>(Ap) : z4;
    float4 rb = bk < K ? *reinterpret_cast<const float4*>(Wp) : z4;
    As[0][ak + 0][ar] = ra.x;
    As[0][ak + 1][ar] = ra.y;
    As[0][ak + 2][ar] = ra.z;
    As[0][ak + 3][ar] = ra.w;
    *reinterpret_cast<float4*>(&Bs[0][bk][bn]) = rb;
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += kBK) {
        const bool more = k0 + kBK < K;
        if (more) {  // K is a multiple of 4: a float4 is either fully inside or fully past K
            ra = k0 + kBK + ak < K ? *reinterpret_cast<const float4*>(Ap + k0 + kBK) : z4;
            rb = k0 + kBK + bk < K ? *reinterpret_cast<const float4*>(Wp + size_t(k0 + kBK) * Npad) : z4;
        }
#pragma unroll
        for (int kk = 0; kk < kBK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[i][q] = fmaf(a[i], b[q], acc[i][q]);
        }
        if (more) {
            As[buf ^ 1][ak + 0][ar] = ra.x;
            As[buf ^ 1][ak + 1][ar] = ra.y;
            As[buf ^ 1][ak + 2][ar] = ra.z;
            As[buf ^ 1][ak + 3][ar] = ra.w;
            *reinterpret_cast<float4*>(&Bs[buf ^ 1][bk][bn]) = rb;
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
        if (r >= M) continue;
#pragma unroll
        for (int hq = 0; hq < 2; ++hq) {
            const int c = n0 + hq * 64 + tx * 4;
            if (c >= N) continue;
            float4 v = make_float4(acc[i][hq * 4 + 0], acc[i][hq * 4 + 1], acc[i][hq * 4 + 2], acc[i][hq * 4 + 3]);
            if (!split) {
                v.x += bias[c + 0];
                v.y += bias[c + 1];
                v.z += bias[c + 2];
                v.w += bias[c + 3];
            }
            if (RELU && !split) {
                v.x = fmaxf(v.x, 0.f);
                v.y = fmaxf(v.y, 0.f);
                v.z = fmaxf(v.z, 0.f);
                v.w = fmaxf(v.w, 0.f);
            }
            *reinterpret_cast<float4*>(C + size_t(r) * N + c) = v;
        }
    }
}

// out = act(sum_z P[z] + bias) over the first M rows (slices added in order).
template <bool RELU>
__global__ void k_splitk_sum(const float* __restrict__ P, int Z, uint64_t slice_stride, const float* __restrict__ bias,
                             float* __restrict__ C, const fdg_batch_counts* cnt, int j, int N) {
    const uint64_t total = uint64_t(d_rows(cnt, j)) * N / 4;
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < total; q += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = q * 4;
        const int c = int(e % N);
        float4 v = *reinterpret_cast<const float4*>(P + e);
        for (int z = 1; z < Z; ++z) {
            const float4 w = *reinterpret_cast<const float4*>(P + z * slice_stride + e);
            v.x += w.x;
            v.y += w.y;
            v.z += w.z;
            v.w += w.w;
        }
        v.x += bias[c];
        v.y += bias[c + 1];
        v.z += bias[c + 2];
        v.w += bias[c + 3];
        if (RELU) {
            v.x = fmaxf(v.x, 0.f);
            v.y = fmaxf(v.y, 0.f);
            v.z = fmaxf(v.z, 0.f);
            v.w = fmaxf(v.w, 0.f);
        }
        *reinterpret_cast<float4*>(C + e) = v;
    }
}

// Softmax cross-entropy of each seed row (warp per row) -> row_loss; optional logits copy.
__global__ void __launch_bounds__(256) k_loss_rows(const float* __restrict__ logits, int C,
                                                   const uint64_t* __restrict__ nodes, const fdg_batch_counts* cnt,
                                                   uint64_t label_seed, float* row_loss, float* logits_out) {
    const uint32_t rows = d_rows(cnt, 0);
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (r >= rows) return;
    const float* x = logits + size_t(r) * C;
    float mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmaxf(mx, x[c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f;
    for (int c = lane; c < C; c += 32) {
        se += expf(x[c] - mx);
        if (logits_out) logits_out[size_t(r) * C + c] = x[c];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    if (lane == 0) {
        const uint32_t label = uint32_t(splitmix64(nodes[r] ^ label_seed) % uint64_t(C));
        row_loss[r] = logf(se) + mx - x[label];
    }
}

constexpr int kLossThreads = 1024;

// Mean of the row losses in a fixed order (deterministic).
__global__ void __launch_bounds__(kLossThreads) k_loss_mean(const float* __restrict__ row_loss,
                                                            const fdg_batch_counts* cnt, float* loss) {
    __shared__ double s_part[kLossThreads];
    const uint32_t rows = d_rows(cnt, 0);
    double t = 0.0;
    for (uint32_t r = threadIdx.x; r < rows; r += kLossThreads) t += double(row_loss[r]);
    s_part[threadIdx.x] = t;
    __syncthreads();
    for (int w = kLossThreads / 2; w; w >>= 1) {
        if (int(threadIdx.x) < w) s_part[threadIdx.x] += s_part[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *loss = rows ? float(s_part[0] / double(rows)) : 0.f;
}

// ------------------------------------------------------------------ backward --
// dZ = (softmax(logits) - onehot(label)) / D_0: gradient of the mean loss.
__global__ void __launch_bounds__(256) k_loss_grad(const float* __restrict__ logits, int C,
                                                   const uint64_t* __restrict__ nodes, const fdg_batch_counts* cnt,
                                                   uint64_t label_seed, float* __restrict__ dZ) {
    const uint32_t rows = d_rows(cnt, 0);
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (r >= rows) return;
    const float* x = logits + size_t(r) * C;
    float mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmaxf(mx, x[c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f;
    for (int c = lane; c < C; c += 32) se += expf(x[c] - mx);
#pragma unroll
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const uint32_t label = uint32_t(splitmix64(nodes[r] ^ label_seed) % uint64_t(C));
    const float inv = 1.f / float(rows);
    for (int c = lane; c < C; c += 32)
        dZ[size_t(r) * C + c] = (expf(x[c] - mx) / se - (uint32_t(c) == label ? 1.f : 0.f)) * inv;
}

// g *= (h > 0) over the first D_j rows of width d (ReLU backward).
__global__ void k_relu_mask(float* __restrict__ g, const float* __restrict__ h, const fdg_batch_counts* cnt, int j,
                            int d) {
    const uint64_t total = uint64_t(d_rows(cnt, j)) * d;
    if (d % 4 == 0) {  // 16-byte accesses, two in flight per thread
        const uint64_t q4 = total / 4, stride = uint64_t(gridDim.x) * blockDim.x;
        float4* g4 = reinterpret_cast<float4*>(g);
        const float4* h4 = reinterpret_cast<const float4*>(h);
        for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < q4; i += 2 * stride) {
            const bool two = i + stride < q4;
            const float4 ha = h4[i], ga = g4[i];
            float4 hb = make_float4(1.f, 1.f, 1.f, 1.f), gb = hb;
            if (two) {
                hb = h4[i + stride];
                gb = g4[i + stride];
            }
            g4[i] = make_float4(ha.x > 0.f ? ga.x : 0.f, ha.y > 0.f ? ga.y : 0.f, ha.z > 0.f ? ga.z : 0.f,
                                ha.w > 0.f ? ga.w : 0.f);
            if (two)
                g4[i + stride] = make_float4(hb.x > 0.f ? gb.x : 0.f, hb.y > 0.f ? gb.y : 0.f, hb.z > 0.f ? gb.z : 0.f,
                                             hb.w > 0.f ? gb.w : 0.f);
        }
        return;
    }
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x)
        if (h[i] <= 0.f) g[i] = 0.f;
}

// Weight gradient A^T . B over the rows R = D_j (A [R x K], B [R x N], row-major), split over
// row slices (blockIdx.z) into partials P[z] [K x N]; the k-tile-0 CTAs also produce the
// column sums of B (bias gradient) into Pb[z] [N]. 64 x 64 outputs per CTA, 4 x 4 per thread.
constexpr int kTn = 64, kTnR = 16;
__global__ void __launch_bounds__(256) k_gemm_tn(const float* __restrict__ A, const float* __restrict__ B,
                                                 const fdg_batch_counts* cnt, int j, int K, int N, float* __restrict__ P,
                                                 float* __restrict__ Pb) {
    __shared__ __align__(16) float As[kTnR][kTn];
    __shared__ __align__(16) float Bs[kTnR][kTn];
    const int R = int(d_rows(cnt, j));
    const int Z = int(gridDim.z), z = int(blockIdx.z);
    const int per = (R + Z - 1) / Z;
    const int r0 = min(R, z * per), r1 = min(R, r0 + per);
    const int k0 = blockIdx.y * kTn, n0 = blockIdx.x * kTn;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int lr = (tid * 4) / kTn, lc = (tid * 4) % kTn;
    const bool bias_cta = blockIdx.y == 0;
    float acc[4][4] = {};
    float bs[4] = {};
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = r0; r < r1; r += kTnR) {
        const int rr = r + lr;
        *reinterpret_cast<float4*>(&As[lr][lc]) =
            (rr < r1 && k0 + lc < K) ? *reinterpret_cast<const float4*>(A + size_t(rr) * K + k0 + lc) : z4;
        *reinterpret_cast<float4*>(&Bs[lr][lc]) =
            (rr < r1 && n0 + lc < N) ? *reinterpret_cast<const float4*>(B + size_t(rr) * N + n0 + lc) : z4;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kTnR; ++q) {
            const float4 a = *reinterpret_cast<const float4*>(&As[q][ty * 4]);
            const float4 b = *reinterpret_cast<const float4*>(&Bs[q][tx * 4]);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[i][c] = fmaf(av[i], bv[c], acc[i][c]);
            if (bias_cta && ty == 0)
#pragma unroll
                for (int c = 0; c < 4; ++c) bs[c] += bv[c];
        }
        __syncthreads();
    }
    float* Pz = P + size_t(z) * K * N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = k0 + ty * 4 + i;
        if (k >= K) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (n0 + tx * 4 + c < N) Pz[size_t(k) * N + n0 + tx * 4 + c] = acc[i][c];
    }
    if (bias_cta && ty == 0)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (n0 + tx * 4 + c < N) Pb[size_t(z) * N + n0 + tx * 4 + c] = bs[c];
}

// Bias gradient slices for the tensor-core weight gradient: Pb[z][c] = sum of column c of
// B over row slice z (the k_wgrad_tc slicing: ceil(ceil(R / 32) / Z) 32-row blocks). A CTA
// is 32 columns x 8 row lanes; the 8 partial sums meet in a fixed order.
__global__ void __launch_bounds__(256) k_colsum(const float* __restrict__ B, const fdg_batch_counts* cnt, int j, int N,
                                                float* Pb) {
    __shared__ float part[8][33];
    const int R = int(d_rows(cnt, j));
    const int Z = int(gridDim.y), z = int(blockIdx.y);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int c = blockIdx.x * 32 + tx;
    const int nkb = (R + 31) / 32, per = ((nkb + Z - 1) / Z) * 32;
    const int r0 = min(R, z * per), r1 = min(R, r0 + per);
    float sum = 0.f;
    if (c < N) {
        int r = r0 + ty;
        for (; r + 24 < r1; r += 32) {  // 4 rows in flight per thread
            const float a = B[size_t(r) * N + c], b = B[size_t(r + 8) * N + c];
            const float d = B[size_t(r + 16) * N + c], e = B[size_t(r + 24) * N + c];
            sum += a;
            sum += b;
            sum += d;
            sum += e;
        }
        for (; r < r1; r += 8) sum += B[size_t(r) * N + c];
    }
    part[ty][tx] = sum;
    __syncthreads();
    if (ty == 0 && c < N) {
        float t = 0.f;
        for (int q = 0; q < 8; ++q) t += part[q][tx];
        Pb[size_t(z) * N + c] = t;
    }
}

// The same slices with 16-byte loads (N % 4 == 0): a CTA is 128 columns (a float4 per lane)
// x 8 row lanes, 4 rows in flight per thread -- four times the bytes in flight per request.
__global__ void __launch_bounds__(256) k_colsum4(const float* __restrict__ B, const fdg_batch_counts* cnt, int j,
                                                 int N, float* Pb) {
    __shared__ float4 part[8][32];
    const int R = int(d_rows(cnt, j));
    const int Z = int(gridDim.y), z = int(blockIdx.y);
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int c = blockIdx.x * 128 + tx * 4;
    const int nkb = (R + 31) / 32, per = ((nkb + Z - 1) / Z) * 32;
    const int r0 = min(R, z * per), r1 = min(R, r0 + per);
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    auto add = [](float4& s, float4 v) {
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
    };
    if (c < N) {
        const float* col = B + c;
        int r = r0 + ty;
        for (; r + 24 < r1; r += 32) {
            const float4 a = *reinterpret_cast<const float4*>(col + size_t(r) * N);
            const float4 b = *reinterpret_cast<const float4*>(col + size_t(r + 8) * N);
            const float4 d = *reinterpret_cast<const float4*>(col + size_t(r + 16) * N);
            const float4 e = *reinterpret_cast<const float4*>(col + size_t(r + 24) * N);
            add(sum, a);
            add(sum, b);
            add(sum, d);
            add(sum, e);
        }
        for (; r < r1; r += 8) add(sum, *reinterpret_cast<const float4*>(col + size_t(r) * N));
    }
    part[ty][tx] = sum;
    __syncthreads();
    if (ty == 0 && c < N) {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < 8; ++q) add(t, part[q][tx]);
        *reinterpret_cast<float4*>(Pb + size_t(z) * N + c) = t;
    }
}

void launch_colsum(const float* B, const fdg_batch_counts* cnt, int j, int N, float* Pb, int Z, cudaStream_t st) {
    if (N % 4 == 0)
        k_colsum4<<<dim3((N + 127) / 128, uint32_t(Z)), 256, 0, st>>>(B, cnt, j, N, Pb);
    else
        k_colsum<<<dim3((N + 31) / 32, uint32_t(Z)), 256, 0, st>>>(B, cnt, j, N, Pb);
}

// G[0 : K N] = sum_z P[z], G[K N : K N + N] = sum_z Pb[z] (slices added in order).
__global__ void k_tn_sum(const float* __restrict__ P, const float* __restrict__ Pb, int Z, int KN, int N,
                         float* __restrict__ G) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < KN + N; i += gridDim.x * blockDim.x) {
        float s = 0.f;
        if (i < KN)
            for (int z = 0; z < Z; ++z) s += P[size_t(z) * KN + i];
        else
            for (int z = 0; z < Z; ++z) s += Pb[size_t(z) * N + (i - KN)];
        G[i] = s;
    }
}

// Input gradient of a layer, self half: dH[v] = v < D_j ? dA[v][d:2d] : 0 for v < D_{j+1}.
__global__ void k_dh_self(const float* __restrict__ dA, int d, const fdg_batch_counts* cnt, int j, float* dH) {
    const uint32_t dst_rows = d_rows(cnt, j), rows = d_rows(cnt, j + 1);
    const uint64_t total = uint64_t(rows) * d / 4;
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < total; q += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t v = q * 4 / d, c = q * 4 - v * d;
        reinterpret_cast<float4*>(dH)[q] = v < dst_rows ? *reinterpret_cast<const float4*>(dA + v * 2 * d + d + c)
                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// Neighbour half: dH[src] += dA[v][0:d] / deg(v) for every edge src -> v, v < D_j
// (warp per destination, vector atomics: sources repeat across destinations).
__global__ void __launch_bounds__(256) k_dh_neigh(const float* __restrict__ dA, int d, const uint2* __restrict__ seg,
                                                  const uint2* __restrict__ edges, const fdg_batch_counts* cnt, int j,
                                                  float* dH) {
    const uint32_t rows = d_rows(cnt, j);
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t v = warp; v < rows; v += nwarps) {
        const uint2 sg = seg[v];
        if (sg.y == sg.x) continue;
        const float inv = 1.0f / float(sg.y - sg.x);
        for (uint32_t c = lane * 4; c < uint32_t(d); c += 128) {
            float4 g = *reinterpret_cast<const float4*>(dA + size_t(v) * 2 * d + c);
            g.x *= inv;
            g.y *= inv;
            g.z *= inv;
            g.w *= inv;
            for (uint32_t e = sg.x; e < sg.y; ++e) atomicAdd(reinterpret_cast<float4*>(dH + size_t(edges[e].x) * d + c), g);
        }
    }
}

// P -= lr * G (SGD over the contiguous parameter block).
__global__ void k_sgd(float* __restrict__ P, const float* __restrict__ G, uint64_t n, float lr) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        P[i] -= lr * G[i];
}

// The forward / backward copies of one layer's master weights Wm [K = 2 d_in x dout] + bias:
// Wpad [K x npad] (CUDA-core GEMM), bpad [npad], Wt [dout x npadT] (backward dA GEMM),
// and the tensor cores' transposed K-major hi / lo split [npad x K].
__global__ void k_derive(const float* __restrict__ Wm, const float* __restrict__ bm, int K, int dout, int npad,
                         int npadT, float* Wpad, float* bpad, float* Wt, float* Whi, float* Wlo, float* Wdhi,
                         float* Wdlo) {
    const int stride = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = t0; i < K * npad; i += stride) {
        const int k = i / npad, n = i - k * npad;
        const float v = n < dout ? Wm[size_t(k) * dout + n] : 0.f;
        Wpad[i] = v;
        if (Whi) {
            const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            Whi[size_t(n) * K + k] = h;
            Wlo[size_t(n) * K + k] = v - h;
        }
    }
    for (int i = t0; i < dout * npadT; i += stride) {
        const int n = i / npadT, k = i - n * npadT;
        Wt[i] = k < K ? Wm[size_t(k) * dout + n] : 0.f;
    }
    for (int i = t0; i < npad; i += stride) bpad[i] = i < dout ? bm[i] : 0.f;
    if (Wdhi)  // backward dA = dOut . W^T on the tensor cores: B operand [K x dout], K-major (Wm's own layout)
        for (int i = t0; i < K * dout; i += stride) {
            const float v = Wm[i], h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            Wdhi[i] = h;
            Wdlo[i] = v - h;
        }
}

}  // namespace

struct Sage {
    Ctx* ctx = nullptr;
    uint32_t L = 0;
    std::vector<uint32_t> dims;     // L + 1
    std::vector<uint32_t> npad;     // per layer: d_out rounded up to kBN
    std::vector<uint32_t> npadT;    // per layer: 2 d_in rounded up to kBN (backward dA GEMM)
    std::vector<uint64_t> bound;    // bound[j] >= D_j, j = 0..L
    // parameters: one contiguous block, per layer [W_neigh; W_self] (2 d_in x d_out, input-major)
    // then b (d_out); gradients G share the layout (a single buffer to all-reduce)
    float* P = nullptr;
    float* G = nullptr;
    std::vector<uint64_t> off;      // per layer offset into P / G
    uint64_t n_params = 0;
    std::vector<float*> W, b;       // derived: [2 d_in x npad], [npad] (CUDA-core forward)
    std::vector<float*> Wt;         // derived: [d_out x npadT] (backward dA = dOut . W^T)
    std::vector<float*> Whi, Wlo;   // derived: transposed K-major hi / lo split (tensor cores)
    std::vector<CUtensorMap> mapA, mapBhi, mapBlo;
    std::vector<uint8_t> tc_ok;     // layer K is a multiple of 32 and the maps were built
    uint2* seg = nullptr;
    std::vector<float*> Al;         // saved layer inputs [mean | self], [D_{L-1-l} x 2 d_in]
    std::vector<float*> Hl;         // saved hidden outputs (post-ReLU), [D_{L-1-l} x d_out]
    float* logits = nullptr;
    float* partial = nullptr;       // forward split-K slices
    uint64_t partial_floats = 0;
    float* row_loss = nullptr;
    float* dbuf[2] = {nullptr, nullptr};  // backward: output gradients of the current / next layer
    float* dA = nullptr;
    float* zeros = nullptr;
    float* tn_part = nullptr;       // backward weight-gradient slices
    uint64_t tn_floats = 0;
    std::vector<uint8_t> set;
    bool forwarded = false;
    // tensor-core weight gradients: MN-major maps of each layer's saved input and output gradient
    std::vector<CUtensorMap> mapAmn, mapDmn;
    // tensor-core input gradients dA = dOut . W^T: K-major maps of dOut and of W's hi / lo split
    std::vector<float*> Wdhi, Wdlo;
    std::vector<CUtensorMap> mapDk, mapWdhi, mapWdlo;
    std::vector<uint8_t> tc_da;
    std::vector<int> wz;            // split-K slices per layer (0: CUDA-core k_gemm_tn)
};

}  // namespace fdg

struct fdg_sage : fdg::Sage {};

using namespace fdg;

namespace {

int tn_slices(uint64_t rows) { return int(std::min<uint64_t>(128, std::max<uint64_t>(1, rows / 512))); }

int derive_layer(fdg_sage* m, uint32_t l, cudaStream_t st) {
    const uint32_t K = 2 * m->dims[l], dout = m->dims[l + 1];
    const int n = int(std::max<uint64_t>(uint64_t(K) * m->npad[l], uint64_t(dout) * m->npadT[l]));
    k_derive<<<std::min(1024, (n + 255) / 256), 256, 0, st>>>(m->P + m->off[l], m->P + m->off[l] + uint64_t(K) * dout,
                                                             int(K), int(dout), int(m->npad[l]), int(m->npadT[l]),
                                                             m->W[l], m->b[l], m->Wt[l], m->Whi[l], m->Wlo[l],
                                                             m->Wdhi[l], m->Wdlo[l]);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

}  // namespace

extern "C" {

int fdg_sage_create(fdg_ctx* ctx, const uint32_t* dims, uint32_t n_layers, const uint32_t* fanouts,
                    uint32_t max_seeds, fdg_sage** out) {
    if (n_layers == 0 || n_layers > FDG_MAX_LAYERS) return fail(FDG_INVALID_ARG, "sage: n_layers must be in [1, 8]");
    if (ctx->row_bytes == 0) return fail(FDG_NOT_LOADED, "sage: no feature table loaded");
    const uint32_t esz = ctx->dtype == 1 ? 2 : 4;
    if (dims[0] * esz != ctx->row_bytes) return fail(FDG_INVALID_ARG, "sage: dims[0] must equal the feature row width");
    for (uint32_t l = 0; l <= n_layers; ++l)
        if (dims[l] == 0 || dims[l] % 4) return fail(FDG_INVALID_ARG, "sage: every dim must be a positive multiple of 4");
    for (uint32_t l = 0; l < n_layers; ++l)
        if (fanouts[l] == 0) return fail(FDG_INVALID_ARG, "fanouts: every entry must be >= 1");
    cudaSetDevice(ctx->device);
    auto m = new fdg_sage();
    m->ctx = ctx;
    m->L = n_layers;
    m->dims.assign(dims, dims + n_layers + 1);
    // D_j <= max_seeds * (1 + f1 + f1 f2 + ...) (Fanouts::max_batch_nodes, sampling.hpp:32-40), <= N
    uint64_t tot = 1, layer = 1;
    for (uint32_t j = 0; j <= n_layers; ++j) {
        m->bound.push_back(std::min<uint64_t>(uint64_t(max_seeds) * tot, std::max<uint64_t>(ctx->num_nodes, 1)));
        if (j < n_layers) {
            layer *= fanouts[j];
            tot += layer;
        }
    }
    auto al = [&](void** p, uint64_t bytes) { return cudaMalloc(p, std::max<uint64_t>(bytes, 16)); };
    uint64_t dmax = 0, amax = 0;  // largest gradient / dA buffers (floats)
    for (uint32_t l = 0; l < n_layers; ++l) {
        m->off.push_back(m->n_params);
        m->n_params += uint64_t(2) * dims[l] * dims[l + 1] + dims[l + 1];
        m->npad.push_back((dims[l + 1] + kBN - 1) / kBN * kBN);
        m->npadT.push_back((2 * dims[l] + kBN - 1) / kBN * kBN);
        const uint64_t rows = m->bound[n_layers - 1 - l];  // layer l+1 writes D_{L-1-l}
        dmax = std::max<uint64_t>(dmax, rows * dims[l + 1]);
        dmax = std::max<uint64_t>(dmax, m->bound[n_layers - l] * dims[l]);  // its input gradient
        amax = std::max<uint64_t>(amax, rows * 2 * dims[l]);
        m->tn_floats = std::max<uint64_t>(m->tn_floats, uint64_t(tn_slices(rows)) * (2 * dims[l] + 1) * dims[l + 1]);
        const uint64_t tiles = uint64_t((2 * dims[l] + 127) / 128) * ((dims[l + 1] + 127) / 128);
        const uint64_t z = std::min<uint64_t>((2 * uint64_t(ctx->sm_count) + tiles - 1) / tiles, (rows + 31) / 32);
        m->wz.push_back(int(std::max<uint64_t>(z, 1)));
        m->tn_floats = std::max<uint64_t>(m->tn_floats, uint64_t(m->wz.back()) * (2 * dims[l] + 1) * dims[l + 1]);
    }
    cudaError_t e = al((void**)&m->seg, m->bound[n_layers - 1] * sizeof(uint2));
    if (e == cudaSuccess) e = al((void**)&m->P, m->n_params * 4);
    if (e == cudaSuccess) e = al((void**)&m->G, m->n_params * 4);
    if (e == cudaSuccess) e = cudaMemset(m->P, 0, m->n_params * 4);
    if (e == cudaSuccess) e = cudaMemset(m->G, 0, m->n_params * 4);
    if (e == cudaSuccess) e = al((void**)&m->logits, m->bound[0] * dims[n_layers] * 4);
    if (e == cudaSuccess) e = al((void**)&m->row_loss, m->bound[0] * 4);
    if (e == cudaSuccess) e = al((void**)&m->dbuf[0], dmax * 4);
    if (e == cudaSuccess) e = al((void**)&m->dbuf[1], dmax * 4);
    if (e == cudaSuccess) e = al((void**)&m->dA, amax * 4);
    if (e == cudaSuccess) e = al((void**)&m->tn_part, m->tn_floats * 4);
    uint32_t zmax = 0;
    for (uint32_t l = 0; l < n_layers; ++l) zmax = std::max(zmax, m->npadT[l]);
    if (e == cudaSuccess) e = al((void**)&m->zeros, uint64_t(zmax) * 4);
    if (e == cudaSuccess) e = cudaMemset(m->zeros, 0, uint64_t(zmax) * 4);
    // split-K slices: at most kMaxSplit x (rows of the largest split layer) x N
    for (uint32_t k = 1; k <= n_layers; ++k) {
        const uint64_t r = m->bound[n_layers - k];
        const int z = splitk_for(r, 2 * dims[k - 1], (dims[k] + kBN - 1) / kBN, ctx->sm_count);
        if (z > 1) m->partial_floats = std::max<uint64_t>(m->partial_floats, uint64_t(z) * r * dims[k]);
    }
    if (e == cudaSuccess && m->partial_floats) e = al((void**)&m->partial, m->partial_floats * 4);
    m->W.assign(n_layers, nullptr);
    m->b.assign(n_layers, nullptr);
    m->Wt.assign(n_layers, nullptr);
    m->Whi.assign(n_layers, nullptr);
    m->Wlo.assign(n_layers, nullptr);
    m->Al.assign(n_layers, nullptr);
    m->Hl.assign(n_layers, nullptr);
    m->mapA.resize(n_layers);
    m->mapBhi.resize(n_layers);
    m->mapBlo.resize(n_layers);
    m->tc_ok.assign(n_layers, 0);
    m->set.assign(n_layers, 0);
    for (uint32_t l = 0; l < n_layers && e == cudaSuccess; ++l) {
        const uint32_t K = 2 * dims[l], np = m->npad[l];
        const uint64_t rows = m->bound[n_layers - 1 - l];
        e = al((void**)&m->W[l], uint64_t(K) * np * 4);
        if (e == cudaSuccess) e = al((void**)&m->b[l], uint64_t(np) * 4);
        if (e == cudaSuccess) e = al((void**)&m->Wt[l], uint64_t(dims[l + 1]) * m->npadT[l] * 4);
        if (e == cudaSuccess) e = al((void**)&m->Al[l], rows * K * 4);
        if (e == cudaSuccess && l + 1 < n_layers) e = al((void**)&m->Hl[l], rows * dims[l + 1] * 4);
        if (e != cudaSuccess || K % 32) continue;
        e = al((void**)&m->Whi[l], uint64_t(np) * K * 4);
        if (e == cudaSuccess) e = al((void**)&m->Wlo[l], uint64_t(np) * K * 4);
        if (e != cudaSuccess) break;
        if (tc_make_map(&m->mapA[l], m->Al[l], rows, K) == FDG_OK &&
            tc_make_map(&m->mapBhi[l], m->Whi[l], np, K) == FDG_OK &&
            tc_make_map(&m->mapBlo[l], m->Wlo[l], np, K) == FDG_OK)
            m->tc_ok[l] = 1;
    }
    if (g_sage_gemm) tc_write_hi(nullptr);  // the kind::tf32 truncation check, once per device, before any run
    m->Wdhi.assign(n_layers, nullptr);
    m->Wdlo.assign(n_layers, nullptr);
    m->mapDk.resize(n_layers);
    m->mapWdhi.resize(n_layers);
    m->mapWdlo.resize(n_layers);
    m->tc_da.assign(n_layers, 0);
    for (uint32_t l = 1; l < n_layers && e == cudaSuccess; ++l) {  // layer 0 needs no input gradient
        const uint64_t rows = m->bound[n_layers - 1 - l];
        const uint32_t K2 = 2 * dims[l];
        e = al((void**)&m->Wdhi[l], uint64_t(K2) * dims[l + 1] * 4);
        if (e == cudaSuccess) e = al((void**)&m->Wdlo[l], uint64_t(K2) * dims[l + 1] * 4);
        if (e != cudaSuccess) break;
        if (tc_make_map(&m->mapDk[l], m->dbuf[(n_layers - 1 - l) % 2], rows, dims[l + 1]) == FDG_OK &&
            tc_make_map(&m->mapWdhi[l], m->Wdhi[l], K2, dims[l + 1]) == FDG_OK &&
            tc_make_map(&m->mapWdlo[l], m->Wdlo[l], K2, dims[l + 1]) == FDG_OK)
            m->tc_da[l] = 1;
    }
    m->mapAmn.resize(n_layers);
    m->mapDmn.resize(n_layers);
    for (uint32_t l = 0; l < n_layers && e == cudaSuccess; ++l) {
        const uint64_t rows = m->bound[n_layers - 1 - l];
        // the backward's output gradient of layer l+1 sits in dbuf[(L-1-l) % 2] (k_loss_grad
        // writes dbuf[0] for the top layer, each layer's input gradient the other buffer)
        float* dout_buf = m->dbuf[(n_layers - 1 - l) % 2];
        if (tc_make_map_mn(&m->mapAmn[l], m->Al[l], rows, 2 * dims[l]) != FDG_OK ||
            tc_make_map_mn(&m->mapDmn[l], dout_buf, rows, dims[l + 1]) != FDG_OK)
            m->wz[l] = 0;
    }
    if (e != cudaSuccess) {
        fdg_sage_destroy(m);
        return cuda_fail(e, "fdg_sage_create", __FILE__, __LINE__);
    }
    *out = m;
    return FDG_OK;
}

int fdg_sage_destroy(fdg_sage* m) {
    if (!m) return FDG_OK;
    cudaSetDevice(m->ctx->device);
    for (void* p : {(void*)m->seg, (void*)m->P, (void*)m->G, (void*)m->logits, (void*)m->partial,
                    (void*)m->row_loss, (void*)m->dbuf[0], (void*)m->dbuf[1], (void*)m->dA, (void*)m->zeros,
                    (void*)m->tn_part})
        cudaFree(p);
    for (auto* v : {&m->W, &m->b, &m->Wt, &m->Whi, &m->Wlo, &m->Al, &m->Hl, &m->Wdhi, &m->Wdlo})
        for (float* p : *v) cudaFree(p);
    delete m;
    return FDG_OK;
}

int fdg_sage_set_layer(fdg_sage* m, uint32_t layer, const float* w_neigh, const float* w_self, const float* bias) {
    if (layer >= m->L) return fail(FDG_OUT_OF_RANGE, "sage_set_layer: layer out of range");
    cudaSetDevice(m->ctx->device);
    const uint32_t din = m->dims[layer], dout = m->dims[layer + 1];
    std::vector<float> blk(uint64_t(2) * din * dout + dout);
    std::memcpy(blk.data(), w_neigh, uint64_t(din) * dout * 4);
    std::memcpy(blk.data() + uint64_t(din) * dout, w_self, uint64_t(din) * dout * 4);
    for (uint32_t c = 0; c < dout; ++c) blk[uint64_t(2) * din * dout + c] = bias ? bias[c] : 0.f;
    FDG_CUDA(cudaMemcpy(m->P + m->off[layer], blk.data(), blk.size() * 4, cudaMemcpyHostToDevice));
    FDG_TRY(derive_layer(m, layer, nullptr));
    FDG_CUDA(cudaDeviceSynchronize());
    m->set[layer] = 1;
    return FDG_OK;
}

int fdg_sage_get_layer(fdg_sage* m, uint32_t layer, int grads, float* w_neigh, float* w_self, float* bias) {
    if (layer >= m->L) return fail(FDG_OUT_OF_RANGE, "sage_get_layer: layer out of range");
    cudaSetDevice(m->ctx->device);
    FDG_CUDA(cudaDeviceSynchronize());
    const uint32_t din = m->dims[layer], dout = m->dims[layer + 1];
    const float* src = (grads ? m->G : m->P) + m->off[layer];
    const uint64_t wn = uint64_t(din) * dout;
    if (w_neigh) FDG_CUDA(cudaMemcpy(w_neigh, src, wn * 4, cudaMemcpyDeviceToHost));
    if (w_self) FDG_CUDA(cudaMemcpy(w_self, src + wn, wn * 4, cudaMemcpyDeviceToHost));
    if (bias) FDG_CUDA(cudaMemcpy(bias, src + 2 * wn, dout * 4, cudaMemcpyDeviceToHost));
    return FDG_OK;
}

int fdg_sage_buffers(fdg_sage* m, float** params_dev, float** grads_dev, uint64_t* n_floats) {
    if (params_dev) *params_dev = m->P;
    if (grads_dev) *grads_dev = m->G;
    if (n_floats) *n_floats = m->n_params;
    return FDG_OK;
}

int fdg_sage_forward(fdg_sage* m, void* stv, const void* x_dev, const uint64_t* nodes_dev, const uint32_t* edges_dev,
                     const fdg_batch_counts* counts_dev, uint64_t label_seed, float* loss_dev, float* logits_dev) {
    for (uint32_t l = 0; l < m->L; ++l)
        if (!m->set[l]) return fail(FDG_NOT_LOADED, "sage_forward: layer " + std::to_string(l) + " has no weights");
    if (!loss_dev) return fail(FDG_INVALID_ARG, "sage_forward: null loss output");
    cudaStream_t st = (cudaStream_t)stv;
    const Ctx& c = *m->ctx;
    const uint32_t L = m->L;
    const uint2* edges = reinterpret_cast<const uint2*>(edges_dev);
    FDG_TRACE("sage", st);
    {
        const uint64_t r = m->bound[L - 1];
        k_seg_clear<<<uint32_t(std::min<uint64_t>((r + 255) / 256, uint64_t(c.sm_count) * 8)), 256, 0, st>>>(
            m->seg, counts_dev, int(L) - 1);
        k_seg<<<c.sm_count * 8, 256, 0, st>>>(edges, counts_dev, m->seg);
    }
    const float* hin = nullptr;
    for (uint32_t k = 1; k <= L; ++k) {
        const int j = int(L - k);  // destinations: D_j
        const uint32_t din = m->dims[k - 1], dout = m->dims[k];
        const uint64_t rows = m->bound[j];
        float* A = m->Al[k - 1];
        const uint32_t agg_blocks = uint32_t(std::min<uint64_t>((rows + 7) / 8, uint64_t(c.sm_count) * 16));
        if (k == 1 && c.dtype == 1)
            k_aggregate<__half><<<agg_blocks, 256, 0, st>>>(static_cast<const __half*>(x_dev), din, m->seg, edges,
                                                            counts_dev, j, A);
        else
            k_aggregate<float><<<agg_blocks, 256, 0, st>>>(k == 1 ? static_cast<const float*>(x_dev) : hin, din,
                                                           m->seg, edges, counts_dev, j, A);
        float* hout = k == L ? m->logits : m->Hl[k - 1];
        if (g_sage_gemm == 1 && m->tc_ok[k - 1]) {
            FDG_TRY(tc_gemm(st, m->mapA[k - 1], m->mapBhi[k - 1], m->mapBlo[k - 1], m->b[k - 1], hout, counts_dev,
                            j, rows, int(dout), int(m->npad[k - 1]), int(2 * din), k != L));
            hin = hout;
            continue;
        }
        const int z = splitk_for(rows, 2 * din, m->npad[k - 1] / kBN, c.sm_count);
        dim3 grid(m->npad[k - 1] / kBN, uint32_t((rows + kBM - 1) / kBM), uint32_t(z));
        float* gout = z > 1 ? m->partial : hout;
        const uint64_t slice = rows * dout;
        if (k == L)
            k_sgemm<false><<<grid, 256, 0, st>>>(A, m->W[k - 1], m->b[k - 1], gout, counts_dev, j, int(dout),
                                                 int(2 * din), int(m->npad[k - 1]), slice);
        else
            k_sgemm<true><<<grid, 256, 0, st>>>(A, m->W[k - 1], m->b[k - 1], gout, counts_dev, j, int(dout),
                                                int(2 * din), int(m->npad[k - 1]), slice);
        if (z > 1) {
            const int sb = int(std::min<uint64_t>((slice / 4 + 255) / 256, uint64_t(c.sm_count) * 8));
            if (k == L)
                k_splitk_sum<false><<<sb, 256, 0, st>>>(m->partial, z, slice, m->b[k - 1], hout, counts_dev, j,
                                                        int(dout));
            else
                k_splitk_sum<true><<<sb, 256, 0, st>>>(m->partial, z, slice, m->b[k - 1], hout, counts_dev, j,
                                                       int(dout));
        }
        hin = hout;
    }
    k_loss_rows<<<uint32_t((m->bound[0] + 7) / 8), 256, 0, st>>>(m->logits, int(m->dims[L]), nodes_dev, counts_dev,
                                                                  label_seed, m->row_loss, logits_dev);
    k_loss_mean<<<1, kLossThreads, 0, st>>>(m->row_loss, counts_dev, loss_dev);
    FDG_CUDA(cudaGetLastError());
    m->forwarded = true;
    return FDG_OK;
}

// Backward of the last forward (same batch, same stream): gradients of the mean loss w.r.t.
// every layer's W_neigh, W_self and b into the gradient buffer.
int fdg_sage_backward(fdg_sage* m, void* stv, const uint64_t* nodes_dev, const uint32_t* edges_dev,
                      const fdg_batch_counts* counts_dev, uint64_t label_seed) {
    if (!m->forwarded) return fail(FDG_NOT_LOADED, "sage_backward: no forward to differentiate");
    cudaStream_t st = (cudaStream_t)stv;
    const Ctx& c = *m->ctx;
    const uint32_t L = m->L;
    const uint2* edges = reinterpret_cast<const uint2*>(edges_dev);
    FDG_TRACE("sage_bwd", st);
    float* cur = m->dbuf[0];
    k_loss_grad<<<uint32_t((m->bound[0] + 7) / 8), 256, 0, st>>>(m->logits, int(m->dims[L]), nodes_dev, counts_dev,
                                                                  label_seed, cur);
    for (uint32_t k = L; k >= 1; --k) {
        const int j = int(L - k);
        const uint32_t din = m->dims[k - 1], dout = m->dims[k], K = 2 * din;
        const uint64_t rows = m->bound[j];
        if (k < L)
            k_relu_mask<<<uint32_t(std::min<uint64_t>((rows * dout + 255) / 256, uint64_t(c.sm_count) * 8)), 256, 0,
                          st>>>(cur, m->Hl[k - 1], counts_dev, j, int(dout));
        // weight + bias gradients: A^T . dOut over the D_j rows, in row slices
        const bool tc = g_sage_gemm == 1 && m->wz[k - 1] > 0;
        const int Z = tc ? m->wz[k - 1] : tn_slices(rows);
        float* Pb = m->tn_part + uint64_t(Z) * K * dout;
        if (tc) {
            FDG_TRY(tc_wgrad(st, m->mapAmn[k - 1], m->mapDmn[k - 1], m->tn_part, counts_dev, j, int(K), int(dout), Z));
            launch_colsum(cur, counts_dev, j, int(dout), Pb, Z, st);
        } else {
            dim3 grid((dout + kTn - 1) / kTn, (K + kTn - 1) / kTn, uint32_t(Z));
            k_gemm_tn<<<grid, 256, 0, st>>>(m->Al[k - 1], cur, counts_dev, j, int(K), int(dout), m->tn_part, Pb);
        }
        const int kn = int(K * dout);
        k_tn_sum<<<std::min(1024, (kn + int(dout) + 255) / 256), 256, 0, st>>>(m->tn_part, Pb, Z, kn, int(dout),
                                                                              m->G + m->off[k - 1]);
        if (k == 1) break;
        // input gradient: dA = dOut . [W_neigh; W_self]^T, then scatter to h^{k-1}
        if (g_sage_gemm == 1 && m->tc_da[k - 1]) {
            FDG_TRY(tc_gemm(st, m->mapDk[k - 1], m->mapWdhi[k - 1], m->mapWdlo[k - 1], m->zeros, m->dA, counts_dev,
                            j, rows, int(K), int(m->npadT[k - 1]), int(dout), false));
        } else {
            dim3 ag(m->npadT[k - 1] / kBN, uint32_t((rows + kBM - 1) / kBM), 1);
            k_sgemm<false><<<ag, 256, 0, st>>>(cur, m->Wt[k - 1], m->zeros, m->dA, counts_dev, j, int(K), int(dout),
                                               int(m->npadT[k - 1]), 0);
        }
        float* nxt = cur == m->dbuf[0] ? m->dbuf[1] : m->dbuf[0];
        const uint64_t in_rows = m->bound[j + 1];
        k_dh_self<<<uint32_t(std::min<uint64_t>((in_rows * din / 4 + 255) / 256, uint64_t(c.sm_count) * 8)), 256, 0,
                    st>>>(m->dA, int(din), counts_dev, j, nxt);
        k_dh_neigh<<<uint32_t(std::min<uint64_t>((rows + 7) / 8, uint64_t(c.sm_count) * 16)), 256, 0, st>>>(
            m->dA, int(din), m->seg, edges, counts_dev, j, nxt);
        cur = nxt;
    }
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

// SGD step from the gradient buffer (after an optional all-reduce), then refresh every
// derived weight copy (CUDA-core, tensor-core and transposed layouts).
int fdg_sage_sgd(fdg_sage* m, void* stv, float lr) {
    cudaStream_t st = (cudaStream_t)stv;
    k_sgd<<<uint32_t(std::min<uint64_t>((m->n_params + 255) / 256, uint64_t(m->ctx->sm_count) * 4)), 256, 0, st>>>(
        m->P, m->G, m->n_params, lr);
    for (uint32_t l = 0; l < m->L; ++l) FDG_TRY(derive_layer(m, l, st));
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

}  // extern "C"

extern "C" {
// Test hook: out[Kin x N] = A^T . B for device A [R x Kin], B [R x N] through the backward's
// weight-gradient engine (option "sage_gemm": tensor cores or CUDA cores), split into Z slices.
int fdg_sage_wgrad_test(const float* A, const float* B, uint32_t R, uint32_t Kin, uint32_t N, uint32_t Z, float* out) {
    fdg_batch_counts h{};
    h.n_nodes = R;
    h.layer_nodes[1] = R;
    fdg_batch_counts* cnt = nullptr;
    float* part = nullptr;
    FDG_CUDA(cudaMalloc(&cnt, sizeof(h)));
    FDG_CUDA(cudaMemcpy(cnt, &h, sizeof(h), cudaMemcpyHostToDevice));
    FDG_CUDA(cudaMalloc(&part, (uint64_t(Z) * (Kin + 1) * N) * 4));
    int rc = FDG_OK;
    if (g_sage_gemm == 1) {
        CUtensorMap ma, mb;
        rc = tc_make_map_mn(&ma, A, R, Kin);
        if (rc == FDG_OK) rc = tc_make_map_mn(&mb, B, R, N);
        if (rc == FDG_OK) rc = tc_wgrad(nullptr, ma, mb, part, cnt, 0, int(Kin), int(N), int(Z));
    } else {
        dim3 grid((N + kTn - 1) / kTn, (Kin + kTn - 1) / kTn, Z);
        k_gemm_tn<<<grid, 256>>>(A, B, cnt, 0, int(Kin), int(N), part, part + uint64_t(Z) * Kin * N);
    }
    if (rc == FDG_OK) {
        launch_colsum(B, cnt, 0, int(N), part + uint64_t(Z) * Kin * N, int(Z), nullptr);
        k_tn_sum<<<256, 256>>>(part, part + uint64_t(Z) * Kin * N, int(Z), int(Kin * N), int(N), out);
        if (cudaDeviceSynchronize() != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "wgrad_test", __FILE__, __LINE__);
    }
    cudaFree(cnt);
    cudaFree(part);
    return rc;
}
}  // extern "C"
