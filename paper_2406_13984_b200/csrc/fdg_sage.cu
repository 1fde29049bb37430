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
#include <string>
#include <vector>

#include "fdg_internal.cuh"

namespace fdg {
// tensor-core GEMM (fdg_sage_tc.cu)
int tc_make_map(CUtensorMap* map, const float* base, uint64_t rows, uint32_t K);
void tc_split_weights(const float* Wcat, uint32_t K, uint32_t dout, uint32_t npad, std::vector<float>& hi,
                      std::vector<float>& lo);
int tc_gemm(cudaStream_t st, const CUtensorMap& tA, const CUtensorMap& tBhi, const CUtensorMap& tBlo,
            const float* bias, float* C, const fdg_batch_counts* cnt, int j, uint64_t rows_bound, int N, int npad,
            int K, bool relu);
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
    float4 ra = *reinterpret_cast<const float4*>(Ap);
    float4 rb = *reinterpret_cast<const float4*>(Wp);
    As[0][ak + 0][ar] = ra.x;
    As[0][ak + 1][ar] = ra.y;
    As[0][ak + 2][ar] = ra.z;
    As[0][ak + 3][ar] = ra.w;
    *reinterpret_cast<float4*>(&Bs[0][bk][bn]) = rb;
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += kBK) {
        const bool more = k0 + kBK < K;
        if (more) {
            ra = *reinterpret_cast<const float4*>(Ap + k0 + kBK);
            rb = *reinterpret_cast<const float4*>(Wp + size_t(k0 + kBK) * Npad);
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

}  // namespace

struct Sage {
    Ctx* ctx = nullptr;
    uint32_t L = 0;
    std::vector<uint32_t> dims;     // L + 1
    std::vector<uint32_t> npad;     // per layer: d_out rounded up to kBN
    std::vector<uint64_t> bound;    // bound[j] >= D_j, j = 0..L
    std::vector<float*> W, b;       // per layer: [2 d_in x npad], [npad]
    uint2* seg = nullptr;
    float* A = nullptr;
    float* H[2] = {nullptr, nullptr};
    float* logits = nullptr;
    float* partial = nullptr;       // split-K slices
    uint64_t partial_floats = 0;
    float* row_loss = nullptr;
    std::vector<uint8_t> set;
    // tensor-core path: transposed K-major W_hi / W_lo and TMA maps per layer
    std::vector<float*> Whi, Wlo;
    std::vector<CUtensorMap> mapA, mapBhi, mapBlo;
    std::vector<uint8_t> tc_ok;     // layer K is a multiple of 32 and the maps were built
};

}  // namespace fdg

struct fdg_sage : fdg::Sage {};

using namespace fdg;

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
    uint32_t max_in = 0, max_out = 0;
    for (uint32_t l = 0; l < n_layers; ++l) {
        max_in = std::max(max_in, dims[l]);
        max_out = std::max(max_out, dims[l + 1]);
    }
    const uint64_t rows = m->bound[n_layers - 1];  // destinations of layer 1
    auto al = [&](void** p, uint64_t bytes) { return cudaMalloc(p, std::max<uint64_t>(bytes, 16)); };
    cudaError_t e = al((void**)&m->seg, rows * sizeof(uint2));
    if (e == cudaSuccess) e = al((void**)&m->A, rows * 2 * max_in * 4);
    if (e == cudaSuccess) e = al((void**)&m->H[0], rows * max_out * 4);
    if (e == cudaSuccess) e = al((void**)&m->H[1], rows * max_out * 4);
    if (e == cudaSuccess) e = al((void**)&m->logits, m->bound[0] * dims[n_layers] * 4);
    if (e == cudaSuccess) e = al((void**)&m->row_loss, m->bound[0] * 4);
    // split-K slices: at most kMaxSplit x (rows of the largest split layer) x N
    for (uint32_t k = 1; k <= n_layers; ++k) {
        const uint64_t r = m->bound[n_layers - k];
        const int z = splitk_for(r, 2 * dims[k - 1], (dims[k] + kBN - 1) / kBN, ctx->sm_count);
        if (z > 1) m->partial_floats = std::max<uint64_t>(m->partial_floats, uint64_t(z) * r * dims[k]);
    }
    if (e == cudaSuccess && m->partial_floats) e = al((void**)&m->partial, m->partial_floats * 4);
    for (uint32_t l = 0; l < n_layers && e == cudaSuccess; ++l) {
        const uint32_t np = (dims[l + 1] + kBN - 1) / kBN * kBN;
        m->npad.push_back(np);
        float *w = nullptr, *bb = nullptr;
        e = al((void**)&w, uint64_t(2) * dims[l] * np * 4);
        if (e == cudaSuccess) e = al((void**)&bb, uint64_t(np) * 4);
        if (e == cudaSuccess) e = cudaMemset(w, 0, uint64_t(2) * dims[l] * np * 4);
        if (e == cudaSuccess) e = cudaMemset(bb, 0, uint64_t(np) * 4);
        m->W.push_back(w);
        m->b.push_back(bb);
    }
    m->set.assign(n_layers, 0);
    m->Whi.assign(n_layers, nullptr);
    m->Wlo.assign(n_layers, nullptr);
    m->mapA.resize(n_layers);
    m->mapBhi.resize(n_layers);
    m->mapBlo.resize(n_layers);
    m->tc_ok.assign(n_layers, 0);
    for (uint32_t l = 0; l < n_layers && e == cudaSuccess; ++l) {
        const uint32_t K = 2 * dims[l];
        if (K % 32) continue;
        e = al((void**)&m->Whi[l], uint64_t(m->npad[l]) * K * 4);
        if (e == cudaSuccess) e = al((void**)&m->Wlo[l], uint64_t(m->npad[l]) * K * 4);
        if (e != cudaSuccess) break;
        const uint64_t rows_l = m->bound[n_layers - 1 - l];  // layer l+1 writes D_{L-1-l}
        if (tc_make_map(&m->mapA[l], m->A, rows_l, K) == FDG_OK &&
            tc_make_map(&m->mapBhi[l], m->Whi[l], m->npad[l], K) == FDG_OK &&
            tc_make_map(&m->mapBlo[l], m->Wlo[l], m->npad[l], K) == FDG_OK)
            m->tc_ok[l] = 1;
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
    cudaFree(m->seg);
    cudaFree(m->A);
    cudaFree(m->H[0]);
    cudaFree(m->H[1]);
    cudaFree(m->logits);
    cudaFree(m->partial);
    cudaFree(m->row_loss);
    for (auto p : m->W) cudaFree(p);
    for (auto p : m->b) cudaFree(p);
    for (auto p : m->Whi) cudaFree(p);
    for (auto p : m->Wlo) cudaFree(p);
    delete m;
    return FDG_OK;
}

int fdg_sage_set_layer(fdg_sage* m, uint32_t layer, const float* w_neigh, const float* w_self, const float* bias) {
    if (layer >= m->L) return fail(FDG_OUT_OF_RANGE, "sage_set_layer: layer out of range");
    cudaSetDevice(m->ctx->device);
    const uint32_t din = m->dims[layer], dout = m->dims[layer + 1], np = m->npad[layer];
    std::vector<float> w(uint64_t(2) * din * np, 0.f), bb(np, 0.f);
    for (uint32_t k = 0; k < din; ++k)
        for (uint32_t c = 0; c < dout; ++c) {
            w[uint64_t(k) * np + c] = w_neigh[uint64_t(k) * dout + c];
            w[uint64_t(din + k) * np + c] = w_self[uint64_t(k) * dout + c];
        }
    for (uint32_t c = 0; c < dout; ++c) bb[c] = bias ? bias[c] : 0.f;
    FDG_CUDA(cudaMemcpy(m->W[layer], w.data(), w.size() * 4, cudaMemcpyHostToDevice));
    if (m->Whi[layer]) {
        std::vector<float> cat(uint64_t(2) * din * dout), hi, lo;
        for (uint32_t k = 0; k < din; ++k)
            for (uint32_t c = 0; c < dout; ++c) {
                cat[uint64_t(k) * dout + c] = w_neigh[uint64_t(k) * dout + c];
                cat[uint64_t(din + k) * dout + c] = w_self[uint64_t(k) * dout + c];
            }
        tc_split_weights(cat.data(), 2 * din, dout, np, hi, lo);
        FDG_CUDA(cudaMemcpy(m->Whi[layer], hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
        FDG_CUDA(cudaMemcpy(m->Wlo[layer], lo.data(), lo.size() * 4, cudaMemcpyHostToDevice));
    }
    FDG_CUDA(cudaMemcpy(m->b[layer], bb.data(), bb.size() * 4, cudaMemcpyHostToDevice));
    m->set[layer] = 1;
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
        const uint32_t agg_blocks = uint32_t(std::min<uint64_t>((rows + 7) / 8, uint64_t(c.sm_count) * 16));
        if (k == 1 && c.dtype == 1)
            k_aggregate<__half><<<agg_blocks, 256, 0, st>>>(static_cast<const __half*>(x_dev), din, m->seg, edges,
                                                            counts_dev, j, m->A);
        else
            k_aggregate<float><<<agg_blocks, 256, 0, st>>>(k == 1 ? static_cast<const float*>(x_dev) : hin, din,
                                                           m->seg, edges, counts_dev, j, m->A);
        float* hout = k == L ? m->logits : m->H[k & 1];
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
            k_sgemm<false><<<grid, 256, 0, st>>>(m->A, m->W[k - 1], m->b[k - 1], gout, counts_dev, j, int(dout),
                                                 int(2 * din), int(m->npad[k - 1]), slice);
        else
            k_sgemm<true><<<grid, 256, 0, st>>>(m->A, m->W[k - 1], m->b[k - 1], gout, counts_dev, j, int(dout),
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
    return FDG_OK;
}

}  // extern "C"
