// fdg_sage_tc.cu -- the train stage's GEMM on the 5th-generation tensor cores.
//
// C[M x N] = act(A[M x K] . W + b) for the GraphSAGE layers (fdg_sage.cu), fp32
// accurate via 3xTF32: every fp32 operand x splits into hi = x with the low 13
// mantissa bits cleared (exact in TF32) and lo = x - hi (exact in fp32), and
//   A . W ~= A_hi . W_hi + A_hi . W_lo + A_lo . W_hi
// accumulates in fp32 in TMEM (the dropped A_lo . W_lo term and lo's own TF32
// rounding are ~2^-20 relative), so the loss stays within 1e-5 of the fp64 oracle.
//
// Persistent CTAs (one per SM) walk the 128 x 128 output tiles, K in 32-element (128-byte) blocks:
//   warp 0 lane 0 : TMA producer -- A block (128 rows x 32) and W_hi / W_lo blocks
//                   (W stored transposed, K-major) into a 3-stage ring, 128-byte
//                   swizzled (the canonical K-major SW128 UMMA layout)
//   warps 4-7     : split the A block: A_lo = A - A_hi into its own tile (elementwise, so
//                   the swizzle is preserved; A_hi is A itself, see kWriteHi), fence to
//                   the async proxy, arrive
//   warps 8-11    : epilogue: tcgen05.ld 32 columns at a time, + bias, ReLU, then through a
//                   swizzled 4 KB smem block per warp into coalesced 128-byte row stores;
//                   two TMEM accumulators let tile i's epilogue overlap tile i+1's MMAs
//   warp 1 lane 0 : MMA issuer -- per K block 4 x 3 tcgen05.mma.kind::tf32
//                   (M=128, N=128, K=8) into one TMEM accumulator; tcgen05.commit
//                   frees the stage, the last commit signals the epilogue
//   warp 2        : TMEM allocation (2 x 128 columns) and release
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "fdg_internal.cuh"

namespace fdg {
namespace {

constexpr int kTcBM = 128, kTcBN = 128, kTcBK = 32, kTcStages = 3;
constexpr int kTcTile = kTcBM * kTcBK * 4;  // 16 KB (A and B tiles alike: 128 rows x 128 bytes)
constexpr int kTcStageBytes = 4 * kTcTile;  // A_hi (TMA lands here), A_lo, W_hi, W_lo
// kind::tf32 reads only the top 19 bits of an fp32 operand (the low 13 mantissa bits are
// ignored: truncation), so the TMA-landed block already is A_hi for the tensor core; the split
// warps only write A_lo = A - trunc(A). That is measured hardware behaviour, not a PTX
// guarantee: tc_write_hi() checks it once per device (the same GEMM with and without the
// explicit A_hi write must agree bit for bit) and turns the write on if it does not hold.
// Also pinned by the 1e-5 parity tests (rounding would be a ~2^-12 relative error).
constexpr int kTcThreads = 384;  // warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4-7 split, 8-11 epilogue
constexpr int kTcEpiBytes = 4 * 32 * 32 * 4;  // epilogue staging: a 32 x 32 fp32 block per epilogue warp
constexpr int kTcSmem = kTcStages * kTcStageBytes + 1024 /* alignment */ + 256 /* barriers */ + kTcEpiBytes;

__device__ __forceinline__ uint32_t d_rows_tc(const fdg_batch_counts* c, int j) {
    uint32_t d = 0;
    for (int i = 0; i <= j + 1 && i < FDG_MAX_LAYERS + 2; ++i) d = max(d, c->layer_nodes[i]);
    return min(d, c->n_nodes);
}

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(sa(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            sa(dst)),
        "l"(map), "r"(sa(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// K-major, 128-byte swizzle UMMA shared-memory descriptor: start >> 4, LBO unused (SW128
// K-major), SBO = 1024 B between 8-row groups, version 1 (sm_100), layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar))
                 : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
// hi = x with the low 13 mantissa bits cleared (exact in TF32), lo = x - hi
__device__ __forceinline__ void split4(float4 v, float4& h, float4& l) {
    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}

// TMEM -> registers: 32 columns of the accumulator, lane = row (32x32b shape).
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Epilogue store of one warp's 32 x 32 block (rows row0.., columns col0..) of out[.. x ld]: the
// row-per-lane registers go through a 4 KB staging block whose 16-byte chunks are XOR-swizzled
// by row (conflict-free both ways), then every store instruction writes four full 128-byte row
// segments (a row per lane wrote 32 half-used sectors). `bcol` = this lane's column's bias.
template <bool RELU, bool BIAS>
__device__ __forceinline__ void store_block(uint32_t stage, const uint32_t (&r)[32], float bcol, int lane,
                                            float* __restrict__ out, size_t ld, int row0, int rows, int col0,
                                            int cols) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        float4 v = make_float4(__uint_as_float(r[q * 4 + 0]), __uint_as_float(r[q * 4 + 1]),
                               __uint_as_float(r[q * 4 + 2]), __uint_as_float(r[q * 4 + 3]));
        if (BIAS) {
            v.x += __shfl_sync(0xffffffffu, bcol, q * 4 + 0);
            v.y += __shfl_sync(0xffffffffu, bcol, q * 4 + 1);
            v.z += __shfl_sync(0xffffffffu, bcol, q * 4 + 2);
            v.w += __shfl_sync(0xffffffffu, bcol, q * 4 + 3);
        }
        if (RELU) {
            v.x = fmaxf(v.x, 0.f);
            v.y = fmaxf(v.y, 0.f);
            v.z = fmaxf(v.z, 0.f);
            v.w = fmaxf(v.w, 0.f);
        }
        sts128(stage + lane * 128 + ((q ^ (lane & 7)) << 4), v);
    }
    __syncwarp();
    const int ch = lane & 7, col = col0 + ch * 4;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int rr = i * 4 + (lane >> 3);
        const float4 v = lds128(stage + rr * 128 + ((ch ^ (rr & 7)) << 4));
        if (row0 + rr < rows && col < cols) *reinterpret_cast<float4*>(out + size_t(row0 + rr) * ld + col) = v;
    }
    __syncwarp();  // the staging block is rewritten by the next call
}

// Persistent: CTA c takes tiles c, c + grid, ... (row-tile major: the column tiles of a row
// tile go to neighbouring CTAs at the same time, so the A block is reused from L2). Two TMEM accumulators (2 x 128
// columns): the epilogue of tile i overlaps the MMAs of tile i + 1.
template <bool RELU>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_sgemm_tc(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tBhi,
               const __grid_constant__ CUtensorMap tBlo, const float* __restrict__ bias, float* __restrict__ C,
               const fdg_batch_counts* cnt, int j, int N, int K, int n_tiles, int write_hi) {
    extern __shared__ uint8_t tc_raw[];
    const int M = int(d_rows_tc(cnt, j));
    const int tiles = (M + kTcBM - 1) / kTcBM * n_tiles;
    if (int(blockIdx.x) >= tiles) return;  // uniform, before any barrier or TMEM allocation
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kTcStages * kTcStageBytes);
    uint64_t* conv = full + kTcStages;
    uint64_t* empty = conv + kTcStages;
    uint64_t* tmem_full = empty + kTcStages;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;     // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto a_hi = [&](int s) { return sm + s * kTcStageBytes; };
    auto a_lo = [&](int s) { return sm + s * kTcStageBytes + kTcTile; };
    auto b_hi = [&](int s) { return sm + s * kTcStageBytes + 2 * kTcTile; };
    auto b_lo = [&](int s) { return sm + s * kTcStageBytes + 3 * kTcTile; };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(conv + s, 128);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tmem_full + a, 1);
            mbar_init(tmem_empty + a, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tmem_slot)), "n"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    const int nk = (K + kTcBK - 1) / kTcBK;  // a ragged last block is zero-filled by TMA (out of bounds)

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            int it = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int m0 = (t / n_tiles) * kTcBM, n0 = (t % n_tiles) * kTcBN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % kTcStages;
                    if (it >= kTcStages) mbar_wait(empty + s, uint32_t((it / kTcStages - 1) & 1));
                    mbar_expect_tx(full + s, 3 * kTcTile);
                    tma_load_2d(a_hi(s), &tA, full + s, kb * kTcBK, m0);
                    tma_load_2d(b_hi(s), &tBhi, full + s, kb * kTcBK, n0);
                    tma_load_2d(b_lo(s), &tBlo, full + s, kb * kTcBK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            // kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(kTcBN >> 3) << 17) |
                                   (uint32_t(kTcBM >> 4) << 24);
            int it = 0, ti = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++ti) {
                const int acc = ti & 1;
                if (ti >= 2) mbar_wait(tmem_empty + acc, uint32_t((ti / 2 - 1) & 1));  // epilogue drained it
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + uint32_t(acc * kTcBN);
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % kTcStages;
                    mbar_wait(conv + s, uint32_t((it / kTcStages) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int k = 0; k < kTcBK / 8; ++k) {  // UMMA_K = 8 tf32 = 32 bytes along the swizzled row
                        const uint64_t dah = umma_desc(sa(a_hi(s)) + k * 32), dal = umma_desc(sa(a_lo(s)) + k * 32);
                        const uint64_t dbh = umma_desc(sa(b_hi(s)) + k * 32), dbl = umma_desc(sa(b_lo(s)) + k * 32);
                        umma_tf32(d, dah, dbh, idesc, (kb | k) ? 1u : 0u);
                        umma_tf32(d, dah, dbl, idesc, 1u);
                        umma_tf32(d, dal, dbh, idesc, 1u);
                    }
                    umma_commit(empty + s);  // the stage is free once these MMAs have read it
                }
                umma_commit(tmem_full + acc);
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---- split A blocks: hi in place, lo into its own tile (same swizzled offsets)
        const int t4 = threadIdx.x - 128;
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % kTcStages;
                mbar_wait(full + s, uint32_t((it / kTcStages) & 1));
                const uint32_t hi = sa(a_hi(s)), lo = sa(a_lo(s));
                float4 v[kTcTile / 16 / 128];
#pragma unroll
                for (int u = 0; u < kTcTile / 16 / 128; ++u) v[u] = lds128(hi + (t4 + u * 128) * 16);  // all loads first
#pragma unroll
                for (int u = 0; u < kTcTile / 16 / 128; ++u) {
                    float4 h, l;
                    split4(v[u], h, l);
                    if (write_hi) sts128(hi + (t4 + u * 128) * 16, h);
                    sts128(lo + (t4 + u * 128) * 16, l);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
                mbar_arrive(conv + s);
            }
        }
    } else if (warp >= 8) {
        // ---- epilogue: TMEM lane = tile row; warp w reads lanes 32 (w % 4) ..
        const int wq = warp & 3;
        const uint32_t stage = sa(sm + kTcStages * kTcStageBytes + 256) + wq * 4096;
        int ti = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++ti) {
            const int acc = ti & 1;
            const int m0 = (t / n_tiles) * kTcBM, n0 = (t % n_tiles) * kTcBN;
            float bl[kTcBN / 32];  // lane's bias per 32-column chunk, loaded before the accumulator wait
#pragma unroll
            for (int c = 0; c < kTcBN / 32; ++c) bl[c] = n0 + c * 32 + lane < N ? bias[n0 + c * 32 + lane] : 0.f;
            mbar_wait(tmem_full + acc, uint32_t((ti / 2) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int c = 0; c < kTcBN / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem + (uint32_t(wq * 32) << 16) + uint32_t(acc * kTcBN + c * 32), r);
                if (c + 1 == kTcBN / 32) {  // every column of this accumulator is in registers: hand it back
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    mbar_arrive(tmem_empty + acc);
                }
                if (n0 + c * 32 < N) store_block<RELU, true>(stage, r, bl[c], lane, C, N, m0 + wq * 32, M, n0 + c * 32, N);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256) : "memory");
    }
}

// ---------------------------------------------------------------------------------
// Weight gradient of the backward pass, dW[Kin x N] = A^T . dOut over the R = D_j rows
// (A = the layer's saved input [R x Kin], dOut [R x N], both row-major), on the tensor
// cores with both operands MN-major: a 32-row block of A is 4 TMA boxes of 32 rows x
// 32 features (128-byte rows, 32-byte swizzle atoms), the MN-major SW128_BASE32B layout
// with LBO = 4 KB between 32-feature blocks and SBO = 512 B between 4-row groups; each
// UMMA (K = 8 rows) starts 1 KB further. Both operands are activations, so the split warps
// split both (hi in place, lo beside) and zero rows past R (stale rows of the buffers).
// Split-K over R: work item = (row slice z, output tile); slices write partial tiles
// P[z] that a fixed-order sum adds (k_tn_sum), so the result is deterministic.
// MN-major tf32 operands only support the "128B swizzle, 32B atom" layout (layout type 1,
// SWIZZLE_128B_BASE32B): 128-byte rows whose four 32-byte chunks are XOR-permuted by
// (row % 4) -- TMA's CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B. K groups are 4 rows (SBO = 512 B),
// 32-feature blocks are the 4 KB TMA boxes (LBO).
__device__ __forceinline__ uint64_t umma_desc_mn(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(4096 >> 4) << 16) | (uint64_t(512 >> 4) << 32) |
           (1ull << 46) | (1ull << 61);
}

__device__ __forceinline__ void split_tile(uint8_t* hi_t, uint8_t* lo_t, int t4, int row0, int R, int write_hi) {
    const uint32_t hi = sa(hi_t), lo = sa(lo_t);
    float4 v[kTcTile / 16 / 128];
#pragma unroll
    for (int u = 0; u < kTcTile / 16 / 128; ++u) v[u] = lds128(hi + (t4 + u * 128) * 16);
#pragma unroll
    for (int u = 0; u < kTcTile / 16 / 128; ++u) {
        const int i = t4 + u * 128;
        const int row = row0 + ((i * 16) & 4095) / 128;  // 4 KB boxes of 32 rows x 128 B
        const bool past = row >= R;  // stale rows of the buffers: zero both halves
        if (past) v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 h, l;
        split4(v[u], h, l);
        if (write_hi || past) sts128(hi + i * 16, h);
        sts128(lo + i * 16, l);
    }
}

__global__ void __launch_bounds__(kTcThreads, 1)
    k_wgrad_tc(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, float* __restrict__ P,
               const fdg_batch_counts* cnt, int j, int Kin, int N, int m_tiles, int n_tiles, int Z, int write_hi) {
    extern __shared__ uint8_t tc_raw[];
    const int R = int(d_rows_tc(cnt, j));
    const int tiles = m_tiles * n_tiles, items = tiles * Z;
    const int nkb = (R + kTcBK - 1) / kTcBK, per = (nkb + Z - 1) / Z;
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kTcStages * kTcStageBytes);
    uint64_t* conv = full + kTcStages;
    uint64_t* empty = conv + kTcStages;
    uint64_t* tmem_full = empty + kTcStages;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;     // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto a_hi = [&](int s) { return sm + s * kTcStageBytes; };
    auto a_lo = [&](int s) { return sm + s * kTcStageBytes + kTcTile; };
    auto b_hi = [&](int s) { return sm + s * kTcStageBytes + 2 * kTcTile; };
    auto b_lo = [&](int s) { return sm + s * kTcStageBytes + 3 * kTcTile; };
    auto kb_range = [&](int z, int& k0, int& k1) {
        k0 = min(nkb, z * per);
        k1 = min(nkb, k0 + per);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(conv + s, 128);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tmem_full + a, 1);
            mbar_init(tmem_empty + a, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tmem_slot)), "n"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer: 4 boxes of A and 4 of B per 32-row block
            int it = 0;
            for (int t = blockIdx.x; t < items; t += gridDim.x) {
                const int tile = t % tiles, z = t / tiles;
                const int m0 = (tile / n_tiles) * kTcBM, n0 = (tile % n_tiles) * kTcBN;
                int k0, k1;
                kb_range(z, k0, k1);
                for (int kb = k0; kb < k1; ++kb, ++it) {
                    const int s = it % kTcStages;
                    if (it >= kTcStages) mbar_wait(empty + s, uint32_t((it / kTcStages - 1) & 1));
                    mbar_expect_tx(full + s, 2 * kTcTile);
                    for (int q = 0; q < 4; ++q) {
                        tma_load_2d(a_hi(s) + q * 4096, &tA, full + s, m0 + 32 * q, kb * kTcBK);
                        tma_load_2d(b_hi(s) + q * 4096, &tB, full + s, n0 + 32 * q, kb * kTcBK);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer (A and B MN-major)
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                                   (uint32_t(kTcBN >> 3) << 17) | (uint32_t(kTcBM >> 4) << 24);
            int it = 0, ti = 0;
            for (int t = blockIdx.x; t < items; t += gridDim.x, ++ti) {
                const int acc = ti & 1;
                int k0, k1;
                kb_range(t / tiles, k0, k1);
                if (ti >= 2) mbar_wait(tmem_empty + acc, uint32_t((ti / 2 - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + uint32_t(acc * kTcBN);
                for (int kb = k0; kb < k1; ++kb, ++it) {
                    const int s = it % kTcStages;
                    mbar_wait(conv + s, uint32_t((it / kTcStages) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int k = 0; k < kTcBK / 8; ++k) {  // 8 rows per UMMA: the next 1 KB row group
                        const uint64_t dah = umma_desc_mn(sa(a_hi(s)) + k * 1024),
                                       dal = umma_desc_mn(sa(a_lo(s)) + k * 1024);
                        const uint64_t dbh = umma_desc_mn(sa(b_hi(s)) + k * 1024),
                                       dbl = umma_desc_mn(sa(b_lo(s)) + k * 1024);
                        umma_tf32(d, dah, dbh, idesc, (kb > k0 || k) ? 1u : 0u);
                        umma_tf32(d, dah, dbl, idesc, 1u);
                        umma_tf32(d, dal, dbh, idesc, 1u);
                    }
                    umma_commit(empty + s);
                }
                umma_commit(tmem_full + acc);  // (an empty slice commits at once: its epilogue writes zeros)
            }
        }
    } else if (warp >= 4 && warp < 8) {
        const int t4 = threadIdx.x - 128;
        int it = 0;
        for (int t = blockIdx.x; t < items; t += gridDim.x) {
            int k0, k1;
            kb_range(t / tiles, k0, k1);
            for (int kb = k0; kb < k1; ++kb, ++it) {
                const int s = it % kTcStages;
                mbar_wait(full + s, uint32_t((it / kTcStages) & 1));
                split_tile(a_hi(s), a_lo(s), t4, kb * kTcBK, R, write_hi);
                split_tile(b_hi(s), b_lo(s), t4, kb * kTcBK, R, write_hi);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(conv + s);
            }
        }
    } else if (warp >= 8) {
        const int wq = warp & 3;
        const uint32_t stage = sa(sm + kTcStages * kTcStageBytes + 256) + wq * 4096;
        int ti = 0;
        for (int t = blockIdx.x; t < items; t += gridDim.x, ++ti) {
            const int acc = ti & 1;
            const int tile = t % tiles, z = t / tiles;
            const int m0 = (tile / n_tiles) * kTcBM, n0 = (tile % n_tiles) * kTcBN;
            int k0, k1;
            kb_range(z, k0, k1);
            mbar_wait(tmem_full + acc, uint32_t((ti / 2) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            float* Pz = P + size_t(z) * Kin * N;  // rows = input features
#pragma unroll
            for (int c = 0; c < kTcBN / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem + (uint32_t(wq * 32) << 16) + uint32_t(acc * kTcBN + c * 32), r);
                if (c + 1 == kTcBN / 32) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    mbar_arrive(tmem_empty + acc);
                }
                if (k1 <= k0) {  // an empty slice writes zeros
#pragma unroll
                    for (int q = 0; q < 32; ++q) r[q] = 0u;
                }
                if (n0 + c * 32 < N) store_block<false, false>(stage, r, 0.f, lane, Pz, N, m0 + wq * 32, Kin, n0 + c * 32, N);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256) : "memory");
    }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    }
    return fn;
}

}  // namespace

// fp32 row-major [rows x K] (K contiguous) as a TMA map with 32 x 128 boxes, 128-byte swizzle.
int tc_make_map(CUtensorMap* map, const float* base, uint64_t rows, uint32_t K) {
    EncodeTiled enc = encode_fn();
    if (!enc) return fail(FDG_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {K, std::max<uint64_t>(rows, 1)};
    const cuuint64_t strides[1] = {uint64_t(K) * 4};
    const cuuint32_t box[2] = {uint32_t(kTcBK), uint32_t(kTcBM)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FDG_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return FDG_OK;
}

// fp32 row-major [rows x cols] as a TMA map with 32 (cols) x 32 (rows) boxes, 128-byte rows
// swizzled in 32-byte atoms: the MN-major operand blocks of k_wgrad_tc.
int tc_make_map_mn(CUtensorMap* map, const float* base, uint64_t rows, uint32_t cols) {
    EncodeTiled enc = encode_fn();
    if (!enc) return fail(FDG_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {cols, std::max<uint64_t>(rows, 1)};
    const cuuint64_t strides[1] = {uint64_t(cols) * 4};
    const cuuint32_t box[2] = {32, uint32_t(kTcBK)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FDG_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return FDG_OK;
}

// Does kind::tf32 truncate the fp32 operand (ignore its low 13 mantissa bits)? One GEMM
// (128 x 32 x 128, A with every mantissa bit set, W exact in tf32, W_lo = 0) with and
// without the explicit A_hi write: equal bits <=> the tensor core saw trunc(A) in both.
// Once per device, on a private stream; 1 (write A_hi) if the check cannot run.
namespace {
int write_hi_check() {
    constexpr int M = 128, K = 32, N = 128;
    std::vector<float> a(M * K), w(N * K);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    auto next = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
    for (auto& v : a) {  // [1, 2) with a random full mantissa, low 13 bits never all zero
        uint32_t b = 0x3F800000u | uint32_t(next() & 0x7FFFFFu) | 1u;
        std::memcpy(&v, &b, 4);
    }
    for (auto& v : w) {  // tf32-exact: low 13 bits clear
        uint32_t b = 0x3F800000u | (uint32_t(next() & 0x7FFFFFu) & ~0x1FFFu);
        std::memcpy(&v, &b, 4);
    }
    fdg_batch_counts cnt{};
    cnt.n_nodes = M;
    cnt.layer_nodes[1] = M;
    float *dA = nullptr, *dW = nullptr, *dZ = nullptr, *dC = nullptr;
    fdg_batch_counts* dcnt = nullptr;
    cudaStream_t st = nullptr;
    int res = 1;
    std::vector<float> c0(M * N), c1(M * N);
    CUtensorMap mA, mW, mZ;
    bool ok = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMalloc(&dA, a.size() * 4) == cudaSuccess && cudaMalloc(&dW, w.size() * 4) == cudaSuccess &&
              cudaMalloc(&dZ, w.size() * 4) == cudaSuccess && cudaMalloc(&dC, 2ull * M * N * 4) == cudaSuccess &&
              cudaMalloc(&dcnt, sizeof(cnt)) == cudaSuccess;
    ok = ok && cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(dW, w.data(), w.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemset(dZ, 0, w.size() * 4) == cudaSuccess && cudaMemset(dC, 0, 2ull * M * N * 4) == cudaSuccess &&
         cudaMemcpy(dcnt, &cnt, sizeof(cnt), cudaMemcpyHostToDevice) == cudaSuccess;
    ok = ok && tc_make_map(&mA, dA, M, K) == FDG_OK && tc_make_map(&mW, dW, N, K) == FDG_OK &&
         tc_make_map(&mZ, dZ, N, K) == FDG_OK;
    ok = ok && cudaFuncSetAttribute(k_sgemm_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem) ==
                   cudaSuccess;
    if (ok) {
        for (int wh = 0; wh < 2; ++wh)  // bias: the zero W_lo block (N floats of zeros)
            k_sgemm_tc<false><<<1, kTcThreads, kTcSmem, st>>>(mA, mW, mZ, dZ, dC + wh * M * N, dcnt, 0, N, K, 1, wh);
        ok = cudaStreamSynchronize(st) == cudaSuccess &&
             cudaMemcpy(c0.data(), dC, c0.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
             cudaMemcpy(c1.data(), dC + M * N, c1.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    if (ok) {
        double err = 0;  // the explicit write must give an fp32-accurate product
        for (int i = 0; i < M; ++i)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += double(a[i * K + k]) * w[n * K + k];
                err = std::max(err, std::abs(c1[i * N + n] - ref) / std::abs(ref));
            }
        if (err < 1e-5) res = std::memcmp(c0.data(), c1.data(), c0.size() * 4) == 0 ? 0 : 1;
    }
    cudaGetLastError();
    cudaFree(dA);
    cudaFree(dW);
    cudaFree(dZ);
    cudaFree(dC);
    cudaFree(dcnt);
    if (st) cudaStreamDestroy(st);
    return res;
}
int g_write_hi[64];
PerDeviceOnce g_write_hi_once;
}  // namespace

int tc_write_hi(cudaStream_t) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_write_hi_once.first()) __atomic_store_n(&g_write_hi[dev & 63], write_hi_check() + 1, __ATOMIC_RELEASE);
    while (!__atomic_load_n(&g_write_hi[dev & 63], __ATOMIC_ACQUIRE)) {
    }
    return g_write_hi[dev & 63] - 1;
}

int tc_wgrad(cudaStream_t st, const CUtensorMap& tA, const CUtensorMap& tB, float* P, const fdg_batch_counts* cnt,
             int j, int Kin, int N, int Z) {
    static PerDeviceOnce attr;
    if (attr.first()) {
        FDG_CUDA(cudaFuncSetAttribute(k_wgrad_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
    }
    int sms = 0, dev = 0;  // per call: the current device may differ between calls
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int m_tiles = (Kin + kTcBM - 1) / kTcBM, n_tiles = (N + kTcBN - 1) / kTcBN;
    const int items = m_tiles * n_tiles * Z;
    k_wgrad_tc<<<std::min(items, sms), kTcThreads, kTcSmem, st>>>(tA, tB, P, cnt, j, Kin, N, m_tiles, n_tiles, Z,
                                                                 tc_write_hi(st));
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

int tc_gemm(cudaStream_t st, const CUtensorMap& tA, const CUtensorMap& tBhi, const CUtensorMap& tBlo,
            const float* bias, float* C, const fdg_batch_counts* cnt, int j, uint64_t rows_bound, int N, int npad,
            int K, bool relu) {
    static PerDeviceOnce attr;
    if (attr.first()) {
        FDG_CUDA(cudaFuncSetAttribute(k_sgemm_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
        FDG_CUDA(cudaFuncSetAttribute(k_sgemm_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
    }
    if (K % 4) return fail(FDG_INVALID_ARG, "tc_gemm: K must be a multiple of 4 (16-byte row stride)");
    int sms = 0, dev = 0;  // per call: the current device may differ between calls
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int n_tiles = npad / kTcBN;
    const uint64_t tiles = (rows_bound + kTcBM - 1) / kTcBM * uint64_t(n_tiles);
    const uint32_t grid = uint32_t(std::min<uint64_t>(tiles, uint64_t(sms)));  // persistent: one CTA per SM
    const int wh = tc_write_hi(st);
    if (relu)
        k_sgemm_tc<true><<<grid, kTcThreads, kTcSmem, st>>>(tA, tBhi, tBlo, bias, C, cnt, j, N, K, n_tiles, wh);
    else
        k_sgemm_tc<false><<<grid, kTcThreads, kTcSmem, st>>>(tA, tBhi, tBlo, bias, C, cnt, j, N, K, n_tiles, wh);
    FDG_CUDA(cudaGetLastError());
    return FDG_OK;
}

}  // namespace fdg
