// Batched FP32 SPD solve of packed Hermitian rows, one system per warp: the default solve of
// the tensor-core half-sweep (replaces batch_solve_into, solver.hpp:204-262, at FP32
// tolerance).
//
// Why a warp per system: the TMEM-resident Cholesky (tc_solve.cu) holds at most 4 systems per
// SM (128 TMEM columns each) and each of its 13 dependent 8-column steps pays a CTA barrier,
// an 8x8 POTRF on one lane and a tcgen05 commit round trip, so it is latency-bound (~38K
// cycles per system). Here every warp owns one system in shared memory (the packed row as
// bulk-copied, 22 KB at f = 100), so 10 systems are in flight per SM, steps need no CTA
// barrier, and the Schur updates run on the warp-level tensor-core path (mma.sync m16n8k8
// tf32: 20-cycle latency, one per 8 cycles per SM sub-partition, scripts/probes/
// mma_sync_probe.cu), which leaves the FMA pipe to the POTRF/TRSM of the other warps.
//
// Per 8-column block b (r0 = 8b), on the panel-blocked packed row (kernels.cuh pb_block):
//   1. every lane loads the 8x8 diagonal block (broadcast) and factors it redundantly
//      (branch-free rsqrt Cholesky; columns >= f are identity padding);
//   2. TRSM: lane l solves rows r0 + l + 32k (<= f) against it in place: the diagonal-block
//      rows become L_cc, the panel rows L, and the augmented row f becomes y = L^-1 b;
//   3. the panel's 8-row groups are read back in mma fragment order and split -P = h + l
//      (tf32 hi/lo); every lower 16x8 tile of the trailing matrix takes
//      D -= Ph Ph^T + Ph Pl^T + Pl Ph^T (three mma.sync; the tile is loaded and stored in
//      accumulator order). Row f is a row, never a column: its update is the forward
//      substitution.
// Tiles are indexed from the bottom-right corner: row group k' = G-1-n (n = absolute 8-row
// group, G groups for rows 0..f) and column block J' = NB-1-J. In those coordinates the
// tiles of a column never change from one step to the next -- step b only decides how many
// columns are still trailing (J' < NB-1-b) -- so the step loop is a runtime loop, every
// fragment index is a compile-time constant, and the code is one step long. Each column's
// tiles are loaded together, go through the three MMA passes together and are stored
// together (independent accumulation chains back to back).
// Back substitution L^T x = y, per block from the last: the block's 8 values of x are solved
// in every lane (L_cc broadcast) over y in place (row f of the packed row), and lane j
// subtracts their contribution from y_j.
// All-zero A gives x = 0 (solver.hpp:215-220); the first non-positive pivot is reported with
// its row, column and value (solver.hpp:230-235) and that row's x is zeroed. The next
// system's packed row is prefetched into L2 when a system starts and bulk-copied into the
// warp's buffer as soon as the back substitution is done with it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace alsk {
namespace {
using namespace tc;

constexpr int WS_MAX_WARPS = 12;
constexpr uint32_t SIGN = 0x80000000u;

__device__ __forceinline__ void mma_m16n8k8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                            uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t tf32_hi_bits(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }
__device__ __forceinline__ void ws_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void ws_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void ws_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    const float4 w = *reinterpret_cast<const float4*>(p + 4);
    v[0] = u.x, v[1] = u.y, v[2] = u.z, v[3] = u.w, v[4] = w.x, v[5] = w.y, v[6] = w.z, v[7] = w.w;
}

// shared memory of one warp: packed row, 1/L[c][c] (8 NB floats), mbarrier
__host__ __device__ inline uint32_t ws_warp_bytes(int f) {
    const int nb = (f + 7) / 8;
    const uint32_t b = static_cast<uint32_t>(packed_stride(f)) * 4u + 32u * static_cast<uint32_t>(nb) + 16u;
    return (b + 127u) & ~127u;
}

// Trailing update of column block J' (J = NB-1-J') at step b: its 16x8 tiles, bottom-aligned.
// fr[k'] holds -P of row group k' (from the bottom) as {hi(t), hi(t+4), lo(t), lo(t+4)}.
template <int NB, int E, int JP>
__device__ __forceinline__ void ws_column(float* buf, int f, const uint32_t (&fr)[NB + E][4], int g8, int t4) {
    constexpr int G = NB + E;
    constexpr int J = NB - 1 - JP;
    constexpr int KD = JP + E;          // k' of the column's diagonal group
    constexpr int P = (KD + 2) / 2;     // tiles: groups k' = 0 .. KD in pairs from the bottom
    constexpr bool TOP_PHANTOM = (KD % 2) == 0;  // the last tile's upper group lies above the diagonal
    float* cb = buf + pb_block(f, J);
    // B operand: +P of the column's own rows (row f, the augmented row, is no column)
    const bool colreal = !(E == 0 && JP == 0) || 8 * J + g8 < f;
    const uint32_t bh0 = colreal ? fr[KD][0] ^ SIGN : 0u, bh1 = colreal ? fr[KD][1] ^ SIGN : 0u;
    const uint32_t bl0 = colreal ? fr[KD][2] ^ SIGN : 0u, bl1 = colreal ? fr[KD][3] ^ SIGN : 0u;
    float d[P][4];
    float2* pu[P];
    float2* pl[P];
    const bool low_ok = 8 * (G - 1) + g8 <= f;  // lower rows of tile 0 (the group holding row f)
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int nu = G - 2 - 2 * p;  // absolute upper group; lower group nu + 1
        pu[p] = reinterpret_cast<float2*>(cb + 8 * (8 * nu + g8 - 8 * J) + 2 * t4);
        pl[p] = reinterpret_cast<float2*>(cb + 8 * (8 * nu + 8 + g8 - 8 * J) + 2 * t4);
        float2 cu = make_float2(0.f, 0.f), cl = make_float2(0.f, 0.f);
        if (!(TOP_PHANTOM && p == P - 1)) cu = *pu[p];
        if (p != 0 || low_ok) cl = *pl[p];
        d[p][0] = cu.x, d[p][1] = cu.y, d[p][2] = cl.x, d[p][3] = cl.y;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) mma_m16n8k8(d[p], fr[2 * p + 1][0], fr[2 * p][0], fr[2 * p + 1][1], fr[2 * p][1], bh0, bh1);
#pragma unroll
    for (int p = 0; p < P; ++p) mma_m16n8k8(d[p], fr[2 * p + 1][0], fr[2 * p][0], fr[2 * p + 1][1], fr[2 * p][1], bl0, bl1);
#pragma unroll
    for (int p = 0; p < P; ++p) mma_m16n8k8(d[p], fr[2 * p + 1][2], fr[2 * p][2], fr[2 * p + 1][3], fr[2 * p][3], bh0, bh1);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        if (!(TOP_PHANTOM && p == P - 1)) *pu[p] = make_float2(d[p][0], d[p][1]);
        if (p != 0 || low_ok) *pl[p] = make_float2(d[p][2], d[p][3]);
    }
}

template <int NB, int E, int JP>
__device__ __forceinline__ void ws_trailing(float* buf, int f, int b, const uint32_t (&fr)[NB + E][4], int g8, int t4) {
    if constexpr (JP <= NB - 2) {
        if (JP < NB - 1 - b) {  // column J = NB-1-JP is trailing (J > b); warp-uniform
            ws_column<NB, E, JP>(buf, f, fr, g8, t4);
            ws_trailing<NB, E, JP + 1>(buf, f, b, fr, g8, t4);
        }
    }
}

// NB = ceil(f / 8) column blocks; E = 1 when f % 8 == 0 (row f starts a group of its own)
template <int NB, int E>
__global__ void __launch_bounds__(WS_MAX_WARPS * 32, 1)
warp_solve_kernel(const float* __restrict__ packed, int64_t count, int f, float* __restrict__ out_x,
                  unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                  double* __restrict__ pivot, int64_t status_base, uint32_t warp_bytes) {
    constexpr int G = NB + E;  // 8-row groups of rows 0 .. f
    extern __shared__ __align__(128) uint8_t ws_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g8 = lane >> 2, t4 = lane & 3;
    const int pks = static_cast<int>(packed_stride(f));
    float* buf = reinterpret_cast<float*>(ws_smem + static_cast<size_t>(warp) * warp_bytes);
    float* dinv = buf + pks;
    uint64_t* bar = reinterpret_cast<uint64_t*>(dinv + 8 * NB);
    const uint32_t row_bytes = static_cast<uint32_t>(pks) * 4u;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    int64_t sys = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
    if (lane == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    __syncwarp();
    if (lane == 0 && sys < count) {
        ws_expect_tx(bar, row_bytes);
        ws_bulk_g2s(smem_u32(buf), packed + sys * pks, row_bytes, bar);
    }
    uint32_t phase = 0;
    for (; sys < count; sys += nwarps, phase ^= 1u) {
        if (lane == 0 && sys + nwarps < count) ws_prefetch_l2(packed + (sys + nwarps) * pks, row_bytes);
        mbar_wait(bar, phase);
        // ---- all-zero A: x = 0. A nonzero diagonal settles it; otherwise scan all of A ----
        bool nz = false;
        for (int i = lane; i < f; i += 32) nz |= buf[pb_index(f, i, i)] != 0.f;
        bool active = __any_sync(~0u, nz);
        if (!active) {
            for (int b = 0; b < NB; ++b)
                for (int r = 8 * b + lane; r < f; r += 32) {
                    float v[8];
                    ld8(buf + pb_block(f, b) + 8 * (r - 8 * b), v);
#pragma unroll
                    for (int k = 0; k < 8; ++k) nz |= v[k] != 0.f;
                }
            active = __any_sync(~0u, nz);
        }
        int bad = 0;
        float badv = 0.f;
        if (active) {
            uint32_t fr[G][4];
            for (int b = 0; b < NB; ++b) {
                const int r0 = 8 * b;
                const int nreal = min(8, f - r0);  // real columns of this block
                float* blk = buf + pb_block(f, b);
                // (1) diagonal block, factored in every lane; rows >= nreal are identity
                float l[8][8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (q < nreal) {
                        ld8(blk + 8 * q, l[q]);
                    } else {
#pragma unroll
                        for (int k = 0; k < 8; ++k) l[q][k] = k == q ? 1.f : 0.f;
                    }
                }
                float dv[8];
                int bad_here = 0;
                float badv_here = 0.f;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float d = l[c][c];
                    if (bad_here == 0 && !(d > 0.f)) {
                        bad_here = c + 1;
                        badv_here = d;
                    }
                    const float ic = rsqrtf(d);
                    dv[c] = ic;
                    l[c][c] = d * ic;
#pragma unroll
                    for (int q = c + 1; q < 8; ++q) l[q][c] *= ic;
#pragma unroll
                    for (int q = c + 1; q < 8; ++q)
#pragma unroll
                        for (int p = c + 1; p <= q; ++p) l[q][p] = fmaf(-l[q][c], l[p][c], l[q][p]);
                }
                if (bad_here) {  // warp-uniform: every lane factored the same block
                    bad = r0 + bad_here;
                    badv = badv_here;
                    break;
                }
                __syncwarp();  // every lane has read the block before the TRSM overwrites it
                if (lane == 0) {
                    *reinterpret_cast<float4*>(dinv + r0) = make_float4(dv[0], dv[1], dv[2], dv[3]);
                    *reinterpret_cast<float4*>(dinv + r0 + 4) = make_float4(dv[4], dv[5], dv[6], dv[7]);
                }
                // (2) TRSM of rows r0 .. f: L[c] = (a[c] - sum_k<c L[k] L_cc[c][k]) / L_cc[c][c]
#pragma unroll
                for (int k = 0; k < (8 * NB + 32) / 32; ++k) {
                    if (r0 + 32 * k > f) break;  // warp-uniform
                    const int i = r0 + lane + 32 * k;
                    if (i <= f) {
                        float* row = blk + 8 * (i - r0);
                        float a[8];
                        ld8(row, a);
                        float L[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            float s = a[c];
#pragma unroll
                            for (int q = 0; q < c; ++q) s = fmaf(-L[q], l[c][q], s);
                            L[c] = s * dv[c];
                        }
                        const int keep = i < r0 + 8 && i != f ? i - r0 : 7;  // diagonal-block row: L_cc, upper part 0
#pragma unroll
                        for (int c = 0; c < 8; ++c) L[c] = (c <= keep && c < nreal) ? L[c] : 0.f;
                        *reinterpret_cast<float4*>(row) = make_float4(L[0], L[1], L[2], L[3]);
                        *reinterpret_cast<float4*>(row + 4) = make_float4(L[4], L[5], L[6], L[7]);
                    }
                }
                __syncwarp();
                if (b == NB - 1) break;
                // (3) panel fragments: row group k' (absolute n = G-1-k'), rows below the block only
#pragma unroll
                for (int kp = 0; kp < G; ++kp) {
                    const int row = 8 * (G - 1 - kp) + g8;
                    float p0 = 0.f, p1 = 0.f;
                    if (row >= r0 + 8 && row <= f) {
                        p0 = -blk[8 * (row - r0) + t4];
                        p1 = -blk[8 * (row - r0) + t4 + 4];
                    }
                    const uint32_t h0 = tf32_hi_bits(p0), h1 = tf32_hi_bits(p1);
                    fr[kp][0] = h0;
                    fr[kp][1] = h1;
                    fr[kp][2] = __float_as_uint(p0 - __uint_as_float(h0));
                    fr[kp][3] = __float_as_uint(p1 - __uint_as_float(h1));
                }
                // (4) trailing update, columns J' = 0 .. NB-2-b
                ws_trailing<NB, E, 0>(buf, f, b, fr, g8, t4);
                __syncwarp();
            }
        }
        if (active && bad == 0) {
            // ---- back substitution L^T x = y over y in place (row f of the packed row) ----
            for (int bb = NB - 1; bb >= 0; --bb) {
                const int k0 = 8 * bb;
                const int nreal = min(8, f - k0);
                const float* lb = buf + pb_block(f, bb);
                float* yrow = buf + pb_block(f, bb) + 8 * (f - k0);
                float yb[8], lc[8][8], dvv[8], xb[8];
                ld8(yrow, yb);
                ld8(dinv + k0, dvv);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (c < nreal) {
                        ld8(lb + 8 * c, lc[c]);
                    } else {
#pragma unroll
                        for (int k = 0; k < 8; ++k) lc[c][k] = 0.f;
                    }
                }
#pragma unroll
                for (int c = 7; c >= 0; --c) {
                    float s = yb[c];
#pragma unroll
                    for (int k = c + 1; k < 8; ++k) s = fmaf(-lc[k][c], xb[k], s);
                    xb[c] = c < nreal ? s * dvv[c] : 0.f;
                }
                // y_j -= sum_c L[k0 + c][j] x_c for j < k0
                for (int j = lane; j < k0; j += 32) {
                    const int J = j >> 3;
                    const int64_t bj = pb_block(f, J);
                    const float* p = buf + bj + 8 * (k0 - 8 * J) + (j & 7);
                    float* yj = buf + bj + 8 * (f - 8 * J) + (j & 7);
                    float s = *yj;
#pragma unroll
                    for (int c = 0; c < 8; ++c) s = fmaf(-p[8 * c], xb[c], s);
                    *yj = s;
                }
                __syncwarp();
                if (lane == 0) {
                    *reinterpret_cast<float4*>(yrow) = make_float4(xb[0], xb[1], xb[2], xb[3]);
                    *reinterpret_cast<float4*>(yrow + 4) = make_float4(xb[4], xb[5], xb[6], xb[7]);
                }
                __syncwarp();
            }
        }
        float xv[(8 * NB + 31) / 32];
        if (active && bad == 0) {
#pragma unroll
            for (int q = 0; q < (8 * NB + 31) / 32; ++q) {
                const int j = lane + 32 * q;
                xv[q] = j < f ? buf[pb_index(f, f, j)] : 0.f;
            }
        }
        __syncwarp();  // the buffer is free: fetch the next system while x is stored
        if (lane == 0 && sys + nwarps < count) {
            fence_proxy_async_smem();
            ws_expect_tx(bar, row_bytes);
            ws_bulk_g2s(smem_u32(buf), packed + (sys + nwarps) * pks, row_bytes, bar);
        }
        float* x = out_x + sys * f;
        if (active && bad == 0) {
#pragma unroll
            for (int q = 0; q < (8 * NB + 31) / 32; ++q) {
                const int j = lane + 32 * q;
                if (j < f) x[j] = xv[q];
            }
            if (lane == 0) column[sys] = 0;
        } else {
            for (int j = lane; j < f; j += 32) x[j] = 0.f;
            if (lane == 0) {
                column[sys] = bad;
                if (bad) {
                    pivot[sys] = static_cast<double>(badv);
                    atomicMin(min_row, static_cast<unsigned long long>(status_base + sys));
                }
            }
        }
    }
}

template <int NB, int E>
void launch_ws(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
               cudaStream_t s) {
    const uint32_t wb = ws_warp_bytes(f);
    const int max_smem = 227 * 1024;
    const int warps = std::max(1, std::min<int>(WS_MAX_WARPS, max_smem / static_cast<int>(wb)));
    const int smem = warps * static_cast<int>(wb);
    ALSK_CUDA(cudaFuncSetAttribute(warp_solve_kernel<NB, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t ctas = (count + warps - 1) / warps;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ctas, num_sms()));
    warp_solve_kernel<NB, E><<<grid, warps * 32, smem, s>>>(packed, count, f, x, st.min_row, st.column + status_off,
                                                           st.pivot + status_off, status_off, wb);
    ALSK_LAUNCHED();
}

}  // namespace

bool warp_solve(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                cudaStream_t s) {
    if (f < 1 || f > 128) return false;
    if (count <= 0) return true;
    const bool e = f % 8 == 0;
    switch ((f + 7) / 8) {
#define ALSK_WS(NB)                                                                        \
    case NB:                                                                               \
        if (e) launch_ws<NB, 1>(packed, count, f, x, st, status_off, s);                   \
        else launch_ws<NB, 0>(packed, count, f, x, st, status_off, s);                     \
        return true;
        ALSK_WS(1) ALSK_WS(2) ALSK_WS(3) ALSK_WS(4) ALSK_WS(5) ALSK_WS(6) ALSK_WS(7) ALSK_WS(8)
        ALSK_WS(9) ALSK_WS(10) ALSK_WS(11) ALSK_WS(12) ALSK_WS(13) ALSK_WS(14) ALSK_WS(15) ALSK_WS(16)
#undef ALSK_WS
        default: return false;
    }
}

}  // namespace alsk
