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
#include <cstdio>

#include "kernels.cuh"
#include "measure.cuh"
#include "tc_common.cuh"

namespace alsk {
namespace {
using namespace tc;

constexpr int WS_MAX_WARPS = 10;
// warps per CTA (one CTA per SM): shared memory allows 10 systems of f <= 104, at most 8 above;
// an SM sub-partition holding 3 warps leaves 168 registers per thread, one holding 2 leaves 255
template <int NB>
constexpr int ws_warps() { return NB >= 14 ? 8 : WS_MAX_WARPS; }
constexpr uint32_t SIGN = 0x80000000u;

__device__ __forceinline__ void mma_m16n8k8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                            uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t tf32_hi_bits(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;\n" : "=f"(r) : "f"(x));
    return r;
}
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

// TRSM of the block's rows r0 .. f in R straight-line rounds of 32 (lane l: rows r0 + l + 32k):
// L[c] = (a[c] - sum_k<c L[k] L_cc[c][k]) / L_cc[c][c], in place. A diagonal-block row gets its
// row of L_cc below the diagonal and finite leftovers above it, which nothing reads; padding
// columns (identity, zero cells) stay 0.
template <int R, int NB>
__device__ __forceinline__ void ws_trsm(float* blk, int r0, int f, int lane, const float (&l)[8][8], const float (&dv)[8]) {
    if constexpr (R <= (8 * NB + 32) / 32) {
        float a[R][8];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int i = r0 + lane + 32 * k;
            if (i <= f) {
                ld8(blk + 8 * (i - r0), a[k]);
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) a[k][c] = 0.f;
            }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int k = 0; k < R; ++k) {
                float s = a[k][c];
#pragma unroll
                for (int q = 0; q < c; ++q) s = fmaf(-a[k][q], l[c][q], s);
                a[k][c] = s * dv[c];
            }
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int i = r0 + lane + 32 * k;
            if (i <= f) {
                float* row = blk + 8 * (i - r0);
                *reinterpret_cast<float4*>(row) = make_float4(a[k][0], a[k][1], a[k][2], a[k][3]);
                *reinterpret_cast<float4*>(row + 4) = make_float4(a[k][4], a[k][5], a[k][6], a[k][7]);
            }
        }
    }
}

// Register-resident columns: the last WS_RES column blocks (J' < WS_RES, the bottom-right
// corner, updated at every step) keep their tiles in registers from the system's start until
// the step before their own (then they are stored for the POTRF/TRSM), which saves most of
// the tiles' shared-memory read-modify-writes.
constexpr int WS_RES = 3;
template <int NB, int E>
struct WsTiles {
    static constexpr int RJ = NB - 1 < WS_RES ? NB - 1 : WS_RES;  // resident columns
    static constexpr int PT = (WS_RES - 1 + E + 2) / 2;           // tiles of the widest one
    float acc[WS_RES][PT][4];
};

// Tile p of column J' (bottom-aligned 16-row tiles): accumulator-order cell pointers and which
// halves exist (upper: not above the diagonal; lower: rows <= f).
template <int NB, int E, int JP>
struct WsTile {
    static constexpr int G = NB + E;
    static constexpr int J = NB - 1 - JP;
    static constexpr int KD = JP + E;              // k' of the column's diagonal group
    static constexpr int P = (KD + 2) / 2;         // tiles: groups k' = 0 .. KD in pairs from the bottom
    static constexpr bool TOP_PHANTOM = (KD % 2) == 0;  // the last tile's upper group lies above the diagonal
    __device__ static float2* up(float* buf, int f, int p, int g8, int t4) {
        return reinterpret_cast<float2*>(buf + pb_block(f, J) + 8 * (8 * (G - 2 - 2 * p) + g8 - 8 * J) + 2 * t4);
    }
    __device__ static bool has_up(int p) { return !(TOP_PHANTOM && p == P - 1); }
    __device__ static bool has_low(int p, int f, int g8) { return p != 0 || 8 * (G - 1) + g8 <= f; }
};

template <int NB, int E, int JP>
__device__ __forceinline__ void ws_tiles_load(float* buf, int f, int g8, int t4, float (&d)[WsTile<NB, E, JP>::P][4]) {
    using T = WsTile<NB, E, JP>;
#pragma unroll
    for (int p = 0; p < T::P; ++p) {
        const float2* pu = T::up(buf, f, p, g8, t4);
        float2 cu = make_float2(0.f, 0.f), cl = make_float2(0.f, 0.f);
        if (T::has_up(p)) cu = pu[0];
        if (T::has_low(p, f, g8)) cl = pu[32];  // 8 rows further
        d[p][0] = cu.x, d[p][1] = cu.y, d[p][2] = cl.x, d[p][3] = cl.y;
    }
}
template <int NB, int E, int JP>
__device__ __forceinline__ void ws_tiles_store(float* buf, int f, int g8, int t4, const float (&d)[WsTile<NB, E, JP>::P][4]) {
    using T = WsTile<NB, E, JP>;
#pragma unroll
    for (int p = 0; p < T::P; ++p) {
        float2* pu = T::up(buf, f, p, g8, t4);
        if (T::has_up(p)) pu[0] = make_float2(d[p][0], d[p][1]);
        if (T::has_low(p, f, g8)) pu[32] = make_float2(d[p][2], d[p][3]);
    }
}

// Fragments of pairs 0 .. N-1 at step b (blk = block b, r0 = 8b), branch-free: a group above
// the panel reads cells of block b's diagonal rows, a row past f cells of block b+1, both
// inside the buffer, and is zeroed.
template <int G, int N>
__device__ __forceinline__ void ws_pairs(const float* blk, int r0, int f, int g8, int t4, uint32_t (&fa)[(G + 1) / 2][8]) {
    constexpr int NP = (G + 1) / 2;
    constexpr int M = N < NP ? N : NP;
    float v[M][2][2];  // [pair][U, D][k0, k1]
#pragma unroll
    for (int p = 0; p < M; ++p)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int kp = 2 * p + 1 - h;
            if (kp >= G) {  // compile time: the upper group of the last pair does not exist
                v[p][h][0] = v[p][h][1] = 0.f;
                continue;
            }
            const int row = 8 * (G - 1 - kp) + g8;
            const float2 x = *reinterpret_cast<const float2*>(blk + 8 * (row - r0) + 2 * t4);
            const bool ok = row >= r0 + 8 && row <= f;
            v[p][h][0] = ok ? -x.x : 0.f;
            v[p][h][1] = ok ? -x.y : 0.f;
        }
#pragma unroll
    for (int p = 0; p < M; ++p) {
        fa[p][0] = tf32_hi_bits(v[p][0][0]);
        fa[p][1] = tf32_hi_bits(v[p][1][0]);
        fa[p][2] = tf32_hi_bits(v[p][0][1]);
        fa[p][3] = tf32_hi_bits(v[p][1][1]);
        fa[p][4] = __float_as_uint(v[p][0][0] - __uint_as_float(fa[p][0]));
        fa[p][5] = __float_as_uint(v[p][1][0] - __uint_as_float(fa[p][1]));
        fa[p][6] = __float_as_uint(v[p][0][1] - __uint_as_float(fa[p][2]));
        fa[p][7] = __float_as_uint(v[p][1][1] - __uint_as_float(fa[p][3]));
    }
}

// Trailing update of column block J' (J = NB-1-J') at step b: its 16x8 tiles, bottom-aligned.
// fa[p] holds -P of the row groups k' = 2p+1 (U, the tile's upper 8 rows) and 2p (D) in MMA
// A-operand order: {hi U k0, hi D k0, hi U k1, hi D k1, lo U k0, lo D k0, lo U k1, lo D k1}, lane
// t carrying the panel columns k0 = 2t, k1 = 2t+1 as MMA k-slots t, t+4 (any k order works
// as long as A and B use the same one). Tile p of every column reads pair p as it is.
template <int NB, int E, int JP>
__device__ __forceinline__ void ws_column(float* buf, int f, const uint32_t (&fa)[(NB + E + 1) / 2][8], int g8, int t4,
                                          WsTiles<NB, E>& rt) {
    using T = WsTile<NB, E, JP>;
    constexpr int P = T::P, KD = T::KD;
    // B operand: +P of the column's own rows (row f, the augmented row, is no column)
    const bool colreal = !(E == 0 && JP == 0) || 8 * T::J + g8 < f;
    constexpr int BP = KD / 2, BO = KD % 2 ? 0 : 1;  // pair and slot of the diagonal group
    const uint32_t bh0 = colreal ? fa[BP][BO] ^ SIGN : 0u, bh1 = colreal ? fa[BP][BO + 2] ^ SIGN : 0u;
    const uint32_t bl0 = colreal ? fa[BP][BO + 4] ^ SIGN : 0u, bl1 = colreal ? fa[BP][BO + 6] ^ SIGN : 0u;
    float d[P][4];
    if constexpr (JP < WsTiles<NB, E>::RJ) {
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) d[p][q] = rt.acc[JP][p][q];
    } else {
        ws_tiles_load<NB, E, JP>(buf, f, g8, t4, d);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) mma_m16n8k8(d[p], fa[p][0], fa[p][1], fa[p][2], fa[p][3], bh0, bh1);
#pragma unroll
    for (int p = 0; p < P; ++p) mma_m16n8k8(d[p], fa[p][0], fa[p][1], fa[p][2], fa[p][3], bl0, bl1);
#pragma unroll
    for (int p = 0; p < P; ++p) mma_m16n8k8(d[p], fa[p][4], fa[p][5], fa[p][6], fa[p][7], bh0, bh1);
    if constexpr (JP < WsTiles<NB, E>::RJ) {
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) rt.acc[JP][p][q] = d[p][q];
    } else {
        ws_tiles_store<NB, E, JP>(buf, f, g8, t4, d);
    }
}

template <int NB, int E, int JP>
__device__ __forceinline__ void ws_trailing(float* buf, int f, int b, const uint32_t (&fa)[(NB + E + 1) / 2][8], int g8, int t4,
                                            WsTiles<NB, E>& rt) {
    if constexpr (JP <= NB - 2) {
        if (JP < NB - 1 - b) {  // column J = NB-1-JP is trailing (J > b); warp-uniform
            ws_column<NB, E, JP>(buf, f, fa, g8, t4, rt);
            ws_trailing<NB, E, JP + 1>(buf, f, b, fa, g8, t4, rt);
        }
    }
}
// resident columns from shared memory (system start)
template <int NB, int E, int JP>
__device__ __forceinline__ void ws_res_load(float* buf, int f, int g8, int t4, WsTiles<NB, E>& rt) {
    if constexpr (JP < WsTiles<NB, E>::RJ) {
        ws_tiles_load<NB, E, JP>(buf, f, g8, t4, reinterpret_cast<float(&)[WsTile<NB, E, JP>::P][4]>(rt.acc[JP]));
        ws_res_load<NB, E, JP + 1>(buf, f, g8, t4, rt);
    }
}
// resident column jp back to shared memory (it is the next step's panel)
template <int NB, int E, int JP>
__device__ __forceinline__ void ws_res_flush(float* buf, int f, int jp, int g8, int t4, WsTiles<NB, E>& rt) {
    if constexpr (JP < WsTiles<NB, E>::RJ) {
        if (jp == JP) ws_tiles_store<NB, E, JP>(buf, f, g8, t4, reinterpret_cast<const float(&)[WsTile<NB, E, JP>::P][4]>(rt.acc[JP]));
        else ws_res_flush<NB, E, JP + 1>(buf, f, jp, g8, t4, rt);
    }
}

// NB = ceil(f / 8) column blocks; E = 1 when f % 8 == 0 (row f starts a group of its own)
template <int NB, int E>
__global__ void __launch_bounds__(ws_warps<NB>() * 32, 1)
warp_solve_kernel(const float* __restrict__ packed, int64_t count, int f, float* __restrict__ out_x,
                  unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                  double* __restrict__ pivot, int64_t status_base, uint32_t warp_bytes,
                  unsigned long long* __restrict__ prof) {
    constexpr int G = NB + E;  // 8-row groups of rows 0 .. f
#ifdef ALSK_MEASURE
    // ALSK_WS_PROF=1: cycles per phase summed over warps (lane 0), measurement builds only
    uint32_t pacc[8] = {}, pt = static_cast<uint32_t>(clock());
#define WS_LAP(slot)                                                 \
    if (prof) {                                                      \
        const uint32_t now_ = static_cast<uint32_t>(clock());        \
        pacc[slot] += now_ - pt;                                     \
        pt = now_;                                                   \
    }
#else
#define WS_LAP(slot)
#endif
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
        WS_LAP(0)
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
        constexpr int Q = (8 * NB + 31) / 32;  // x values per lane
        float xv[Q];
        WS_LAP(1)
        if (active) {
            uint32_t fa[(G + 1) / 2][8];
            WsTiles<NB, E> rt;
            ws_res_load<NB, E, 0>(buf, f, g8, t4, rt);
            for (int b = 0; b < NB; ++b) {
                const int r0 = 8 * b;
                const int nreal = min(8, f - r0);  // real columns of this block
                float* blk = buf + pb_block(f, b);
                // (1) diagonal block, factored in every lane; rows >= nreal are identity. Only
                //     the lower triangle is read: the upper cells hold leftovers of the updates.
                float l[8][8];
                if (nreal == 8) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) ld8(blk + 8 * q, l[q]);
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (q < nreal) {
                            ld8(blk + 8 * q, l[q]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 8; ++k) l[q][k] = k == q ? 1.f : 0.f;
                        }
                    }
                }
                float dv[8], piv[8];
                bool ok = true;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float d = l[c][c];
                    piv[c] = d;
                    ok &= d > 0.f;
                    const float ic = rsqrt_ftz(d);
                    dv[c] = ic;
                    l[c][c] = d * ic;
#pragma unroll
                    for (int q = c + 1; q < 8; ++q) l[q][c] *= ic;
#pragma unroll
                    for (int q = c + 1; q < 8; ++q)
#pragma unroll
                        for (int p = c + 1; p <= q; ++p) l[q][p] = fmaf(-l[q][c], l[p][c], l[q][p]);
                }
                if (!ok) {  // warp-uniform (every lane factored the same block): the first bad pivot
#pragma unroll
                    for (int c = 7; c >= 0; --c)
                        if (!(piv[c] > 0.f)) {
                            bad = r0 + c + 1;
                            badv = piv[c];
                        }
                    break;
                }
                WS_LAP(2)
                __syncwarp();  // every lane has read the block before the TRSM overwrites it
                if (lane == 0) {
                    *reinterpret_cast<float4*>(dinv + r0) = make_float4(dv[0], dv[1], dv[2], dv[3]);
                    *reinterpret_cast<float4*>(dinv + r0 + 4) = make_float4(dv[4], dv[5], dv[6], dv[7]);
                }
                // (2) TRSM of rows r0 .. f (straight-line rounds of 32 rows)
                switch ((f - r0) >> 5) {
                    case 0: ws_trsm<1, NB>(blk, r0, f, lane, l, dv); break;
                    case 1: ws_trsm<2, NB>(blk, r0, f, lane, l, dv); break;
                    case 2: ws_trsm<3, NB>(blk, r0, f, lane, l, dv); break;
                    case 3: ws_trsm<4, NB>(blk, r0, f, lane, l, dv); break;
                    default: ws_trsm<5, NB>(blk, r0, f, lane, l, dv); break;
                }
                __syncwarp();
                WS_LAP(3)
                if (b == NB - 1) break;
                // (3) panel fragments of the pairs in use (2p <= G-1-b; group G-1-b, one above
                //     the panel, is the phantom half of column b+1's top tile and is zeroed)
                switch ((G - 1 - b) >> 1) {
#define ALSK_WS_PAIRS(N) \
    case N - 1: ws_pairs<G, N>(blk, r0, f, g8, t4, fa); break;
                    ALSK_WS_PAIRS(1) ALSK_WS_PAIRS(2) ALSK_WS_PAIRS(3) ALSK_WS_PAIRS(4) ALSK_WS_PAIRS(5)
                    ALSK_WS_PAIRS(6) ALSK_WS_PAIRS(7) ALSK_WS_PAIRS(8)
                    default: ws_pairs<G, 9>(blk, r0, f, g8, t4, fa); break;
#undef ALSK_WS_PAIRS
                }
                // (4) trailing update, columns J' = 0 .. NB-2-b
                WS_LAP(4)
                ws_trailing<NB, E, 0>(buf, f, b, fa, g8, t4, rt);
                ws_res_flush<NB, E, 0>(buf, f, NB - 2 - b, g8, t4, rt);
                __syncwarp();
                WS_LAP(5)
            }
        }
        if (active && bad == 0) {
            // ---- back substitution L^T x = y; lane owns y_j / x_j, j = lane + 32 q ----
            int lbase[Q];  // offset of L[0][j] relative to 8 k0 + 8 c: pb_block(J) - 64 J + (j & 7)
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int j = min(lane + 32 * q, f - 1);
                const int J = j >> 3;
                lbase[q] = static_cast<int>(pb_block(f, J)) - 64 * J + (j & 7);
                xv[q] = lane + 32 * q < f ? buf[pb_index(f, f, j)] : 0.f;
            }
            for (int bb = NB - 1; bb >= 0; --bb) {
                const int k0 = 8 * bb, q0 = k0 >> 5, sl = k0 & 31;
                const int nreal = min(8, f - k0);
                const float* lb = buf + pb_block(f, bb);
                float ysel = xv[0];
#pragma unroll
                for (int q = 1; q < Q; ++q) ysel = q0 == q ? xv[q] : ysel;
                float yb[8], lc[8][8], dvv[8], xb[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) yb[c] = __shfl_sync(~0u, ysel, sl + c);
                ld8(dinv + k0, dvv);
                if (nreal == 8) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) ld8(lb + 8 * c, lc[c]);
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (c < nreal) {
                            ld8(lb + 8 * c, lc[c]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 8; ++k) lc[c][k] = 0.f;
                        }
                    }
                }
#pragma unroll
                for (int c = 7; c >= 0; --c) {  // the newest x (x_c+1) enters last: one FMA on the chain
                    float s = yb[c];
#pragma unroll
                    for (int k = 7; k > c; --k) s = fmaf(-lc[k][c], xb[k], s);
                    xb[c] = c < nreal ? s * dvv[c] : 0.f;
                }
                // y_j -= sum_c L[k0 + c][j] x_c for j < k0 (lanes past it read a safe cell)
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    if (32 * q >= k0) break;  // warp-uniform: no lane of this slice is above the block
                    const bool upd = lane + 32 * q < k0;
                    const float* p = buf + (upd ? lbase[q] + 8 * k0 : 0);
                    float s0 = xv[q], s1 = 0.f;  // two chains; rows k0+c >= f do not exist
#pragma unroll                                       // (their cells may hold anything: masked, not 0*x)
                    for (int c = 0; c < 8; c += 2) {
                        s0 = fmaf(c < nreal ? -p[8 * c] : 0.f, xb[c], s0);
                        s1 = fmaf(c + 1 < nreal ? -p[8 * c + 8] : 0.f, xb[c + 1], s1);
                    }
                    xv[q] = upd ? s0 + s1 : xv[q];
                }
                // the owners of x_k0 .. x_k0+7 take them
                const int oc = lane - sl;  // binary select tree (a dynamic index would go to local memory)
                const float x01 = oc & 1 ? xb[1] : xb[0], x23 = oc & 1 ? xb[3] : xb[2];
                const float x45 = oc & 1 ? xb[5] : xb[4], x67 = oc & 1 ? xb[7] : xb[6];
                const float x03 = oc & 2 ? x23 : x01, x47 = oc & 2 ? x67 : x45;
                const float xs = oc & 4 ? x47 : x03;
                const bool own = lane >= sl && lane < sl + 8;
#pragma unroll
                for (int q = 0; q < Q; ++q) xv[q] = (own && q == q0) ? xs : xv[q];
            }
        }
        WS_LAP(6)
        __syncwarp();  // the buffer is free: fetch the next system while x is stored
        if (lane == 0 && sys + nwarps < count) {
            fence_proxy_async_smem();
            ws_expect_tx(bar, row_bytes);
            ws_bulk_g2s(smem_u32(buf), packed + (sys + nwarps) * pks, row_bytes, bar);
        }
        float* x = out_x + sys * f;
        if (active && bad == 0) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
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
        WS_LAP(7)
    }
#ifdef ALSK_MEASURE
    if (prof && lane == 0)
#pragma unroll
        for (int q = 0; q < 8; ++q) atomicAdd(prof + q, static_cast<unsigned long long>(pacc[q]));
#endif
#undef WS_LAP
}

template <int NB, int E>
void launch_ws(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
               cudaStream_t s) {
    const uint32_t wb = ws_warp_bytes(f);
    const int max_smem = 227 * 1024;
    const int warps = std::max(1, std::min<int>(ws_warps<NB>(), max_smem / static_cast<int>(wb)));
    const int smem = warps * static_cast<int>(wb);
    ALSK_CUDA(cudaFuncSetAttribute(warp_solve_kernel<NB, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t ctas = (count + warps - 1) / warps;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ctas, num_sms()));
    static const bool want_prof = measure_env("ALSK_WS_PROF") != nullptr;
    unsigned long long* prof = nullptr;
    DevBuf pbuf;
    if (want_prof) {
        pbuf.alloc(8 * sizeof(unsigned long long), s);
        ALSK_CUDA(cudaMemsetAsync(pbuf.as<void>(), 0, 8 * sizeof(unsigned long long), s));
        prof = pbuf.as<unsigned long long>();
    }
    warp_solve_kernel<NB, E><<<grid, warps * 32, smem, s>>>(packed, count, f, x, st.min_row, st.column + status_off,
                                                           st.pivot + status_off, status_off, wb, prof);
    ALSK_LAUNCHED();
    if (want_prof) {
        unsigned long long h[8];
        ALSK_CUDA(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s));
        ALSK_CUDA(cudaStreamSynchronize(s));
        const double per = 1e3 * static_cast<double>(count);
        std::fprintf(stderr,
                     "[ws-prof f=%d systems=%lld warps/CTA=%d grid=%u] kcyc per system per warp: load-wait %.2f "
                     "zero %.2f potrf %.2f trsm %.2f frags %.2f trailing %.2f backsub %.2f store %.2f\n",
                     f, static_cast<long long>(count), warps, grid, h[0] / per, h[1] / per, h[2] / per, h[3] / per,
                     h[4] / per, h[5] / per, h[6] / per, h[7] / per);
    }
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
