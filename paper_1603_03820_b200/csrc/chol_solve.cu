// Batched FP32 SPD solve of packed Hermitian rows: one matrix per CTA, resident in
// registers as 8x8 tiles of the augmented lower matrix [A | b] (rows < f: A lower; row f:
// b), blocked right-looking Cholesky, forward substitution folded into the factorization
// (the augmented row becomes y = L^{-1} b), blocked back substitution L^T x = y on the same
// register tiles. Shared memory holds only one block column at a time.
//
// Replaces batch_solve_into (solver.hpp:204-262) for the tensor-core half-sweep (FP32,
// tolerance-checked): all-zero A gives x = 0 (solver.hpp:215-220); a non-positive pivot is
// reported with the failing row, column and pivot like the reference's NumericalError
// (solver.hpp:230-235) and the row's x is zeroed.
//
// Per block column bc: the diagonal-tile owner factors its 8x8 block (rsqrt on the critical
// path), the panel owners solve their tiles against it with the block's operands hoisted
// into registers, every trailing tile takes the rank-8 downdate (8 LDS.128 broadcasts per
// 64 FFMA). Back substitution: per block row (last to first) the tiles below the diagonal
// contribute L^T x partials through shared memory and the diagonal owner solves its 8x8
// upper-triangular system.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace alsk {
namespace {

__device__ __forceinline__ void tile_of(int t, int nb, int& bi, int& bj) {  // column-major lower tiles
    int c = 0;
    while (t >= nb - c) {
        t -= nb - c;
        ++c;
    }
    bj = c;
    bi = c + t;
}

template <int NB>
struct SolveSmem {
    static constexpr int FP = 8 * NB;
    float panel[8 * FP];  // k-major panel of the current block column: panel[c*FP + row]
    float lcc[64];        // factored diagonal block, row-major
    float dall[FP];       // 1 / L[c][c] for every real column
    float ys[FP];         // y = L^{-1} b
    float xs[FP];         // solution
    float red[NB * 8];    // back-substitution partials, one 8-vector per block row
    int flags[4];         // [0] breakdown column + 1, [1] pivot bits
};

template <int NB>
__global__ void __launch_bounds__(((NB * (NB + 1) / 2 + 31) / 32) * 32)
packed_solve_kernel(const float* __restrict__ packed, int f, float* __restrict__ out_x,
                    unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                    double* __restrict__ pivot, int64_t status_base) {
    constexpr int FP = 8 * NB;
    constexpr int NTILES = NB * (NB + 1) / 2;
    __shared__ __align__(16) SolveSmem<NB> sm;
    const int e = threadIdx.x;
    const int64_t row = blockIdx.x;
    const float* pk = packed + row * packed_stride(f);
    float* x = out_x + row * static_cast<int64_t>(f);
    const bool active = e < NTILES;
    int bi = 0, bj = 0;
    if (active) tile_of(e, NB, bi, bj);
    const int ia = 8 * bi, jb = 8 * bj;
    const int nbc = (f + 7) >> 3;  // block columns holding real columns
    const int fb = f >> 3, fr = f & 7;  // block row / offset of the augmented row

    float acc[8][8];
    int nz = 0;
#pragma unroll
    for (int ii = 0; ii < 8; ++ii)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int i = ia + ii, j = jb + jj;
            float v = 0.f;
            if (active && j < f) {
                if (i < f && j <= i) {
                    v = __ldg(pk + pb_index(f, i, j));
                    nz |= v != 0.f;
                } else if (i == f) {
                    v = __ldg(pk + pb_index(f, f, j));
                }
            }
            acc[ii][jj] = v;
        }
    if (e == 0) sm.flags[0] = 0;
    if (!__syncthreads_or(nz)) {  // all-zero A (solver.hpp:215-220)
        for (int i = e; i < f; i += blockDim.x) x[i] = 0.f;
        if (e == 0) column[row] = 0;
        return;
    }

    for (int bc = 0; bc < nbc; ++bc) {
        // (1) diagonal tile: 8x8 Cholesky of the real columns, rsqrt on the critical path
        if (active && bi == bc && bj == bc) {
            int bad = 0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (bad || 8 * bc + c >= f) continue;
                const float d = acc[c][c];
                if (!(d > 0.f)) {
                    bad = 8 * bc + c + 1;
                    sm.flags[1] = __float_as_int(d);
                    continue;
                }
                const float inv = rsqrtf(d);
                acc[c][c] = d * inv;
                sm.dall[8 * bc + c] = inv;
#pragma unroll
                for (int r = c + 1; r < 8; ++r) acc[r][c] *= inv;
#pragma unroll
                for (int r = c + 1; r < 8; ++r)
#pragma unroll
                    for (int q = c + 1; q <= r; ++q) acc[r][q] = fmaf(-acc[r][c], acc[q][c], acc[r][q]);
            }
            if (bad) sm.flags[0] = bad;
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int c = 0; c < 8; c += 4)
                    *reinterpret_cast<float4*>(&sm.lcc[r * 8 + c]) =
                        make_float4(acc[r][c], acc[r][c + 1], acc[r][c + 2], acc[r][c + 3]);
        }
        __syncthreads();
        if (sm.flags[0]) {  // breakdown: report, zero the row (uniform)
            if (e == 0) {
                column[row] = sm.flags[0];
                pivot[row] = static_cast<double>(__int_as_float(sm.flags[1]));
                atomicMin(min_row, static_cast<unsigned long long>(status_base + row));
            }
            for (int i = e; i < f; i += blockDim.x) x[i] = 0.f;
            return;
        }
        // (2) panel tiles: L_ic = P * L_cc^{-T}, operands hoisted from shared memory
        if (active && bj == bc && bi > bc) {
            float lc[8][8], di[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float4 a = *reinterpret_cast<const float4*>(&sm.lcc[c * 8]);
                const float4 b = *reinterpret_cast<const float4*>(&sm.lcc[c * 8 + 4]);
                lc[c][0] = a.x, lc[c][1] = a.y, lc[c][2] = a.z, lc[c][3] = a.w;
                lc[c][4] = b.x, lc[c][5] = b.y, lc[c][6] = b.z, lc[c][7] = b.w;
                di[c] = (8 * bc + c < f) ? sm.dall[8 * bc + c] : 0.f;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    float s0 = acc[r][c], s1 = 0.f;  // two partial sums shorten the chain
#pragma unroll
                    for (int k = 0; k < c; ++k) {
                        if (k & 1) s1 = fmaf(-acc[r][k], lc[c][k], s1);
                        else s0 = fmaf(-acc[r][k], lc[c][k], s0);
                    }
                    acc[r][c] = (s0 + s1) * di[c];
                }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                float4* dst = reinterpret_cast<float4*>(&sm.panel[c * FP + ia]);
                dst[0] = make_float4(acc[0][c], acc[1][c], acc[2][c], acc[3][c]);
                dst[1] = make_float4(acc[4][c], acc[5][c], acc[6][c], acc[7][c]);
            }
        }
        __syncthreads();
        // (3) trailing tiles: rank-8 downdate with the published panel
        if (active && bj > bc) {
#pragma unroll 2
            for (int k = 0; k < 8; ++k) {
                const float4 a0 = *reinterpret_cast<const float4*>(&sm.panel[k * FP + ia]);
                const float4 a1 = *reinterpret_cast<const float4*>(&sm.panel[k * FP + ia + 4]);
                const float4 b0 = *reinterpret_cast<const float4*>(&sm.panel[k * FP + jb]);
                const float4 b1 = *reinterpret_cast<const float4*>(&sm.panel[k * FP + jb + 4]);
                const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(-a[i], b[j], acc[i][j]);
            }
        }
        // the panel is rewritten only after the next diagonal barrier
    }
    if (e == 0) column[row] = 0;

    // y = L^{-1} b sits in the augmented row of block row fb
    if (active && bi == fb) {
#pragma unroll
        for (int r = 0; r < 8; ++r)  // static indices keep acc in registers
            if (r == fr) {
#pragma unroll
                for (int jj = 0; jj < 8; ++jj)
                    if (jb + jj < f) sm.ys[jb + jj] = acc[r][jj];
            }
    }
    __syncthreads();
    // back substitution L^T x = y, block rows from last to first
    for (int bk = nbc - 1; bk >= 0; --bk) {
        if (active && bj == bk && bi > bk && bi < nbc) {
            float p[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) p[c] = 0.f;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int i = ia + r;
                if (i >= f) continue;  // augmented row and padding
                const float xi = sm.xs[i];
#pragma unroll
                for (int c = 0; c < 8; ++c) p[c] = fmaf(acc[r][c], xi, p[c]);
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) sm.red[bi * 8 + c] = p[c];
        }
        __syncthreads();
        if (active && bi == bk && bj == bk) {
            float s[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) s[c] = (8 * bk + c < f) ? sm.ys[8 * bk + c] : 0.f;
            for (int b2 = bk + 1; b2 < nbc; ++b2)
#pragma unroll
                for (int c = 0; c < 8; ++c) s[c] -= sm.red[b2 * 8 + c];
            float xv[8];
#pragma unroll
            for (int c = 7; c >= 0; --c) {
                float t = s[c];
#pragma unroll
                for (int r = c + 1; r < 8; ++r)
                    if (8 * bk + r < f) t = fmaf(-acc[r][c], xv[r], t);
                xv[c] = (8 * bk + c < f) ? t * sm.dall[8 * bk + c] : 0.f;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (8 * bk + c < f) sm.xs[8 * bk + c] = xv[c];
        }
        __syncthreads();
    }
    for (int i = e; i < f; i += blockDim.x) x[i] = sm.xs[i];
}

template <int NB>
void launch(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t off, cudaStream_t s) {
    constexpr int GT = ((NB * (NB + 1) / 2 + 31) / 32) * 32;
    constexpr int64_t kMaxGrid = 1LL << 30;
    for (int64_t c0 = 0; c0 < count; c0 += kMaxGrid) {
        const int64_t n = std::min<int64_t>(count - c0, kMaxGrid);
        packed_solve_kernel<NB><<<static_cast<unsigned>(n), GT, 0, s>>>(
            packed + c0 * packed_stride(f), f, x + c0 * f, st.min_row,
            st.column + off + c0, st.pivot + off + c0, off + c0);
        ALSK_LAUNCHED();
    }
}

}  // namespace

bool packed_solve_tiles(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                  cudaStream_t s) {
    const int nb = (f + 1 + 7) / 8;
#define ALSK_PS_CASE(NBV)                                     \
    if (nb <= NBV) {                                          \
        launch<NBV>(packed, count, f, x, st, status_off, s);  \
        return true;                                          \
    }
    ALSK_PS_CASE(2)
    ALSK_PS_CASE(4)
    ALSK_PS_CASE(7)
    ALSK_PS_CASE(10)
    ALSK_PS_CASE(13)
    ALSK_PS_CASE(15)
#undef ALSK_PS_CASE
    return false;
}

}  // namespace alsk
