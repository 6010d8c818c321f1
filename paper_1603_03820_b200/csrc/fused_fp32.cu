// FP32 fused half-sweep kernel: get_hermitian + get_bias + Cholesky + both triangular
// solves for one row per CTA, without materialising A_u in HBM.
//
// Replaces, for precision ALSK_PREC_FP32, the loop body of update_x (solver.hpp:336-344):
// assemble_mo_rows (solver.hpp:99-157) followed by batch_solve_into (solver.hpp:204-262).
//
// Design (B200):
//  * Augmented outer product. Each gathered factor row theta_v is staged in shared memory
//    as theta'_v = [theta_v, r_uv, 0...] (length FP = 8*NB >= f+1). The lower triangle of
//    sum theta' theta'^T holds A_u in rows/cols < f and B_u in row f, so the bias is the
//    same FMA stream as the Hermitian (cuMF's get_bias folded into get_hermitian).
//  * Register blocking. Thread t owns one 8x8 tile (bi,bj), bj<=bi, of the lower
//    triangle: 64 FP32 accumulators, 4 LDS.128 per 64 FFMA. f=100 -> NB=13, 91 tiles,
//    96 threads. The 8-float block halves are XOR-swizzled by bit 2 of the block index so
//    eight consecutive tiles of a quarter-warp hit eight distinct 16-byte bank groups.
//  * Gather. Factor rows are copied global->shared with cp.async (LDGSTS, 16 B per lane,
//    L2-only .cg) into a double-buffered chunk of 32 nonzeros, overlapping the next
//    chunk's gather with the current chunk's FMAs.
//  * Cholesky in registers. The factorisation is a sequence of rank-1 downdates, i.e. the
//    same outer product with the current column of L: per column c the owners publish
//    column c to shared memory, one barrier, every thread downdates its tile. The
//    augmented row turns into y = L^{-1} B on the way (forward substitution for free).
//  * Back substitution L^T x = y by warp 0 from a packed copy of L in shared memory
//    (aliasing the gather buffers), column-oriented with warp shuffles.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace alsk {
namespace {

constexpr int KC = 32;  // nonzeros per staged chunk

template <int NB>
struct FusedShape {
    static constexpr int FP = NB * 8;                     // padded augmented width
    static constexpr int NTILES = NB * (NB + 1) / 2;      // lower-triangular 8x8 tiles
    static constexpr int NT = ((NTILES + 31) / 32) * 32;  // threads per CTA
    static constexpr int LDT = FP;                        // row stride of a staged chunk
    static constexpr int TILE_FLOATS = 2 * KC * LDT;      // double-buffered gather area
    static constexpr int LPK_FLOATS = FP * (FP + 1) / 2 + FP;  // packed L + y (upper bound)
    static constexpr int UNION_FLOATS = TILE_FLOATS > LPK_FLOATS ? TILE_FLOATS : LPK_FLOATS;
    // + column exchange buffer (2*FP) + dinv (FP)
    static constexpr size_t SMEM = (UNION_FLOATS + 3 * FP) * sizeof(float);
};

__device__ __forceinline__ int swz_block_half(int blk, int h) { return 2 * blk + (h ^ ((blk >> 2) & 1)); }
// physical float offset of logical column c within a staged row
__device__ __forceinline__ int phys_col(int c) {
    const int blk = c >> 3, h = (c >> 2) & 1, q = c & 3;
    return 4 * swz_block_half(blk, h) + q;
}

__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__device__ __forceinline__ void tile_coords(int t, int& bi, int& bj) {
    int b = 0;
    while ((b + 1) * (b + 2) / 2 <= t) ++b;
    bi = b;
    bj = t - b * (b + 1) / 2;
}

// Stage nonzeros [k, k+cnt) of the current row into buffer `dst` (KC x LDT floats).
template <int NB>
__device__ __forceinline__ void stage_chunk(float* dst, const int32_t* __restrict__ col_idx,
                                            const float* __restrict__ values,
                                            const float* __restrict__ theta, int64_t col_lo,
                                            int f, bool vec16, int64_t k, int cnt) {
    using S = FusedShape<NB>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = S::NT / 32;
    if (vec16) {
        const int q4 = f >> 2;  // 16-byte pieces per factor row
        for (int kk = warp; kk < cnt; kk += NW) {
            const int64_t v = static_cast<int64_t>(col_idx[k + kk]) - col_lo;
            const float* src = theta + v * f;
            float* row = dst + kk * S::LDT;
            for (int c4 = lane; c4 < q4; c4 += 32) {
                const int c = c4 * 4;
                cp_async16(row + phys_col(c), src + c);
            }
            if (lane == 31) row[phys_col(f)] = values[k + kk];
        }
    } else {
        for (int kk = warp; kk < cnt; kk += NW) {
            const int64_t v = static_cast<int64_t>(col_idx[k + kk]) - col_lo;
            const float* src = theta + v * f;
            float* row = dst + kk * S::LDT;
            for (int c = lane; c < f; c += 32) cp_async4(row + phys_col(c), src + c);
            if (lane == 31) row[phys_col(f)] = values[k + kk];
        }
    }
}

// Zero the padding columns (f+1 .. FP-1) of both staging buffers; column f is rewritten
// with r_uv per staged nonzero, columns < f by the gather.
template <int NB>
__device__ __forceinline__ void zero_padding(float* tile, int f) {
    using S = FusedShape<NB>;
    const int pad = S::FP - (f + 1);
    if (pad <= 0) return;
    for (int e = threadIdx.x; e < 2 * KC * pad; e += S::NT) {
        const int row = e / pad, c = f + 1 + (e - row * pad);
        tile[row * S::LDT + phys_col(c)] = 0.f;
    }
}

// Accumulate the augmented outer products of the current row into acc (8x8 tile).
template <int NB>
__device__ __forceinline__ void accumulate_row(float (&acc)[8][8], float* tile,
                                               const int32_t* __restrict__ col_idx,
                                               const float* __restrict__ values,
                                               const float* __restrict__ theta, int64_t col_lo,
                                               int f, bool vec16, int64_t k0, int64_t k1,
                                               bool active, int offA0, int offA1, int offB0,
                                               int offB1) {
    using S = FusedShape<NB>;
    const int64_t n = k1 - k0;
    if (n <= 0) return;
    const int nchunks = static_cast<int>((n + KC - 1) / KC);
    stage_chunk<NB>(tile, col_idx, values, theta, col_lo, f, vec16, k0,
                    static_cast<int>((n < KC ? n : (int64_t)KC)));
    cp_async_commit();
    for (int ch = 0; ch < nchunks; ++ch) {
        float* cur = tile + (ch & 1) * KC * S::LDT;
        const int cnt = static_cast<int>(((n - (int64_t)ch * KC) < KC ? (n - (int64_t)ch * KC) : (int64_t)KC));
        if (ch + 1 < nchunks) {
            const int64_t kn = k0 + static_cast<int64_t>(ch + 1) * KC;
            stage_chunk<NB>(tile + ((ch + 1) & 1) * KC * S::LDT, col_idx, values, theta, col_lo, f,
                            vec16, kn, static_cast<int>(((k1 - kn) < KC ? (k1 - kn) : (int64_t)KC)));
            cp_async_commit();
            cp_async_wait_1();
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
        if (active) {
#pragma unroll 2
            for (int kk = 0; kk < cnt; ++kk) {
                const float* trow = cur + kk * S::LDT;
                const float4 a0 = *reinterpret_cast<const float4*>(trow + offA0);
                const float4 a1 = *reinterpret_cast<const float4*>(trow + offA1);
                const float4 b0 = *reinterpret_cast<const float4*>(trow + offB0);
                const float4 b1 = *reinterpret_cast<const float4*>(trow + offB1);
                const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
        }
        __syncthreads();  // buffer `cur` is restaged two chunks later
    }
}

template <int NB, bool SOLVE>
__global__ void __launch_bounds__(FusedShape<NB>::NT, (NB >= 14 ? 2 : 4))
fused_update_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                    const float* __restrict__ values, int64_t col_lo,
                    const float* __restrict__ theta, int f, float lambda, int64_t rb,
                    float* __restrict__ out_x, float* __restrict__ out_a, float* __restrict__ out_b,
                    unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                    double* __restrict__ pivot, int64_t status_base) {
    using S = FusedShape<NB>;
    extern __shared__ __align__(16) float smem[];
    float* tile = smem;                      // union: gather chunks | packed L
    float* colbuf = smem + S::UNION_FLOATS;  // 2 x FP
    float* dinv = colbuf + 2 * S::FP;        // FP

    const int tid = threadIdx.x;
    const int64_t row = blockIdx.x;
    const int64_t u = rb + row;
    const int64_t k0 = row_ptr[u], k1 = row_ptr[u + 1];
    const bool active = tid < S::NTILES;
    int bi = 0, bj = 0;
    if (active) tile_coords(tid, bi, bj);
    const int offA0 = 4 * swz_block_half(bi, 0), offA1 = 4 * swz_block_half(bi, 1);
    const int offB0 = 4 * swz_block_half(bj, 0), offB1 = 4 * swz_block_half(bj, 1);
    const bool vec16 = ((f & 3) == 0) && ((reinterpret_cast<uintptr_t>(theta) & 15) == 0);

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    zero_padding<NB>(tile, f);
    accumulate_row<NB>(acc, tile, col_idx, values, theta, col_lo, f, vec16, k0, k1, active, offA0,
                       offA1, offB0, offB1);

    // lambda * n_u on the diagonal (solver.hpp:141,152), float arithmetic
    const float reg = lambda * static_cast<float>(k1 - k0);
    if (active && bi == bj) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (8 * bi + i < f) acc[i][i] += reg;
    }

    if constexpr (!SOLVE) {
        if (!active) return;
        float* a_out = out_a + row * static_cast<int64_t>(f) * f;
        float* b_out = out_b + row * f;
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const int i = 8 * bi + ii, j = 8 * bj + jj;
                if (j > i || j >= f || i > f) continue;
                if (i == f) {
                    b_out[j] = acc[ii][jj];
                } else {
                    a_out[i * f + j] = acc[ii][jj];
                    a_out[j * f + i] = acc[ii][jj];
                }
            }
        return;
    } else {
        // all-zero A (empty row with lambda*0, or zero factors) => x = 0 (solver.hpp:215-220)
        int nz = 0;
        if (active) {
#pragma unroll
            for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int i = 8 * bi + ii, j = 8 * bj + jj;
                    if (i < f && j <= i) nz |= (acc[ii][jj] != 0.f);
                }
        }
        float* x = out_x + row * f;
        if (!__syncthreads_or(nz)) {
            for (int i = tid; i < f; i += S::NT) x[i] = 0.f;
            if (tid == 0) column[row] = 0;
            return;
        }

        // ---- in-register right-looking Cholesky of the augmented system ----
        bool broke = false;
        for (int c = 0; c < f; ++c) {
            const int bc = c >> 3, jc = c & 7;
            float* cb = colbuf + (c & 1) * S::FP;
            if (active && bj == bc) {
#pragma unroll
                for (int jj = 0; jj < 8; ++jj)
                    if (jj == jc) {
#pragma unroll
                        for (int ii = 0; ii < 8; ++ii) cb[8 * bi + ii] = acc[ii][jj];
                    }
            }
            __syncthreads();
            const float d = cb[c];
            if (!(d > 0.f)) {  // uniform across the CTA
                if (tid == 0) {
                    column[row] = c + 1;
                    pivot[row] = static_cast<double>(d);
                    atomicMin(min_row, static_cast<unsigned long long>(status_base + row));
                }
                broke = true;
                break;
            }
            const float rinv = rsqrtf(d);
            if (tid == 0) dinv[c] = rinv;
            if (active && bj >= bc) {
                float li[8], lj[8];
#pragma unroll
                for (int ii = 0; ii < 8; ++ii) li[ii] = cb[8 * bi + ii] * rinv;
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) lj[jj] = cb[8 * bj + jj] * rinv;
                const bool diag = (bi == bj);
#pragma unroll
                for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const bool upd = (8 * bj + jj > c) && (!diag || ii >= jj);
                        if (upd) acc[ii][jj] = fmaf(-li[ii], lj[jj], acc[ii][jj]);
                    }
                if (bj == bc) {
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        if (jj == jc) {
#pragma unroll
                            for (int ii = 0; ii < 8; ++ii) acc[ii][jj] = li[ii];
                        }
                }
            }
        }
        if (broke) {
            for (int i = tid; i < f; i += S::NT) x[i] = 0.f;
            return;
        }
        if (tid == 0) column[row] = 0;

        // ---- dump packed L (rows < f) and y (row f) into the gather area ----
        float* lpk = tile;
        if (active) {
#pragma unroll
            for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int i = 8 * bi + ii, j = 8 * bj + jj;
                    if (i <= f && j < f && j <= i) lpk[i * (i + 1) / 2 + j] = acc[ii][jj];
                }
        }
        __syncthreads();

        // ---- back substitution L^T x = y, warp 0, column oriented ----
        if (tid < 32) {
            const int lane = tid;
            constexpr int G = (S::FP + 31) / 32;
            const float* yrow = lpk + f * (f + 1) / 2;
            float yv[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int j = g * 32 + lane;
                yv[g] = j < f ? yrow[j] : 0.f;
            }
#pragma unroll
            for (int g = G - 1; g >= 0; --g) {
                for (int t = 31; t >= 0; --t) {
                    const int i = g * 32 + t;
                    if (i >= f) continue;
                    const float xi = __shfl_sync(0xffffffffu, yv[g], t) * dinv[i];
                    if (lane == t) yv[g] = xi;
                    const float* lrow = lpk + i * (i + 1) / 2;
#pragma unroll
                    for (int gg = 0; gg <= g; ++gg) {
                        const int j = gg * 32 + lane;
                        if (j < i) yv[gg] = fmaf(-lrow[j], xi, yv[gg]);
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int j = g * 32 + lane;
                if (j < f) x[j] = yv[g];
            }
        }
    }
}

template <int NB, bool SOLVE>
void launch_fused(const DevCsr& r, const float* theta, int f, float lambda, int64_t rb, int64_t re,
                  float* x, float* a, float* b, const SolveStatus* st, cudaStream_t s) {
    using S = FusedShape<NB>;
    auto k = fused_update_kernel<NB, SOLVE>;
    ALSK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    constexpr int64_t kMaxGrid = 1LL << 30;
    for (int64_t b0 = rb; b0 < re; b0 += kMaxGrid) {
        const int64_t n = std::min<int64_t>(re - b0, kMaxGrid);
        const int64_t off = b0 - rb;
        k<<<static_cast<unsigned>(n), S::NT, S::SMEM, s>>>(
            r.row_ptr, r.col_idx, r.values, r.col_offset, theta, f, lambda, b0,
            x ? x + off * f : nullptr, a ? a + off * f * f : nullptr, b ? b + off * f : nullptr,
            st ? st->min_row : nullptr, st ? st->column + off : nullptr,
            st ? st->pivot + off : nullptr, off);
        ALSK_LAUNCHED();
    }
}

template <bool SOLVE>
bool dispatch(const DevCsr& r, const float* theta, int f, float lambda, int64_t rb, int64_t re,
              float* x, float* a, float* b, const SolveStatus* st, cudaStream_t s) {
    const int need = (f + 1 + 7) / 8;
    if (re <= rb) return true;
#define ALSK_FUSED_CASE(NBV)                                                     \
    if (need <= NBV) {                                                          \
        launch_fused<NBV, SOLVE>(r, theta, f, lambda, rb, re, x, a, b, st, s); \
        return true;                                                            \
    }
    ALSK_FUSED_CASE(2)
    ALSK_FUSED_CASE(4)
    ALSK_FUSED_CASE(7)
    ALSK_FUSED_CASE(10)
    ALSK_FUSED_CASE(13)
    ALSK_FUSED_CASE(16)
#undef ALSK_FUSED_CASE
    return false;
}

}  // namespace

bool update_fused_fp32(const DevCsr& r, const float* theta, int f, float lambda, int64_t rb,
                       int64_t re, float* x_out, const SolveStatus& st, cudaStream_t s) {
    return dispatch<true>(r, theta, f, lambda, rb, re, x_out, nullptr, nullptr, &st, s);
}

bool hermitian_fused_fp32(const DevCsr& r, const float* theta, int f, float lambda, int64_t rb,
                          int64_t re, float* A, float* B, cudaStream_t s) {
    return dispatch<false>(r, theta, f, lambda, rb, re, nullptr, A, B, nullptr, s);
}

}  // namespace alsk
