// FP32 fused half-sweep kernel: get_hermitian + get_bias + Cholesky + both triangular
// solves for one row per CTA, without materialising A_u in HBM.
//
// Replaces, for precision ALSK_PREC_FP32, the loop body of update_x (solver.hpp:336-344):
// assemble_mo_rows (solver.hpp:99-157) followed by batch_solve_into (solver.hpp:204-262).
//
// Design (B200):
//  * Augmented outer product. Each gathered factor row theta_v (stride ldt = f rounded up
//    to a multiple of 4, zero padded) is staged in shared memory as
//    theta'_v = [theta_v, 0.., r_uv at column `aug` = ldt, 0..] of width FP = 8*NB. The
//    lower triangle of sum theta' theta'^T holds A_u in rows/cols < f and B_u in row aug,
//    so the bias is the same FMA stream as the Hermitian.
//  * Register blocking. Thread t owns one 8x8 tile (bi,bj), bj<=bi, of the lower
//    triangle: 64 FP32 accumulators, 4 LDS.128 per 64 FFMA. f=100 -> NB=13, 91 tiles,
//    96 threads.
//  * Gather by TMA bulk copies. Lane k of warp 0 issues one cp.async.bulk (global ->
//    shared, ldt*4 bytes, completion counted on the stage's mbarrier) for the k-th
//    nonzero of a 32-nonzero chunk; a 3-stage ring keeps two chunks in flight while the
//    FMAs consume the third. Stages are handed back through per-stage "empty" mbarriers
//    (one arrive per warp), so warps never wait on each other inside the stream.
//  * Blocked Cholesky in registers. Per 8-column block: the diagonal-tile owner factors
//    its 8x8 block and publishes it; the panel owners solve their tiles against it
//    (forward substitution, 8 independent rows each) and publish the panel transposed;
//    every trailing tile takes the rank-8 downdate, which is the Hermitian inner loop
//    again. Two barriers per block column. The augmented row becomes y = L^{-1} B.
//  * Back substitution L^T x = y by warp 0 from a packed copy of L in shared memory
//    (aliasing the stage ring), column-oriented with warp shuffles.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "measure.cuh"

namespace alsk {
namespace {

constexpr int KC = 32;     // nonzeros per staged chunk (one bulk copy per lane of warp 0)
constexpr int STAGES = 3;  // ring depth

template <int NB>
struct FusedShape {
    static constexpr int FP = NB * 8;                     // padded augmented width
    static constexpr int NTILES = NB * (NB + 1) / 2;      // lower-triangular 8x8 tiles
    static constexpr int NT = ((NTILES + 31) / 32) * 32;  // threads per CTA
    static constexpr int LDT = FP;                        // row stride of a staged chunk
    static constexpr int RING_FLOATS = STAGES * KC * LDT;
    static constexpr int LPK_FLOATS = FP * (FP + 1) / 2 + FP;  // packed L + y (upper bound)
    static constexpr int UNION_FLOATS = RING_FLOATS > LPK_FLOATS ? RING_FLOATS : LPK_FLOATS;
    // + panel (8 x FP) + diag block (64) + dinv (FP) + flags (8) + mbarriers (STAGES x 2 floats)
    static constexpr int EXTRA_FLOATS = 8 * FP + 64 + FP + 8 + 4 * STAGES + 2;
    static constexpr size_t SMEM = (UNION_FLOATS + EXTRA_FLOATS) * sizeof(float) + 16;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// Column-major enumeration of the lower-triangular tiles: column bj holds tiles
// (bj..NB-1, bj). The trailing tiles of block column bc (bj > bc) are then a suffix of the
// enumeration and the panel tiles a contiguous run, so the Cholesky phases occupy as few
// warps as possible.
__device__ __forceinline__ void tile_coords_colmajor(int t, int nb, int& bi, int& bj) {
    int c = 0;
    while (t >= nb - c) {
        t -= nb - c;
        ++c;
    }
    bj = c;
    bi = c + t;
}

// acc[ii][jj] += sign * sum_k  rowsA[k][ia+ii] * rowsB[k][jb+jj]  over k in [0,cnt) of a
// k-major buffer with row stride LDT (the Hermitian inner loop; also the rank-8 downdate).
template <int LDT, bool NEG>
__device__ __forceinline__ void outer_accumulate(float (&acc)[8][8], const float* buf, int cnt, int ia, int jb) {
#pragma unroll 2
    for (int kk = 0; kk < cnt; ++kk) {
        const float* trow = buf + kk * LDT;
        const float4 a0 = *reinterpret_cast<const float4*>(trow + ia);
        const float4 a1 = *reinterpret_cast<const float4*>(trow + ia + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(trow + jb);
        const float4 b1 = *reinterpret_cast<const float4*>(trow + jb + 4);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(NEG ? -a[i] : a[i], b[j], acc[i][j]);
    }
}

// Issue the bulk copies of chunk `ch` (nonzeros [k0+ch*KC, ...)) into its ring stage.
// Called by all lanes of warp 0.
template <int NB>
__device__ __forceinline__ void issue_chunk(float* ring, uint64_t* bars, const int32_t* __restrict__ col_idx,
                                            const float* __restrict__ values, const float* __restrict__ theta,
                                            int64_t col_lo, int ldt, int aug, int64_t k0, int64_t n, int ch) {
    using S = FusedShape<NB>;
    const int lane = threadIdx.x & 31;
    const int64_t kb = k0 + static_cast<int64_t>(ch) * KC;
    const int64_t left = n - static_cast<int64_t>(ch) * KC;
    const int cnt = static_cast<int>(left < KC ? left : KC);
    const int st = ch % STAGES;
    float* buf = ring + st * KC * S::LDT;
    const uint32_t row_bytes = static_cast<uint32_t>(ldt) * 4u;
    float* row = buf + lane * S::LDT;
    int64_t v = 0;
    if (lane < cnt) {
        v = static_cast<int64_t>(col_idx[kb + lane]) - col_lo;
        row[aug] = values[kb + lane];
    }
    __syncwarp();  // the rating writes happen-before lane 0's releasing arrive
    if (lane == 0) mbar_expect_tx(&bars[st], row_bytes * static_cast<uint32_t>(cnt));
    __syncwarp();
    if (lane < cnt) bulk_g2s(row, theta + v * ldt, row_bytes, &bars[st]);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int NB, bool SOLVE>
__global__ void __launch_bounds__(FusedShape<NB>::NT, (NB >= 14 ? 2 : 4))
fused_update_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                    const float* __restrict__ values, int64_t col_lo, const float* __restrict__ theta,
                    int f, int ldt, float lambda, int64_t rb, float* __restrict__ out_x,
                    float* __restrict__ out_a, float* __restrict__ out_b,
                    unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                    double* __restrict__ pivot, int64_t status_base) {
    using S = FusedShape<NB>;
    extern __shared__ __align__(16) float smem[];
    float* ring = smem;                            // STAGES x KC x LDT  | later: packed L + y
    float* panel = smem + S::UNION_FLOATS;         // 8 x FP (k-major: panel[k*FP + row])
    float* dblk = panel + 8 * S::FP;               // 8 x 8 factored diagonal block
    float* dinv = dblk + 64;                       // FP: 1 / L[c][c]
    int* flags = reinterpret_cast<int*>(dinv + S::FP);  // [0] breakdown column+1, [1] pivot bits
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(flags + 8) + 7) & ~static_cast<uintptr_t>(7));

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int aug = ldt;  // augmented (rating) column
    const int64_t row = blockIdx.x;
    const int64_t u = rb + row;
    const int64_t k0 = row_ptr[u], k1 = row_ptr[u + 1];
    const int64_t n = k1 - k0;
    const bool active = tid < S::NTILES;
    int bi = 0, bj = 0;
    if (active) tile_coords_colmajor(tid, NB, bi, bj);
    const int ia = 8 * bi, jb = 8 * bj;

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    // zero the ring once (padding columns must read as 0); init stage barriers
    for (int e = tid; e < S::RING_FLOATS / 4; e += S::NT) reinterpret_cast<float4*>(ring)[e] = make_float4(0, 0, 0, 0);
    uint64_t* empty = bars + STAGES;  // consumer release: one arrive per warp
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&empty[s], S::NT / 32);
        }
        flags[0] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();

    // ---- Hermitian + bias: stream the row's factor rows through the TMA ring ----
    const int nchunks = static_cast<int>((n + KC - 1) / KC);
    if (warp == 0) {
        for (int ch = 0; ch < STAGES - 1 && ch < nchunks; ++ch)
            issue_chunk<NB>(ring, bars, col_idx, values, theta, col_lo, ldt, aug, k0, n, ch);
    }
    for (int ch = 0; ch < nchunks; ++ch) {
        const int nx = ch + STAGES - 1;
        if (warp == 0 && nx < nchunks) {
            // refill the stage consumed at iteration ch-1 once every warp released it
            mbar_wait(&empty[nx % STAGES], static_cast<uint32_t>(((nx / STAGES) - 1) & 1));
            issue_chunk<NB>(ring, bars, col_idx, values, theta, col_lo, ldt, aug, k0, n, nx);
        }
        const int st = ch % STAGES;
        mbar_wait(&bars[st], static_cast<uint32_t>((ch / STAGES) & 1));
        const int64_t left = n - static_cast<int64_t>(ch) * KC;
        const int cnt = static_cast<int>(left < KC ? left : KC);
        if (active) outer_accumulate<S::LDT, false>(acc, ring + st * KC * S::LDT, cnt, ia, jb);
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[st]);
    }
    __syncthreads();  // all chunks consumed before the ring is reused

    // lambda * n_u on the diagonal (solver.hpp:141,152), float arithmetic
    const float reg = lambda * static_cast<float>(n);
    if (active && bi == bj) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (ia + i < f) acc[i][i] += reg;
    }

    if constexpr (!SOLVE) {
        if (!active) return;
        float* a_out = out_a + row * static_cast<int64_t>(f) * f;
        float* b_out = out_b + row * f;
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const int i = ia + ii, j = jb + jj;
                if (j > i || j >= f) continue;
                if (i == aug) {
                    b_out[j] = acc[ii][jj];
                } else if (i < f) {
                    a_out[i * f + j] = acc[ii][jj];
                    a_out[j * f + i] = acc[ii][jj];
                }
            }
        return;
    } else {
        float* x = out_x + row * f;
        // all-zero A (empty row with lambda*0, or zero factors) => x = 0 (solver.hpp:215-220)
        int nz = 0;
        if (active) {
#pragma unroll
            for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                for (int jj = 0; jj < 8; ++jj)
                    if (ia + ii < f && jb + jj <= ia + ii) nz |= (acc[ii][jj] != 0.f);
        }
        if (!__syncthreads_or(nz)) {
            for (int i = tid; i < f; i += S::NT) x[i] = 0.f;
            if (tid == 0) column[row] = 0;
            return;
        }

        // ---- blocked right-looking Cholesky in registers ----
        const int nbc = (f + 7) >> 3;  // block columns holding real columns
        for (int bc = 0; bc < nbc; ++bc) {
            // (A) diagonal tile owner factors its 8x8 block (real columns only)
            if (active && bi == bc && bj == bc) {
                int bad = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (bad || 8 * bc + c >= f) continue;
                    const float d = acc[c][c];
                    if (!(d > 0.f)) {
                        bad = 8 * bc + c + 1;
                        flags[1] = __float_as_int(d);
                        continue;
                    }
                    const float l = sqrtf(d), inv = 1.0f / l;
                    acc[c][c] = l;
                    dinv[8 * bc + c] = inv;
#pragma unroll
                    for (int r = c + 1; r < 8; ++r) acc[r][c] *= inv;
#pragma unroll
                    for (int r = c + 1; r < 8; ++r)
#pragma unroll
                        for (int q = c + 1; q <= r; ++q) acc[r][q] = fmaf(-acc[r][c], acc[q][c], acc[r][q]);
                }
                flags[0] = bad;
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int c = 0; c < 8; ++c) dblk[r * 8 + c] = acc[r][c];
            }
            __syncthreads();
            if (flags[0]) {  // uniform: breakdown at column flags[0]-1
                if (tid == 0) {
                    column[row] = flags[0];
                    pivot[row] = static_cast<double>(__int_as_float(flags[1]));
                    atomicMin(min_row, static_cast<unsigned long long>(status_base + row));
                }
                for (int i = tid; i < f; i += S::NT) x[i] = 0.f;
                return;
            }
            // (B) panel tiles (bi > bc, bj == bc): L_panel = P * L_cc^{-T}, row by row forward
            //     substitution; publish transposed (k-major) for the rank-8 downdate
            if (active && bj == bc && bi > bc) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float di = (8 * bc + c < f) ? dinv[8 * bc + c] : 0.f;
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        float s = acc[r][c];
#pragma unroll
                        for (int k = 0; k < c; ++k) s = fmaf(-acc[r][k], dblk[c * 8 + k], s);
                        acc[r][c] = s * di;
                    }
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    float4* dst = reinterpret_cast<float4*>(panel + c * S::FP + ia);
                    dst[0] = make_float4(acc[0][c], acc[1][c], acc[2][c], acc[3][c]);
                    dst[1] = make_float4(acc[4][c], acc[5][c], acc[6][c], acc[7][c]);
                }
            }
            __syncthreads();
            // (C) trailing tiles (bj > bc): rank-8 downdate with the published panel
            if (active && bj > bc) outer_accumulate<S::FP, true>(acc, panel, 8, ia, jb);
        }
        if (tid == 0) column[row] = 0;

        // ---- dump packed L (rows < f) and y (row aug) into the ring area ----
        __syncthreads();
        float* lpk = ring;
        float* yrow = lpk + f * (f + 1) / 2;
        if (active) {
#pragma unroll
            for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const int i = ia + ii, j = jb + jj;
                    if (j >= f || j > i) continue;
                    if (i < f) lpk[i * (i + 1) / 2 + j] = acc[ii][jj];
                    else if (i == aug) yrow[j] = acc[ii][jj];
                }
        }
        __syncthreads();

        // ---- back substitution L^T x = y, warp 0, column oriented ----
        if (tid < 32) {
            const int lane = tid;
            constexpr int G = (S::FP + 31) / 32;
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
void launch_fused(const DevCsr& r, const float* theta, int f, int ldt, float lambda, int64_t rb, int64_t re,
                  float* x, float* a, float* b, const SolveStatus* st, cudaStream_t s) {
    using S = FusedShape<NB>;
    auto k = fused_update_kernel<NB, SOLVE>;
    ALSK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    constexpr int64_t kMaxGrid = 1LL << 30;
    for (int64_t b0 = rb; b0 < re; b0 += kMaxGrid) {
        const int64_t cnt = std::min<int64_t>(re - b0, kMaxGrid);
        const int64_t off = b0 - rb;
        k<<<static_cast<unsigned>(cnt), S::NT, S::SMEM, s>>>(
            r.row_ptr, r.col_idx, r.values, r.col_offset, theta, f, ldt, lambda, b0,
            x ? x + off * f : nullptr, a ? a + off * f * f : nullptr, b ? b + off * f : nullptr,
            st ? st->min_row : nullptr, st ? st->column + off : nullptr, st ? st->pivot + off : nullptr, off);
        ALSK_LAUNCHED();
    }
}

// theta with a row stride that is a multiple of 4 floats and a 16-byte aligned base, as the
// bulk copies require; copies (zero padded) only when the caller's layout does not qualify.
struct StridedTheta {
    const float* ptr;
    int ldt;
    DevBuf owned;
};

void strided_theta(StridedTheta& t, const float* theta, int64_t theta_rows, int f, cudaStream_t s) {
    t.ptr = theta;
    t.ldt = f;
    const bool ok = (f % 4 == 0) && ((reinterpret_cast<uintptr_t>(theta) & 15) == 0);
    if (ok) return;
    t.ldt = (f + 3) & ~3;
    const int64_t rows = std::max<int64_t>(theta_rows, 1);
    t.owned.alloc(sizeof(float) * rows * t.ldt, s);
    ALSK_CUDA(cudaMemsetAsync(t.owned.as<void>(), 0, sizeof(float) * rows * t.ldt, s));
    if (theta_rows > 0)
        ALSK_CUDA(cudaMemcpy2DAsync(t.owned.as<float>(), sizeof(float) * t.ldt, theta, sizeof(float) * f,
                                    sizeof(float) * f, theta_rows, cudaMemcpyDeviceToDevice, s));
    t.ptr = t.owned.as<float>();
}

// ---- small ranks: one thread (short rows) or one warp (longer rows) per row ------------
// The f=10 shapes (ML-1M, SparkALS: ~5 ratings per user, ~1,500 per item) are bound by the
// gather of 4(f+2) bytes per rating from HBM; a CTA per row spends its time in launch and
// synchronisation instead. Here a thread (WARP = false) or a warp (WARP = true: lanes take
// every 32nd rating, then a fixed butterfly reduction) accumulates the lower triangle and
// B in registers (FP32), adds lambda n_u, and runs the Cholesky and both triangular solves
// in registers. Same results contract as the fused kernel (FP32 tolerance; all-zero A ->
// x = 0, solver.hpp:215-220; first non-positive pivot reported, solver.hpp:230-235).
// Cholesky of the packed lower triangle a (lambda term included) and both triangular solves
// of b, in registers; x row t written by `writer`. All-zero A -> x = 0 (solver.hpp:215-220);
// the first non-positive pivot is reported (solver.hpp:230-235).
template <int F>
__device__ __forceinline__ void small_chol_solve(float* a, float* b, bool writer, int64_t t, float* __restrict__ x,
                                                 unsigned long long* __restrict__ min_row,
                                                 int32_t* __restrict__ column, double* __restrict__ pivot,
                                                 int64_t status_base) {
    constexpr int NA = F * (F + 1) / 2;
    bool nz = false;
#pragma unroll
    for (int q = 0; q < NA; ++q) nz |= a[q] != 0.f;
    float* xr = x + t * F;
    if (!nz) {
        if (writer) {
#pragma unroll
            for (int i = 0; i < F; ++i) xr[i] = 0.f;
            column[t] = 0;
        }
        return;
    }
    // right-looking Cholesky in registers; a non-positive pivot poisons what follows, which
    // the check below discards
    float piv[F], dv[F];
#pragma unroll
    for (int c = 0; c < F; ++c) {
        const float d = a[c * (c + 1) / 2 + c];
        piv[c] = d;
        const float ic = rsqrtf(d);
        dv[c] = ic;
        a[c * (c + 1) / 2 + c] = d * ic;
#pragma unroll
        for (int q = c + 1; q < F; ++q) a[q * (q + 1) / 2 + c] *= ic;
#pragma unroll
        for (int q = c + 1; q < F; ++q)
#pragma unroll
            for (int p = c + 1; p <= q; ++p)
                a[q * (q + 1) / 2 + p] = fmaf(-a[q * (q + 1) / 2 + c], a[p * (p + 1) / 2 + c], a[q * (q + 1) / 2 + p]);
    }
    int bad = 0;
    float badv = 0.f;
#pragma unroll
    for (int c = F - 1; c >= 0; --c)
        if (!(piv[c] > 0.f)) {
            bad = c + 1;
            badv = piv[c];
        }
    if (bad) {
        if (writer) {
            column[t] = bad;
            pivot[t] = static_cast<double>(badv);
            atomicMin(min_row, static_cast<unsigned long long>(status_base + t));
#pragma unroll
            for (int i = 0; i < F; ++i) xr[i] = 0.f;
        }
        return;
    }
    // L y = b, then L^T x = y
#pragma unroll
    for (int i = 0; i < F; ++i) {
        float s = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s = fmaf(-a[i * (i + 1) / 2 + k], b[k], s);
        b[i] = s * dv[i];
    }
#pragma unroll
    for (int i = F - 1; i >= 0; --i) {
        float s = b[i];
#pragma unroll
        for (int k = i + 1; k < F; ++k) s = fmaf(-a[k * (k + 1) / 2 + i], b[k], s);
        b[i] = s * dv[i];
    }
    if (writer) {
#pragma unroll
        for (int i = 0; i < F; ++i) xr[i] = b[i];
        column[t] = 0;
    }
}


// Factor-row loads of the small-rank kernel (read-only path) with a 64-byte L2 prefetch
// size (`.L2::64B`): a 40-byte row at a 40-byte stride otherwise pulls whole 128-byte lines
// from DRAM (SparkALS Theta half: 528 -> 328 GB read per launch; time unchanged, the kernel
// is latency-bound).
#ifndef SMALL_L2_64B
#define SMALL_L2_64B 1
#endif
__device__ __forceinline__ float2 ld_row2(const float2* p) {
#if SMALL_L2_64B
    float2 v;
    asm volatile("ld.global.nc.L2::64B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

template <int F, bool WARP, bool PARTIAL>
__global__ void __launch_bounds__(128)
small_update_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                    const float* __restrict__ values, int64_t col_lo, const float* __restrict__ theta, int ldt,
                    float lambda, int64_t rb, int64_t count, float* __restrict__ x,
                    unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                    double* __restrict__ pivot, int64_t status_base) {
    const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t t = WARP ? gt >> 5 : gt;
    const int lane = WARP ? static_cast<int>(threadIdx.x & 31) : 0;
    if (t >= count) return;  // warp-uniform in the WARP variant
    const int64_t u = rb + t;
    constexpr int NA = F * (F + 1) / 2;
    constexpr int NQ = (F + 3) / 4;
    float a[NA], b[F];
#pragma unroll
    for (int q = 0; q < NA; ++q) a[q] = 0.f;
#pragma unroll
    for (int q = 0; q < F; ++q) b[q] = 0.f;
    const int64_t k0 = row_ptr[u], k1 = row_ptr[u + 1];
    // SU ratings per lane per round: every index, value and row load of the round is issued
    // before the first product, so a thread has SU gathers in flight instead of one dependent
    // col_idx -> row chain. Slots past the row end load nothing and add exact zeros, so the
    // sums keep the one-rating-at-a-time order.
    constexpr int SU = F <= 12 ? 4 : 2;
    constexpr int64_t step = WARP ? 32 : 1;
    // The next round's indices and ratings are loaded while this round's rows arrive and
    // multiply, so a round waits for one load latency instead of two.
    int nv[SU];
    float nr[SU];
#pragma unroll
    for (int j = 0; j < SU; ++j) {
        const int64_t kj = k0 + lane + j * step;
        const bool ok = kj < k1;
        nv[j] = ok ? __ldg(col_idx + kj) - static_cast<int>(col_lo) : 0;
        nr[j] = ok ? __ldg(values + kj) : 0.f;
    }
    for (int64_t k = k0 + lane; k < k1; k += SU * step) {
        int vv[SU];
        float rr[SU];
#pragma unroll
        for (int j = 0; j < SU; ++j) {
            vv[j] = nv[j];
            rr[j] = nr[j];
            const int64_t kj = k + (SU + j) * step;
            const bool ok = kj < k1;
            nv[j] = ok ? __ldg(col_idx + kj) - static_cast<int>(col_lo) : 0;
            nr[j] = ok ? __ldg(values + kj) : 0.f;
        }
        // the caller's rows in place (no padded copy): 16-, 8- or 4-byte loads by F's alignment
        float th[SU][4 * NQ];
#pragma unroll
        for (int j = 0; j < SU; ++j) {
            const bool ok = k + j * step < k1;
            const float* src = theta + static_cast<int64_t>(ok ? vv[j] : 0) * ldt;
            if constexpr (F % 4 == 0) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const float4 w = ok ? __ldg(reinterpret_cast<const float4*>(src) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
                    th[j][4 * q] = w.x, th[j][4 * q + 1] = w.y, th[j][4 * q + 2] = w.z, th[j][4 * q + 3] = w.w;
                }
            } else if constexpr (F % 2 == 0) {
#pragma unroll
                for (int q = 0; q < F / 2; ++q) {
                    float2 w = make_float2(0.f, 0.f);
                    if (ok) w = ld_row2(reinterpret_cast<const float2*>(src) + q);
                    th[j][2 * q] = w.x, th[j][2 * q + 1] = w.y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < F; ++q) th[j][q] = ok ? __ldg(src + q) : 0.f;
            }
        }
#pragma unroll
        for (int j = 0; j < SU; ++j) {
            if (k + j * step >= k1) break;  // past the row end
#pragma unroll
            for (int i = 0; i < F; ++i) {
                b[i] = fmaf(rr[j], th[j][i], b[i]);
#pragma unroll
                for (int c = 0; c <= i; ++c) a[i * (i + 1) / 2 + c] = fmaf(th[j][i], th[j][c], a[i * (i + 1) / 2 + c]);
            }
        }
    }
    if constexpr (WARP) {  // every lane ends with the same sums (fixed butterfly order)
#pragma unroll
        for (int q = 0; q < NA; ++q)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
#pragma unroll
        for (int q = 0; q < F; ++q)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) b[q] += __shfl_xor_sync(0xffffffffu, b[q], o);
    }
    const bool writer = lane == 0;
    const float reg = lambda * static_cast<float>(k1 - k0);  // float arithmetic as solver.hpp:141,152
#pragma unroll
    for (int i = 0; i < F; ++i) a[i * (i + 1) / 2 + i] += reg;
    if constexpr (PARTIAL) {
        // data-parallel partial (parallel.hpp:408-411): packed [lower(A) row-major | b],
        // lambda n_u^local on the diagonal, reduced across ranks before the solve
        if (writer) {
            float* o = x + t * (NA + F);
#pragma unroll
            for (int q = 0; q < NA; ++q) o[q] = a[q];
#pragma unroll
            for (int q = 0; q < F; ++q) o[NA + q] = b[q];
        }
    } else {
        small_chol_solve<F>(a, b, writer, t, x, min_row, column, pivot, status_base);
    }
}

// Solve of reduced small-rank packed rows ([lower(A) | b], NA + F floats): a thread per row.
template <int F>
__global__ void __launch_bounds__(128)
small_solve_packed_kernel(const float* __restrict__ packed, int64_t count, float* __restrict__ x,
                          unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                          double* __restrict__ pivot) {
    constexpr int NA = F * (F + 1) / 2;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count) return;
    float a[NA], b[F];
    const float* p = packed + t * (NA + F);
#pragma unroll
    for (int q = 0; q < NA; ++q) a[q] = p[q];
#pragma unroll
    for (int q = 0; q < F; ++q) b[q] = p[NA + q];
    small_chol_solve<F>(a, b, true, t, x, min_row, column, pivot, 0);
}

template <bool WARP, bool PARTIAL = false>
bool launch_small(const DevCsr& r, const float* theta, int f, int ldt, float lambda, int64_t rb, int64_t re,
                  float* x, const SolveStatus& st, cudaStream_t s) {
    const int64_t count = re - rb;
    const int64_t threads = WARP ? count * 32 : count;
    const unsigned grid = static_cast<unsigned>((threads + 127) / 128);
#define ALSK_SMALL_CASE(FV)                                                                                  \
    case FV:                                                                                                 \
        small_update_kernel<FV, WARP, PARTIAL><<<grid, 128, 0, s>>>(r.row_ptr, r.col_idx, r.values, r.col_offset, \
                                                                    theta, ldt, lambda, rb, count, x, st.min_row, \
                                                                    st.column, st.pivot, 0);                      \
        ALSK_LAUNCHED();                                                                                     \
        return true;
    switch (f) {
        ALSK_SMALL_CASE(1)
        ALSK_SMALL_CASE(2)
        ALSK_SMALL_CASE(3)
        ALSK_SMALL_CASE(4)
        ALSK_SMALL_CASE(5)
        ALSK_SMALL_CASE(6)
        ALSK_SMALL_CASE(7)
        ALSK_SMALL_CASE(8)
        ALSK_SMALL_CASE(9)
        ALSK_SMALL_CASE(10)
        ALSK_SMALL_CASE(11)
        ALSK_SMALL_CASE(12)
        ALSK_SMALL_CASE(13)
        ALSK_SMALL_CASE(14)
        ALSK_SMALL_CASE(15)
        default:
            return false;
    }
#undef ALSK_SMALL_CASE
}

template <bool SOLVE>
bool dispatch(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
              int64_t re, float* x, float* a, float* b, const SolveStatus* st, cudaStream_t s) {
    const int ldt = (f + 3) & ~3;
    const int need = (ldt + 1 + 7) / 8;
    if (need > 16) return false;
    if (re <= rb) return true;
    StridedTheta th;
    strided_theta(th, theta, theta_rows, f, s);
#define ALSK_FUSED_CASE(NBV)                                                                     \
    if (need <= NBV) {                                                                          \
        launch_fused<NBV, SOLVE>(r, th.ptr, f, th.ldt, lambda, rb, re, x, a, b, st, s);         \
        return true;                                                                            \
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

bool update_fused_fp32(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
                       int64_t re, float* x_out, const SolveStatus& st, cudaStream_t s) {
    // small ranks: a thread per row when rows average under 32 ratings, else a warp per row
    static const bool no_small = measure_env("ALSK_NO_SMALL_F") != nullptr;  // A/B switch
    if (!no_small && f <= 15 && r.rows > 0) {
        if (re <= rb) return true;
        // rows read in place at stride f (a factor is never copied: at SparkALS scale X is
        // 26 GB); only an under-aligned base pointer forces the padded copy
        const uintptr_t need = f % 4 == 0 ? 15 : (f % 2 == 0 ? 7 : 3);
        const float* tp = theta;
        int ldt = f;
        StridedTheta th;
        if (reinterpret_cast<uintptr_t>(theta) & need) {
            strided_theta(th, theta, theta_rows, f, s);
            tp = th.ptr;
            ldt = th.ldt;
        }
        const bool ok = r.nnz < 32 * r.rows ? launch_small<false>(r, tp, f, ldt, lambda, rb, re, x_out, st, s)
                                            : launch_small<true>(r, tp, f, ldt, lambda, rb, re, x_out, st, s);
        if (ok) return true;
    }
    return dispatch<true>(r, theta, theta_rows, f, lambda, rb, re, x_out, nullptr, nullptr, &st, s);
}

// Data-parallel partial Hermitians for small ranks (f <= 15): packed [lower(A) | b] rows of
// f(f+1)/2 + f floats with lambda n_u^local on the diagonal (parallel.hpp:408-411).
bool partial_small_fp32(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
                        int64_t re, float* out, cudaStream_t s) {
    if (f < 1 || f > 15) return false;
    if (re <= rb) return true;
    const uintptr_t need = f % 4 == 0 ? 15 : (f % 2 == 0 ? 7 : 3);
    const float* tp = theta;
    int ldt = f;
    StridedTheta th;
    if (reinterpret_cast<uintptr_t>(theta) & need) {
        strided_theta(th, theta, theta_rows, f, s);
        tp = th.ptr;
        ldt = th.ldt;
    }
    SolveStatus none{};
    return r.nnz < 32 * r.rows ? launch_small<false, true>(r, tp, f, ldt, lambda, rb, re, out, none, s)
                               : launch_small<true, true>(r, tp, f, ldt, lambda, rb, re, out, none, s);
}

bool solve_small_packed(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, cudaStream_t s) {
    if (count <= 0) return true;
    const unsigned grid = static_cast<unsigned>((count + 127) / 128);
#define ALSK_SMALL_SOLVE(FV)                                                                               \
    case FV:                                                                                               \
        small_solve_packed_kernel<FV><<<grid, 128, 0, s>>>(packed, count, x, st.min_row, st.column, st.pivot); \
        ALSK_LAUNCHED();                                                                                   \
        return true;
    switch (f) {
        ALSK_SMALL_SOLVE(1)
        ALSK_SMALL_SOLVE(2)
        ALSK_SMALL_SOLVE(3)
        ALSK_SMALL_SOLVE(4)
        ALSK_SMALL_SOLVE(5)
        ALSK_SMALL_SOLVE(6)
        ALSK_SMALL_SOLVE(7)
        ALSK_SMALL_SOLVE(8)
        ALSK_SMALL_SOLVE(9)
        ALSK_SMALL_SOLVE(10)
        ALSK_SMALL_SOLVE(11)
        ALSK_SMALL_SOLVE(12)
        ALSK_SMALL_SOLVE(13)
        ALSK_SMALL_SOLVE(14)
        ALSK_SMALL_SOLVE(15)
        default:
            return false;
    }
#undef ALSK_SMALL_SOLVE
}

bool hermitian_fused_fp32(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
                          int64_t re, float* A, float* B, cudaStream_t s) {
    return dispatch<false>(r, theta, theta_rows, f, lambda, rb, re, nullptr, A, B, nullptr, s);
}

}  // namespace alsk
