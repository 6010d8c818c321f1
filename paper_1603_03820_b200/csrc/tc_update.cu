// Tensor-core half-sweep (ALSK_PREC_TF32X2): get_hermitian + get_bias on tcgen05 (kind::tf32,
// two-term split), Cholesky + both triangular solves on the CUDA cores, one persistent CTA
// per SM, nothing per-row materialised in HBM.
//
// Replaces, for this precision, the loop body of update_x (solver.hpp:336-344):
// assemble_mo_rows (solver.hpp:99-157) followed by batch_solve_into (solver.hpp:204-262).
//
// Arithmetic. The gathered rows are augmented with the rating, theta'_k = [theta_k, r_k]
// (f+1 features), and every entry is split x = h + l, h = rna_tf32(x), l = rna_tf32(x - h).
// One MMA per 8-rating k-step, D += H^T [H | 2L] (M = 128, N = 2*NF, NF = round16(f+1)), so
// with D = [D0 | D1]:   sym(D0 + D1) = H^T H + H^T L + L^T H = sum_k theta'_k theta'_k^T
// up to the dropped L^T L term (2^-22 relative). Rows < f of that symmetric matrix are A_u
// (solver.hpp:130-140), row f is B_u (the bias rides along, solver.hpp:137).
// The tensor core's FP32 accumulation truncates, which biases long sums; rows longer than
// SEG_CHUNKS x 32 ratings are therefore accumulated in segments, each drained from TMEM and
// added into shared memory with round-to-nearest FP32 adds.
//
// Warp roles (448 threads, 1 CTA per SM, rows j = blockIdx.x + t*gridDim.x):
//   warps 0-7  : two epilogue groups of 4 warps (group g takes rows with t%2 == g). TMEM ->
//                registers -> shared memory (segment sums, symmetrisation, lambda n_u) ->
//                8x8 tiles in registers -> blocked right-looking Cholesky -> back
//                substitution -> x_u.
//   warps 8-11 : split warps: read the TMA-landed rating-major rows, split tf32 hi/lo and
//                write them transposed into the K-major operand tile (lane = rating), with
//                zero padding of partial k-groups.
//   warp 12    : MMA issuer (one thread), owns the TMEM allocation (2 buffers x 256 columns).
//   warp 13    : TMA issuer: cp.async.bulk.tensor tile::gather4, 4 factor rows x 32
//                features per instruction, into a 128B-swizzled rating-major staging ring.
// Pipelines: staging ring (raw_full / raw_empty, 4 deep), operand ring (hl_full / hl_empty,
// 2 deep, released by tcgen05.commit) and the TMEM double buffer (tfull / tempty), one TMEM
// job per row segment.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace alsk {
namespace {
using namespace tc;

constexpr int KC = 32;                   // ratings per stage (four k-groups of 8)
constexpr int MNB = 4;                   // feature blocks of 32 (M = 128 rows)
constexpr int RAW_BYTES = KC * MNB * 128;   // 16 KB: one staged chunk, rating-major
constexpr int HL_BYTES = 256 * KC * 4;      // 32 KB: H rows [0,NF) then 2L rows [NF,2NF), K-major
constexpr int HL_STAGES = 2;
constexpr int SEG_CHUNKS = 16;              // TMEM accumulation segment: 16 x 32 ratings
constexpr int NTHREADS = 448;
constexpr int TMEM_COLS = 512;           // two buffers x 256 columns (D0 @ +0, D1 @ +NF)

// ---- shared-memory plan (host and device agree) ----
struct TcPlan {
    int f, sld, stages, nb;
    int s_floats, grp_floats;
    size_t ring_bytes, grp_bytes, bar_off, total;
    __host__ __device__ TcPlan(int f_, int nb_, int stages_) : f(f_), stages(stages_), nb(nb_) {
        sld = (f + 1) | 1;  // >= f+1 columns (A and B); odd: row writes and column reads conflict-free
        s_floats = ((f + 1) * sld + 3) & ~3;  // keep the float4 panel 16-byte aligned
        const int fp = 8 * nb;
        grp_floats = (s_floats + 8 * fp + 64 + fp + 8 + 3) & ~3;
        ring_bytes = static_cast<size_t>(stages) * RAW_BYTES + static_cast<size_t>(HL_STAGES) * HL_BYTES;
        grp_bytes = static_cast<size_t>(grp_floats) * 4;
        bar_off = (ring_bytes + 2 * grp_bytes + 15) & ~static_cast<size_t>(15);
        total = bar_off + static_cast<size_t>(2 * stages + 2 * HL_STAGES + 6) * 8 + 16 + 1024;  // + align slack
    }
};

__device__ __forceinline__ void tile_coords_colmajor(int t, int nb, int& bi, int& bj) {
    int c = 0;
    while (t >= nb - c) {
        t -= nb - c;
        ++c;
    }
    bj = c;
    bi = c + t;
}

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

__device__ __forceinline__ void tma_gather4(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int col, int r0,
                                            int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ int chunk_count(int64_t n, int64_t c0) {
    const int64_t left = n - c0;
    return left < KC ? static_cast<int>(left) : KC;
}

struct RowIter {  // the CTA's row sequence j = blockIdx.x + t * gridDim.x
    int64_t j, nrows;
    __device__ RowIter(int64_t nrows_) : j(blockIdx.x), nrows(nrows_) {}
    __device__ bool more() const { return j < nrows; }
    __device__ void next() { j += gridDim.x; }
};

// One epilogue group's Cholesky of the augmented tile set (rows < f: A lower; row f: B) and
// the back substitution; x written to xrow. Mirrors fused_fp32.cu's blocked algorithm with
// group-scoped named barriers. Returns the breakdown column+1 (0 = ok).
template <int NB>
__device__ __forceinline__ void group_solve(float (&acc)[8][8], bool active, int bi, int bj, int e, int f,
                                            float* lpk, float* panel, float* dblk, float* dinv, int* flags,
                                            uint32_t bar_id, float* __restrict__ xrow, int32_t* col_out,
                                            double* piv_out, unsigned long long* min_row, int64_t status_row) {
    constexpr int FP = 8 * NB;
    const int ia = 8 * bi, jb = 8 * bj;
    const int aug = f;
    // all-zero A => x = 0 (solver.hpp:215-220)
    int nz = 0;
    if (active) {
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
                if (ia + ii < f && jb + jj <= ia + ii) nz |= (acc[ii][jj] != 0.f);
    }
    if (e == 0) flags[2] = 0;
    named_barrier(bar_id, 128);
    if (nz) flags[2] = 1;
    named_barrier(bar_id, 128);
    if (!flags[2]) {
        for (int i = e; i < f; i += 128) xrow[i] = 0.f;
        if (e == 0) *col_out = 0;
        named_barrier(bar_id, 128);
        return;
    }
    const int nbc = (f + 7) >> 3;
    for (int bc = 0; bc < nbc; ++bc) {
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
        named_barrier(bar_id, 128);
        if (flags[0]) {
            if (e == 0) {
                *col_out = flags[0];
                *piv_out = static_cast<double>(__int_as_float(flags[1]));
                atomicMin(min_row, static_cast<unsigned long long>(status_row));
            }
            for (int i = e; i < f; i += 128) xrow[i] = 0.f;
            named_barrier(bar_id, 128);
            if (e == 0) flags[0] = 0;
            named_barrier(bar_id, 128);
            return;
        }
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
                float4* dst = reinterpret_cast<float4*>(panel + c * FP + ia);
                dst[0] = make_float4(acc[0][c], acc[1][c], acc[2][c], acc[3][c]);
                dst[1] = make_float4(acc[4][c], acc[5][c], acc[6][c], acc[7][c]);
            }
        }
        named_barrier(bar_id, 128);
        if (active && bj > bc) outer_accumulate<FP, true>(acc, panel, 8, ia, jb);
    }
    if (e == 0) *col_out = 0;
    // packed L (rows < f) and y (row aug) for the back substitution
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
    named_barrier(bar_id, 128);
    if (e < 32) {
        const int lane = e;
        constexpr int G = (FP + 31) / 32;
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
            if (j < f) xrow[j] = yv[g];
        }
    }
    named_barrier(bar_id, 128);  // lpk / dinv reused by the group's next row
}

__device__ __forceinline__ int64_t row_segments(int64_t n) {
    const int64_t nch = (n + KC - 1) / KC;
    return (nch + SEG_CHUNKS - 1) / SEG_CHUNKS;
}

template <int NB, bool SOLVE>
__global__ void __launch_bounds__(NTHREADS, 1)
tc_update_kernel(const __grid_constant__ CUtensorMap tmap, const int64_t* __restrict__ row_ptr,
                 const int32_t* __restrict__ col_idx, const float* __restrict__ values, int64_t col_lo, int f,
                 float lambda, int64_t rb, int64_t nrows, int stages, float* __restrict__ out_x,
                 float* __restrict__ out_a, float* __restrict__ out_b, unsigned long long* __restrict__ min_row,
                 int32_t* __restrict__ column, double* __restrict__ pivot, int64_t status_base) {
    constexpr int FP = 8 * NB;
    constexpr int NTILES = NB * (NB + 1) / 2;
    static_assert(NTILES <= 128, "tile set must fit one 128-thread epilogue group");
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    const TcPlan P(f, NB, stages);
    // augmented features per operand half; a multiple of 16 keeps every 16-column TMEM load of
    // the second half aligned
    const int NF = (f + 1 + 15) & ~15;
    uint8_t* ring = base;                                          // stages x RAW_BYTES
    uint8_t* hl = base + static_cast<size_t>(stages) * RAW_BYTES;  // HL_STAGES x HL_BYTES
    float* grp0 = reinterpret_cast<float*>(base + P.ring_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + P.bar_off);
    uint64_t* raw_full = bars;
    uint64_t* raw_empty = bars + stages;
    uint64_t* hl_full = bars + 2 * stages;
    uint64_t* hl_empty = hl_full + HL_STAGES;
    // tfull[2*g + b]: a job for group g finished in TMEM buffer b. One barrier per (owner,
    // buffer) pair: jobs on a buffer drain in order, so each owner's barrier is at most one
    // phase ahead of it and parity waits cannot alias.
    uint64_t* tfull = hl_empty + HL_STAGES;
    uint64_t* tempty = tfull + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&raw_full[s], 1);
            mbar_init(&raw_empty[s], 4);
        }
        for (int s = 0; s < HL_STAGES; ++s) {
            mbar_init(&hl_full[s], 4);
            mbar_init(&hl_empty[s], 1);
        }
        for (int b = 0; b < 4; ++b) mbar_init(&tfull[b], 1);
        for (int b = 0; b < 2; ++b) mbar_init(&tempty[b], 4);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < static_cast<int>(P.ring_bytes / 16); i += NTHREADS)
        reinterpret_cast<float4*>(ring)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (warp == 12) tmem_alloc<TMEM_COLS>(tmem_slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 13) {
        // ---------------- TMA issuer ----------------
        const int nblk = (f + 31) >> 5;  // feature blocks of 32 holding real features
        uint32_t ctr = 0;
        for (RowIter it(nrows); it.more(); it.next()) {
            const int64_t u = rb + it.j;
            const int64_t k0 = row_ptr[u], n = row_ptr[u + 1] - k0;
            for (int64_t c0 = 0; c0 < n; c0 += KC, ++ctr) {
                const int s = ctr % stages;
                const uint32_t ph = (ctr / stages) & 1u;
                const int cnt = chunk_count(n, c0);
                int v = 0;
                if (lane < cnt) v = col_idx[k0 + c0 + lane] - static_cast<int>(col_lo);
                const int v_first = __shfl_sync(0xffffffffu, v, lane & ~3);
                if (lane >= cnt) v = v_first;  // pad a partial quad with a valid row
                const int q0 = __shfl_sync(0xffffffffu, v, (lane & 7) * 4 + 0);
                const int q1 = __shfl_sync(0xffffffffu, v, (lane & 7) * 4 + 1);
                const int q2 = __shfl_sync(0xffffffffu, v, (lane & 7) * 4 + 2);
                const int q3 = __shfl_sync(0xffffffffu, v, (lane & 7) * 4 + 3);
                const int nquads = (cnt + 3) >> 2;
                if (lane == 0) {
                    mbar_wait(&raw_empty[s], ph ^ 1u);
                    mbar_expect_tx(&raw_full[s], static_cast<uint32_t>(nquads * nblk * 512));
                }
                __syncwarp();
                if (lane < nquads) {
                    const uint32_t dst = smem_u32(ring + s * RAW_BYTES) + (lane >> 1) * (MNB * 1024) + (lane & 1) * 512;
                    for (int b = 0; b < nblk; ++b) tma_gather4(&tmap, dst + b * 1024, &raw_full[s], b * 32, q0, q1, q2, q3);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 8 && warp < 12) {
        // ---------------- split warps ----------------
        // lane = rating slot k of the chunk; warp pw handles feature chunks c16 = pw + 4t.
        // Every offset below is a per-thread constant plus a multiple of t.
        const int pw = warp - 8;
        const int k = lane;
        const uint32_t raw_k = static_cast<uint32_t>((k >> 3) * (MNB * 1024) + (k & 7) * 128);
        const uint32_t raw_sw0 = static_cast<uint32_t>(((pw ^ (k & 7))) << 4);
        const uint32_t raw_sw1 = static_cast<uint32_t>((((pw + 4) ^ (k & 7))) << 4);
        uint32_t kq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r8 = 4 * (pw & 1) + q;  // feature & 7
            kq[q] = static_cast<uint32_t>((pw >> 1) * 1024 + r8 * 128 + ((((k >> 2) ^ r8)) << 4) + (k & 3) * 4);
        }
        const uint32_t l_off = static_cast<uint32_t>(NF * 128);
        uint32_t ctr = 0;
        for (RowIter it(nrows); it.more(); it.next()) {
            const int64_t u = rb + it.j;
            const int64_t k0 = row_ptr[u], n = row_ptr[u + 1] - k0;
            for (int64_t c0 = 0; c0 < n; c0 += KC, ++ctr) {
                const int s = ctr % stages;
                const int hs = ctr % HL_STAGES;
                const int cnt = chunk_count(n, c0);
                const bool valid = k < cnt;
                const float r = valid ? values[k0 + c0 + k] : 0.f;
                const float r_hi = tf32_rna(r), r_lo2 = 2.f * tf32_rna(r - r_hi);
                mbar_wait(&raw_full[s], (ctr / stages) & 1u);
                mbar_wait(&hl_empty[hs], ((ctr / HL_STAGES) & 1u) ^ 1u);
                const uint8_t* raw = ring + s * RAW_BYTES + raw_k;
                uint8_t* H = hl + hs * HL_BYTES;
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int c16 = pw + 4 * t;
                    if (4 * c16 > f) break;  // uniform per warp
                    const float4 x = *reinterpret_cast<const float4*>(raw + (t >> 1) * 1024 + ((t & 1) ? raw_sw1 : raw_sw0));
                    const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int feat = 4 * c16 + q;
                        float h, l2;
                        if (feat < f) {
                            h = tf32_rna(xv[q]);
                            l2 = 2.f * tf32_rna(xv[q] - h);
                        } else {
                            h = feat == f ? r_hi : 0.f;
                            l2 = feat == f ? r_lo2 : 0.f;
                        }
                        uint8_t* dst = H + kq[q] + t * 2048;
                        *reinterpret_cast<float*>(dst) = valid ? h : 0.f;
                        *reinterpret_cast<float*>(dst + l_off) = valid ? l2 : 0.f;
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&raw_empty[s]);
                    mbar_arrive(&hl_full[hs]);
                }
            }
        }
    } else if (warp == 12) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc = idesc_tf32(128, 2 * NF);
        uint32_t ctr = 0, job = 0;
        int t = 0;
        for (RowIter it(nrows); it.more(); it.next(), ++t) {
            const int64_t u = rb + it.j;
            const int64_t n = row_ptr[u + 1] - row_ptr[u];
            const int owner = t & 1;
            int64_t c0 = 0;
            while (c0 < n) {  // one TMEM job per segment of SEG_CHUNKS chunks
                const uint32_t b = job & 1u;
                const uint32_t dcol = tmem + b * 256u;
                if (lane == 0) mbar_wait(&tempty[b], ((job >> 1) & 1u) ^ 1u);
                __syncwarp();
                tc_fence_after();
                for (int sc = 0; sc < SEG_CHUNKS && c0 < n; ++sc, c0 += KC, ++ctr) {
                    const int hs = ctr % HL_STAGES;
                    const int cnt = chunk_count(n, c0);
                    if (lane == 0) {
                        mbar_wait(&hl_full[hs], (ctr / HL_STAGES) & 1u);
                        tc_fence_after();
                        const uint32_t hb = smem_u32(hl + hs * HL_BYTES);
                        const int ksteps = (cnt + 7) >> 3;
                        for (int kb = 0; kb < ksteps; ++kb) {
                            const uint64_t d = sdesc_sw128(hb + kb * 32, 16, 1024);
                            mma_tf32(dcol, d, d, idesc, (sc > 0 || kb > 0) ? 1u : 0u);
                        }
                        mma_commit(&hl_empty[hs]);
                    }
                    __syncwarp();
                }
                if (lane == 0) mma_commit(&tfull[2 * owner + b]);
                __syncwarp();
                ++job;
            }
        }
    } else {
        // ---------------- epilogue groups ----------------
        const int g = warp >> 2;
        const int e = threadIdx.x & 127;  // TMEM lane = matrix row owned in the readback
        const uint32_t bar_id = 1 + g;
        float* S = grp0 + g * P.grp_floats;
        float* panel = S + P.s_floats;
        float* dblk = panel + 8 * FP;
        float* dinv = dblk + 64;
        int* flags = reinterpret_cast<int*>(dinv + FP);
        const int sld = P.sld;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int nch16 = (f + 1 + 15) >> 4;  // 16-column TMEM chunks covering features 0..f
        const bool active = e < NTILES;
        int bi = 0, bj = 0;
        if (active) tile_coords_colmajor(e, NB, bi, bj);
        const int ia = 8 * bi, jb = 8 * bj;
        if (e == 0) flags[0] = flags[1] = flags[2] = 0;
        float* Srow = S + e * sld;
        uint32_t job = 0, use[2] = {0u, 0u};
        int t = 0;
        for (RowIter it(nrows); it.more(); it.next(), ++t) {
            const int64_t u = rb + it.j;
            const int64_t n = row_ptr[u + 1] - row_ptr[u];
            const uint32_t nseg = static_cast<uint32_t>(row_segments(n));
            if ((t & 1) != g) {
                job += nseg;
                continue;
            }
            const int64_t row = it.j;
            float acc[8][8];
#pragma unroll
            for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) acc[ii][jj] = 0.f;
            if (n > 0) {
                for (uint32_t sg = 0; sg < nseg; ++sg, ++job) {
                    const uint32_t b = job & 1u;
                    const uint32_t dcol = tmem + b * 256u + lane_base;
                    mbar_wait(&tfull[2 * g + b], use[b] & 1u);
                    ++use[b];
                    tc_fence_after();
                    for (int c = 0; c < nch16; ++c) {
                        float d0[16], d1[16];
                        tmem_ld16(dcol + c * 16, d0);
                        tmem_ld16(dcol + NF + c * 16, d1);
                        tmem_ld_wait();
                        if (e <= f) {
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) {
                                const int j = c * 16 + jj;
                                if (j <= f) Srow[j] = (sg ? Srow[j] : 0.f) + (d0[jj] + d1[jj]);
                            }
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if ((e & 31) == 0) mbar_arrive(&tempty[b]);
                }
                named_barrier(bar_id, 128);
                // symmetrise in place: lower A (+ lambda n_u on the diagonal, float arithmetic as
                // solver.hpp:141,152) and B in row f
                if (e < f) {
                    for (int j = 0; j < e; ++j) Srow[j] = 0.5f * (Srow[j] + S[j * sld + e]);
                    Srow[e] += lambda * static_cast<float>(n);
                } else if (e == f) {
                    for (int j = 0; j < f; ++j) Srow[j] = 0.5f * (Srow[j] + S[j * sld + f]);
                }
                named_barrier(bar_id, 128);
                if constexpr (!SOLVE) {
                    float* a_out = out_a + row * static_cast<int64_t>(f) * f;
                    float* b_out = out_b + row * static_cast<int64_t>(f);
                    for (int idx = e; idx < f * f; idx += 128) {
                        const int i = idx / f, j = idx - i * f;
                        a_out[idx] = j <= i ? S[i * sld + j] : S[j * sld + i];
                    }
                    for (int j = e; j < f; j += 128) b_out[j] = S[f * sld + j];
                    named_barrier(bar_id, 128);
                    continue;
                }
#pragma unroll
                for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const int i = ia + ii, j = jb + jj;
                        if (active && j < f && (j <= i || i == f) && i <= f) acc[ii][jj] = S[i * sld + j];
                    }
                named_barrier(bar_id, 128);  // S becomes the packed-L scratch
            }
            if constexpr (!SOLVE) {
                float* a_out = out_a + row * static_cast<int64_t>(f) * f;
                for (int idx = e; idx < f * f; idx += 128) a_out[idx] = 0.f;
                for (int j = e; j < f; j += 128) out_b[row * static_cast<int64_t>(f) + j] = 0.f;
            } else {
                group_solve<NB>(acc, active, bi, bj, e, f, S, panel, dblk, dinv, flags, bar_id,
                                out_x + row * static_cast<int64_t>(f), column + row, pivot + row, min_row,
                                status_base + row);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 12) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// ---- host side ----
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw Failure(ALSK_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
    return fn;
}

// 2-D map over the factor rows: dim0 = ldt features (contiguous), dim1 = rows; box 32 x 1
// (gather4 fetches 4 rows of the box), 128-byte swizzle, out-of-bounds reads as zero.
CUtensorMap factor_map(const float* theta, int64_t rows, int ldt) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ldt), static_cast<cuuint64_t>(std::max<int64_t>(rows, 1))};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldt) * 4};
    const cuuint32_t box[2] = {32, 1};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(theta), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Failure(ALSK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

template <int NB, bool SOLVE>
void launch_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, int ldt, float lambda, int64_t rb,
               int64_t re, float* x, float* a, float* b, const SolveStatus* st, cudaStream_t s) {
    int stages = 4;
    while (stages > 2 && TcPlan(f, NB, stages).total > 227 * 1024) --stages;
    const TcPlan P(f, NB, stages);
    auto k = tc_update_kernel<NB, SOLVE>;
    ALSK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P.total)));
    const CUtensorMap map = factor_map(theta, theta_rows, ldt);
    const int64_t nrows = re - rb;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(nrows, num_sms()));
    k<<<grid, NTHREADS, P.total, s>>>(map, r.row_ptr, r.col_idx, r.values, r.col_offset, f, lambda, rb, nrows, stages,
                                       x, a, b, st ? st->min_row : nullptr, st ? st->column : nullptr,
                                       st ? st->pivot : nullptr, 0);
    ALSK_LAUNCHED();
}

struct Strided {
    const float* ptr;
    int ldt;
    DevBuf owned;
};
void strided(Strided& t, const float* theta, int64_t rows, int f, cudaStream_t s) {
    t.ptr = theta;
    t.ldt = f;
    if (f % 4 == 0 && (reinterpret_cast<uintptr_t>(theta) & 15) == 0) return;
    t.ldt = (f + 3) & ~3;
    const int64_t nr = std::max<int64_t>(rows, 1);
    t.owned.alloc(sizeof(float) * nr * t.ldt, s);
    ALSK_CUDA(cudaMemsetAsync(t.owned.as<void>(), 0, sizeof(float) * nr * t.ldt, s));
    if (rows > 0)
        ALSK_CUDA(cudaMemcpy2DAsync(t.owned.as<float>(), sizeof(float) * t.ldt, theta, sizeof(float) * f,
                                    sizeof(float) * f, rows, cudaMemcpyDeviceToDevice, s));
    t.ptr = t.owned.as<float>();
}

template <bool SOLVE>
bool dispatch_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb, int64_t re,
                 float* x, float* a, float* b, const SolveStatus* st, cudaStream_t s) {
    if (!tc_supported(f)) return false;
    if (re <= rb) return true;
    Strided th;
    strided(th, theta, theta_rows, f, s);
    const int nb = (f + 1 + 7) / 8;
#define ALSK_TC_CASE(NBV)                                                                          \
    if (nb <= NBV) {                                                                               \
        launch_tc<NBV, SOLVE>(r, th.ptr, theta_rows, f, th.ldt, lambda, rb, re, x, a, b, st, s);  \
        return true;                                                                               \
    }
    ALSK_TC_CASE(5)
    ALSK_TC_CASE(7)
    ALSK_TC_CASE(10)
    ALSK_TC_CASE(13)
    ALSK_TC_CASE(15)
#undef ALSK_TC_CASE
    return false;
}

}  // namespace

bool tc_supported(int f) { return f >= 16 && f <= 119; }  // 2*round16(f+1) <= 256, tiles <= 128

bool update_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb, int64_t re,
               float* x_out, const SolveStatus& st, cudaStream_t s) {
    return dispatch_tc<true>(r, theta, theta_rows, f, lambda, rb, re, x_out, nullptr, nullptr, &st, s);
}

bool hermitian_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb, int64_t re,
                  float* A, float* B, cudaStream_t s) {
    return dispatch_tc<false>(r, theta, theta_rows, f, lambda, rb, re, nullptr, A, B, nullptr, s);
}

}  // namespace alsk
