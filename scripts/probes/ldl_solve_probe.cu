// PROBE RECORD (not built into the library): a register-resident LDL^T batched solve, two
// mirrored systems per CTA. Fully unrolled it needs ~11K FFMA + ~110K other SASS
// instructions for f = 100 (2 MB of code per CTA pass, 12 minutes of ptxas, 400 B of
// spills at 128 registers): the instruction stream alone would exceed the work, so the
// design was dropped before measuring (batched solve).
// Batched FP32 SPD solve of packed Hermitian rows on the CUDA cores, with each matrix held
// in registers: the solve of the tensor-core half-sweep (batch_solve_into, solver.hpp:204-262,
// at FP32 tolerance).
//
// Why registers: a 100x100 Cholesky is 13 dependent 8-column steps on the TMEM path
// (tc_solve.cu) and TMEM fits only 4 systems per SM, so that kernel is latency-bound. Here a
// CTA of R threads (R = f rounded up + the augmented row) factors TWO systems at once and
// 4 CTAs share an SM, so 8 systems are in flight and the FMA pipes stay busy.
//
// Layout: thread t owns row t of system A and row R-1-t of system B ("mirrored" rows), so
// every thread holds exactly R + 1 values (t + 1 of A's lower triangle, R - t of B's), the
// element (row, col j) sitting at the compile-time register slot j (A) or R - j (B). The
// last row of each system is the augmented row b^T; rows between f and R-2 are identity
// padding (they do not couple to the real rows).
//
// Right-looking LDL^T, one column per step: the rows at or below the pivot publish their
// column-c entry to shared memory (double-buffered, so one CTA barrier per step), every row
// forms s = a[c] / d_c and updates its entries a[j] -= s * col[j] for c < j <= row, and
// keeps s as L's multiplier. On the augmented row this is the forward substitution: its
// multipliers end up as z = D^-1 L^-1 b. The factors are then dumped to shared memory and
// one warp per system solves L^T x = z column by column. Numerics: FP32 FMA throughout (no
// tensor-core split), the same contract as the other FP32 solves: all-zero A gives x = 0
// (solver.hpp:215-220); the first non-positive pivot d_c (the Cholesky pivot squared) is
// reported as column c with that row's x zeroed (solver.hpp:230-235).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <utility>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace alsk {
namespace {
using namespace tc;

template <int R>
struct LdlPlan {
    static constexpr int NT = (R + 31) / 32 * 32;  // threads per CTA
    static constexpr int NW = NT / 32;
    static constexpr int Q = (R - 1 + 31) / 32;    // back-substitution values per lane
    static constexpr int TRI = (R - 1) * R / 2;     // lower triangle of the R-1 matrix rows (incl. diagonal)
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// element (i, j <= i) of a system in my row numbering, read from its packed row in shared
// memory (panel-blocked, kernels.cuh pb_index; packed row f is b)
template <int R>
__device__ __forceinline__ float sys_elem(const float* pk, int f, int i, int j) {
    if (i == R - 1) return j < f ? pk[pb_index(f, f, j)] : 0.f;
    if (i >= f) return i == j ? 1.f : 0.f;  // identity padding
    return pk[pb_index(f, i, j)];
}

// Compile-time loops: every register slot index below is a constant, so the rows stay in
// registers (a loop the compiler declines to unroll would move them to local memory).
template <class F, int... Is>
__device__ __forceinline__ void static_for_impl(F&& fn, std::integer_sequence<int, Is...>) {
    (fn(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& fn) {
    static_for_impl(fn, std::make_integer_sequence<int, N>{});
}

template <int R>
__global__ void __launch_bounds__(LdlPlan<R>::NT, 4)
ldl_solve_kernel(const float* __restrict__ packed, int64_t count, int f, int64_t pks, int64_t stride,
                 float* __restrict__ out_x,
                 unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                 double* __restrict__ pivot, int64_t status_base) {
    using P = LdlPlan<R>;
    extern __shared__ __align__(16) float sm[];
    // stride: floats per staged system (>= the packed row and the factor dump, multiple of 4)
    float* stage = sm;                                // [2][stride]: packed rows, then L / D / z
    float* col = sm + 2 * stride;                     // [2 systems][2 parities][NT]
    __shared__ uint64_t bar;
    __shared__ int bad[2];
    __shared__ float badv[2];

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const int rB = R - 1 - t;                   // my row of system B
    const int tmaxA = min(32 * warp + 31, R - 1);  // highest A row in my warp
    const int rmaxB = R - 1 - 32 * warp;           // highest B row in my warp
    const bool live = t < R;
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int64_t npairs = (count + 1) / 2;
    uint32_t phase = 0;
    for (int64_t pair = blockIdx.x; pair < npairs; pair += gridDim.x, phase ^= 1u) {
        const int64_t gA = 2 * pair, gB = gA + 1;
        const bool hasB = gB < count;
        if (t == 0) {
            const uint32_t bytes = static_cast<uint32_t>(pks * 4);
            expect_tx(&bar, bytes * (hasB ? 2u : 1u));
            bulk_g2s(smem_u32(stage), packed + gA * pks, bytes, &bar);
            if (hasB) bulk_g2s(smem_u32(stage + stride), packed + gB * pks, bytes, &bar);
            bad[0] = bad[1] = 0;
        }
        mbar_wait(&bar, phase);
        // my two rows into registers: slot k <= t is A[t][k], slot k > t is B[rB][R - k]
        float a[R + 1];
        bool nzA = false, nzB = false;
        static_for<R + 1>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            float v = 0.f;
            if (live) {
                if (k <= t) {
                    v = sys_elem<R>(stage, f, t, k);
                    nzA |= (t < f && v != 0.f);
                } else if (hasB) {
                    v = sys_elem<R>(stage + stride, f, rB, R - k);
                    nzB |= (rB < f && v != 0.f);
                } else {
                    v = (rB == R - k && rB < R - 1) ? 1.f : 0.f;  // a missing B solves as identity
                }
            }
            a[k] = v;
        });
        const bool actA = __syncthreads_or(nzA) != 0;  // all-zero A: x = 0 (solver.hpp:215-220)
        const bool actB = __syncthreads_or(nzB) != 0;
        // ---- LDL^T, one column per step ----
        static_for<R - 1>([&](auto cc) {
            constexpr int c = decltype(cc)::value;
            float* cA = col + (0 * 2 + (c & 1)) * P::NT;
            float* cB = col + (1 * 2 + (c & 1)) * P::NT;
            if (live && t >= c) cA[t] = a[c];
            if (live && rB >= c) cB[rB] = a[R - c];
            asm volatile("bar.sync 1, %0;\n" ::"r"(P::NT) : "memory");
            const float dA = cA[c], dB = cB[c];
            if (t == c && !(dA > 0.f) && bad[0] == 0) {
                bad[0] = c + 1;
                badv[0] = dA;
            }
            if (rB == c && !(dB > 0.f) && bad[1] == 0) {
                bad[1] = c + 1;
                badv[1] = dB;
            }
            const float sA = (t > c) ? __fdiv_rn(a[c], dA) : 0.f;
            const float sB = (rB > c) ? __fdiv_rn(a[R - c], dB) : 0.f;
            // a[j] -= s col[j] for j in (c, row]; warp-uniform skips of quads beyond the warp's rows
            constexpr int J0 = (c + 1) & ~3;
            static_for<(R - 1 - J0 + 3) / 4>([&](auto qq) {
                constexpr int j4 = J0 + 4 * decltype(qq)::value;
                if (j4 <= tmaxA) {
                    const float4 v = *reinterpret_cast<const float4*>(cA + j4);
                    const float vv[4] = {v.x, v.y, v.z, v.w};
                    static_for<4>([&](auto q) {
                        constexpr int j = j4 + decltype(q)::value;
                        if constexpr (j > c && j < R - 1)
                            if (t >= j) a[j] = fmaf(-sA, vv[decltype(q)::value], a[j]);
                    });
                }
                if (j4 <= rmaxB) {
                    const float4 v = *reinterpret_cast<const float4*>(cB + j4);
                    const float vv[4] = {v.x, v.y, v.z, v.w};
                    static_for<4>([&](auto q) {
                        constexpr int j = j4 + decltype(q)::value;
                        if constexpr (j > c && j < R - 1)
                            if (rB >= j) a[R - j] = fmaf(-sB, vv[decltype(q)::value], a[R - j]);
                    });
                }
            });
            if (t > c) a[c] = sA;
            if (rB > c) a[R - c] = sB;
        });
        __syncthreads();  // the packed rows are consumed: the stage takes the factors
        // dump: row i < R-1 -> [L[i][0..i-1], d_i] at i(i+1)/2; the augmented row -> z at TRI
        if (live) {
            static_for<R + 1>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if (k <= t) {
                    const int idx = t < R - 1 ? t * (t + 1) / 2 + k : P::TRI + k;
                    if (k < R - 1 || t < R - 1) stage[idx] = a[k];
                } else {
                    constexpr int j = R - k;
                    const int idx = rB < R - 1 ? rB * (rB + 1) / 2 + j : P::TRI + j;
                    if (j < R - 1 || rB < R - 1) stage[stride + idx] = a[k];
                }
            });
        }
        __syncthreads();
        // ---- L^T x = z, one warp per system ----
        for (int sys = warp; sys < 2; sys += P::NW) {
            const int64_t g = sys == 0 ? gA : gB;
            if (g >= count) continue;
            const float* L = stage + sys * stride;
            const bool act = sys == 0 ? actA : actB;
            const int b = bad[sys];
            float x[P::Q];
#pragma unroll
            for (int q = 0; q < P::Q; ++q) {
                const int i = 32 * q + lane;
                x[q] = i < R - 1 ? L[P::TRI + i] : 0.f;
            }
            for (int i = R - 2; i > 0; --i) {
                float xi = 0.f;
#pragma unroll
                for (int q = 0; q < P::Q; ++q)
                    if (q == (i >> 5)) xi = x[q];
                xi = __shfl_sync(0xffffffffu, xi, i & 31);
                const float* Li = L + i * (i + 1) / 2;
#pragma unroll
                for (int q = 0; q < P::Q; ++q) {
                    const int k = 32 * q + lane;
                    if (k < i) x[q] = fmaf(-Li[k], xi, x[q]);
                }
            }
            float* xo = out_x + g * f;
#pragma unroll
            for (int q = 0; q < P::Q; ++q) {
                const int i = 32 * q + lane;
                if (i < f) xo[i] = (act && b == 0) ? x[q] : 0.f;
            }
            if (lane == 0) {
                if (act && b != 0) {
                    column[g] = b;
                    pivot[g] = static_cast<double>(badv[sys]);
                    atomicMin(min_row, static_cast<unsigned long long>(status_base + g));
                } else {
                    column[g] = 0;
                }
            }
        }
        __syncthreads();  // the stage is refilled by the next pair's bulk copies
    }
}

template <int R>
void launch_ldl(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                cudaStream_t s) {
    using P = LdlPlan<R>;
    const int64_t pks = packed_stride(f);
    const int64_t stride = (pks + 3) & ~int64_t(3);
    const size_t dump = static_cast<size_t>(P::TRI + R);
    const size_t smem =
        sizeof(float) * (2 * static_cast<size_t>(std::max<int64_t>(stride, (dump + 3) & ~size_t(3))) + 4 * P::NT);
    auto k = ldl_solve_kernel<R>;
    ALSK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 0;
    ALSK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, P::NT, smem));
    const int64_t npairs = (count + 1) / 2;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(npairs, std::max(occ, 1) * int64_t(num_sms()))));
    k<<<grid, P::NT, smem, s>>>(packed, count, f, pks, std::max<int64_t>(stride, (dump + 3) & ~size_t(3)), x,
                                st.min_row, st.column + status_off,
                                st.pivot + status_off, status_off);
    ALSK_LAUNCHED();
}

}  // namespace

// R = f rounded up to a multiple of 4, plus the augmented row (identity padding in between).
bool packed_solve_ldl(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                      cudaStream_t s) {
    if (count <= 0) return true;
    const int r = ((f + 3) / 4) * 4 + 1;
    switch (r) {
        case 101: launch_ldl<101>(packed, count, f, x, st, status_off, s); return true;
        default: return false;
    }
}

}  // namespace alsk
