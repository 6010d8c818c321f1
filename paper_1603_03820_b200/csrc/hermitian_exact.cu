// Reference-order Hermitian assembly (materialised) and reference-order batched Cholesky.
//
// These kernels reproduce the reference's default accumulate_double=true path bit for
// bit: every A/B entry is one thread's sequential double sum over the row's nonzeros in
// ascending order (a float*float product is exact in double, so FMA vs mul+add cannot
// differ), lambda*n_u is added last on the diagonal and the result rounded once to float
// (solver.hpp:99-157). The Cholesky is left-looking like batch_solve_into (solver.hpp:
// 223-246): each entry's sum in ascending column order with separately rounded multiply and
// subtract; the forward and back substitutions (solver.hpp:249-259) run one thread per
// system in the same order.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "kernels.cuh"
#include "measure.cuh"

namespace alsk {
namespace {

constexpr int kChunk = 64;  // nonzeros staged per shared-memory tile

// Lower-triangular tile enumeration: t -> (bi, bj), bj <= bi, row-major.
__device__ __forceinline__ void tile_coords(int t, int& bi, int& bj) {
    int b = 0;
    while ((b + 1) * (b + 2) / 2 <= t) ++b;
    bi = b;
    bj = t - b * (b + 1) / 2;
}

// One CTA per row (grid.x) and tile pass (grid.y). Thread owns a TBxTB tile of the
// augmented (f+1)x(f+1) lower triangle: row f of the augmented matrix is B = sum r*theta.
template <class Acc, class OutT, int TB>
__global__ void herm_mat_kernel(const int64_t* __restrict__ row_ptr,
                                const int32_t* __restrict__ col_idx,
                                const float* __restrict__ values, int64_t col_lo,
                                const float* __restrict__ theta, int f, int nb, double lambda,
                                int64_t rb, OutT* __restrict__ A, OutT* __restrict__ B, int packed) {
    extern __shared__ float tile[];  // kChunk x fp
    const int fp = nb * TB;
    const int64_t u = rb + blockIdx.x;
    const int64_t k0 = row_ptr[u], k1 = row_ptr[u + 1];
    const int t = blockIdx.y * blockDim.x + threadIdx.x;
    const int ntiles = nb * (nb + 1) / 2;
    const bool active = t < ntiles;
    int bi = 0, bj = 0;
    if (active) tile_coords(t, bi, bj);

    Acc acc[TB][TB];
#pragma unroll
    for (int i = 0; i < TB; ++i)
#pragma unroll
        for (int j = 0; j < TB; ++j) acc[i][j] = Acc(0);

    for (int64_t k = k0; k < k1; k += kChunk) {
        const int cnt = static_cast<int>(((k1 - k) < kChunk ? (k1 - k) : (int64_t)kChunk));
        __syncthreads();
        // a warp per staged rating, lanes over the features: no index division, and each
        // lane's loads of a round are issued before its stores (double-buffering the tile
        // with cp.async measured slower: 9.85 vs 9.70 ms per Netflix launch)
        {
            const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
            for (int kk = threadIdx.x >> 5; kk < cnt; kk += nw) {
                const int64_t row = static_cast<int64_t>(col_idx[k + kk]) - col_lo;
                const float rv = values[k + kk];
                const float* src = theta + row * f;
                float* dst = tile + kk * fp;
                for (int c0 = 0; c0 < fp; c0 += 128) {
                    float v[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = c0 + lane + 32 * q;
                        v[q] = c < f ? src[c] : (c == f ? rv : 0.f);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = c0 + lane + 32 * q;
                        if (c < fp) dst[c] = v[q];
                    }
                }
            }
        }
        __syncthreads();
        if (active) {
#pragma unroll 4
            for (int kk = 0; kk < cnt; ++kk) {
                const float* trow = tile + kk * fp;
                Acc a[TB], b[TB];
#pragma unroll
                for (int i = 0; i < TB; ++i) a[i] = static_cast<Acc>(trow[bi * TB + i]);
#pragma unroll
                for (int j = 0; j < TB; ++j) b[j] = static_cast<Acc>(trow[bj * TB + j]);
#pragma unroll
                for (int i = 0; i < TB; ++i)
#pragma unroll
                    for (int j = 0; j < TB; ++j) acc[i][j] += a[i] * b[j];
            }
        }
    }
    if (!active) return;
    const Acc reg = static_cast<Acc>(lambda) * static_cast<Acc>(k1 - k0);
    const int64_t out_row = u - rb;
    if (packed) {  // lower-packed A then B
        OutT* o = A + out_row * (static_cast<int64_t>(f) * (f + 1) / 2 + f);
#pragma unroll
        for (int ii = 0; ii < TB; ++ii)
#pragma unroll
            for (int jj = 0; jj < TB; ++jj) {
                const int i = bi * TB + ii, j = bj * TB + jj;
                if (j > i || j >= f || i > f) continue;
                o[i * (i + 1) / 2 + j] = static_cast<OutT>(i == j ? acc[ii][jj] + reg : acc[ii][jj]);
            }
        return;
    }
    OutT* a_out = A + out_row * static_cast<int64_t>(f) * f;
    OutT* b_out = B + out_row * f;
#pragma unroll
    for (int ii = 0; ii < TB; ++ii) {
#pragma unroll
        for (int jj = 0; jj < TB; ++jj) {
            const int i = bi * TB + ii, j = bj * TB + jj;
            if (j > i || j >= f || i > f) continue;
            if (i == f) {
                b_out[j] = static_cast<OutT>(acc[ii][jj]);
            } else if (i == j) {
                a_out[i * f + i] = static_cast<OutT>(acc[ii][jj] + reg);
            } else {
                const OutT val = static_cast<OutT>(acc[ii][jj]);
                a_out[i * f + j] = val;
                a_out[j * f + i] = val;
            }
        }
    }
}

__global__ void check_columns_kernel(const int64_t* __restrict__ row_ptr,
                                     const int32_t* __restrict__ col_idx, int64_t kb, int64_t ke,
                                     int64_t col_lo, int64_t col_hi,
                                     unsigned long long* __restrict__ first_bad) {
    for (int64_t k = kb + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < ke;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t v = col_idx[k];
        if (v < col_lo || v >= col_hi) atomicMin(first_bad, static_cast<unsigned long long>(k));
    }
}

// One CTA per system. Shared: packed lower L (double), rhs/forward vector s (double),
// x (float).
// Back substitution does not run here: it is one serial chain of f(f-1)/2 subtractions per
// system (the reference's order), which would hold the whole CTA. The kernel hands each
// system to backsub_exact_kernel instead, through `work` (subst_stride(f) doubles per
// system): b (f doubles), then for i = f-1 down to 0 the diagonal L[i][i] followed by
// L[j][i], j = i+1..f-1 -- column i of L, read in ascending column order by the forward
// substitution and in the stored order by the back substitution. A system that needs no
// substitution (all-zero or broken; x already written) gets 0 as its first diagonal.
// Element e of system t sits at subst_at(t, e): interleaved by 32 systems, so the
// substitution warp's loads of one element are a single 256-byte access.
__host__ __device__ inline int64_t subst_stride(int f) { return static_cast<int64_t>(f) * (f + 1) / 2 + f; }
__device__ __forceinline__ int64_t subst_at(int64_t t, int64_t e, int64_t per) {
    return (t >> 5) * (per * 32) + e * 32 + (t & 31);
}

// One CTA per system, left-looking Cholesky in the reference's order (solver.hpp:222-244):
// for column c every row r >= c forms s = a_rc - sum_{t<c} l_rt l_ct, t ascending, each
// product and difference rounded separately -- one thread per row with the running sum in a
// register (no trailing-matrix stores); the diagonal row checks s > 0 and every thread takes
// the square root, the other rows divide. L is held column-major packed (column t = rows
// t..f-1, contiguous), so a warp's l_rt loads are consecutive doubles and l_ct is a
// broadcast. Both substitutions run in backsub_exact_kernel (a single lane's chain here cost
// 11% of this kernel's time in shared-memory wavefronts and issue slots).
constexpr int SE_U = 8;  // dot products formed ahead of their in-order subtractions

__global__ void solve_exact_kernel(const float* __restrict__ A, const float* __restrict__ Bv,
                                   int f, int64_t row_base, float* __restrict__ X,
                                   unsigned long long* __restrict__ min_row,
                                   int32_t* __restrict__ column, double* __restrict__ pivot,
                                   double* __restrict__ work, unsigned long long* __restrict__ prof) {
#ifdef ALSK_MEASURE
    long long t_lap = clock64();  // ALSK_SE_PROF=1: cycles per phase (thread 0), measurement builds
#define SE_LAP(slot)                                                    \
    if (prof && threadIdx.x == 0) {                                     \
        const long long now_ = clock64();                               \
        atomicAdd(prof + (slot), static_cast<unsigned long long>(now_ - t_lap)); \
        t_lap = now_;                                                   \
    }
#else
#define SE_LAP(slot)
#endif
    extern __shared__ double sm[];
    double* L = sm;                    // f(f+1)/2, column-major packed: l_rt at colstart(t) + r
    double* y = L + f * (f + 1) / 2;   // f: b (as double)
    double* piv = y + f;               // the current column's pivot
    const int64_t row = blockIdx.x;
    const float* a = A + row * static_cast<int64_t>(f) * f;
    const float* b = Bv + row * f;
    float* x = X + row * f;
    const int64_t per = subst_stride(f);
    const int tid = threadIdx.x, nt = blockDim.x;
    // column t starts at colstart(t) - t + t = t(f-1) - t(t-1)/2 (+ r for row r)
    auto colstart = [f](int t) { return t * (f - 1) - t * (t - 1) / 2; };

    // all-zero test over the full f*f storage (solver.hpp:215-220), then the lower triangle
    int nonzero = 0;
    for (int e = tid; e < f * f; e += nt) nonzero |= (a[e] != 0.0f);
    {
        const int lane = tid & 31, nw = nt >> 5;
        for (int i = tid >> 5; i < f; i += nw)  // a warp per row (L2-warm re-read)
            for (int j = lane; j <= i; j += 32) L[colstart(j) + i] = static_cast<double>(a[static_cast<int64_t>(i) * f + j]);
    }
    for (int i = tid; i < f; i += nt) y[i] = static_cast<double>(b[i]);
    if (!__syncthreads_or(nonzero)) {
        for (int i = tid; i < f; i += nt) x[i] = 0.0f;
        if (tid == 0) {
            column[row] = 0;
            work[subst_at(row, f, per)] = 0.0;
        }
        return;
    }

    SE_LAP(0)
    bool broke = false;
    for (int c = 0; c < f; ++c) {
        for (int r = c + tid; r < f; r += nt) {
            double acc = L[colstart(c) + r];
            int off = 0;
            int t = 0;
            for (; t + SE_U <= c; t += SE_U) {  // products formed ahead; only the subtractions chain
                double p[SE_U];
#pragma unroll
                for (int q = 0; q < SE_U; ++q) {
                    p[q] = __dmul_rn(L[off + r], L[off + c]);
                    off += f - 1 - (t + q);
                }
#pragma unroll
                for (int q = 0; q < SE_U; ++q) acc = __dsub_rn(acc, p[q]);
            }
            for (; t < c; ++t) {
                acc = __dsub_rn(acc, __dmul_rn(L[off + r], L[off + c]));
                off += f - 1 - t;
            }
            if (r == c) *piv = acc;
            else L[colstart(c) + r] = acc;
        }
        __syncthreads();
        const double d = *piv;
        if (!(d > 0.0)) {  // CTA-uniform
            if (tid == 0) {
                column[row] = c + 1;
                pivot[row] = d;
                atomicMin(min_row, static_cast<unsigned long long>(row_base + row));
            }
            broke = true;
            break;
        }
        const double lcc = sqrt(d);
        for (int r = c + 1 + tid; r < f; r += nt) L[colstart(c) + r] = __ddiv_rn(L[colstart(c) + r], lcc);
        if (tid == 0) L[colstart(c) + c] = lcc;
        __syncthreads();
    }
    SE_LAP(1)
    if (broke) {
        for (int i = tid; i < f; i += nt) x[i] = 0.0f;
        if (tid == 0) work[subst_at(row, f, per)] = 0.0;
        return;
    }
    if (tid == 0) column[row] = 0;
    __syncthreads();
    SE_LAP(2)
    // hand off to backsub_exact_kernel: b, then per column i (descending) the diagonal and
    // column i below it -- one contiguous run of the column-major L
    double* wk = work + subst_at(row, 0, per);
    for (int i = tid; i < f; i += nt) wk[32 * i] = y[i];
    int64_t e = f;
    for (int i = f - 1; i >= 0; --i) {
        const int n = f - i;
        const double* col = L + colstart(i) + i;
        for (int jj = tid; jj < n; jj += nt) wk[32 * (e + jj)] = col[jj];
        e += n;
    }
    SE_LAP(3)
#undef SE_LAP
}

// Forward and back substitution, one thread per system (solver.hpp:249-259), each a chain
// the reference's order makes serial: y_i = (b_i - sum_{j<i} l_ij y_j) / l_ii with the
// subtractions in ascending j (applied column by column: for j ascending, y_j = s_j / l_jj,
// then s_i -= l_ij y_j for i > j -- the same per-entry order), then for i = f-1 down to 0
// x_i = float((y_i - sum_{j>i} l_ji double(x_j)) / l_ii), ascending j, each product and
// difference rounded separately. Systems run side by side (thousands per SM) instead of on
// one thread of a CTA. s/y/x live in one shared-memory array, [i][thread] (conflict-free):
// x_j overwrites y_j once y_j is consumed.
constexpr int BS_THREADS = 64;
constexpr int BS_G = 8;  // back-substitution products formed per group (16, and grouping the
                          // forward updates, measured slower)
__global__ void __launch_bounds__(BS_THREADS) backsub_exact_kernel(const double* __restrict__ work, int f, int64_t count,
                                                                   float* __restrict__ X) {
    extern __shared__ double ysh[];
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const int64_t per = subst_stride(f);
    const double* b = work + subst_at(t, 0, per);  // element e at b[32 * e]
    const double* cols = b + 32 * f;                 // column f-1 first
    if (!(cols[0] > 0.0)) return;  // all-zero or broken system: x already written
    double* ys = ysh + threadIdx.x;
    const int bd = blockDim.x;
    for (int i = 0; i < f; ++i) ys[i * bd] = b[32 * i];
    // forward: column j starts (f-1-j)(f-j)/2 elements into the column stream
    for (int j = 0; j < f; ++j) {
        const double* c = cols + 32 * ((static_cast<int64_t>(f - 1 - j) * (f - j)) / 2);
        const double yj = __ddiv_rn(ys[j * bd], c[0]);
        ys[j * bd] = yj;
        for (int i = j + 1; i < f; ++i) ys[i * bd] = __dsub_rn(ys[i * bd], __dmul_rn(c[32 * (i - j)], yj));
    }
    // back substitution over the stream in stored order (column f-1 first)
    const double* u = cols;
    for (int i = f - 1; i >= 0; --i) {
        const double d = u[0];
        double acc = ys[i * bd];
        const double* c = u + 32;
        const int n = f - 1 - i;
        int k = 0;
        for (; k + BS_G <= n; k += BS_G) {  // products formed ahead; only the subtractions chain
            double p[BS_G];
#pragma unroll
            for (int q = 0; q < BS_G; ++q) p[q] = __dmul_rn(c[32 * (k + q)], ys[(i + 1 + k + q) * bd]);
#pragma unroll
            for (int q = 0; q < BS_G; ++q) acc = __dsub_rn(acc, p[q]);
        }
        for (; k < n; ++k) acc = __dsub_rn(acc, __dmul_rn(c[32 * k], ys[(i + 1 + k) * bd]));
        ys[i * bd] = static_cast<double>(static_cast<float>(__ddiv_rn(acc, d)));
        u += 32 * (n + 1);
    }
    float* x = X + t * f;
    for (int i = 0; i < f; ++i) x[i] = static_cast<float>(ys[i * bd]);
}

}  // namespace

void check_columns_async(const DevCsr& r, int64_t kb, int64_t ke, int64_t col_lo, int64_t col_hi,
                         unsigned long long* first_bad, cudaStream_t s) {
    if (ke <= kb) return;
    const int64_t n = ke - kb;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, num_sms() * 8));
    check_columns_kernel<<<grid, 256, 0, s>>>(r.row_ptr, r.col_idx, kb, ke, col_lo, col_hi, first_bad);
    ALSK_LAUNCHED();
}

void fail_bad_column(const DevCsr& r, unsigned long long entry, int64_t col_lo, int64_t col_hi, cudaStream_t s) {
    int32_t v = 0;
    d2h(&v, r.col_idx + entry, 1, s);
    ALSK_CUDA(cudaStreamSynchronize(s));
    fail_input("column " + std::to_string(v) + " outside partition [" + std::to_string(col_lo) + ", " +
               std::to_string(col_hi) + ")");
}

void check_columns(const DevCsr& r, int64_t rb, int64_t re, int64_t col_lo, int64_t col_hi,
                   cudaStream_t s) {
    if (re <= rb) return;
    int64_t kb = 0, ke = 0;
    d2h(&kb, r.row_ptr + rb, 1, s);
    d2h(&ke, r.row_ptr + re, 1, s);
    ALSK_CUDA(cudaStreamSynchronize(s));
    if (ke <= kb) return;
    DevBuf flag(sizeof(unsigned long long), s);
    ALSK_CUDA(cudaMemsetAsync(flag.as<void>(), 0xff, sizeof(unsigned long long), s));
    const int64_t n = ke - kb;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, num_sms() * 8));
    check_columns_kernel<<<grid, 256, 0, s>>>(r.row_ptr, r.col_idx, kb, ke, col_lo, col_hi,
                                              flag.as<unsigned long long>());
    ALSK_LAUNCHED();
    unsigned long long bad = 0;
    d2h(&bad, flag.as<unsigned long long>(), 1, s);
    ALSK_CUDA(cudaStreamSynchronize(s));
    if (bad != ~0ull) fail_bad_column(r, bad, col_lo, col_hi, s);
}

namespace {
template <class Acc, class OutT>
void launch_herm(const DevCsr& r, const float* theta, int f, double lambda, int64_t rb, int64_t re,
                 OutT* A, OutT* B, bool packed, cudaStream_t s) {
    const int64_t count = re - rb;
    if (count <= 0) return;
    constexpr int TB = 6;  // per-thread tile: 4x4 9.53, 5x5 8.81, 6x6 7.26, 7x7 8.15, 8x8 11.0 ms per Netflix launch
    const int nb = (f + 1 + TB - 1) / TB;
    const int ntiles = nb * (nb + 1) / 2;
    const int threads = std::min(512, ((ntiles + 31) / 32) * 32);
    const int passes = (ntiles + threads - 1) / threads;
    const size_t smem = static_cast<size_t>(kChunk) * nb * TB * sizeof(float);
    if (smem > 200 * 1024) fail_input("rank " + std::to_string(f) + " too large for device assembly");
    auto k = herm_mat_kernel<Acc, OutT, TB>;
    ALSK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t per_a = packed ? static_cast<int64_t>(f) * (f + 1) / 2 + f : static_cast<int64_t>(f) * f;
    for (int64_t b0 = 0; b0 < count; b0 += 65535 * 16) {
        const int64_t n = std::min<int64_t>(count - b0, 65535 * 16);
        dim3 grid(static_cast<unsigned>(n), static_cast<unsigned>(passes));
        k<<<grid, threads, smem, s>>>(r.row_ptr, r.col_idx, r.values, r.col_offset, theta, f, nb, lambda,
                                      rb + b0, A + b0 * per_a, packed ? nullptr : B + b0 * f, packed ? 1 : 0);
        ALSK_LAUNCHED();
    }
}
}  // namespace

void hermitian_materialize(const DevCsr& r, const float* theta, int f, double lambda,
                           bool acc_double, int64_t rb, int64_t re, float* A, float* B,
                           cudaStream_t s) {
    if (acc_double) launch_herm<double, float>(r, theta, f, lambda, rb, re, A, B, false, s);
    else launch_herm<float, float>(r, theta, f, lambda, rb, re, A, B, false, s);
}

void hermitian_materialize_d(const DevCsr& r, const float* theta, int f, double lambda, bool acc_double,
                             int64_t rb, int64_t re, double* A, double* B, bool packed, cudaStream_t s) {
    if (acc_double) launch_herm<double, double>(r, theta, f, lambda, rb, re, A, B, packed, s);
    else launch_herm<float, double>(r, theta, f, lambda, rb, re, A, B, packed, s);
}

void solve_exact(const float* A, const float* B, int64_t count, int f, bool /*zero_row_policy*/,
                 float* X, const SolveStatus& st, cudaStream_t s) {
    // Both policies write a zero row for a broken system; the host raises for `fail`.
    if (count <= 0) return;
    const size_t smem = (static_cast<size_t>(f) * (f + 1) / 2 + f + 1) * sizeof(double);
    if (f > 256 || smem > 220 * 1024) fail_input("rank " + std::to_string(f) + " too large for device solve");
    ALSK_CUDA(cudaFuncSetAttribute(solve_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int threads = f <= 32 ? 32 : (f <= 64 ? 64 : 128);
    // the hand-off scratch bounds a launch: ~4 GB of (y, L) streams at a time, whole groups
    // of 32 systems
    const int64_t per = subst_stride(f);
    const int64_t chunk = std::max<int64_t>(32, std::min<int64_t>(1LL << 30, (int64_t{4} << 30) / (per * 8)) & ~int64_t{31});
    DevBuf work(sizeof(double) * per * ((std::min(count, chunk) + 31) & ~int64_t{31}), s);
    constexpr int BT = BS_THREADS;
    const size_t bsmem = static_cast<size_t>(BT) * f * sizeof(double);
    ALSK_CUDA(cudaFuncSetAttribute(backsub_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
    for (int64_t b0 = 0; b0 < count; b0 += chunk) {
        const int64_t n = std::min<int64_t>(count - b0, chunk);
        static const bool want_prof = measure_env("ALSK_SE_PROF") != nullptr;
        DevBuf pb;
        if (want_prof) {
            pb.alloc(4 * sizeof(unsigned long long), s);
            ALSK_CUDA(cudaMemsetAsync(pb.as<void>(), 0, 4 * sizeof(unsigned long long), s));
        }
        solve_exact_kernel<<<static_cast<unsigned>(n), threads, smem, s>>>(
            A + static_cast<size_t>(b0) * f * f, B + static_cast<size_t>(b0) * f, f,
            b0, X + static_cast<size_t>(b0) * f, st.min_row, st.column + b0,
            st.pivot + b0, work.as<double>(), want_prof ? pb.as<unsigned long long>() : nullptr);
        ALSK_LAUNCHED();
        backsub_exact_kernel<<<static_cast<unsigned>((n + BT - 1) / BT), BT, bsmem, s>>>(
            work.as<double>(), f, n, X + static_cast<size_t>(b0) * f);
        ALSK_LAUNCHED();
        if (want_prof) {
            unsigned long long h[4];
            d2h(h, pb.as<unsigned long long>(), 4, s);
            ALSK_CUDA(cudaStreamSynchronize(s));
            std::fprintf(stderr, "[se-prof f=%d systems=%lld threads=%d] kcyc per system: load %.1f factor %.1f - %.1f hand-off %.1f\n",
                         f, static_cast<long long>(n), threads, h[0] / 1e3 / n, h[1] / 1e3 / n, h[2] / 1e3 / n,
                         h[3] / 1e3 / n);
        }
    }
}

}  // namespace alsk
