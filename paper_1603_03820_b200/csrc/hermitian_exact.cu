// Reference-order Hermitian assembly (materialised) and reference-order batched Cholesky.
//
// These kernels reproduce the reference's default accumulate_double=true path bit for
// bit: every A/B entry is one thread's sequential double sum over the row's nonzeros in
// ascending order (a float*float product is exact in double, so FMA vs mul+add cannot
// differ), lambda*n_u is added last on the diagonal and the result rounded once to float
// (solver.hpp:99-157). The Cholesky is right-looking, but each entry still receives its
// updates in ascending column order with separately rounded multiply and subtract, which
// is exactly the left-looking order of batch_solve_into (solver.hpp:223-246).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "kernels.cuh"
#include "measure.cuh"

namespace alsk {
namespace {

constexpr int kChunk = 32;  // nonzeros staged per shared-memory tile

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
        for (int e = threadIdx.x; e < cnt * fp; e += blockDim.x) {
            const int kk = e / fp, c = e - kk * fp;
            float v = 0.f;
            if (c < f) {
                const int64_t row = static_cast<int64_t>(col_idx[k + kk]) - col_lo;
                v = theta[row * f + c];
            } else if (c == f) {
                v = values[k + kk];
            }
            tile[kk * fp + c] = v;
        }
        __syncthreads();
        if (active) {
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

// Packed lower-triangular index.
__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }

// One CTA per system. Shared: packed lower L (double), rhs/forward vector s (double),
// x (float).
__global__ void solve_exact_kernel(const float* __restrict__ A, const float* __restrict__ Bv,
                                   int f, int64_t row_base, float* __restrict__ X,
                                   unsigned long long* __restrict__ min_row,
                                   int32_t* __restrict__ column, double* __restrict__ pivot,
                                   unsigned long long* __restrict__ prof) {
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
    double* L = sm;                        // f(f+1)/2
    double* s = L + f * (f + 1) / 2;       // f
    float* xs = reinterpret_cast<float*>(s + f);
    uint8_t* tri = reinterpret_cast<uint8_t*>(xs + f);  // (i, j) of the (f-1)-triangle, row-major
    const int64_t row = blockIdx.x;
    const float* a = A + row * static_cast<int64_t>(f) * f;
    const float* b = Bv + row * f;
    float* x = X + row * f;
    const int tid = threadIdx.x, nt = blockDim.x;

    // all-zero test over the full f*f storage (solver.hpp:215-220)
    int nonzero = 0;
    for (int e = tid; e < f * f; e += nt) nonzero |= (a[e] != 0.0f);
    if (!__syncthreads_or(nonzero)) {
        for (int i = tid; i < f; i += nt) x[i] = 0.0f;
        if (tid == 0) column[row] = 0;
        return;
    }
    for (int i = tid; i < f; i += nt) {
        for (int j = 0; j <= i; ++j) L[pk(i, j)] = static_cast<double>(a[i * f + j]);
        s[i] = static_cast<double>(b[i]);
    }
    for (int i = tid; i < f - 1; i += nt)
        for (int j = 0; j <= i; ++j) {
            tri[2 * pk(i, j)] = static_cast<uint8_t>(i);
            tri[2 * pk(i, j) + 1] = static_cast<uint8_t>(j);
        }
    __syncthreads();

    SE_LAP(0)
    bool broke = false;
    for (int c = 0; c < f; ++c) {
        // every thread reads the pivot and takes its square root itself (the same value in
        // every thread), so no single-thread phase and barrier precede the divisions
        const double d = L[pk(c, c)];
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
        for (int r = c + 1 + tid; r < f; r += nt) L[pk(r, c)] = __ddiv_rn(L[pk(r, c)], lcc);
        __syncthreads();  // every thread has read d: the diagonal can take L[c][c] now
        if (tid == 0) L[pk(c, c)] = lcc;
        // trailing update of entries (r, q), c < q <= r, enumerated flat over the threads
        // (row-major lower triangle: entry k of the (f-c-1)-triangle is tri[k]; the first
        // T(T+1)/2 entries of the largest triangle are exactly the smaller ones), so short
        // rows leave no lanes idle. Each entry still takes its updates in ascending c, one
        // separately rounded multiply-subtract per column: the reference's order.
        const int T = f - c - 1, nent = T * (T + 1) / 2;
        for (int k = tid; k < nent; k += nt) {
            const int r = c + 1 + tri[2 * k], q = c + 1 + tri[2 * k + 1];
            const int rb = r * (r + 1) / 2;
            L[rb + q] = __dsub_rn(L[rb + q], __dmul_rn(L[rb + c], L[q * (q + 1) / 2 + c]));
        }
        __syncthreads();
    }
    SE_LAP(1)
    if (broke) {
        for (int i = tid; i < f; i += nt) x[i] = 0.0f;
        return;
    }
    if (tid == 0) column[row] = 0;
    // forward substitution, column oriented: s_i -= L[i][j]*y_j for j ascending
    // (same per-entry order as the reference's row-oriented loop, solver.hpp:249-253).
    if (tid < 32) {
        for (int j = 0; j < f; ++j) {
            const double yj = __ddiv_rn(s[j], L[pk(j, j)]);
            __syncwarp();
            if (tid == 0) s[j] = yj;
            for (int i = j + 1 + tid; i < f; i += 32) s[i] = __dsub_rn(s[i], __dmul_rn(L[pk(i, j)], yj));
            __syncwarp();
        }
        SE_LAP(2)
        // back substitution reads the already-rounded float x[j] (solver.hpp:254-259);
        // its order (j ascending from i+1) is inherently sequential.
        // Products of 8 consecutive j are formed ahead of their (in-order) subtractions, so
        // only the subtraction chain is serial.
        if (tid == 0) {
            for (int i = f - 1; i >= 0; --i) {
                double acc = s[i];
                int j = i + 1;
                for (; j + 8 <= f; j += 8) {
                    double p[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) p[u] = __dmul_rn(L[pk(j + u, i)], static_cast<double>(xs[j + u]));
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc = __dsub_rn(acc, p[u]);
                }
                for (; j < f; ++j) acc = __dsub_rn(acc, __dmul_rn(L[pk(j, i)], static_cast<double>(xs[j])));
                xs[i] = static_cast<float>(__ddiv_rn(acc, L[pk(i, i)]));
            }
        }
        __syncwarp();
        SE_LAP(3)
        for (int i = tid; i < f; i += 32) x[i] = xs[i];
    }
#undef SE_LAP
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
    constexpr int TB = 4;
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
    const size_t smem = (static_cast<size_t>(f) * (f + 1) / 2 + f) * sizeof(double) + f * sizeof(float) +
                        static_cast<size_t>(f) * (f - 1) + 16;  // + the (f-1)-triangle's (i, j) bytes
    if (f > 256 || smem > 220 * 1024) fail_input("rank " + std::to_string(f) + " too large for device solve");
    ALSK_CUDA(cudaFuncSetAttribute(solve_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int threads = f <= 32 ? 32 : (f <= 64 ? 64 : 128);
    for (int64_t b0 = 0; b0 < count; b0 += (1LL << 30)) {
        const int64_t n = std::min<int64_t>(count - b0, 1LL << 30);
        static const bool want_prof = measure_env("ALSK_SE_PROF") != nullptr;
        DevBuf pb;
        if (want_prof) {
            pb.alloc(4 * sizeof(unsigned long long), s);
            ALSK_CUDA(cudaMemsetAsync(pb.as<void>(), 0, 4 * sizeof(unsigned long long), s));
        }
        solve_exact_kernel<<<static_cast<unsigned>(n), threads, smem, s>>>(
            A + static_cast<size_t>(b0) * f * f, B + static_cast<size_t>(b0) * f, f,
            b0, X + static_cast<size_t>(b0) * f, st.min_row, st.column + b0,
            st.pivot + b0, want_prof ? pb.as<unsigned long long>() : nullptr);
        ALSK_LAUNCHED();
        if (want_prof) {
            unsigned long long h[4];
            d2h(h, pb.as<unsigned long long>(), 4, s);
            ALSK_CUDA(cudaStreamSynchronize(s));
            std::fprintf(stderr, "[se-prof f=%d systems=%lld threads=%d] kcyc per system: load %.1f factor %.1f forward %.1f back %.1f\n",
                         f, static_cast<long long>(n), threads, h[0] / 1e3 / n, h[1] / 1e3 / n, h[2] / 1e3 / n,
                         h[3] / 1e3 / n);
        }
    }
}

}  // namespace alsk
