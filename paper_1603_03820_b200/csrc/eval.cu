// Objective and RMSE on the device (solver.hpp:358-406).
//
// Each rating's residual is computed exactly like dot_rows (solver.hpp:265-270): an
// index-ascending double dot over float operands. The sums over ratings/rows use a
// deterministic two-level reduction (fixed per-block order, then one block over the
// partials), so results are run-to-run reproducible and differ from the reference's serial
// sum only by double reassociation (~1e-16 relative).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace alsk {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 8;

__device__ __forceinline__ double dot_rows(const float* __restrict__ a, const float* __restrict__ b, int f) {
    double s = 0.0;
    for (int i = 0; i < f; ++i) s += static_cast<double>(a[i]) * static_cast<double>(b[i]);
    return s;
}

// The same dot with 16-byte operand loads (f % 4 == 0, 16-byte aligned rows): the products
// are still added one by one in ascending index order, so the result is bit-identical to
// dot_rows; a lane's gathered row costs f/4 load instructions instead of f.
__device__ __forceinline__ double dot_rows4(const float* __restrict__ a, const float* __restrict__ b, int f) {
    const float4* a4 = reinterpret_cast<const float4*>(a);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    double s = 0.0;
    for (int i = 0; i < f / 4; ++i) {
        const float4 p = a4[i], q = __ldg(b4 + i);
        s += static_cast<double>(p.x) * static_cast<double>(q.x);
        s += static_cast<double>(p.y) * static_cast<double>(q.y);
        s += static_cast<double>(p.z) * static_cast<double>(q.z);
        s += static_cast<double>(p.w) * static_cast<double>(q.w);
    }
    return s;
}

template <bool VEC>
__device__ __forceinline__ double dot_any(const float* __restrict__ a, const float* __restrict__ b, int f) {
    if constexpr (VEC) return dot_rows4(a, b, f);
    else return dot_rows(a, b, f);
}

inline bool vec4_ok(const float* a, const float* b, int f) {
    return f % 4 == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0;
}

// Deterministic block reduction of one double per thread; result in thread 0.
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    __syncthreads();
    return t;
}

// Squared residuals over the CSR; one warp per row, lanes over the row's ratings.
template <bool VEC>
__global__ void loss_sq_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                               const float* __restrict__ values, int64_t rows,
                               const float* __restrict__ x, const float* __restrict__ theta, int f,
                               double* __restrict__ partial) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    double acc = 0.0;
    for (int64_t u = warp0; u < rows; u += nwarps) {
        const float* xu = x + u * f;
        for (int64_t k = row_ptr[u] + lane; k < row_ptr[u + 1]; k += 32) {
            const double d = static_cast<double>(values[k]) -
                             dot_any<VEC>(xu, theta + static_cast<int64_t>(col_idx[k]) * f, f);
            acc += d * d;
        }
    }
    const double t = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// Regularisation term: sum over rows of n * |row|^2 (rows with n==0 skipped).
__global__ void reg_kernel(const int64_t* __restrict__ counts_ptr, const int64_t* __restrict__ counts,
                           int64_t rows, const float* __restrict__ fac, int f,
                           double* __restrict__ partial) {
    double acc = 0.0;
    for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < rows;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t n = counts_ptr ? counts_ptr[u + 1] - counts_ptr[u] : counts[u];
        if (n == 0) continue;
        const float* r = fac + u * f;
        double norm2 = 0.0;
        for (int i = 0; i < f; ++i) norm2 += static_cast<double>(r[i]) * static_cast<double>(r[i]);
        acc += static_cast<double>(n) * norm2;
    }
    const double t = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void final_sum_kernel(const double* __restrict__ partial, int n, double* __restrict__ out) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
    const double t = block_sum(acc);
    if (threadIdx.x == 0) *out = t;
}

__global__ void col_count_kernel(const int32_t* __restrict__ col_idx, int64_t nnz,
                                 unsigned long long* __restrict__ counts) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(counts + col_idx[k], 1ull);
}

template <bool VEC>
__global__ void rmse_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                            const float* __restrict__ values, int64_t count,
                            const float* __restrict__ x, int64_t x_rows,
                            const float* __restrict__ theta, int64_t theta_rows, int f,
                            double* __restrict__ partial, unsigned long long* __restrict__ first_bad) {
    double acc = 0.0;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < count;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = rows[t], c = cols[t];
        if (r < 0 || r >= x_rows || c < 0 || c >= theta_rows) {
            atomicMin(first_bad, static_cast<unsigned long long>(t));
            continue;
        }
        const double d = static_cast<double>(values[t]) - dot_any<VEC>(x + r * f, theta + c * f, f);
        acc += d * d;
    }
    const double t = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

int blocks_for(int64_t work, int per_block) {
    const int64_t b = (work + per_block - 1) / per_block;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, kMaxBlocks)));
}

double reduce_partials(const double* partial, int n, cudaStream_t s) {
    DevBuf out(sizeof(double), s);
    final_sum_kernel<<<1, kThreads, 0, s>>>(partial, n, out.as<double>());
    ALSK_LAUNCHED();
    double h = 0.0;
    d2h(&h, out.as<double>(), 1, s);
    ALSK_CUDA(cudaStreamSynchronize(s));
    return h;
}

}  // namespace

void column_counts(const DevCsr& r, int64_t* col_nnz, cudaStream_t s) {
    ALSK_CUDA(cudaMemsetAsync(col_nnz, 0, sizeof(int64_t) * r.cols, s));
    if (r.nnz == 0) return;
    col_count_kernel<<<blocks_for(r.nnz, kThreads), kThreads, 0, s>>>(
        r.col_idx, r.nnz, reinterpret_cast<unsigned long long*>(col_nnz));
    ALSK_LAUNCHED();
}

double loss_device(const DevCsr& r, const int64_t* col_nnz, const float* x, const float* theta,
                   int f, double lambda, cudaStream_t s) {
    DevBuf partial(sizeof(double) * 3 * kMaxBlocks, s);
    double* p = partial.as<double>();
    const int b1 = blocks_for(r.rows * 32, kThreads);
    if (vec4_ok(x, theta, f))
        loss_sq_kernel<true><<<b1, kThreads, 0, s>>>(r.row_ptr, r.col_idx, r.values, r.rows, x, theta, f, p);
    else
        loss_sq_kernel<false><<<b1, kThreads, 0, s>>>(r.row_ptr, r.col_idx, r.values, r.rows, x, theta, f, p);
    ALSK_LAUNCHED();
    const int b2 = blocks_for(r.rows, kThreads);
    reg_kernel<<<b2, kThreads, 0, s>>>(r.row_ptr, nullptr, r.rows, x, f, p + kMaxBlocks);
    ALSK_LAUNCHED();
    const int b3 = blocks_for(r.cols, kThreads);
    reg_kernel<<<b3, kThreads, 0, s>>>(nullptr, col_nnz, r.cols, theta, f, p + 2 * kMaxBlocks);
    ALSK_LAUNCHED();
    const double sq = reduce_partials(p, b1, s);
    const double reg_x = reduce_partials(p + kMaxBlocks, b2, s);
    const double reg_t = reduce_partials(p + 2 * kMaxBlocks, b3, s);
    return sq + lambda * (reg_x + reg_t);
}

double rmse_device(const int64_t* rows, const int64_t* cols, const float* values, int64_t count,
                   const float* x, int64_t x_rows, const float* theta, int64_t theta_rows, int f,
                   cudaStream_t s) {
    if (count <= 0) fail_input("empty test set");
    DevBuf partial(sizeof(double) * kMaxBlocks, s);
    DevBuf bad(sizeof(unsigned long long), s);
    ALSK_CUDA(cudaMemsetAsync(bad.as<void>(), 0xff, sizeof(unsigned long long), s));
    const int b = blocks_for(count, kThreads);
    if (vec4_ok(x, theta, f))
        rmse_kernel<true><<<b, kThreads, 0, s>>>(rows, cols, values, count, x, x_rows, theta, theta_rows, f,
                                                 partial.as<double>(), bad.as<unsigned long long>());
    else
        rmse_kernel<false><<<b, kThreads, 0, s>>>(rows, cols, values, count, x, x_rows, theta, theta_rows, f,
                                                  partial.as<double>(), bad.as<unsigned long long>());
    ALSK_LAUNCHED();
    unsigned long long first_bad = 0;
    d2h(&first_bad, bad.as<unsigned long long>(), 1, s);
    const double sq = reduce_partials(partial.as<double>(), b, s);
    if (first_bad != ~0ull) {
        int64_t rr = 0, cc = 0;
        d2h(&rr, rows + first_bad, 1, s);
        d2h(&cc, cols + first_bad, 1, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
        fail_input("test pair (" + std::to_string(rr) + ", " + std::to_string(cc) +
                   ") outside factor shapes");
    }
    return std::sqrt(sq / static_cast<double>(count));
}

}  // namespace alsk
