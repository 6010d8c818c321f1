// CSR invariant check in HBM for the device loaders (binary cache, block stream): the
// reference's validate() (sparse.hpp:105-125) after a raw upload, so the host only reads and
// copies. One warp per row: row_ptr non-decreasing, every column in [0, cols), strictly
// increasing within the row; the first failing row (atomicMin) is returned and the host
// rebuilds the reference's message from that row alone (row_ptr ends are checked on the
// host first). Reads 4 bytes per rating + 8 per row: an HBM-bound pass (about 0.06 ms per
// 10^8 ratings at 7 TB/s).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"

namespace alsk {
namespace {

__global__ void csr_check_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t rows,
                                 int64_t cols, int64_t nnz, unsigned long long* __restrict__ first_bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < rows; u += warps) {
        const int64_t b = rp[u], e0 = rp[u + 1];
        bool bad = e0 < b;
        const int64_t e = e0 < nnz ? e0 : nnz;
        for (int64_t k0 = b; !bad && k0 < e; k0 += 32) {
            const int64_t k = k0 + lane;
            bool f = false;
            if (k < e) {
                const int32_t v = ci[k];
                f = v < 0 || v >= cols || (k > b && ci[k - 1] >= v);
            }
            bad = __any_sync(0xffffffffu, f);
        }
        if (bad && lane == 0) atomicMin(first_bad, static_cast<unsigned long long>(u));
    }
}

}  // namespace

// First row violating the CSR invariants, or -1. Synchronizes `s`.
int64_t csr_first_bad_row(const int64_t* rp, const int32_t* ci, int64_t rows, int64_t cols, int64_t nnz,
                          cudaStream_t s) {
    if (rows <= 0) return -1;
    DevBuf flag(sizeof(unsigned long long), s);
    ALSK_CUDA(cudaMemsetAsync(flag.as<void>(), 0xff, sizeof(unsigned long long), s));
    int dev = 0, sms = 148;
    ALSK_CUDA(cudaGetDevice(&dev));
    ALSK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t want = (rows * 32 + 255) / 256;
    const unsigned grid = static_cast<unsigned>(want < int64_t(sms) * 8 ? want : int64_t(sms) * 8);
    csr_check_kernel<<<grid, 256, 0, s>>>(rp, ci, rows, cols, nnz, flag.as<unsigned long long>());
    ALSK_LAUNCHED();
    unsigned long long h = ~0ULL;
    ALSK_CUDA(cudaMemcpyAsync(&h, flag.as<void>(), sizeof h, cudaMemcpyDeviceToHost, s));
    ALSK_CUDA(cudaStreamSynchronize(s));
    return h == ~0ULL ? -1 : static_cast<int64_t>(h);
}

}  // namespace alsk
