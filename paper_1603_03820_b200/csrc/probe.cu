// FP32 FFMA throughput probe: the roofline denominator for the Hermitian (MEASURED_PEAKS.json
// carries HBM and bf16 tensor peaks only). Every thread runs 16 independent FFMA chains with
// register operands (the same 3-register FFMA form the Hermitian inner loop issues).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace alsk {
namespace {
constexpr int kChains = 16;
__global__ void __launch_bounds__(512) ffma_probe_kernel(float* out, int iters, float b, float c) {
    float a[kChains];
#pragma unroll
    for (int j = 0; j < kChains; ++j) a[j] = threadIdx.x * 1e-3f + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int j = 0; j < kChains; ++j) a[j] = fmaf(a[j], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kChains; ++j) s += a[j];
    if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keep the chains live
}
}  // namespace
}  // namespace alsk

extern "C" double alsk_fp32_peak_probe(void) {
    using namespace alsk;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0.0;
    const int sms = num_sms();
    const int blocks = sms * 4, threads = 512, iters = 4096;
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float) * blocks * threads) != cudaSuccess) return 0.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        ffma_probe_kernel<<<blocks, threads>>>(out, iters, 0.99999f, 1e-6f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        count_launch();
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * blocks * threads * double(iters) * 8 * kChains;
        if (ms > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return best;
}
