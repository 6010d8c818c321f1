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

// Throughput of the Hermitian register-blocked inner loop alone (no gather, no barriers):
// 96-thread CTAs, 8x8 tiles of a 13x13 lower-triangular tile set, operands from a shared
// buffer of 32 staged rows. Separates the loop's issue efficiency from the pipeline.
// variant 0: FFMA, unroll 2 (the v2 kernel's loop); 1: FFMA, operands software-pipelined;
// 2: FFMA2 (fma.rn.f32x2, a_i broadcast), unroll 2; 3: FFMA2 + software pipelining;
// 4: FFMA2 dependent-chain peak (like the FFMA peak probe).
namespace alsk {
namespace {
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a, float b0, float b1) {
    unsigned long long c = (static_cast<unsigned long long>(__float_as_uint(d1)) << 32) | __float_as_uint(d0);
    const unsigned long long bb = (static_cast<unsigned long long>(__float_as_uint(b1)) << 32) | __float_as_uint(b0);
    const unsigned long long aa = (static_cast<unsigned long long>(__float_as_uint(a)) << 32) | __float_as_uint(a);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(aa), "l"(bb));
    d0 = __uint_as_float(static_cast<unsigned>(c));
    d1 = __uint_as_float(static_cast<unsigned>(c >> 32));
}

template <int V>
__global__ void __launch_bounds__(96, 4) herm_loop_probe_kernel(float* out, int reps) {
    __shared__ __align__(16) float buf[33 * 104];
    for (int e = threadIdx.x; e < 33 * 104; e += 96) buf[e] = 1e-3f * (e % 97);
    __syncthreads();
    int b = 0, t = threadIdx.x < 91 ? threadIdx.x : 0;
    while ((b + 1) * (b + 2) / 2 <= t) ++b;
    const int ia = 8 * b, jb = 8 * (t - b * (b + 1) / 2);
    float acc[8][8] = {};
    if (V == 4) {
        float a = threadIdx.x * 1e-3f;
        for (int r = 0; r < reps * 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; j += 2) ffma2(acc[i][j], acc[i][j + 1], a, 0.999f, 0.998f);
    } else {
        for (int r = 0; r < reps; ++r) {
            if (V == 0 || V == 2) {
#pragma unroll 2
                for (int kk = 0; kk < 32; ++kk) {
                    const float* trow = buf + kk * 104;
                    const float4 a0 = *reinterpret_cast<const float4*>(trow + ia);
                    const float4 a1 = *reinterpret_cast<const float4*>(trow + ia + 4);
                    const float4 b0 = *reinterpret_cast<const float4*>(trow + jb);
                    const float4 b1 = *reinterpret_cast<const float4*>(trow + jb + 4);
                    const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (V == 0) {
#pragma unroll
                            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 8; j += 2) ffma2(acc[i][j], acc[i][j + 1], a[i], bb[j], bb[j + 1]);
                        }
                    }
                }
            } else {
                float4 a0 = *reinterpret_cast<const float4*>(buf + ia), a1 = *reinterpret_cast<const float4*>(buf + ia + 4);
                float4 b0 = *reinterpret_cast<const float4*>(buf + jb), b1 = *reinterpret_cast<const float4*>(buf + jb + 4);
#pragma unroll 2
                for (int kk = 0; kk < 32; ++kk) {
                    const float* nrow = buf + (kk + 1) * 104;
                    const float4 na0 = *reinterpret_cast<const float4*>(nrow + ia);
                    const float4 na1 = *reinterpret_cast<const float4*>(nrow + ia + 4);
                    const float4 nb0 = *reinterpret_cast<const float4*>(nrow + jb);
                    const float4 nb1 = *reinterpret_cast<const float4*>(nrow + jb + 4);
                    const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (V == 1) {
#pragma unroll
                            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 8; j += 2) ffma2(acc[i][j], acc[i][j + 1], a[i], bb[j], bb[j + 1]);
                        }
                    }
                    a0 = na0; a1 = na1; b0 = nb0; b1 = nb1;
                }
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j];
    if (s == 1234.5f) out[blockIdx.x] = s;
}
}  // namespace
}  // namespace alsk

extern "C" double alsk_herm_loop_probe(int ctas_per_sm, int variant) {
    using namespace alsk;
    const int blocks = num_sms() * ctas_per_sm, reps = 2000;
    float* out = nullptr;
    if (cudaMalloc(&out, sizeof(float) * blocks) != cudaSuccess) return 0.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        switch (variant) {
            case 0: herm_loop_probe_kernel<0><<<blocks, 96>>>(out, reps); break;
            case 1: herm_loop_probe_kernel<1><<<blocks, 96>>>(out, reps); break;
            case 2: herm_loop_probe_kernel<2><<<blocks, 96>>>(out, reps); break;
            case 3: herm_loop_probe_kernel<3><<<blocks, 96>>>(out, reps); break;
            default: herm_loop_probe_kernel<4><<<blocks, 96>>>(out, reps); break;
        }
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) return -1.0;
        count_launch();
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        // useful FMAs: 91 tiles x 64 per k-step (the 5 idle threads do not count);
        // variant 4 counts all 96 threads x 64 x 16 per rep
        const double flops = variant == 4 ? 2.0 * blocks * 96.0 * 64.0 * 16.0 * reps
                                          : 2.0 * blocks * 91.0 * 64.0 * 32.0 * reps;
        if (ms > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return best;
}
