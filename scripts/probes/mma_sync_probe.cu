// Probe (not part of the library): legacy warp-level mma.sync m16n8k8 tf32 on sm_100a --
// throughput (independent accumulators, W warps per SM) and latency (one dependent chain).
// usage: mma_sync_probe <warps_per_cta> <chains>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <int C>
__global__ void k(int iters, float* sink, long long* cyc) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(0.001f * (threadIdx.x + i));
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.002f * (threadIdx.x + i));
    float d[C][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < C; ++c) mma(d[c], a, b);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int C>
void run(int warps, int iters) {
    int sms = 148;
    float* sink; long long* cyc;
    cudaMalloc(&sink, sizeof(float) * sms * warps * 32);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    k<C><<<sms, warps * 32>>>(iters, sink, cyc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<C><<<sms, warps * 32>>>(iters, sink, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c0; cudaMemcpy(&c0, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    double mmas_per_sm = double(iters) * C * warps;
    double flops = mmas_per_sm * sms * 16 * 8 * 8 * 2;
    printf("chains=%d warps/SM=%d: %.2f cycles per mma per warp (latency if chains=1), SM rate %.3f mma/clk, %.1f TFLOP/s tf32\n",
           C, warps, double(c0) / (double(iters) * C), mmas_per_sm / double(c0), flops / (ms * 1e9));
    cudaFree(sink); cudaFree(cyc);
}
int main() {
    int iters = 20000;
    run<1>(1, iters);
    run<4>(1, iters);
    run<8>(1, iters);
    for (int w : {4, 8, 16, 32}) run<4>(w, iters / 4);
    for (int w : {4, 8, 16}) run<8>(w, iters / 4);
    return 0;
}
