// Bring-up probe (not part of the library): tcgen05.mma kind::tf32 issue rate from one
// thread, K-major SW128 operands resident in smem (one CTA per SM, 148 CTAs).
// usage: mma_rate_probe <N> <ksteps_per_stage>
#include <cstdio>
#include <cstdlib>
#include "../../paper_1603_03820_b200/csrc/tc_common.cuh"
using namespace alsk::tc;

__global__ void k(int N, int kst, int iters, long long* cyc) {
    extern __shared__ uint8_t sm[];
    uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)base)[i] = 0.001f * (i & 7);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_tf32(128, N);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int kb = 0; kb < kst; ++kb) {
                uint64_t d = sdesc_sw128(smem_u32(base) + (kb & 3) * 32 + (kb >> 2) * 32768, 16, 1024);
                mma_tf32(tmem + (it & 1) * 256, d, d, id, kb > 0);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main(int argc, char** argv) {
    int N = argc > 1 ? atoi(argv[1]) : 224, kst = argc > 2 ? atoi(argv[2]) : 4, iters = 2000;
    long long* d; cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
    k<<<148, 128, 66 * 1024 + 1024>>>(N, kst, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double mmas = double(iters) * kst;
    printf("N=%d kst=%d: %s  %.1f clk/MMA  -> %.1f MAC/clk/SM (tf32 nominal ~1900)\n", N, kst, cudaGetErrorString(e),
           mx / mmas, 128.0 * N * 8 / (mx / mmas));
    return 0;
}
