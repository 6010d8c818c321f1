// Bring-up probe (not part of the library): tcgen05.mma kind::tf32 M=128 N=224 K=8 issue
// rate when every MMA reads a different k-slice of a 4-stage operand ring (no reuse), for
// K-major SWIZZLE_128B (k-slices 32 B apart inside 128 B rows) vs SWIZZLE_32B (one 32 B
// row per k-slice) layouts, optionally with 8 warps hammering shared memory meanwhile.
// usage: mma_rate2_probe <layout 128|32> <noise 0|1>
#include <cstdio>
#include <cstdlib>
#include "../../paper_1603_03820_b200/csrc/tc_common.cuh"
using namespace alsk::tc;
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__global__ void k(int layout, int noise, int iters, long long* cyc, float* sink) {
    extern __shared__ uint8_t sm[];
    uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<256>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    for (int i = threadIdx.x; i < 4 * 32768 / 4; i += blockDim.x) ((float*)base)[i] = 0.001f * (i & 7);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_tf32(128, 224);
        for (int it = 0; it < iters; ++it) {
            const uint32_t stage = smem_u32(base) + (it & 3) * 32768;
            for (int kb = 0; kb < 4; ++kb) {
                uint64_t d;
                if (layout == 128) d = sdesc(stage + kb * 32, 16, 1024, 2);       // SW128: 8 rows x 128 B atoms
                else d = sdesc(stage + kb * 8192, 16, 256, 6);                     // SW32: 8 rows x 32 B atoms
                mma_tf32(tmem, d, d, id, kb > 0);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    } else if (noise && warp >= 2) {
        float acc = 0.f;
        uint8_t* nb = base + 4 * 32768;
        for (int it = 0; it < iters * 8; ++it) {
            float4 v = *reinterpret_cast<float4*>(nb + ((threadIdx.x * 16 + it * 512) & 16383));
            acc += v.x;
            *reinterpret_cast<float4*>(nb + ((threadIdx.x * 16 + it * 1024 + 256) & 16383)) = make_float4(acc, 0, 0, 0);
        }
        if (acc == 1.5f) sink[0] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}
int main(int argc, char** argv) {
    const int layout = atoi(argv[1]), noise = atoi(argv[2]), iters = 2000;
    long long* d; float* sink; cudaMalloc(&d, 148 * 8); cudaMalloc(&sink, 4);
    const int smem = 4 * 32768 + 16384 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 320, smem>>>(layout, noise, iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("layout SW%d noise %d: %s  %.1f clk/MMA (N=224 ideal 112)\n", layout, noise, cudaGetErrorString(e), mx / (iters * 4.0));
    return 0;
}
