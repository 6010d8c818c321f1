// Bring-up probe (not part of the library): round-trip latency of a small tcgen05.mma batch
// as the batched solve uses it: thread 0 issues `nmma` MMAs (M = 128, K = 8, tf32, N = n)
// + tcgen05.commit, all 128 threads wait on the mbarrier (spinning try_wait), a named
// barrier, repeat. Reports clocks per round trip with 1 or 4 CTAs per SM, and the same loop
// with the MMA replaced by a plain mbarrier arrive (barrier overhead only).
#include <cstdio>
#include <cstdlib>
#include "../../paper_1603_03820_b200/csrc/tc_common.cuh"
using namespace alsk::tc;

__device__ uint64_t desc0(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((128 >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((256 >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    return d;
}

__global__ void __launch_bounds__(128) k(int iters, int n, int nmma, int mode, long long* out) {
    extern __shared__ uint8_t sm[];
    uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<128>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    for (int i = threadIdx.x; i < 8192 / 4; i += 128) ((float*)base)[i] = 0.001f * (i & 7);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint64_t a = desc0(smem_u32(base)), b = desc0(smem_u32(base + 4096));
    const uint32_t id = idesc_tf32(128, n);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 4) {
            if (threadIdx.x == 0) {
                tc_fence_after();
                for (int q = 0; q < nmma; ++q) mma_tf32(tmem, a, b, id, 1u);
                mma_commit(&bar);
            }
            __syncwarp();
            const long long s0 = clock64();
            const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 120;
            uint32_t r[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "r"(ta) : "memory");
            tmem_ld_wait();
            const long long s1 = clock64();
            if (r[0] == 12345u && r[7] == 7u) out[0] = 1;
            if (threadIdx.x == 32) out[gridDim.x + blockIdx.x] += s1 - s0;
            mbar_wait(&bar, ph);
            ph ^= 1u;
            tc_fence_before();
            named_barrier(1, 128);
            continue;
        }
        if (mode >= 2) {
            const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (it & 7) * 8;
            uint32_t r[8];
            if (mode == 2) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                             : "r"(ta) : "memory");
                tmem_ld_wait();
                if (r[0] == 12345u && r[7] == 7u) out[0] = 1;
            } else {
                for (int q = 0; q < 8; ++q) r[q] = it + q;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta),
                             "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            }
            named_barrier(1, 128);
            continue;
        }
        if (threadIdx.x == 0) {
            tc_fence_after();
            if (mode == 0) {
                for (int q = 0; q < nmma; ++q) mma_tf32(tmem, a, b, id, 1u);
                mma_commit(&bar);
            } else {
                mbar_arrive(&bar);
            }
        }
        mbar_wait(&bar, ph);
        ph ^= 1u;
        tc_fence_before();
        named_barrier(1, 128);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<128>(tmem); }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d;
    cudaMalloc(&d, sizeof(long long) * 8 * sms);
    long long* h = new long long[8 * sms];
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50000);
    const int ns[] = {16, 112};
    for (int cps : {1, 4})
        for (int mode : {4, 3, 2, 1, 0})
            for (int n : ns)
                for (int nmma : {1, 3}) {
                    if (mode >= 1 && mode <= 3 && (n != 16 || nmma != 1)) continue;
                    const int grid = cps * sms;
                    cudaMemset(d, 0, sizeof(long long) * 8 * sms);
                    k<<<grid, 128, 50000>>>(2000, n, nmma, mode, d);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                    cudaMemcpy(h, d, sizeof(long long) * 2 * grid, cudaMemcpyDeviceToHost);
                    double s = 0, s2 = 0;
                    for (int i = 0; i < grid; ++i) s += h[i], s2 += h[grid + i];
                    if (mode == 4) printf("   (ld8 under a running MMA: %.1f clk)\n", s2 / grid / 2000);
                    printf("CTAs/SM %d %-12s N=%3d x%d: %8.1f clk per round trip\n", cps,  mode == 4 ? "mma+ld8" : mode == 3 ? "tmem st8" : mode == 2 ? "tmem ld8" : mode ? "arrive-only" : "mma+commit",
                           n, nmma, s / grid);
                }
    return 0;
}
