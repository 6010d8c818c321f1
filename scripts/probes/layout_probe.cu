// Bring-up probe (not part of the library): K-major tf32 operand layouts for a K = 8 panel
// (128 rows x 32 bytes). Stages A (128 x 8) in the layout under test, issues one
// tcgen05.mma D = A A^T (M = 128, N = 112; then a second MMA with B starting at row `boff`
// and N = 16 into columns boff..boff+15 of a cleared D), reads TMEM back and compares with
// a double host reference.
//   layout 0: SWIZZLE_128B (1024-byte atoms of 8 rows x 128 B; only the first 32 B used)
//   layout 1: SWIZZLE_NONE, core matrix 8 rows x 16 B, LBO = 128 (K), SBO = 256 (M/N)
//   layout 2: SWIZZLE_NONE with LBO/SBO swapped in the descriptor (to tell them apart)
//   layout 3: SWIZZLE_32B, 256-byte atoms of 8 rows x 32 B, chunk ^= (row >> 2) & 1, SBO = 256
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include "../../paper_1603_03820_b200/csrc/tc_common.cuh"
using namespace alsk::tc;

constexpr int N = 112;

__device__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

__device__ uint32_t offset(int layout, int i, int k) {  // byte offset of (row i, k) in the tile
    const int c = k >> 2, w = (k & 3) * 4;
    switch (layout) {
        case 0: return (i >> 3) * 1024 + (i & 7) * 128 + ((c ^ (i & 7)) << 4) + w;
        case 1: return (i >> 3) * 256 + c * 128 + (i & 7) * 16 + w;
        case 2: return (i >> 3) * 256 + c * 128 + (i & 7) * 16 + w;
        default: return (i >> 3) * 256 + (i & 7) * 32 + ((c ^ ((i >> 2) & 1)) << 4) + w;
    }
}

__global__ void k(const float* A, float* D, float* D2, int layout, int boff) {
    extern __shared__ uint8_t sm[];
    uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc<256>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    for (int idx = threadIdx.x; idx < 16384 / 4; idx += 128) ((float*)base)[idx] = 0.f;
    __syncthreads();
    for (int k8 = 0; k8 < 8; ++k8) *(float*)(base + offset(layout, threadIdx.x, k8)) = A[threadIdx.x * 8 + k8];
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        uint32_t lbo = 16, sbo = 1024, lay = 2;
        if (layout == 1) lbo = 128, sbo = 256, lay = 0;
        if (layout == 2) lbo = 256, sbo = 128, lay = 0;
        if (layout == 3) lbo = 16, sbo = 256, lay = 6;
        const uint32_t sa = smem_u32(base);
        const uint64_t a = desc(sa, lbo, sbo, lay);
        const uint32_t rowstep = layout == 0 ? 1024 : 256;  // bytes per 8-row group
        const uint64_t b2 = desc(sa + (boff / 8) * rowstep, lbo, sbo, lay);
        mma_tf32(tmem, a, a, idesc_tf32(128, N), 0u);
        mma_tf32(tmem + 128, a, b2, idesc_tf32(128, 16), 0u);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const uint32_t lb = (uint32_t)(warp * 32) << 16;
    for (int c = 0; c < N / 16; ++c) {
        float d[16];
        tmem_ld16(tmem + lb + c * 16, d);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * N + c * 16 + j] = d[j];
    }
    {
        float d[16];
        tmem_ld16(tmem + lb + 128, d);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) D2[(warp * 32 + lane) * 16 + j] = d[j];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

static float tf32r(float x) { unsigned u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
    float* A = new float[128 * 8];
    srand(3);
    for (int i = 0; i < 128 * 8; ++i) A[i] = tf32r((float)rand() / RAND_MAX - 0.5f);
    for (int i = N; i < 128; ++i) for (int k = 0; k < 8; ++k) A[i * 8 + k] = tf32r((float)rand() / RAND_MAX - 0.5f);
    float *dA, *dD, *dD2;
    cudaMalloc(&dA, 128 * 8 * 4); cudaMalloc(&dD, 128 * N * 4); cudaMalloc(&dD2, 128 * 16 * 4);
    cudaMemcpy(dA, A, 128 * 8 * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    float* D = new float[128 * N]; float* D2 = new float[128 * 16];
    const int boff = 24;
    for (int layout = 0; layout < 4; ++layout) {
        cudaMemset(dD, 0, 128 * N * 4); cudaMemset(dD2, 0, 128 * 16 * 4);
        k<<<1, 128, 20000>>>(dA, dD, dD2, layout, boff);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("layout %d: kernel %s\n", layout, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(D2, dD2, 128 * 16 * 4, cudaMemcpyDeviceToHost);
        double e1 = 0, e2 = 0, s = 0;
        for (int i = 0; i < 128; ++i) {
            for (int j = 0; j < N; ++j) {
                double r = 0;
                for (int q = 0; q < 8; ++q) r += (double)A[i * 8 + q] * A[j * 8 + q];
                e1 = fmax(e1, fabs(r - D[i * N + j])); s = fmax(s, fabs(r));
            }
            for (int j = 0; j < 16; ++j) {
                double r = 0;
                for (int q = 0; q < 8; ++q) r += (double)A[i * 8 + q] * A[(boff + j) * 8 + q];
                e2 = fmax(e2, fabs(r - D2[i * 16 + j]));
            }
        }
        printf("layout %d: max|D-ref| = %.3e (scale %.3e)   offset-B (row %d, N=16) max err = %.3e\n", layout, e1, s,
               boff, e2);
    }
    return 0;
}
