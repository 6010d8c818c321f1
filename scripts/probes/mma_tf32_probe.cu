// Bring-up probe (not part of the library): one CTA stages a K x 128 tf32 block H (and L)
// in the 128B-swizzled MN-major layout of tc_common.cuh, issues K/8 x {H^T H, H^T L}
// tcgen05.mma (M=128, N=112), reads TMEM back, and compares with a double host reference.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../../paper_1603_03820_b200/csrc/tc_common.cuh"
using namespace alsk::tc;

constexpr int K = 32, N = 112;
__global__ void k(const float* H, const float* L, float* D0, float* D1, int trunc_mode, uint32_t idv, int* nzc) {
    extern __shared__ uint8_t sm[];
    uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    uint8_t* Hs = base; uint8_t* Ls = base + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    const bool kmaj = (idv >> 15 & 3) == 0;
    if (kmaj) {
        for (int idx = threadIdx.x; idx < K * 128; idx += 128) {
            const int kk = idx / 128, i = idx % 128;
            const int off = (i / 8) * 1024 + (i % 8) * 128 + (((kk / 4) ^ (i % 8)) * 16) + (kk % 4) * 4;
            *(float*)(Hs + off) = H[kk * 128 + i];
            *(float*)(Ls + off) = L[kk * 128 + i];
        }
    } else
    for (int idx = threadIdx.x; idx < K * 32; idx += 128) {
        const int kk = idx / 32, c16 = idx % 32;
        float4 h = *(const float4*)(H + kk * 128 + 4 * c16), l = *(const float4*)(L + kk * 128 + 4 * c16);
        *(float4*)(Hs + sw128_offset<4>(kk, c16)) = h;
        *(float4*)(Ls + sw128_offset<4>(kk, c16)) = l;
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    {  // TMEM store/load round trip in columns 256..271
        float v[16];
        const uint32_t lb0 = (uint32_t)(warp * 32) << 16;
        uint32_t r[16];
        for (int j = 0; j < 16; ++j) r[j] = __float_as_uint((float)((warp * 32 + lane) * 1000 + j));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     :: "r"(tmem + lb0 + 256), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tmem_ld16(tmem + lb0 + 256, v);
        tmem_ld_wait();
        if (lane == 5 && warp == 1) printf("tmem base %08x: st/ld lane 37 col 3 -> %g (want 37003)\n", tmem, v[3]);
    }
    if (threadIdx.x == 0) {
        const uint32_t id = idv;
        for (int kb = 0; kb < K / 8; ++kb) {
            uint64_t a = kmaj ? sdesc_sw128(smem_u32(Hs) + kb * 32, 16, 1024) : sdesc_sw128(smem_u32(Hs) + kb * 4096, 1024, 4096);
            uint64_t b = kmaj ? sdesc_sw128(smem_u32(Ls) + kb * 32, 16, 1024) : sdesc_sw128(smem_u32(Ls) + kb * 4096, 1024, 4096);
            mma_tf32(tmem, a, a, id, kb > 0);
            mma_tf32(tmem + 128, a, b, id, kb > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (trunc_mode == 7) { long long t0 = clock64(); while (clock64() - t0 < 20000000) {} }
    const uint32_t lb = (uint32_t)(warp * 32) << 16;
    int nz = 0;
    for (int c = 0; c < 32; ++c) { float t[16]; tmem_ld16(tmem + lb + c * 16, t); tmem_ld_wait(); for (int j = 0; j < 16; ++j) nz += (t[j] != 0.f); }
    atomicAdd(nzc, nz);
    for (int c = 0; c < N / 16; ++c) {
        float d0[16], d1[16];
        tmem_ld16(tmem + lb + c * 16, d0);
        tmem_ld16(tmem + lb + 128 + c * 16, d1);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) {
            D0[(warp * 32 + lane) * N + c * 16 + j] = d0[j];
            D1[(warp * 32 + lane) * N + c * 16 + j] = d1[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

static float tf32r(float x) { unsigned u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }
static float tf32t(float x) { unsigned u; memcpy(&u, &x, 4); u &= 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }

int main(int argc, char** argv) {
    const int raw0 = argc > 1 ? atoi(argv[1]) : 0; const int raw = raw0 == 1;  // 1: feed raw fp32 H (tests hw truncation vs rounding)
    float *H = new float[K * 128], *L = new float[K * 128];
    srand(7);
    for (int i = 0; i < K * 128; ++i) {
        float x = (float)rand() / RAND_MAX;
        H[i] = raw ? x : tf32r(x);
        L[i] = tf32r(((float)rand() / RAND_MAX - 0.5f) * 1e-3f);
    }
    float *dH, *dL, *dD0, *dD1; int* nzc; cudaMalloc(&nzc, 4); cudaMemset(nzc, 0, 4);
    uint32_t idv = idesc_tf32_mn(128, N);
    const int var = argc > 2 ? atoi(argv[2]) : 0;
    if (var == 1) idv = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((N >> 3) << 17) | ((128 >> 4) << 23);
    if (var == 3) idv = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
    if (var == 2) idv = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);  // K-major flags
    printf("variant %d idesc=%08x\n", var, idv);
    cudaMalloc(&dH, K * 512); cudaMalloc(&dL, K * 512); cudaMalloc(&dD0, 128 * N * 4); cudaMalloc(&dD1, 128 * N * 4);
    cudaMemcpy(dH, H, K * 512, cudaMemcpyHostToDevice); cudaMemcpy(dL, L, K * 512, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    k<<<1, 128, 40000>>>(dH, dL, dD0, dD1, raw0, idv, nzc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e) return 1;
    int hnz = 0; cudaMemcpy(&hnz, nzc, 4, cudaMemcpyDeviceToHost); printf("nonzero TMEM words: %d of %d\n", hnz, 128 * 512);
    float* D0 = new float[128 * N]; float* D1 = new float[128 * N];
    cudaMemcpy(D0, dD0, 128 * N * 4, cudaMemcpyDeviceToHost); cudaMemcpy(D1, dD1, 128 * N * 4, cudaMemcpyDeviceToHost);
    for (int mode = 0; mode < 3; ++mode) {  // 0: exact operands, 1: truncated H, 2: rounded H
        double e0 = 0, e1 = 0, s0 = 0;
        for (int i = 0; i < 128; ++i) for (int j = 0; j < N; ++j) {
            double r0 = 0, r1 = 0;
            for (int kk = 0; kk < K; ++kk) {
                auto hv = [&](int f) { float v = H[kk * 128 + f]; return mode == 1 ? tf32t(v) : mode == 2 ? tf32r(v) : v; };
                r0 += (double)hv(i) * hv(j);
                r1 += (double)hv(i) * L[kk * 128 + j];
            }
            e0 = fmax(e0, fabs(r0 - D0[i * N + j])); e1 = fmax(e1, fabs(r1 - D1[i * N + j])); s0 = fmax(s0, fabs(r0));
        }
        printf("raw=%d ref-mode=%d  max|D0-ref|=%.3e (scale %.3e)  max|D1-ref|=%.3e\n", raw, mode, e0, s0, e1);
    }
    printf("D0[0][0..3] = %g %g %g %g ; D0[5][7]=%g D0[7][5]=%g\n", D0[0], D0[1], D0[2], D0[3], D0[5 * N + 7], D0[7 * N + 5]);
    return 0;
}
