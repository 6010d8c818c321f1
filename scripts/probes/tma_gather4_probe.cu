// Bring-up probe (not part of the library): does tile::gather4 with a 128B-swizzled box
// land at a 512-byte (not 1024-byte) aligned destination, and what bytes does it count?
// usage: tma_gather4_probe <dst_offset_bytes> <cols>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap map, int off, float* out, unsigned* tx) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 512; i += blockDim.x) ((float*)base)[i] = -1.f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(512));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(base + off)),
            "l"((uint64_t)&map), "r"(0), "r"(3), "r"(7), "r"(11), "r"(60), "r"(su32(&bar))
            : "memory");
        uint32_t done = 0;
        long long t0 = clock64();
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(su32(&bar)));
            if (clock64() - t0 > 4000000000ll) { *tx = 0xdead; break; }
        }
        if (done) *tx = 1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = ((float*)base)[i];
}

int main(int argc, char** argv) {
    int off = argc > 1 ? atoi(argv[1]) : 0, cols = argc > 2 ? atoi(argv[2]) : 32;
    const int rows = 64;
    float* h = (float*)malloc(rows * cols * 4);
    for (int r = 0; r < rows; ++r) for (int c = 0; c < cols; ++c) h[r * cols + c] = r * 1000 + c;
    float *g, *out; unsigned* tx;
    cudaMalloc(&g, rows * cols * 4); cudaMalloc(&out, 2048); cudaMalloc(&tx, 4);
    cudaMemcpy(g, h, rows * cols * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
    CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode=%d off=%d cols=%d\n", (int)r, off, cols);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096);
    k<<<1, 128, 4096>>>(m, off, out, tx);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e) return 1;
    float o[512]; unsigned t;
    cudaMemcpy(o, out, 2048, cudaMemcpyDeviceToHost); cudaMemcpy(&t, tx, 4, cudaMemcpyDeviceToHost);
    printf("tx-done=%x\n", t);
    for (int row = 0; row < 8; ++row) {
        printf("row %d:", row);
        for (int ch = 0; ch < 8; ++ch) printf(" [%g]", o[row * 32 + ch * 4]);
        printf("\n");
    }
    return 0;
}
