// Bring-up probe (not part of the library): gathered-row copy rate into shared memory.
// Each CTA (one per SM) repeatedly stages 32 random rows of 400 B (f=100 floats) from a
// table of `rows` rows into a 4-deep ring, with W issuing warps, by one of:
//  0: cp.async 16 B, lane = rating (25 instructions per chunk)
//  1: cp.async 16 B, lane = 16-byte piece (32 instructions per chunk)
//  2: cp.async.bulk 400 B per rating (one instruction, 32 lanes)
//  3: LDG.128 + STS.128, lane = piece (8 rows in flight per warp)
// usage: gather_probe <mode> <warps> <rows>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../../paper_1603_03820_b200/csrc/tc_common.cuh"
using namespace alsk::tc;

constexpr int ROWB = 400, KC = 32, CH = 8 * 1664;
constexpr int STMAX = 12;

__global__ void k(const __grid_constant__ CUtensorMap tmap, const float* tab, const int* idx, int nidx, int mode, int chunks, long long* cyc, float* sink, int ST, int nrows, int seqrows, int spin) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[STMAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) mbar_init(&full[s], (mode == 2 || mode >= 4) ? 1 : 32 * W);
        fence_barrier_init();
    }
    __syncthreads();
    long long t0 = clock64();
    float acc = 0.f;
    for (int c = 0; c < chunks; ++c) {
        const int s = c % ST;
        uint8_t* st = sm + s * CH;
        if (c >= ST) {  // wait for the chunk issued ST ago, consume one value
            if (spin) {
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(done) : "r"(smem_u32(&full[s])), "r"(((c / ST) - 1) & 1) : "memory");
            } else mbar_wait(&full[s], ((c / ST) - 1) & 1);
            acc += *reinterpret_cast<float*>(st + lane * 4);
            __syncthreads();
        }
        const int base = (blockIdx.x * 977 + c * 32) % (nidx - 32);
        if (mode == 0) {
            for (int r = warp; r < 1; r += W) {}
            // each warp takes ratings lane (all 32) for its share of pieces
            const int v = seqrows ? (int)((unsigned)(base + lane) % (unsigned)nrows) : (int)(((unsigned)(base + lane) * 2654435761u) % (unsigned)nrows);
            for (int p = warp; p < 25; p += W)
                cp_async16(smem_u32(st + lane * ROWB + p * 16), tab + (int64_t)v * 100 + 4 * p);
            cp_async_arrive_noinc(&full[s]);
        } else if (mode == 1) {
            const int v = seqrows ? (int)((unsigned)(base + lane) % (unsigned)nrows) : (int)(((unsigned)(base + lane) * 2654435761u) % (unsigned)nrows);
            for (int i = warp; i < 32; i += W) {
                const int vi = __shfl_sync(0xffffffffu, v, i);
                if (lane < 25) cp_async16(smem_u32(st + i * ROWB + lane * 16), tab + (int64_t)vi * 100 + 4 * lane);
            }
            cp_async_arrive_noinc(&full[s]);
        } else if (mode == 2) {
            if (warp == 0) {
                const int v = seqrows ? (int)((unsigned)(base + lane) % (unsigned)nrows) : (int)(((unsigned)(base + lane) * 2654435761u) % (unsigned)nrows);
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(32 * ROWB));
                __syncwarp();
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(st + lane * ROWB)), "l"(tab + (int64_t)v * 100), "r"(ROWB), "r"(smem_u32(&full[s]))
                             : "memory");
            }
        } else if (mode == 5) {
            if (threadIdx.x == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(32 * ROWB));
                const int64_t off = ((int64_t)blockIdx.x * chunks + c) % ((int64_t)nrows - 64) * 100;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(st)), "l"(tab + (off & ~31)), "r"(32 * ROWB), "r"(smem_u32(&full[s]))
                             : "memory");
            }
        } else if (mode == 4) {
            if (warp == 0) {
                const int v = seqrows ? (int)((unsigned)(base + lane) % (unsigned)nrows) : (int)(((unsigned)(base + lane) * 2654435761u) % (unsigned)nrows);
                const int q0 = __shfl_sync(0xffffffffu, v, (lane & 7) * 4 + 0), q1 = __shfl_sync(0xffffffffu, v, (lane & 7) * 4 + 1);
                const int q2 = __shfl_sync(0xffffffffu, v, (lane & 7) * 4 + 2), q3 = __shfl_sync(0xffffffffu, v, (lane & 7) * 4 + 3);
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(32 * ROWB));
                __syncwarp();
                if (lane < 8)
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(st + lane * 1664)),
                                 "l"((uint64_t)&tmap), "r"(0), "r"(q0), "r"(q1), "r"(q2), "r"(q3), "r"(smem_u32(&full[s])) : "memory");
            }
        } else {
            const int v = seqrows ? (int)((unsigned)(base + lane) % (unsigned)nrows) : (int)(((unsigned)(base + lane) * 2654435761u) % (unsigned)nrows);
            for (int i0 = warp * 8; i0 < 32; i0 += W * 8) {
                float4 x[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int vi = __shfl_sync(0xffffffffu, v, i0 + j);
                    x[j] = lane < 25 ? ldg_nc_f4(tab + (int64_t)vi * 100 + 4 * lane) : make_float4(0, 0, 0, 0);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (lane < 25) *reinterpret_cast<float4*>(st + (i0 + j) * ROWB + lane * 16) = x[j];
            }
            __syncwarp();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        }
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    if (acc == 1234.5f) sink[0] = acc;
}

int main(int argc, char** argv) {
    const int mode = atoi(argv[1]), W = atoi(argv[2]);
    const long rows = atol(argv[3]);
    const int ST = argc > 4 ? atoi(argv[4]) : 4;
    const int nidx = 1 << 22, chunks = 4000;
    float* tab; int* idx; long long* cyc; float* sink;
    cudaMalloc(&tab, rows * 400); cudaMemset(tab, 0, rows * 400);
    cudaMalloc(&idx, nidx * 4); cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 4);
    int* h = (int*)malloc(nidx * 4); srand(1);
    for (int i = 0; i < nidx; ++i) h[i] = (int)(((long)rand() * 7919L) % rows);
    cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[2] = {100, (cuuint64_t)rows}, str[1] = {400};
    cuuint32_t box[2] = {100, 1}, es[2] = {1, 1};
    CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode failed %d\n", (int)r);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH);
    for (int rep = 0; rep < 2; ++rep) k<<<148, 32 * W, ST * CH>>>(m, tab, idx, nidx, mode, chunks, cyc, sink, ST, (int)rows, argc > 5 ? atoi(argv[5]) : 0, argc > 6 ? atoi(argv[6]) : 0);
    cudaError_t e = cudaDeviceSynchronize();
    long long hc[148]; cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = hc[i] > mx ? hc[i] : mx;
    printf("mode %d warps %d st %d rows %ld: %s  %.1f clk/rating  %.0f GB/s chip\n", mode, W, ST, rows, cudaGetErrorString(e),
           mx / (chunks * 32.0), 400.0 * chunks * 32 * 148 / (mx / 1.965e9) / 1e9);
    return 0;
}
