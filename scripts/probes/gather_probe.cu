// Bring-up probe (not part of the library): gathered-row copy rate into shared memory.
// NOTE (round 2): its ~46-50 cycles per row for every mechanism was an artifact of this
// harness (one CTA per SM, one mbarrier and a CTA barrier per chunk); l2bw_probe.cu
// measures the same copies with many warps: 17 B/clk per SM for lane = rating cp.async,
// 38-45 for lane = piece cp.async, 67 for TMA tile::gather4.
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

__global__ void k(const __grid_constant__ CUtensorMap tmap, const float* tab, const int* idx, int nidx, int mode, int chunks, long long* cyc, float* sink, int ST, int nrows, int seqrows, int spin, int nbulk) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[STMAX];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) mbar_init(&full[s], mode == 6 ? 32 * W + 1 : (mode == 2 || mode >= 4) ? 1 : 32 * W);
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
        } else if (mode == 6) {
            // mixed: rows [0, nbulk) by TMA bulk copies (one per row, warp 0), the rest by
            // cp.async 16 B with lane = rating
            const int v = (int)(((unsigned)(base + lane) * 2654435761u) % (unsigned)nrows);
            if (warp == 0) {
                if (lane == 0 && nbulk > 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(nbulk * ROWB));
                else if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
                __syncwarp();
                if (lane < nbulk)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     smem_u32(st + lane * ROWB)), "l"(tab + (int64_t)v * 100), "r"(ROWB), "r"(smem_u32(&full[s]))
                                 : "memory");
            }
            if (lane >= nbulk)
                for (int p = warp; p < 25; p += W)
                    cp_async16(smem_u32(st + lane * ROWB + p * 16), tab + (int64_t)v * 100 + 4 * p);
            cp_async_arrive_noinc(&full[s]);
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

// mode 7: LDG.128 gathers straight into registers, lane = rating, warp w loads pieces
// w, w+W, ... of every row, DEP chunks in flight per warp; no shared memory at all.
template <int NP, int DEP>
__global__ void k7(const float* tab, int nrows, int chunks, long long* cyc, float* sink) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    float4 buf[DEP][NP];
    float acc = 0.f;
    long long t0 = clock64();
    auto issue = [&](int c, float4 (&b)[NP]) {
        const int base = (blockIdx.x * 977 + c * 32);
        const int v = (int)(((unsigned)(base + lane) * 2654435761u) % (unsigned)nrows);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int p = warp + q * W;
            b[q] = p < 25 ? ldg_nc_f4(tab + (int64_t)v * 100 + 4 * p) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
#pragma unroll
    for (int d = 0; d < DEP; ++d) issue(d, buf[d]);
    for (int c0 = 0; c0 < chunks; c0 += DEP) {
#pragma unroll
        for (int d = 0; d < DEP; ++d) {
#pragma unroll
            for (int q = 0; q < NP; ++q) acc += buf[d][q].x + buf[d][q].y + buf[d][q].z + buf[d][q].w;
            issue(c0 + d + DEP, buf[d]);
        }
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    if (acc == 1234.5f) sink[0] = acc;
}

// mode 8: like mode 7, plus every gathered piece is written into a 4-deep rating-major
// staging ring in shared memory with st.async (completion counted as transaction bytes on
// the stage's mbarrier, no release fence in the loading warps); warp 0 lane 0 consumes
// (waits for the stage and re-arms it). Stage s of chunk c must have been consumed before
// chunk c+4 writes it: the writers wait on an `empty` barrier (acquire only).
__device__ __forceinline__ uint32_t mapa_self(uint32_t a) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
    return r;
}
template <int NP, int DEP>
__global__ void __cluster_dims__(1, 1, 1) k8(const float* tab, int nrows, int chunks, long long* cyc, float* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[4], empty[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 4; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const uint32_t stage_bytes = 32 * 25 * 16;
    float4 buf[DEP][NP];
    float acc = 0.f;
    long long t0 = clock64();
    auto issue = [&](int c, float4 (&b)[NP]) {
        const int base = (blockIdx.x * 977 + c * 32);
        const int v = (int)(((unsigned)(base + lane) * 2654435761u) % (unsigned)nrows);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int p = warp + q * W;
            b[q] = p < 25 ? ldg_nc_f4(tab + (int64_t)v * 100 + 4 * p) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
#pragma unroll
    for (int d = 0; d < DEP; ++d) issue(d, buf[d]);
    for (int c0 = 0; c0 < chunks; c0 += DEP) {
#pragma unroll
        for (int d = 0; d < DEP; ++d) {
            const int c = c0 + d, s = c & 3;
            if (c >= 4) mbar_wait(&empty[s], ((c >> 2) - 1) & 1);
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(stage_bytes) : "memory");
            uint8_t* st = sm + s * 32 * 400;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const int p = warp + q * W;
                if (p < 25)
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                                     mapa_self(smem_u32(st + lane * 400 + p * 16))), "f"(buf[d][q].x), "f"(buf[d][q].y), "f"(buf[d][q].z),
                                 "f"(buf[d][q].w), "r"(mapa_self(smem_u32(&full[s]))) : "memory");
            }
            issue(c + DEP, buf[d]);
            if (threadIdx.x == 0) {  // consumer: wait for the stage, read one value, free it
                mbar_wait(&full[s], (c >> 2) & 1);
                acc += *reinterpret_cast<float*>(st);
                mbar_arrive(&empty[s]);
            }
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
    if (mode == 8) {
        cudaFuncSetAttribute(k8<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 400);
        cudaFuncSetAttribute(k8<4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 400);
        for (int rep = 0; rep < 2; ++rep) {
            if (W == 8 && ST == 2) k8<4, 2><<<148, 256, 4 * 32 * 400>>>(tab, (int)rows, chunks, cyc, sink);
            else if (W == 8 && ST == 3) k8<4, 3><<<148, 256, 4 * 32 * 400>>>(tab, (int)rows, chunks, cyc, sink);
            else { printf("unsupported W/ST for mode 8\n"); return 1; }
        }
    } else if (mode == 7) {
        for (int rep = 0; rep < 2; ++rep) {
            if (W == 8 && ST == 2) k7<4, 2><<<148, 256>>>(tab, (int)rows, chunks, cyc, sink);
            else if (W == 8 && ST == 3) k7<4, 3><<<148, 256>>>(tab, (int)rows, chunks, cyc, sink);
            else if (W == 8 && ST == 4) k7<4, 4><<<148, 256>>>(tab, (int)rows, chunks, cyc, sink);
            else if (W == 13 && ST == 4) k7<2, 4><<<148, 416>>>(tab, (int)rows, chunks, cyc, sink);
            else if (W == 13 && ST == 6) k7<2, 6><<<148, 416>>>(tab, (int)rows, chunks, cyc, sink);
            else if (W == 16 && ST == 4) k7<2, 4><<<148, 512>>>(tab, (int)rows, chunks, cyc, sink);
            else { printf("unsupported W/ST for mode 7\n"); return 1; }
        }
    } else
    for (int rep = 0; rep < 2; ++rep) k<<<148, 32 * W, ST * CH>>>(m, tab, idx, nidx, mode, chunks, cyc, sink, ST, (int)rows, argc > 5 ? atoi(argv[5]) : 0, argc > 6 ? atoi(argv[6]) : 0, argc > 7 ? atoi(argv[7]) : 0);
    cudaError_t e = cudaDeviceSynchronize();
    long long hc[148]; cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = hc[i] > mx ? hc[i] : mx;
    printf("nbulk %d mode %d warps %d st %d rows %ld: %s  %.1f clk/rating  %.0f GB/s chip\n", argc > 7 ? atoi(argv[7]) : 0,
           mode, W, ST, rows, cudaGetErrorString(e), mx / (chunks * 32.0), 400.0 * chunks * 32 * 148 / (mx / 1.965e9) / 1e9);
    return 0;
}
