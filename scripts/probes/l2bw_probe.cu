// Bring-up probe (not part of the library): L2 -> SM bandwidth with many warps per SM.
// A 17,770 x 100 float table (7.1 MB, L2-resident, the Netflix Theta) is read by every SM:
//  mode 0: streaming LDG.128 over the table (coalesced), U loads in flight per thread
//  mode 1: random 400-byte rows, a warp per row (25 lanes x 16 B), U rows in flight per warp
//  mode 2: the same rows by cp.async.cg 16 B into a per-warp shared ring (L2 only)
//  mode 3: the same with cp.async.ca (L1-allocating)
//  mode 4: lane = row (32 rows per instruction, 25 instructions per 32 rows), cp.async.ca,
//          stride 104 floats, double-buffered per warp with wait_group (tc_update's loader pattern)
//  mode 5: mode 3 with completion on a per-warp mbarrier (cp.async.mbarrier.arrive.noinc)
//  mode 6: mode 4 with completion on a per-warp mbarrier
//  mode 7: TMA tile::gather4 (4 rows per instruction, lane 0 of each warp issues 8 per 32 rows),
//          double-buffered per warp on mbarrier transaction counts
// Prints bytes per clock per SM and chip TB/s. usage: l2bw_probe <mode> <threads/CTA> <CTAs/SM>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

constexpr int ROWS = 17770, F = 100, U = 4, ITERS = 2048;

__device__ __forceinline__ unsigned hashu(unsigned x) { return x * 2654435761u; }

__global__ void k(const __grid_constant__ CUtensorMap tmap, const float4* __restrict__ tab, int mode, float* sink, long long* cyc) {
    extern __shared__ __align__(16) float4 ring[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
    const unsigned gw = blockIdx.x * W + warp;
    float acc = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    if (mode == 0) {
        const int n4 = ROWS * F / 4;
        unsigned i = (blockIdx.x * blockDim.x + threadIdx.x) * 7u;
        for (int it = 0; it < ITERS; ++it) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcg(tab + (i + u * 32u * 1024u) % n4);
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
            i += blockDim.x * U * 13u;
        }
    } else if (mode == 1) {
        for (int it = 0; it < ITERS; ++it) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned r = hashu(gw * 131071u + it * U + u) % ROWS;
                v[u] = lane < 25 ? __ldcg(tab + r * 25 + lane) : make_float4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
        }
    } else if (mode == 7) {
        float* my = reinterpret_cast<float*>(ring) + warp * (2 * 8 * 416);  // 4-row groups padded to 1664 B
        __shared__ uint64_t bar7[32][2];
        if (lane == 0) {
            for (int b = 0; b < 2; ++b)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar7[warp][b])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        __syncwarp();
        for (int it = 0; it < ITERS / 8; ++it) {
            const int slot = it & 1;
            const unsigned r = hashu(gw * 131071u + it * 32 + lane) % ROWS;
            const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar7[warp][slot]));
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(32 * 400) : "memory");
            __syncwarp();
            const int g = lane & 7;
            const unsigned q0 = __shfl_sync(0xffffffffu, r, g * 4), q1 = __shfl_sync(0xffffffffu, r, g * 4 + 1);
            const unsigned q2 = __shfl_sync(0xffffffffu, r, g * 4 + 2), q3 = __shfl_sync(0xffffffffu, r, g * 4 + 3);
            if (lane < 8) {
                const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(my + (slot * 8 + g) * 416));
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"((uint64_t)&tmap), "r"(0), "r"(q0), "r"(q1),
                             "r"(q2), "r"(q3), "r"(b) : "memory");
            }
            if (it > 0) {
                const unsigned pb = static_cast<unsigned>(__cvta_generic_to_shared(&bar7[warp][slot ^ 1]));
                const unsigned par = ((it - 1) >> 1) & 1;
                asm volatile("{ .reg .pred p; W7: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W7; }" ::"r"(pb), "r"(par) : "memory");
            }
            acc += my[((slot ^ 1) * 8 + (lane >> 2)) * 416 + (lane & 3) * 100];
        }
        {
            const int it = ITERS / 8;
            const unsigned pb = static_cast<unsigned>(__cvta_generic_to_shared(&bar7[warp][(it - 1) & 1]));
            const unsigned par = ((it - 1) >> 1) & 1;
            asm volatile("{ .reg .pred p; W8: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W8; }" ::"r"(pb), "r"(par) : "memory");
        }
    } else if (mode == 4 || mode == 6) {
        float* my = reinterpret_cast<float*>(ring) + warp * (2 * 32 * 104);
        __shared__ uint64_t bar[32][2];
        if (mode == 6 && lane == 0) {
            for (int b = 0; b < 2; ++b)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[warp][b])), "r"(32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        __syncwarp();
        for (int it = 0; it < ITERS / 8; ++it) {  // 32 rows per round = 8 rounds of U=4 rows
            const int slot = it & 1;
            const unsigned r = hashu(gw * 131071u + it * 32 + lane) % ROWS;
            const unsigned dst0 = static_cast<unsigned>(__cvta_generic_to_shared(my + (slot * 32 + lane) * 104));
            for (int c = 0; c < 25; ++c)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst0 + c * 16), "l"(tab + r * 25 + c));
            if (mode == 4) {
                asm volatile("cp.async.commit_group;");
                asm volatile("cp.async.wait_group 1;");
            } else {
                const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[warp][slot]));
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(b));
                if (it > 0) {
                    const unsigned pb = static_cast<unsigned>(__cvta_generic_to_shared(&bar[warp][slot ^ 1]));
                    const unsigned par = ((it - 1) >> 1) & 1;
                    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(pb), "r"(par) : "memory");
                }
            }
            __syncwarp();
            acc += my[((slot ^ 1) * 32 + lane) * 104];
        }
        if (mode == 4) asm volatile("cp.async.wait_group 0;");
    } else {
        float4* my = ring + warp * (U * 2 * 32);
        __shared__ uint64_t bar5[32][2];
        if (mode == 5 && lane == 0) {
            for (int b = 0; b < 2; ++b)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar5[warp][b])), "r"(32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        __syncwarp();
        for (int it = 0; it < ITERS; ++it) {
            const int slot = it & 1;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned r = hashu(gw * 131071u + it * U + u) % ROWS;
                if (lane < 25) {
                    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(my + (slot * U + u) * 32 + lane));
                    if (mode == 2)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(tab + r * 25 + lane));
                    else
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(tab + r * 25 + lane));
                }
            }
            if (mode != 5) {
                asm volatile("cp.async.commit_group;");
                asm volatile("cp.async.wait_group 1;");
            } else {
                const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar5[warp][slot]));
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(b));
                if (it > 0) {
                    const unsigned pb = static_cast<unsigned>(__cvta_generic_to_shared(&bar5[warp][slot ^ 1]));
                    const unsigned par = ((it - 1) >> 1) & 1;
                    asm volatile("{ .reg .pred p; W5: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W5; }" ::"r"(pb), "r"(par) : "memory");
                }
            }
            __syncwarp();
            acc += my[((slot ^ 1) * U) * 32 + lane].x;
        }
        if (mode != 5) asm volatile("cp.async.wait_group 0;");
    }
    const long long t1 = clock64();
    if (acc == 12345.f) sink[0] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main(int argc, char** argv) {
    const int mode = atoi(argv[1]), threads = atoi(argv[2]), per_sm = atoi(argv[3]);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float4* tab;
    float* sink;
    long long* cyc;
    cudaMalloc(&tab, (size_t)ROWS * F * 4);
    cudaMemset(tab, 0, (size_t)ROWS * F * 4);
    cudaMalloc(&sink, 4);
    const int grid = sms * per_sm;
    cudaMalloc(&cyc, grid * 8);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    CUtensorMap tm;
    cuuint64_t dims[2] = {100, (cuuint64_t)ROWS}, str[1] = {400};
    cuuint32_t box[2] = {100, 1}, es[2] = {1, 1};
    CUresult cr = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr) printf("encode failed %d\n", (int)cr);
    const int smem = mode == 7 ? (threads / 32) * 2 * 8 * 1664 : (mode == 4 || mode == 6) ? (threads / 32) * 2 * 32 * 104 * 4 : mode >= 2 ? (threads / 32) * U * 2 * 32 * 16 : 0;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k<<<grid, threads, smem>>>(tm, tab, mode, sink, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<grid, threads, smem>>>(tm, tab, mode, sink, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> c(grid);
    cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto x : c) mx = x > mx ? x : mx;
    const double warps = (double)grid * threads / 32;
    const double bytes = mode == 0 ? (double)grid * threads * ITERS * U * 16
                       : (mode == 4 || mode == 6 || mode == 7) ? warps * (ITERS / 8) * 32 * 400 : warps * ITERS * U * 400;
    printf("mode %d threads %d ctas/sm %d err %s: %.3f ms, %.2f TB/s, %.1f B/clk/SM (max cta cycles %lld)\n", mode,
           threads, per_sm, cudaGetErrorString(cudaGetLastError()), ms, bytes / ms / 1e9, bytes / sms / (double)mx, mx);
    return 0;
}
