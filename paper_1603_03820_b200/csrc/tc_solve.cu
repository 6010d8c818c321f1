// Batched FP32 SPD solve of packed Hermitian rows with the matrix resident in TMEM and the
// Schur-complement updates on the tensor core (the batched Cholesky of the tensor-core
// half-sweep; replaces batch_solve_into, solver.hpp:204-262, at FP32 tolerance).
//
// One CTA of 128 threads per matrix at a time (persistent over rows, 4 CTAs per SM, 128
// TMEM columns each). Thread i owns TMEM lane i = row i of the augmented matrix
// [A lower ; b^T] (rows < f: A, row f: b). Per 8-column block bc:
//   1. every lane reads its 8 entries of the block column from TMEM (tcgen05.ld);
//   2. the 8 diagonal-block rows go through shared memory, one thread factors the 8x8 block
//      (rsqrt) and publishes L_cc and 1/diag;
//   3. each lane below the block solves its own row against it (TRSM); the augmented row
//      becomes y = L^{-1} b (forward substitution for free); L goes back to TMEM;
//   4. the panel P (rows below the block, K = 8) is split P = Ph + Pl (tf32 hi/lo) into two
//      K-major 128B-swizzled tiles and one thread issues D -= Ph Ph^T + Ph Pl^T + Pl Ph^T
//      as three negated tcgen05.mma (M = 128, N = round16(f), K = 8).
// Back substitution L^T x = y: the lanes dump L (packed lower) into the idle operand tiles
// and one warp runs the column-oriented solve with the right-hand side in registers.
// The next row's packed data is bulk-copied into shared memory while the current one is
// factored. All-zero A gives x = 0 (solver.hpp:215-220); a non-positive pivot is reported
// with row, column and pivot (solver.hpp:230-235) and the row's x is zeroed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace alsk {
namespace {
using namespace tc;

constexpr int TS_THREADS = 128;
constexpr int TS_TMEM_COLS = 128;
constexpr int TILE_BYTES = 128 * 128;  // one K-major SW128 operand tile: 128 rows x 128 B (K=8 used)

struct TsPlan {
    int pks, rowbuf_bytes;
    size_t ph, pl, rowbuf, misc, total;
    __host__ __device__ explicit TsPlan(int f) {
        pks = static_cast<int>(packed_stride(f));
        rowbuf_bytes = pks * 4;
        ph = 0;
        pl = TILE_BYTES;
        rowbuf = 2 * TILE_BYTES;
        misc = rowbuf + ((rowbuf_bytes + 127) & ~127);
        // blk[64] ys[128] xs[128] dinv[128] red[32*8] + 2 mbarriers + tmem slot + flags
        total = misc + (64 + 128 * 3 + 256) * 4 + 64 + 1024;
    }
};

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ float rna_tf32(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u); }

__global__ void __launch_bounds__(TS_THREADS, 4)
tc_solve_kernel(const float* __restrict__ packed, int64_t count, int f, float* __restrict__ out_x,
                unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                double* __restrict__ pivot, int64_t status_base) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const TsPlan P(f);
    uint8_t* Ph = base + P.ph;
    uint8_t* Pl = base + P.pl;
    float* rowbuf = reinterpret_cast<float*>(base + P.rowbuf);
    float* blk = reinterpret_cast<float*>(base + P.misc);
    float* ys = blk + 64;
    float* xs = ys + 128;
    float* dinv = xs + 128;
    float* red = dinv + 128;  // [32][8]: back-substitution partials (4 warps x 8 lane groups)
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 256);
    uint64_t* load_bar = bars;
    uint64_t* mma_bar = bars + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
    int* flags = reinterpret_cast<int*>(tmem_slot + 1);  // [0] breakdown column + 1, [1] pivot bits

    const int i = threadIdx.x;  // matrix row == TMEM lane
    const int warp = i >> 5, lane = i & 31;
    const int nbc = (f + 7) >> 3;
    const int N = (f + 15) & ~15;
    const uint32_t idesc_neg = idesc_tf32(128, N) | (1u << 13);  // D -= A * B^T
    const uint32_t row_bytes = static_cast<uint32_t>(P.rowbuf_bytes);

    if (warp == 0) tmem_alloc<TS_TMEM_COLS>(tmem_slot);
    if (i == 0) {
        mbar_init(load_bar, 1);
        mbar_init(mma_bar, 1);
        fence_barrier_init();
    }
    for (int t = i; t < 2 * TILE_BYTES / 16; t += TS_THREADS)
        reinterpret_cast<float4*>(Ph)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tlane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    uint32_t load_phase = 0, mma_phase = 0;
    int64_t row = blockIdx.x;
    if (i == 0 && row < count) {
        expect_tx(load_bar, row_bytes);
        bulk_g2s(smem_u32(rowbuf), packed + row * P.pks, row_bytes, load_bar);
    }
    // row i's operand slots in the K-major tiles (two 16-byte chunks, 128B swizzle)
    const uint32_t prow = static_cast<uint32_t>((i >> 3) * 1024 + (i & 7) * 128);
    const uint32_t pc0 = prow + ((0u ^ (i & 7)) << 4), pc1 = prow + ((1u ^ (i & 7)) << 4);

#ifdef ALSK_TS_DEBUG
#define TSDBG(...) do { if (threadIdx.x == 0 && blockIdx.x == 0) printf(__VA_ARGS__); } while (0)
#else
#define TSDBG(...) do {} while (0)
#endif
    TSDBG("start tmem=%x\n", tmem);
#ifdef ALSK_TS_DEBUG
    long long tt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define TLAP(k) do { const long long now_ = clock64(); tt[k] += now_ - tq; tq = now_; } while (0)
#else
#define TLAP(k) do {} while (0)
#endif
    for (; row < count; row += gridDim.x) {
        mbar_wait(load_bar, load_phase);
        load_phase ^= 1u;
        // ---- fill TMEM with my row (lower part; row f = b) ----
        int nz = 0;
        for (int c0 = 0; c0 < N; c0 += 8) {
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int j = c0 + q;
                float t = 0.f;
                if (i < f && j <= i) {
                    t = rowbuf[i * (i + 1) / 2 + j];
                    nz |= t != 0.f;
                } else if (i == f && j < f) {
                    t = rowbuf[f * (f + 1) / 2 + j];
                }
                v[q] = t;
            }
            tmem_st8(tlane + c0, v);
        }
        tmem_st_wait();
        tc_fence_before();
        nz = __syncthreads_or(nz);
        if (i == 0) {
            flags[0] = 0;
            if (row + gridDim.x < count) {  // rowbuf is free: prefetch the next row
                expect_tx(load_bar, row_bytes);
                bulk_g2s(smem_u32(rowbuf), packed + (row + gridDim.x) * P.pks, row_bytes, load_bar);
            }
        }
        float* x = out_x + row * static_cast<int64_t>(f);
        if (!nz) {  // all-zero A (solver.hpp:215-220)
            if (i < f) x[i] = 0.f;
            if (i == 0) column[row] = 0;
            continue;
        }
        bool broken = false;
        for (int bc = 0; bc < nbc; ++bc) {
            const int r0 = 8 * bc;
            
            TLAP(7);
            tc_fence_after();
            float a[8];
            tmem_ld8(tlane + r0, a);
            tmem_ld_wait();
            TLAP(0);
            // (1) the diagonal rows hand their block to one thread of their warp, which factors
            //     it (rsqrt) and publishes L_cc and 1/diag; everyone else waits at the barrier
            const int dw = r0 >> 5;  // warp holding lanes r0 .. r0+7
            if (i >= r0 && i < r0 + 8) {
                *reinterpret_cast<float4*>(&blk[(i - r0) * 8]) = make_float4(a[0], a[1], a[2], a[3]);
                *reinterpret_cast<float4*>(&blk[(i - r0) * 8 + 4]) = make_float4(a[4], a[5], a[6], a[7]);
            }
            if (warp == dw) __syncwarp();
            if (i == (r0 & ~31) + (r0 & 31)) {  // lane r0 of its warp
                float l[8][8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const float4 u = *reinterpret_cast<const float4*>(&blk[r * 8]);
                    const float4 w = *reinterpret_cast<const float4*>(&blk[r * 8 + 4]);
                    l[r][0] = u.x, l[r][1] = u.y, l[r][2] = u.z, l[r][3] = u.w;
                    l[r][4] = w.x, l[r][5] = w.y, l[r][6] = w.z, l[r][7] = w.w;
                }
                int bad = 0;
                float badv = 0.f;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float d = l[c][c];
                    const bool live = !bad && r0 + c < f;
                    if (live && !(d > 0.f)) {
                        bad = r0 + c + 1;
                        badv = d;
                    }
                    const bool ok = live && d > 0.f;
                    const float ic = ok ? rsqrtf(d) : 0.f;
                    dinv[r0 + c] = ic;
                    if (ok) {
                        l[c][c] = d * ic;
#pragma unroll
                        for (int r = c + 1; r < 8; ++r) l[r][c] *= ic;
#pragma unroll
                        for (int r = c + 1; r < 8; ++r)
#pragma unroll
                            for (int q = c + 1; q <= r; ++q) l[r][q] = fmaf(-l[r][c], l[q][c], l[r][q]);
                    }
                }
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    *reinterpret_cast<float4*>(&blk[r * 8]) = make_float4(l[r][0], l[r][1], l[r][2], l[r][3]);
                    *reinterpret_cast<float4*>(&blk[r * 8 + 4]) = make_float4(l[r][4], l[r][5], l[r][6], l[r][7]);
                }
                flags[0] = bad;
                flags[1] = __float_as_int(badv);
            }
            __syncthreads();
            TLAP(1);
            if (flags[0]) {  // uniform
                if (i == 0) {
                    column[row] = flags[0];
                    pivot[row] = static_cast<double>(__int_as_float(flags[1]));
                    atomicMin(min_row, static_cast<unsigned long long>(status_base + row));
                }
                if (i < f) x[i] = 0.f;
                broken = true;
                break;
            }
            // (2) my row of L for this block column; lanes outside keep their entries (upper-part
            //     or padding cells that are never read)
            float L[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) L[c] = a[c];
            const bool diag_row = i >= r0 && i < r0 + 8 && i < f;
            const bool below = (i >= r0 + 8 && i < f) || (i == f && i >= r0);
            if (diag_row) {
                const float4 u = *reinterpret_cast<const float4*>(&blk[(i - r0) * 8]);
                const float4 w = *reinterpret_cast<const float4*>(&blk[(i - r0) * 8 + 4]);
                const float v[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
#pragma unroll
                for (int c = 0; c < 8; ++c) L[c] = (c <= i - r0) ? v[c] : 0.f;
            } else if (below) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float4 u = *reinterpret_cast<const float4*>(&blk[c * 8]);
                    const float4 w = *reinterpret_cast<const float4*>(&blk[c * 8 + 4]);
                    const float lc[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
                    float s = a[c];
#pragma unroll
                    for (int k = 0; k < c; ++k) s = fmaf(-L[k], lc[k], s);
                    L[c] = (r0 + c < f) ? s * dinv[r0 + c] : 0.f;
                }
            }
            tmem_st8(tlane + r0, L);  // .sync.aligned: every lane of the warp stores
            if (i == f) {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (r0 + c < f) ys[r0 + c] = L[c];
            }
            const bool update = bc + 1 < nbc;  // no trailing columns after the last block
            if (update) {
                // panel operand: rows below the block only (factored rows contribute nothing)
                float h[8], lo[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float pv = (i >= r0 + 8 && i <= f) ? L[c] : 0.f;
                    h[c] = rna_tf32(pv);
                    lo[c] = rna_tf32(pv - h[c]);
                }
                *reinterpret_cast<float4*>(Ph + pc0) = make_float4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<float4*>(Ph + pc1) = make_float4(h[4], h[5], h[6], h[7]);
                *reinterpret_cast<float4*>(Pl + pc0) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                *reinterpret_cast<float4*>(Pl + pc1) = make_float4(lo[4], lo[5], lo[6], lo[7]);
                TLAP(2);
                fence_proxy_async_smem();
            }
            TLAP(6);
            tmem_st_wait();
            tc_fence_before();
            __syncthreads();
            TLAP(3);
            if (update) {
                if (i == 0) {
                    tc_fence_after();
                    const uint64_t dh = sdesc_sw128(smem_u32(Ph), 16, 1024);
                    const uint64_t dl = sdesc_sw128(smem_u32(Pl), 16, 1024);
                    mma_tf32(tmem, dh, dh, idesc_neg, 1u);
                    mma_tf32(tmem, dh, dl, idesc_neg, 1u);
                    mma_tf32(tmem, dl, dh, idesc_neg, 1u);
                    mma_commit(mma_bar);
                }
                mbar_wait(mma_bar, mma_phase);
                mma_phase ^= 1u;
                TLAP(4);
            }
        }
        TLAP(7);
        if (broken) {
            tc_fence_before();
            __syncthreads();
            continue;
        }
        if (i == 0) column[row] = 0;
        // ---- back substitution L^T x = y ----
        // every lane dumps its row of L (columns 0..i) from TMEM into a packed lower copy in
        // the (now idle) operand tiles; warp 0 then runs the column-oriented solve with the
        // right-hand side spread over its lanes
        float* lpk = reinterpret_cast<float*>(Ph);  // f(f+1)/2 floats <= 2 tiles
        for (int c0 = 0; c0 < 8 * nbc; c0 += 8) {
            float lb[8];
            tc_fence_after();
            tmem_ld8(tlane + c0, lb);
            tmem_ld_wait();
            if (i < f) {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c0 + c <= i) lpk[i * (i + 1) / 2 + c0 + c] = lb[c];
            }
        }
        __syncthreads();
        if (warp == 0) {
            constexpr int G = 4;  // 128 / 32 values per lane
            float yv[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int j = g * 32 + lane;
                yv[g] = j < f ? ys[j] : 0.f;
            }
#pragma unroll
            for (int g = G - 1; g >= 0; --g) {
                for (int t = 31; t >= 0; --t) {
                    const int ii = g * 32 + t;
                    if (ii >= f) continue;  // uniform
                    const float xi = __shfl_sync(0xffffffffu, yv[g], t) * dinv[ii];
                    if (lane == t) yv[g] = xi;
                    const float* lrow = lpk + ii * (ii + 1) / 2;
#pragma unroll
                    for (int gg = 0; gg <= g; ++gg) {
                        const int j = gg * 32 + lane;
                        if (j < ii) yv[gg] = fmaf(-lrow[j], xi, yv[gg]);
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int j = g * 32 + lane;
                if (j < f) xs[j] = yv[g];
            }
        }
        __syncthreads();
        TLAP(5);
        if (i < f) x[i] = xs[i];
#ifdef ALSK_TS_DEBUG
        if (threadIdx.x == 0 && blockIdx.x == 0)
            printf("row %lld: ld %lld diag+bar %lld trsm+split %lld fence %lld bar %lld mma %lld backsub %lld other %lld\n",
                   (long long)row, tt[0], tt[1], tt[2], tt[6], tt[3], tt[4], tt[5], tt[7]);
        for (int k = 0; k < 8; ++k) tt[k] = 0;
#endif
        tc_fence_before();
        __syncthreads();  // TMEM and the shared scratch are reused by the next row
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<TS_TMEM_COLS>(tmem);
    }
}

}  // namespace

bool packed_solve(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                  cudaStream_t s) {
    static const bool tiles = std::getenv("ALSK_SOLVE_TILES") != nullptr;  // A/B switch for measurements
    if (tiles || f < 8 || f > 127) return packed_solve_tiles(packed, count, f, x, st, status_off, s);
    if (count <= 0) return true;
    const TsPlan P(f);
    ALSK_CUDA(cudaFuncSetAttribute(tc_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(P.total)));
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(count, 4LL * num_sms()));
    tc_solve_kernel<<<grid, TS_THREADS, P.total, s>>>(packed, count, f, x, st.min_row, st.column + status_off,
                                                      st.pivot + status_off, status_off);
    ALSK_LAUNCHED();
    return true;
}

}  // namespace alsk
