// Batched FP32 SPD solve of packed Hermitian rows with the matrices resident in TMEM and the
// Schur-complement updates on the tensor core (the batched Cholesky of the tensor-core
// half-sweep; replaces batch_solve_into, solver.hpp:204-262, at FP32 tolerance).
//
// A CTA of 128 threads factors RPC systems side by side (persistent over groups of RPC rows,
// 4/RPC CTAs per SM, 128 TMEM columns per system; RPC = 1 by default, 2 measured slower). Thread i owns TMEM lane i = row i of every
// augmented matrix [A lower ; b^T] (rows < f: A, row f: b). Per 8-column block bc, for all
// RPC systems at once (every barrier and MMA round trip is shared between them):
//   1. every lane reads its 8 entries of the block column from TMEM (tcgen05.ld);
//   2. the 8 diagonal-block rows go through shared memory; one thread per system (in
//      different warps) factors the 8x8 block (rsqrt) and publishes L_cc and 1/diag;
//   3. each lane below the block solves its own row against it (TRSM); the augmented row
//      becomes y = L^{-1} b (forward substitution for free); L goes back to TMEM;
//   4. the panel P (rows below the block, K = 8) is split P = Ph + Pl (tf32 hi/lo) into two
//      K-major 128B-swizzled tiles and one thread issues D -= Ph Ph^T + Ph Pl^T + Pl Ph^T
//      as three negated tcgen05.mma (M = 128, N = round16(f), K = 8) per system.
// Back substitution L^T x = y: the lanes dump L (packed lower) into the idle operand tiles
// and one warp per system runs the column-oriented solve with the right-hand side in
// registers. The next group's packed rows are bulk-copied into shared memory while the
// current one is factored. All-zero A gives x = 0 (solver.hpp:215-220); a non-positive pivot
// is reported with row, column and pivot (solver.hpp:230-235) and that row's x is zeroed.
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
constexpr int TILE_BYTES = 128 * 128;      // one K-major SW128 operand tile: 128 rows x 128 B (K=8 used)

template <int RPC>
struct TsPlan {
    int pks, rowbuf_bytes;
    size_t tiles, rowbuf, misc, total;
    __host__ __device__ explicit TsPlan(int f) {
        pks = static_cast<int>(packed_stride(f));
        rowbuf_bytes = pks * 4;
        tiles = 0;                                          // RPC x (Ph, Pl)
        rowbuf = static_cast<size_t>(RPC) * 2 * TILE_BYTES;  // RPC packed rows
        misc = rowbuf + static_cast<size_t>(RPC) * ((rowbuf_bytes + 127) & ~127);
        // per system: blk[64] ys[128] xs[128] dinv[128]; flags; 2 mbarriers + tmem slot
        total = misc + static_cast<size_t>(RPC) * (64 + 128 * 3 + 4) * 4 + 64 + 1024;
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

struct SysSmem {  // per-system scratch in shared memory
    float* blk;   // 8x8 diagonal block (row-major), then L_cc
    float* ys;    // y = L^{-1} b
    float* xs;    // x
    float* dinv;  // 1 / L[c][c]
    int* flags;   // [0] breakdown column + 1, [1] pivot bits
};

template <int RPC>
__global__ void __launch_bounds__(TS_THREADS, 4 / RPC)
tc_solve_kernel(const float* __restrict__ packed, int64_t count, int f, float* __restrict__ out_x,
                unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                double* __restrict__ pivot, int64_t status_base) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    constexpr int TS_TMEM_COLS = 128 * RPC;
    const TsPlan<RPC> P(f);
    const int rbb = (P.rowbuf_bytes + 127) & ~127;
    SysSmem ss[RPC];
    uint8_t* Ph[RPC];
    uint8_t* Pl[RPC];
    float* rowbuf[RPC];
    {
        float* m = reinterpret_cast<float*>(base + P.misc);
#pragma unroll
        for (int r = 0; r < RPC; ++r) {
            Ph[r] = base + P.tiles + static_cast<size_t>(r) * 2 * TILE_BYTES;
            Pl[r] = Ph[r] + TILE_BYTES;
            rowbuf[r] = reinterpret_cast<float*>(base + P.rowbuf + static_cast<size_t>(r) * rbb);
            ss[r].blk = m;
            ss[r].ys = m + 64;
            ss[r].xs = m + 192;
            ss[r].dinv = m + 320;
            ss[r].flags = reinterpret_cast<int*>(m + 448);
            m += 452;
        }
    }
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + P.misc + static_cast<size_t>(RPC) * 452 * 4 + 8 * 0);
    bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bars) + 7) & ~static_cast<uintptr_t>(7));
    uint64_t* load_bar = bars;
    uint64_t* mma_bar = bars + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

    const int i = threadIdx.x;  // matrix row == TMEM lane
    const int warp = i >> 5, lane = i & 31;
    const int nbc = (f + 7) >> 3;
    const int N = (f + 15) & ~15;
    const uint32_t idesc_neg = idesc_tf32(128, N) | (1u << 13);  // D -= A * B^T
    const uint32_t row_bytes = static_cast<uint32_t>(P.rowbuf_bytes);
    const int64_t ngroups = (count + RPC - 1) / RPC;

    if (warp == 0) tmem_alloc<TS_TMEM_COLS>(tmem_slot);
    if (i == 0) {
        mbar_init(load_bar, 1);
        mbar_init(mma_bar, 1);
        fence_barrier_init();
    }
    for (int t = i; t < RPC * 2 * TILE_BYTES / 16; t += TS_THREADS)
        reinterpret_cast<float4*>(base + P.tiles)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tlane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    uint32_t load_phase = 0, mma_phase = 0;

    auto issue_load = [&](int64_t g) {  // thread 0: bulk-copy the group's packed rows
        const int64_t r0 = g * RPC;
        const int nr = static_cast<int>(std::min<int64_t>(RPC, count - r0));
        expect_tx(load_bar, row_bytes * static_cast<uint32_t>(nr));
        for (int r = 0; r < nr; ++r)
            bulk_g2s(smem_u32(base + P.rowbuf) + r * rbb, packed + (r0 + r) * P.pks, row_bytes, load_bar);
    };
    int64_t g = blockIdx.x;
    if (i == 0 && g < ngroups) issue_load(g);
    // row i's operand slots in the K-major tiles (two 16-byte chunks, 128B swizzle)
    const uint32_t prow = static_cast<uint32_t>((i >> 3) * 1024 + (i & 7) * 128);
    const uint32_t pc0 = prow + ((0u ^ (i & 7)) << 4), pc1 = prow + ((1u ^ (i & 7)) << 4);

    // fill TMEM with my row of each system of group gg (lower part; row f = b); nz[r] flags a
    // nonzero A entry in my row
    auto fill = [&](int64_t gg, int (&nz)[RPC]) {
        mbar_wait(load_bar, load_phase);
        load_phase ^= 1u;
        const int64_t rr0 = gg * RPC;
#pragma unroll
        for (int r = 0; r < RPC; ++r) {
            const bool exists = rr0 + r < count;
            nz[r] = 0;
            for (int c0 = 0; c0 < N; c0 += 8) {
                float v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int j = c0 + q;
                    float t = 0.f;
                    if (exists) {
                        if (i < f && j <= i) {
                            t = rowbuf[r][i * (i + 1) / 2 + j];
                            nz[r] |= t != 0.f;
                        } else if (i == f && j < f) {
                            t = rowbuf[r][f * (f + 1) / 2 + j];
                        }
                    }
                    v[q] = t;
                }
                tmem_st8(tlane + r * 128 + c0, v);
            }
        }
        tmem_st_wait();
    };
    int nzr[RPC];
    if (g < ngroups) fill(g, nzr);
    for (; g < ngroups; g += gridDim.x) {
        const int64_t row0 = g * RPC;
        bool active[RPC];
#pragma unroll
        for (int r = 0; r < RPC; ++r) {
            active[r] = __syncthreads_or(nzr[r]) != 0;  // all-zero A: x = 0 (solver.hpp:215-220)
            if (row0 + r < count && !active[r]) {
                if (i < f) out_x[(row0 + r) * f + i] = 0.f;
                if (i == 0) column[row0 + r] = 0;
            }
        }
        tc_fence_before();
        __syncthreads();
        if (i == 0 && g + gridDim.x < ngroups) issue_load(g + gridDim.x);  // rowbufs are free

        for (int bc = 0; bc < nbc; ++bc) {
            const int r0 = 8 * bc;
            bool any = false;
#pragma unroll
            for (int r = 0; r < RPC; ++r) any |= active[r];
            if (!any) break;
            tc_fence_after();
            float a[RPC][8];
#pragma unroll
            for (int r = 0; r < RPC; ++r) tmem_ld8(tlane + r * 128 + r0, a[r]);
            tmem_ld_wait();
            // (1) diagonal rows -> shared memory; the block is factored by a lane of the warp
            //     that holds those rows (a warp sync suffices: the rest of the CTA waits at the
            //     barrier after the factorization)
            const int dwarp = r0 >> 5;
            if (i >= r0 && i < r0 + 8) {
#pragma unroll
                for (int r = 0; r < RPC; ++r) {
                    *reinterpret_cast<float4*>(&ss[r].blk[(i - r0) * 8]) = make_float4(a[r][0], a[r][1], a[r][2], a[r][3]);
                    *reinterpret_cast<float4*>(&ss[r].blk[(i - r0) * 8 + 4]) = make_float4(a[r][4], a[r][5], a[r][6], a[r][7]);
                }
            }
            if (warp == dwarp) __syncwarp();
#pragma unroll
            for (int r = 0; r < RPC; ++r) {
                if (i != 32 * dwarp + ((r0 & 31) + 8 * r) % 32 || !active[r]) continue;
                float* blk = ss[r].blk;
                float l[8][8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 u = *reinterpret_cast<const float4*>(&blk[q * 8]);
                    const float4 w = *reinterpret_cast<const float4*>(&blk[q * 8 + 4]);
                    l[q][0] = u.x, l[q][1] = u.y, l[q][2] = u.z, l[q][3] = u.w;
                    l[q][4] = w.x, l[q][5] = w.y, l[q][6] = w.z, l[q][7] = w.w;
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
                    ss[r].dinv[r0 + c] = ic;
                    if (ok) {
                        l[c][c] = d * ic;
#pragma unroll
                        for (int q = c + 1; q < 8; ++q) l[q][c] *= ic;
#pragma unroll
                        for (int q = c + 1; q < 8; ++q)
#pragma unroll
                            for (int p = c + 1; p <= q; ++p) l[q][p] = fmaf(-l[q][c], l[p][c], l[q][p]);
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    *reinterpret_cast<float4*>(&blk[q * 8]) = make_float4(l[q][0], l[q][1], l[q][2], l[q][3]);
                    *reinterpret_cast<float4*>(&blk[q * 8 + 4]) = make_float4(l[q][4], l[q][5], l[q][6], l[q][7]);
                }
                ss[r].flags[0] = bad;
                ss[r].flags[1] = __float_as_int(badv);
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < RPC; ++r) {
                if (active[r] && ss[r].flags[0]) {  // breakdown (uniform)
                    const int64_t row = row0 + r;
                    if (i == 0) {
                        column[row] = ss[r].flags[0];
                        pivot[row] = static_cast<double>(__int_as_float(ss[r].flags[1]));
                        atomicMin(min_row, static_cast<unsigned long long>(status_base + row));
                    }
                    if (i < f) out_x[row * f + i] = 0.f;
                    active[r] = false;
                }
            }
            const bool update = bc + 1 < nbc;  // no trailing columns after the last block
            const bool diag_row = i >= r0 && i < r0 + 8 && i < f;
            const bool below = (i >= r0 + 8 && i < f) || (i == f && i >= r0);
#pragma unroll
            for (int r = 0; r < RPC; ++r) {
                // (2) my row of L; lanes outside keep their entries (upper-part or padding
                //     cells that are never read)
                float L[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) L[c] = a[r][c];
                const float* blk = ss[r].blk;
                if (active[r] && diag_row) {
                    const float4 u = *reinterpret_cast<const float4*>(&blk[(i - r0) * 8]);
                    const float4 w = *reinterpret_cast<const float4*>(&blk[(i - r0) * 8 + 4]);
                    const float v[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int c = 0; c < 8; ++c) L[c] = (c <= i - r0) ? v[c] : 0.f;
                } else if (active[r] && below) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 u = *reinterpret_cast<const float4*>(&blk[c * 8]);
                        const float4 w = *reinterpret_cast<const float4*>(&blk[c * 8 + 4]);
                        const float lc[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
                        float s = a[r][c];
#pragma unroll
                        for (int k = 0; k < c; ++k) s = fmaf(-L[k], lc[k], s);
                        L[c] = (r0 + c < f) ? s * ss[r].dinv[r0 + c] : 0.f;
                    }
                }
                tmem_st8(tlane + r * 128 + r0, L);  // .sync.aligned: every lane of the warp stores
                if (active[r] && i == f) {
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        if (r0 + c < f) ss[r].ys[r0 + c] = L[c];
                }
                if (update && active[r]) {
                    // panel operand: rows below the block only (factored rows contribute nothing)
                    float h[8], lo[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float pv = (i >= r0 + 8 && i <= f) ? L[c] : 0.f;
                        h[c] = rna_tf32(pv);
                        lo[c] = rna_tf32(pv - h[c]);
                    }
                    *reinterpret_cast<float4*>(Ph[r] + pc0) = make_float4(h[0], h[1], h[2], h[3]);
                    *reinterpret_cast<float4*>(Ph[r] + pc1) = make_float4(h[4], h[5], h[6], h[7]);
                    *reinterpret_cast<float4*>(Pl[r] + pc0) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                    *reinterpret_cast<float4*>(Pl[r] + pc1) = make_float4(lo[4], lo[5], lo[6], lo[7]);
                }
            }
            if (update) fence_proxy_async_smem();
            tmem_st_wait();
            tc_fence_before();
            __syncthreads();
            if (update) {
                bool issued = false;
                if (i == 0) {
                    tc_fence_after();
#pragma unroll
                    for (int r = 0; r < RPC; ++r) {
                        if (!active[r]) continue;
                        const uint64_t dh = sdesc_sw128(smem_u32(Ph[r]), 16, 1024);
                        const uint64_t dl = sdesc_sw128(smem_u32(Pl[r]), 16, 1024);
                        const uint32_t d = tmem + r * 128;
                        mma_tf32(d, dh, dh, idesc_neg, 1u);
                        mma_tf32(d, dh, dl, idesc_neg, 1u);
                        mma_tf32(d, dl, dh, idesc_neg, 1u);
                        issued = true;
                    }
                    if (issued) mma_commit(mma_bar);
                    else mbar_arrive(mma_bar);  // nothing to wait for; keep the phase count
                }
                mbar_wait(mma_bar, mma_phase);
                mma_phase ^= 1u;
            }
        }
        // ---- back substitution L^T x = y ----
        // every lane dumps its row of L (columns 0..i) of each system from TMEM into a packed
        // lower copy in that system's (now idle) operand tiles; warp r then runs system r's
        // column-oriented solve with the right-hand side spread over its lanes
        for (int c0 = 0; c0 < 8 * nbc; c0 += 8) {
            tc_fence_after();
            float lb[RPC][8];
#pragma unroll
            for (int r = 0; r < RPC; ++r) tmem_ld8(tlane + r * 128 + c0, lb[r]);
            tmem_ld_wait();
            if (i < f) {
#pragma unroll
                for (int r = 0; r < RPC; ++r) {
                    if (!active[r]) continue;
                    float* lpk = reinterpret_cast<float*>(Ph[r]);
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        if (c0 + c <= i) lpk[i * (i + 1) / 2 + c0 + c] = lb[r][c];
                }
            }
        }
        __syncthreads();
        // back substitution of system r by warp r, overlapped with the next group's TMEM fill
        // by the other warps (each warp fills its own lanes once it is free); the barrier at
        // the top of the next iteration orders the tiles' reuse
#pragma unroll
        for (int r = 0; r < RPC; ++r) {
            if (warp != r || !active[r]) continue;
            const float* lpk = reinterpret_cast<const float*>(Ph[r]);
            const float* ys = ss[r].ys;
            const float* dinv = ss[r].dinv;
            constexpr int G = 4;  // 128 / 32 values per lane
            float yv[G];
#pragma unroll
            for (int gq = 0; gq < G; ++gq) {
                const int j = gq * 32 + lane;
                yv[gq] = j < f ? ys[j] : 0.f;
            }
#pragma unroll
            for (int gq = G - 1; gq >= 0; --gq) {
                for (int t = 31; t >= 0; --t) {
                    const int ii = gq * 32 + t;
                    if (ii >= f) continue;  // uniform
                    const float xi = __shfl_sync(0xffffffffu, yv[gq], t) * dinv[ii];
                    if (lane == t) yv[gq] = xi;
                    const float* lrow = lpk + ii * (ii + 1) / 2;
#pragma unroll
                    for (int gg = 0; gg <= gq; ++gg) {
                        const int j = gg * 32 + lane;
                        if (j < ii) yv[gg] = fmaf(-lrow[j], xi, yv[gg]);
                    }
                }
            }
            float* x = out_x + (row0 + r) * f;
#pragma unroll
            for (int gq = 0; gq < G; ++gq) {
                const int j = gq * 32 + lane;
                if (j < f) x[j] = yv[gq];
            }
            if (lane == 0) column[row0 + r] = 0;
        }
        if (g + gridDim.x < ngroups) {
            tc_fence_after();
            fill(g + gridDim.x, nzr);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<TS_TMEM_COLS>(tmem);
    }
}

template <int RPC>
void launch_solve(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                  cudaStream_t s) {
    const TsPlan<RPC> P(f);
    ALSK_CUDA(cudaFuncSetAttribute(tc_solve_kernel<RPC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(P.total)));
    const int64_t groups = (count + RPC - 1) / RPC;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(groups, static_cast<int64_t>(4 / RPC) * num_sms()));
    tc_solve_kernel<RPC><<<grid, TS_THREADS, P.total, s>>>(packed, count, f, x, st.min_row, st.column + status_off,
                                                           st.pivot + status_off, status_off);
    ALSK_LAUNCHED();
}

}  // namespace

bool packed_solve(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                  cudaStream_t s) {
    static const bool tiles = std::getenv("ALSK_SOLVE_TILES") != nullptr;  // A/B switches for measurements
    static const bool pairs = std::getenv("ALSK_SOLVE_PAIRS") != nullptr;
    if (tiles || f < 8 || f > 127) return packed_solve_tiles(packed, count, f, x, st, status_off, s);
    if (count <= 0) return true;
    if (pairs) launch_solve<2>(packed, count, f, x, st, status_off, s);
    else launch_solve<1>(packed, count, f, x, st, status_off, s);
    return true;
}

}  // namespace alsk
