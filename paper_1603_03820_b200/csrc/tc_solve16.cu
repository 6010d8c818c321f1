// Batched FP32 SPD solve with 16-column steps (the TMEM Cholesky of tc_solve.cu with half the
// dependent steps; replaces batch_solve_into, solver.hpp:204-262, at FP32 tolerance).
//
// Same roles as tc_solve.cu (4 CTAs per SM, 128 factor threads = TMEM lanes, one
// back-substitution warp, mbarrier hand-off of L and y). Per 16-column block (r0 = 16 bc):
//   1. every lane reads its 16 entries of the block column from TMEM;
//   2. the 16 diagonal rows (one warp) factor the 16x16 diagonal block without a CTA barrier:
//      POTRF of the top-left 8x8 (one lane) -> the 8 lower rows solve against it and update
//      their own 8x8 Schur block from each other's rows (shared memory, warp syncs) ->
//      POTRF of that block (one lane) -> M = diag(1/L) L for the whole 16x16 block;
//   3. every lane at or below the block solves its row against M (TRSM over 16 columns;
//      the augmented row becomes y); L goes back to TMEM;
//   4. the panel (rows below, K = 16) is split hi/lo into two 8 KB K-major tiles and one
//      thread issues six negated MMAs (two K halves x Ph Ph^T + Ph Pl^T + Pl Ph^T).
// The packed rows are read straight from global memory (prefetched into L2 one system
// ahead), which leaves the shared memory for the 16-wide tiles at 4 CTAs per SM.
// Measurement build only (ALSK_MEASURE): measured slower than tc_solve.cu;
// the product library gets the stub at the end of this file.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "measure.cuh"
#include "tc_common.cuh"

#ifdef ALSK_MEASURE

namespace alsk {
namespace {
using namespace tc;

constexpr int S16_FACTOR = 128;
constexpr int S16_THREADS = S16_FACTOR + 32;
constexpr int S16_BS_WARP = S16_FACTOR / 32;
constexpr uint32_t S16_BAR = 1;
// K = 16 panel tile, K-major without swizzle: 4 core matrices (16 B) per 8-row group along K
// (LBO = 128 B apart), 8-row groups SBO = 512 B apart; 128 rows = 8 KB
constexpr int P16_BYTES = 8192;
constexpr uint32_t P16_LBO = 128, P16_SBO = 512;

struct S16Plan {
    int pks;
    size_t lbuf, vec, blk, bars, total;
    __host__ __device__ explicit S16Plan(int f) {
        pks = static_cast<int>(packed_stride(f));
        const size_t pkb = (static_cast<size_t>(pks) * 4 + 127) & ~static_cast<size_t>(127);
        lbuf = 2 * P16_BYTES;           // Ph, Pl, then the hand-off buffer
        vec = lbuf + pkb;               // dinv[2][128]
        blk = vec + 2 * 128 * 4;        // a16[16][16], M[16][16], L21[8][8], flags, meta
        bars = blk + (256 + 256 + 64) * 4 + 32;
        total = bars + 8 * 8 + 1024;
    }
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_st8x(uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8x(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __uint_as_float(r[q]);
}
__device__ __forceinline__ void tmem_st_wait16() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ bool bar_red_or16(uint32_t id, uint32_t threads, bool v) {
    uint32_t r;
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.u32 q, %1, 0;\n bar.red.or.pred p, %2, %3, q;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(r)
        : "r"(static_cast<uint32_t>(v)), "r"(id), "r"(threads)
        : "memory");
    return r != 0;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ float rna16(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u); }
__device__ __forceinline__ uint64_t p16_desc(uint32_t tile) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((tile >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((P16_LBO >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((P16_SBO >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;
    return d;
}
// single-thread 8x8 right-looking Cholesky of the block at `a` (row stride 16); writes
// M = diag(1/L) L (rows of padding columns zero, row stride 16) and 1/diag; returns the first
// real column with a non-positive pivot (+1) and its pivot
__device__ __forceinline__ int potrf8(const float* a, float* m_out, float* dinv, int base, int f, float& badv) {
    float l[8][8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float4 u = *reinterpret_cast<const float4*>(&a[q * 16]);
        const float4 w = *reinterpret_cast<const float4*>(&a[q * 16 + 4]);
        l[q][0] = u.x, l[q][1] = u.y, l[q][2] = u.z, l[q][3] = u.w;
        l[q][4] = w.x, l[q][5] = w.y, l[q][6] = w.z, l[q][7] = w.w;
    }
    float piv[8], dv[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float d = l[c][c];
        piv[c] = d;
        const float ic = rsqrtf(d);
        dv[c] = ic;
        l[c][c] = d * ic;
#pragma unroll
        for (int q = c + 1; q < 8; ++q) l[q][c] *= ic;
#pragma unroll
        for (int q = c + 1; q < 8; ++q)
#pragma unroll
            for (int p = c + 1; p <= q; ++p) l[q][p] = fmaf(-l[q][c], l[p][c], l[q][p]);
    }
    int bad = 0;
    badv = 0.f;
#pragma unroll
    for (int c = 7; c >= 0; --c)
        if (base + c < f && !(piv[c] > 0.f)) {
            bad = base + c + 1;
            badv = piv[c];
        }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const bool real = base + c < f;
        float m[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m[k] = !real ? 0.f : (k < c ? l[c][k] * dv[c] : (k == c ? dv[c] : 0.f));
        *reinterpret_cast<float4*>(&m_out[c * 16]) = make_float4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<float4*>(&m_out[c * 16 + 4]) = make_float4(m[4], m[5], m[6], m[7]);
    }
    *reinterpret_cast<float4*>(&dinv[base]) = make_float4(dv[0], dv[1], dv[2], dv[3]);
    *reinterpret_cast<float4*>(&dinv[base + 4]) = make_float4(dv[4], dv[5], dv[6], dv[7]);
    return bad;
}

__global__ void __launch_bounds__(S16_THREADS, 4)
tc_solve16_kernel(const float* __restrict__ packed, int64_t count, int f, float* __restrict__ out_x,
                  unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                  double* __restrict__ pivot, int64_t status_base, uint32_t sleep_ns, uint32_t mma_first_ns,
                  uint32_t bs_ns) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const S16Plan P(f);
    uint8_t* Ph = base;
    uint8_t* Pl = base + P16_BYTES;
    float* lbuf = reinterpret_cast<float*>(base + P.lbuf);
    float* dinvb = reinterpret_cast<float*>(base + P.vec);
    float* a16 = reinterpret_cast<float*>(base + P.blk);  // diagonal rows [16][16]
    float* M16 = a16 + 256;                                // M = diag(1/L) L, [16][16]
    float* L21 = M16 + 256;                                // [8][8]
    int* flags = reinterpret_cast<int*>(L21 + 64);         // [0] bad, [1] pivot bits, [2] bad of the first half, [3] its pivot
    int* meta = flags + 4;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + P.bars);
    uint64_t* mma_bar = bars;
    uint64_t* lfull = bars + 1;
    uint64_t* lfree = bars + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);

    const int i = threadIdx.x;
    const int warp = i >> 5, lane = i & 31;
    const int nbc8 = (f + 7) >> 3;     // 8-column blocks (packed layout, dump)
    const int nbc16 = (f + 15) >> 4;   // 16-column steps
    const int N = (f + 15) & ~15;
    const uint32_t row_bytes = static_cast<uint32_t>(P.pks) * 4;

    if (warp == 0) tmem_alloc<128>(tmem_slot);
    if (i == 0) {
        mbar_init(mma_bar, 1);
        mbar_init(lfull, 1);
        mbar_init(lfree, 1);
        fence_barrier_init();
    }
    for (int t = i; t < 2 * P16_BYTES / 16; t += S16_THREADS)
        reinterpret_cast<float4*>(base)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto wait = [&](uint64_t* bar, uint32_t ph, uint32_t ns) {
        if (ns == 0) mbar_wait(bar, ph);
        else mbar_wait_sleep(bar, ph, ns);
    };

    if (warp == S16_BS_WARP) {
        // ---------------- back substitution (as tc_solve.cu) ----------------
        uint32_t t = 0;
        for (int64_t g = blockIdx.x; g < count; g += gridDim.x, ++t) {
            wait(lfull, t & 1u, bs_ns);
            if (meta[0]) {
                const float* dinv = dinvb + 128 * (t & 1u);
                constexpr int G = 4;
                int lb[G];
                float yv[G];
#pragma unroll
                for (int gq = 0; gq < G; ++gq) {
                    const int j = min(gq * 32 + lane, f - 1);
                    lb[gq] = static_cast<int>(pb_index(f, 0, j));
                    yv[gq] = gq * 32 + lane < f ? lbuf[lb[gq] + 8 * f] : 0.f;
                }
#pragma unroll
                for (int gq = G - 1; gq >= 0; --gq) {
                    for (int s = 31; s >= 0; --s) {
                        const int ii = gq * 32 + s;
                        if (ii >= f) continue;
                        const float xi = __shfl_sync(0xffffffffu, yv[gq], s) * dinv[ii];
                        if (lane == s) yv[gq] = xi;
#pragma unroll
                        for (int gg = 0; gg <= gq; ++gg) {
                            const int j = gg * 32 + lane;
                            if (j < ii) yv[gg] = fmaf(-lbuf[lb[gg] + 8 * ii], xi, yv[gg]);
                        }
                    }
                }
                float* x = out_x + g * f;
#pragma unroll
                for (int gq = 0; gq < G; ++gq) {
                    const int j = gq * 32 + lane;
                    if (j < f) x[j] = yv[gq];
                }
                if (lane == 0) column[g] = 0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(lfree);
        }
    } else {
        // ---------------- factor threads ----------------
        const uint32_t tlane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        const int wtop = 32 * warp + 31;
        const uint32_t sPh = smem_u32(Ph), sPl = smem_u32(Pl);
        const uint32_t prow = static_cast<uint32_t>((i >> 3) * P16_SBO + (i & 7) * 16);  // + chunk * LBO
        uint32_t ph_mma = 0;
        // my row of system gg from global memory into TMEM (four 8-column blocks per batch of
        // loads in flight); nz: a nonzero A entry in my row
        auto fill = [&](int64_t gg, int& nz) {
            const float* src = packed + gg * P.pks;
            uint32_t bits = 0;
            for (int b0 = 0; b0 < nbc8 && 8 * b0 <= wtop; b0 += 4) {
                float4 u[4][2];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int b = b0 + q;
                    if (b < nbc8 && i >= 8 * b && i <= f) {
                        const float4* p = reinterpret_cast<const float4*>(src + pb_block(f, b) + 8 * (i - 8 * b));
                        u[q][0] = ldg_nc_f4(reinterpret_cast<const float*>(p));
                        u[q][1] = ldg_nc_f4(reinterpret_cast<const float*>(p + 1));
                    } else {
                        u[q][0] = u[q][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int b = b0 + q;
                    if (b >= nbc8 || 8 * b > wtop) break;  // warp-uniform
                    const float v[8] = {u[q][0].x, u[q][0].y, u[q][0].z, u[q][0].w,
                                        u[q][1].x, u[q][1].y, u[q][1].z, u[q][1].w};
#pragma unroll
                    for (int k = 0; k < 8; ++k) bits |= __float_as_uint(v[k]) << 1;
                    tmem_st8x(tlane + 8 * b, v);
                }
            }
            nz = i < f && bits != 0;
            tmem_st_wait16();
        };
        int64_t g = blockIdx.x;
        if (i == 0 && g + gridDim.x < count) prefetch_l2(packed + (g + gridDim.x) * P.pks, row_bytes);
        int nz = 0;
        if (g < count) fill(g, nz);
        uint32_t t = 0;
        for (; g < count; g += gridDim.x, ++t) {
            float* dinv = dinvb + 128 * (t & 1u);
            tc_fence_before();
            bool active = bar_red_or16(S16_BAR, S16_FACTOR, nz != 0);  // all-zero A: x = 0 (solver.hpp:215-220)
            tc_fence_after();
            if (i == 0 && g + 2 * gridDim.x < count) prefetch_l2(packed + (g + 2 * gridDim.x) * P.pks, row_bytes);
            if (!active) {
                if (i < f) out_x[g * f + i] = 0.f;
                if (i == 0) column[g] = 0;
            }
            for (int bc = 0; active && bc < nbc16; ++bc) {
                const int r0 = 16 * bc;
                const bool wlive = wtop >= r0;
                float a[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) a[c] = 0.f;
                if (wlive) {
                    tc_fence_after();
                    tmem_ld16(tlane + r0, a);
                    tmem_ld_wait();
                }
                // ---- the 16x16 diagonal block, inside the warp that holds its rows ----
                const bool drow = i >= r0 && i < r0 + 16;
                if (drow) {
#pragma unroll
                    for (int c = 0; c < 16; c += 4)
                        *reinterpret_cast<float4*>(&a16[(i - r0) * 16 + c]) = make_float4(a[c], a[c + 1], a[c + 2], a[c + 3]);
                }
                if (warp == (r0 >> 5)) {
                    const bool has2 = r0 + 8 < f;  // the lower half holds real columns
                    __syncwarp();
                    if (i == r0) {
                        float bv;
                        const int bad = potrf8(a16, M16, dinv, r0, f, bv);
                        flags[2] = bad;
                        flags[3] = __float_as_int(bv);
                        if (!has2) {
                            flags[0] = bad;
                            flags[1] = __float_as_int(bv);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {  // rows 8..15 of M (padding) and M's upper right
                                *reinterpret_cast<float4*>(&M16[(8 + q) * 16]) = make_float4(0.f, 0.f, 0.f, 0.f);
                                *reinterpret_cast<float4*>(&M16[(8 + q) * 16 + 4]) = make_float4(0.f, 0.f, 0.f, 0.f);
                                *reinterpret_cast<float4*>(&M16[(8 + q) * 16 + 8]) = make_float4(0.f, 0.f, 0.f, 0.f);
                                *reinterpret_cast<float4*>(&M16[(8 + q) * 16 + 12]) = make_float4(0.f, 0.f, 0.f, 0.f);
                            }
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            *reinterpret_cast<float4*>(&M16[q * 16 + 8]) = make_float4(0.f, 0.f, 0.f, 0.f);
                            *reinterpret_cast<float4*>(&M16[q * 16 + 12]) = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                    }
                    if (has2) {
                        __syncwarp();
                        const bool low = i >= r0 + 8 && i < r0 + 16;
                        float l21[8];
                        if (low) {  // my row against L11: the first 8 entries of my L row
#pragma unroll
                            for (int c = 0; c < 8; ++c) {
                                const float4 u = *reinterpret_cast<const float4*>(&M16[c * 16]);
                                const float4 w = *reinterpret_cast<const float4*>(&M16[c * 16 + 4]);
                                const float mc[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
                                float s = a[c] * mc[c];
#pragma unroll
                                for (int k = 0; k < c; ++k) s = fmaf(-l21[k], mc[k], s);
                                l21[c] = s;
                            }
                            const int q = i - r0 - 8;
                            *reinterpret_cast<float4*>(&L21[q * 8]) = make_float4(l21[0], l21[1], l21[2], l21[3]);
                            *reinterpret_cast<float4*>(&L21[q * 8 + 4]) = make_float4(l21[4], l21[5], l21[6], l21[7]);
                        }
                        __syncwarp();
                        if (low) {  // my row of the Schur block A22 - L21 L21^T
                            const int q = i - r0 - 8;
                            float s22[8];
#pragma unroll
                            for (int p = 0; p < 8; ++p) {
                                const float4 u = *reinterpret_cast<const float4*>(&L21[p * 8]);
                                const float4 w = *reinterpret_cast<const float4*>(&L21[p * 8 + 4]);
                                float s = a[8 + p];
                                s = fmaf(-l21[0], u.x, s);
                                s = fmaf(-l21[1], u.y, s);
                                s = fmaf(-l21[2], u.z, s);
                                s = fmaf(-l21[3], u.w, s);
                                s = fmaf(-l21[4], w.x, s);
                                s = fmaf(-l21[5], w.y, s);
                                s = fmaf(-l21[6], w.z, s);
                                s = fmaf(-l21[7], w.w, s);
                                s22[p] = s;
                            }
                            *reinterpret_cast<float4*>(&a16[(8 + q) * 16 + 8]) = make_float4(s22[0], s22[1], s22[2], s22[3]);
                            *reinterpret_cast<float4*>(&a16[(8 + q) * 16 + 12]) = make_float4(s22[4], s22[5], s22[6], s22[7]);
                        }
                        __syncwarp();
                        if (i == r0 + 8) {
                            float bv;
                            const int bad2 = potrf8(a16 + 8 * 16 + 8, M16 + 8 * 16 + 8, dinv, r0 + 8, f, bv);
                            const int bad1 = flags[2];
                            flags[0] = bad1 ? bad1 : bad2;
                            flags[1] = bad1 ? flags[3] : __float_as_int(bv);
                        }
                        __syncwarp();
                        if (low) {  // M21 row = L21 row / L[c][c] of my column
                            const int q = i - r0 - 8;
                            const float sc = i < f ? dinv[i] : 0.f;
                            *reinterpret_cast<float4*>(&M16[(8 + q) * 16]) =
                                make_float4(l21[0] * sc, l21[1] * sc, l21[2] * sc, l21[3] * sc);
                            *reinterpret_cast<float4*>(&M16[(8 + q) * 16 + 4]) =
                                make_float4(l21[4] * sc, l21[5] * sc, l21[6] * sc, l21[7] * sc);
                        }
                    }
                }
                named_barrier(S16_BAR, S16_FACTOR);
                if (flags[0]) {  // breakdown (uniform)
                    if (i == 0) {
                        column[g] = flags[0];
                        pivot[g] = static_cast<double>(__int_as_float(flags[1]));
                        atomicMin(min_row, static_cast<unsigned long long>(status_base + g));
                    }
                    if (i < f) out_x[g * f + i] = 0.f;
                    active = false;
                    break;
                }
                const bool update = bc + 1 < nbc16;
                // ---- TRSM over the 16 columns ----
                float L[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) L[c] = a[c];
                if (i >= r0 && i <= f) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        float mc[16];
#pragma unroll
                        for (int k = 0; k <= c; k += 4) {
                            const float4 u = *reinterpret_cast<const float4*>(&M16[c * 16 + k]);
                            mc[k] = u.x, mc[k + 1] = u.y, mc[k + 2] = u.z, mc[k + 3] = u.w;
                        }
                        float s = a[c] * mc[c];
#pragma unroll
                        for (int k = 0; k < c; ++k) s = fmaf(-L[k], mc[k], s);
                        L[c] = (i - r0 >= c || i == f) ? s : 0.f;
                    }
                }
                if (wlive) tmem_st16(tlane + r0, L);
                if (update) {
                    // panel: rows below the 16-block, K = 16, split hi/lo into the tiles
                    if (wlive) {
                        const bool prow_on = i >= r0 + 16 && i <= f;
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc) {
                            float h[4], lo[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float pv = prow_on ? L[4 * cc + q] : 0.f;
                                h[q] = rna16(pv);
                                lo[q] = pv - h[q];
                            }
                            *reinterpret_cast<float4*>(Ph + prow + cc * P16_LBO) = make_float4(h[0], h[1], h[2], h[3]);
                            *reinterpret_cast<float4*>(Pl + prow + cc * P16_LBO) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                        }
                    }
                    fence_proxy_async_smem();
                }
                tmem_st_wait16();
                tc_fence_before();
                named_barrier(S16_BAR, S16_FACTOR);
                if (update) {
                    if (i == 0) {
                        tc_fence_after();
                        const uint32_t id = idesc_tf32(128, N) | (1u << 13);
#pragma unroll
                        for (int kh = 0; kh < 2; ++kh) {  // K halves: 2 core matrices = 256 bytes apart
                            const uint64_t dh = p16_desc(sPh + kh * 2 * P16_LBO), dl = p16_desc(sPl + kh * 2 * P16_LBO);
                            mma_tf32(tmem, dh, dh, id, 1u);
                            mma_tf32(tmem, dh, dl, id, 1u);
                            mma_tf32(tmem, dl, dh, id, 1u);
                        }
                        mma_commit(mma_bar);
                    }
                    uint32_t done;
                    asm volatile(
                        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                        : "=r"(done)
                        : "r"(smem_u32(mma_bar)), "r"(ph_mma)
                        : "memory");
                    if (!done) {
                        __nanosleep(mma_first_ns);
                        wait(mma_bar, ph_mma, sleep_ns);
                    }
                    ph_mma ^= 1u;
                }
            }
            // hand the factor to the back-substitution warp
            if (t > 0) wait(lfree, (t - 1) & 1u, sleep_ns);
            if (active) {
                for (int b = 0; b < nbc8 && 8 * b <= wtop; ++b) {
                    tc_fence_after();
                    float lv[8];
                    tmem_ld8x(tlane + 8 * b, lv);
                    tmem_ld_wait();
                    if (i >= 8 * b && i <= f) {
                        float4* dst = reinterpret_cast<float4*>(lbuf + pb_block(f, b) + 8 * (i - 8 * b));
                        dst[0] = make_float4(lv[0], lv[1], lv[2], lv[3]);
                        dst[1] = make_float4(lv[4], lv[5], lv[6], lv[7]);
                    }
                }
            }
            if (i == 0) meta[0] = active ? 1 : 0;
            named_barrier(S16_BAR, S16_FACTOR);
            if (i == 0) mbar_arrive(lfull);
            if (g + gridDim.x < count) {
                tc_fence_after();
                fill(g + gridDim.x, nz);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

}  // namespace

bool packed_solve16(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                    cudaStream_t s) {
    if (f < 16 || f > 127) return false;
    if (count <= 0) return true;
    const S16Plan P(f);
    const int smem = static_cast<int>(std::max<size_t>(P.total, 46 * 1024));
    ALSK_CUDA(cudaFuncSetAttribute(tc_solve16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int resident = 0;
    // CTAs that fit an SM's shared memory (228 KB, 1 KB reserved per CTA + 1 KB static);
    // cudaOccupancyMaxActiveBlocksPerMultiprocessor reports 1 for this kernel, which is not
    // what the hardware runs
    resident = static_cast<int>((228 * 1024) / (smem + 2 * 1024));
    const int per_sm = std::max(1, std::min(4, resident));
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(count, per_sm * static_cast<int64_t>(num_sms())));
    static const std::array<uint32_t, 3> w = [] {  // poll sleep, MMA first sleep, back-substitution poll (ns)
        std::array<uint32_t, 3> v{32u, 200u, 1000u};
        if (const char* e = measure_env("ALSK_TS16_WAITS")) {
            unsigned a = 0, b = 0, c = 0;
            if (std::sscanf(e, "%u,%u,%u", &a, &b, &c) == 3) v = {a, b, c};
        }
        return v;
    }();
    tc_solve16_kernel<<<grid, S16_THREADS, smem, s>>>(packed, count, f, x, st.min_row, st.column + status_off,
                                                      st.pivot + status_off, status_off, w[0], w[1], w[2]);
    ALSK_LAUNCHED();
    return true;
}

}  // namespace alsk

#else  // !ALSK_MEASURE

namespace alsk {
bool packed_solve16(const float*, int64_t, int, float*, const SolveStatus&, int64_t, cudaStream_t) { return false; }
}  // namespace alsk

#endif  // ALSK_MEASURE
