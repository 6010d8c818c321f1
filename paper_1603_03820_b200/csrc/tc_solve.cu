// Batched FP32 SPD solve of packed Hermitian rows with the matrices resident in TMEM and the
// Schur-complement updates on the tensor core (the batched Cholesky of the tensor-core
// half-sweep; replaces batch_solve_into, solver.hpp:204-262, at FP32 tolerance).
//
// A CTA (persistent, 4 per SM, one system at a time in 128 TMEM columns) has 128 factor
// threads and one back-substitution warp. Factor thread i owns TMEM lane i = row i of the
// augmented matrix [A lower ; b^T] (rows < f: A, row f: b). Per 8-column block bc:
//   1. every lane reads its 8 entries of the block column from TMEM (tcgen05.ld);
//   2. the 8 diagonal-block rows go through shared memory; the lane of the first of them
//      factors the 8x8 block (rsqrt, branch-free; the breakdown check follows) and publishes
//      M = diag(1/L_cc) L_cc (row c of L_cc scaled by 1/L[c][c], diagonal = 1/L[c][c]);
//   3. every lane at or below the block solves its own row against it (TRSM:
//      L[c] = a[c] M[c][c] - sum_k<c L[k] M[c][k]; on a diagonal-block row this also yields
//      its L_cc row); the augmented row becomes y = L^{-1} b (forward substitution for
//      free); L goes back to TMEM;
//   4. the panel P (rows below the block, K = 8) is split P = Ph + Pl (tf32 hi/lo) into two
//      K-major tiles (no swizzle, 4 KB each) and one thread issues D -= Ph Ph^T + Ph Pl^T +
//      Pl Ph^T as three negated tcgen05.mma (M = 128, N = round16(f), K = 8).
// Warps whose rows all lie above the current block skip its TMEM traffic (upper part).
// Back substitution L^T x = y: the factor threads dump L and y (panel-blocked like the input,
// kernels.cuh) into a shared buffer and hand it to the back-substitution warp (mbarriers
// lfull / lfree), which solves it with the right-hand side in registers while the factor
// threads fill TMEM with the next system (its packed rows were bulk-copied into shared
// memory during the factorization: two 16-byte loads per lane and block).
// All-zero A gives x = 0 (solver.hpp:215-220); a non-positive pivot is reported with row,
// column and pivot (solver.hpp:230-235) and that row's x is zeroed.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"
#include "measure.cuh"
#include "tc_common.cuh"

namespace alsk {
namespace {
using namespace tc;

constexpr int TS_FACTOR = 128;              // factor threads (thread i <-> TMEM lane i)
constexpr int TS_THREADS = TS_FACTOR + 32;  // + the back-substitution warp
constexpr int BS_WARP = TS_FACTOR / 32;
constexpr uint32_t BAR_FACTOR = 1;          // named barrier of the factor threads
// K = 8 panel tile, K-major without swizzle: core matrices of 8 rows x 16 bytes; the two
// K halves of a row group are LBO = 128 bytes apart, row groups SBO = 256 bytes apart
constexpr int PT_BYTES = 4096;
constexpr uint32_t PT_LBO = 128, PT_SBO = 256;
constexpr int TS_PROF_SLOTS = 16;

struct TsPlan {
    int pks;
    size_t rowbuf, lbuf, vec, blk, bars, total;
    __host__ __device__ explicit TsPlan(int f) {
        pks = static_cast<int>(packed_stride(f));
        const size_t pkb = (static_cast<size_t>(pks) * 4 + 127) & ~static_cast<size_t>(127);
        rowbuf = 2 * PT_BYTES;  // Ph at 0, Pl at PT_BYTES
        lbuf = rowbuf + pkb;    // L and y of the system handed to the back substitution
        vec = lbuf + pkb;       // dinv[2][128]
        blk = vec + 2 * 128 * 4;  // 8x8 block, flags, meta
        bars = blk + 64 * 4 + 32;
        total = bars + 8 * 8 + 1024;  // mbarriers + TMEM slot, 1 KB alignment slack
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
// barrier over `threads` threads of barrier `id`, returning the OR of v over them
__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t threads, bool v) {
    uint32_t r;
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.u32 q, %1, 0;\n bar.red.or.pred p, %2, %3, q;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(r)
        : "r"(static_cast<uint32_t>(v)), "r"(id), "r"(threads)
        : "memory");
    return r != 0;
}
// waits of the factor threads: parked in try_wait (ns == 0) or nanosleep back-off
// a wait known to take at least ~first_ns: one test, one long sleep, then short polls
__device__ __forceinline__ void ts_wait_first(uint64_t* bar, uint32_t parity, uint32_t first_ns, uint32_t ns) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(first_ns);
    mbar_wait_sleep(bar, parity, ns);
}
__device__ __forceinline__ void ts_wait(uint64_t* bar, uint32_t parity, uint32_t ns) {
    if (ns == 0) mbar_wait_park(bar, parity);
    else mbar_wait_sleep(bar, parity, ns);
}
__device__ __forceinline__ float rna_tf32(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u); }
// panel tile descriptor starting at row `row` (a multiple of 8)
__device__ __forceinline__ uint64_t pt_desc(uint32_t tile, int row) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>(((tile + (row >> 3) * PT_SBO) >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((PT_LBO >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((PT_SBO >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version (Blackwell); layout bits 61-63 = 0: no swizzle
    return d;
}
// D[:, col .. col+n) -= Ph Ph^T + Ph Pl^T + Pl Ph^T restricted to B rows col .. col+n
__device__ __forceinline__ void schur_mma(uint32_t tmem, uint32_t ph, uint32_t pl, int col, int n) {
    const uint32_t id = idesc_tf32(128, n) | (1u << 13);  // negate A: D -= A B^T
    const uint64_t ah = pt_desc(ph, 0), al = pt_desc(pl, 0), bh = pt_desc(ph, col), bl = pt_desc(pl, col);
    mma_tf32(tmem + col, ah, bh, id, 1u);
    mma_tf32(tmem + col, ah, bl, id, 1u);
    mma_tf32(tmem + col, al, bh, id, 1u);
}

// PROF: clock64() per phase, factor thread `opts` (slots 0-7) and the back-substitution warp's lane 0
// (8-9), into prof[blockIdx.x * TS_PROF_SLOTS + slot] (ALSK_TS_PROF=<thread>).
template <bool PROF>
__global__ void __launch_bounds__(TS_THREADS, 4)
tc_solve_kernel(const float* __restrict__ packed, int64_t count, int f, float* __restrict__ out_x,
                unsigned long long* __restrict__ min_row, int32_t* __restrict__ column,
                double* __restrict__ pivot, int64_t status_base, long long* __restrict__ prof,
                uint32_t sleep_ns, uint32_t opts, uint32_t mma_first_ns, uint32_t bs_ns) {
    uint32_t pcy[TS_PROF_SLOTS] = {};  // 32-bit: one launch of one CTA stays far below 2^32 cycles
    uint32_t tq = PROF ? static_cast<uint32_t>(clock()) : 0u;
    const uint32_t tstart = tq;
    auto lap = [&](int slot) {
        if constexpr (PROF) {
            const uint32_t now = static_cast<uint32_t>(clock());
            pcy[slot] += now - tq;
            tq = now;
        }
    };
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const TsPlan P(f);
    uint8_t* Ph = base;
    uint8_t* Pl = base + PT_BYTES;
    float* rowbuf = reinterpret_cast<float*>(base + P.rowbuf);
    float* lbuf = reinterpret_cast<float*>(base + P.lbuf);
    float* dinvb = reinterpret_cast<float*>(base + P.vec);  // [2][128]: 1 / L[c][c] of the systems in flight
    float* blk = reinterpret_cast<float*>(base + P.blk);     // 8x8 diagonal block, then M
    int* flags = reinterpret_cast<int*>(blk + 64);         // [0] breakdown column + 1, [1] pivot bits
    int* meta = flags + 4;                                 // [0] 1: system handed to the back substitution
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + P.bars);
    uint64_t* load_bar = bars;  // packed rows of the next system landed
    uint64_t* mma_bar = bars + 1;  // Schur update done (tiles free, trailing columns final)
    uint64_t* lfull = bars + 2;    // L / y / 1/diag of a system ready for the back substitution
    uint64_t* lfree = bars + 3;    // back substitution done with them
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

    const int i = threadIdx.x;
    const int warp = i >> 5, lane = i & 31;
    const int nbc = (f + 7) >> 3;
    const int N = (f + 15) & ~15;

    if (warp == 0) tmem_alloc<128>(tmem_slot);
    if (i == 0) {
        mbar_init(load_bar, 1);
        mbar_init(mma_bar, 1);
        mbar_init(lfull, 1);
        mbar_init(lfree, 1);
        fence_barrier_init();
    }
    for (int t = i; t < 2 * PT_BYTES / 16; t += TS_THREADS)
        reinterpret_cast<float4*>(base)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == BS_WARP) {
        // ---------------- back substitution L^T x = y, one system at a time ----------------
        uint32_t t = 0;
        for (int64_t g = blockIdx.x; g < count; g += gridDim.x, ++t) {
            ts_wait(lfull, t & 1u, bs_ns);  // long wait: leave the issue slots to the factor warps
            lap(9);
            if (meta[0]) {
                const float* dinv = dinvb + 128 * (t & 1u);
                constexpr int G = 4;  // 128 / 32 values per lane
                // lane j's cells of row ii of the panel-blocked dump sit at lb[g] + 8 ii
                int lb[G];
                float yv[G];
#pragma unroll
                for (int gq = 0; gq < G; ++gq) {
                    const int j = min(gq * 32 + lane, f - 1);
                    lb[gq] = static_cast<int>(pb_index(f, 0, j));
                    yv[gq] = gq * 32 + lane < f ? lbuf[lb[gq] + 8 * f] : 0.f;  // y = row f
                }
#pragma unroll
                for (int gq = G - 1; gq >= 0; --gq) {
                    for (int s = 31; s >= 0; --s) {
                        const int ii = gq * 32 + s;
                        if (ii >= f) continue;  // uniform
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
            lap(8);
        }
    } else {
        // ---------------- factor threads ----------------
        const uint32_t tlane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        // last row of my warp: TMEM blocks right of it are the upper part for the whole warp
        // (never read), so the warp skips their loads and stores
        const int wtop = 32 * warp + 31;
        const uint32_t row_bytes = static_cast<uint32_t>(P.pks) * 4;
        const uint32_t sPh = smem_u32(Ph), sPl = smem_u32(Pl);
        // row i's two 16-byte K chunks in the panel tiles
        const uint32_t pc0 = static_cast<uint32_t>((i >> 3) * PT_SBO + (i & 7) * 16), pc1 = pc0 + PT_LBO;
        uint32_t ph_load = 0, ph_mma = 0;
        auto issue_load = [&](int64_t gg) {  // thread 0: bulk-copy a system's packed row
            expect_tx(load_bar, row_bytes);
            bulk_g2s(smem_u32(rowbuf), packed + gg * P.pks, row_bytes, load_bar);
        };
        // my row of the system in rowbuf into TMEM (panel-blocked; row f = b); nz: a nonzero
        // A entry in my row
        auto fill = [&](int& nz) {
            ts_wait(load_bar, ph_load, sleep_ns);
            ph_load ^= 1u;
            uint32_t bits = 0;
            for (int b = 0; b < nbc && 8 * b <= wtop; ++b) {
                float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if (i >= 8 * b && i <= f) {
                    const float4* src = reinterpret_cast<const float4*>(rowbuf + pb_block(f, b) + 8 * (i - 8 * b));
                    const float4 u = src[0], w = src[1];
                    v[0] = u.x, v[1] = u.y, v[2] = u.z, v[3] = u.w, v[4] = w.x, v[5] = w.y, v[6] = w.z, v[7] = w.w;
#pragma unroll
                    for (int q = 0; q < 8; ++q) bits |= __float_as_uint(v[q]) << 1;  // +-0 -> 0
                }
                tmem_st8(tlane + 8 * b, v);
            }
            nz = i < f && bits != 0;
            tmem_st_wait();
        };
        int64_t g = blockIdx.x;
        if (i == 0 && g < count) issue_load(g);
        int nz = 0;
        if (g < count) fill(nz);
        lap(6);
        uint32_t t = 0;
        for (; g < count; g += gridDim.x, ++t) {
            float* dinv = dinvb + 128 * (t & 1u);
            tc_fence_before();
            bool active = bar_red_or(BAR_FACTOR, TS_FACTOR, nz != 0);  // all-zero A: x = 0 (solver.hpp:215-220)
            tc_fence_after();
            if (i == 0 && g + gridDim.x < count) issue_load(g + gridDim.x);  // rowbuf is free
            if (!active) {
                if (i < f) out_x[g * f + i] = 0.f;
                if (i == 0) column[g] = 0;
            }
            lap(10);
            for (int bc = 0; active && bc < nbc; ++bc) {
                const int r0 = 8 * bc;
                const bool wlive = wtop >= r0;  // warp-uniform: some row of my warp at or below the block
                tc_fence_after();
                float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if (wlive) {
                    tmem_ld8(tlane + r0, a);
                    tmem_ld_wait();
                }
                // (1) diagonal rows -> shared memory; the lane of row r0 factors the block (a
                //     warp sync suffices: the rest of the CTA waits at the barrier below)
                if (i >= r0 && i < r0 + 8) {
                    *reinterpret_cast<float4*>(&blk[(i - r0) * 8]) = make_float4(a[0], a[1], a[2], a[3]);
                    *reinterpret_cast<float4*>(&blk[(i - r0) * 8 + 4]) = make_float4(a[4], a[5], a[6], a[7]);
                }
                if (warp == (r0 >> 5)) __syncwarp();
                lap(0);
                if (i == r0) {
                    float l[8][8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 u = *reinterpret_cast<const float4*>(&blk[q * 8]);
                        const float4 w = *reinterpret_cast<const float4*>(&blk[q * 8 + 4]);
                        l[q][0] = u.x, l[q][1] = u.y, l[q][2] = u.z, l[q][3] = u.w;
                        l[q][4] = w.x, l[q][5] = w.y, l[q][6] = w.z, l[q][7] = w.w;
                    }
                    // branch-free right-looking 8x8 Cholesky; a non-positive pivot poisons what
                    // follows it, which the check below discards with the whole system
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
                    float badv = 0.f;
#pragma unroll
                    for (int c = 7; c >= 0; --c)  // first real column with a non-positive pivot
                        if (r0 + c < f && !(piv[c] > 0.f)) {
                            bad = r0 + c + 1;
                            badv = piv[c];
                        }
                    // M = diag(1/L_cc) L_cc, rows of padding columns zero
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const bool real = r0 + c < f;  // padding rows of M stay exactly zero
                        float m[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) m[k] = !real ? 0.f : (k < c ? l[c][k] * dv[c] : (k == c ? dv[c] : 0.f));
                        *reinterpret_cast<float4*>(&blk[c * 8]) = make_float4(m[0], m[1], m[2], m[3]);
                        *reinterpret_cast<float4*>(&blk[c * 8 + 4]) = make_float4(m[4], m[5], m[6], m[7]);
                        dinv[r0 + c] = dv[c];
                    }
                    flags[0] = bad;
                    flags[1] = __float_as_int(badv);
                }
                named_barrier(BAR_FACTOR, TS_FACTOR);
                lap(1);
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
                lap(12);
                const bool update = bc + 1 < nbc;  // no trailing columns after the last block
                // (2) my row of L (rows at or below the block, including row f = y); lanes above
                //     keep their entries (upper-part or padding cells that are never read)
                float L[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) L[c] = a[c];
                if (i >= r0 && i <= f) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 u = *reinterpret_cast<const float4*>(&blk[c * 8]);
                        const float4 w = *reinterpret_cast<const float4*>(&blk[c * 8 + 4]);
                        const float mc[8] = {u.x, u.y, u.z, u.w, w.x, w.y, w.z, w.w};
                        float s = a[c] * mc[c];
#pragma unroll
                        for (int k = 0; k < c; ++k) s = fmaf(-L[k], mc[k], s);
                        L[c] = (i - r0 >= c || i == f) ? s : 0.f;  // diagonal-block rows: lower part
                    }
                }
                lap(13);
                if (wlive) tmem_st8(tlane + r0, L);  // .sync.aligned: every lane of the warp stores
                lap(2);
                if (update) {
                    // panel operand: rows below the block only (factored rows contribute nothing)
                    float h[8], lo[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float pv = (i >= r0 + 8 && i <= f) ? L[c] : 0.f;
                        h[c] = rna_tf32(pv);
                        lo[c] = pv - h[c];  // exact; the MMA reads its leading tf32 bits
                    }
                    if (wlive) {  // rows of a dead warp were zeroed when its rows left the panel
                        *reinterpret_cast<float4*>(Ph + pc0) = make_float4(h[0], h[1], h[2], h[3]);
                        *reinterpret_cast<float4*>(Ph + pc1) = make_float4(h[4], h[5], h[6], h[7]);
                        *reinterpret_cast<float4*>(Pl + pc0) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                        *reinterpret_cast<float4*>(Pl + pc1) = make_float4(lo[4], lo[5], lo[6], lo[7]);
                    }
                    fence_proxy_async_smem();
                }
                tmem_st_wait();
                tc_fence_before();
                named_barrier(BAR_FACTOR, TS_FACTOR);
                lap(3);
                if (update) {
                    if (i == 0) {
                        tc_fence_after();
                        schur_mma(tmem, sPh, sPl, 0, N);
                        mma_commit(mma_bar);
                    }
                    ts_wait_first(mma_bar, ph_mma, mma_first_ns, sleep_ns);  // MMA round trip >= ~500 cycles
                    ph_mma ^= 1u;
                }
                lap(4);
            }
            // hand the factor to the back-substitution warp: L (packed lower) into lbuf once
            // it is done with the previous system
            if (t > 0) ts_wait(lfree, (t - 1) & 1u, sleep_ns);
            if (active) {
                for (int b = 0; b < nbc && 8 * b <= wtop; ++b) {
                    tc_fence_after();
                    float lv[8];
                    tmem_ld8(tlane + 8 * b, lv);
                    tmem_ld_wait();
                    if (i >= 8 * b && i <= f) {
                        float4* dst = reinterpret_cast<float4*>(lbuf + pb_block(f, b) + 8 * (i - 8 * b));
                        dst[0] = make_float4(lv[0], lv[1], lv[2], lv[3]);
                        dst[1] = make_float4(lv[4], lv[5], lv[6], lv[7]);
                    }
                }
            }
            if (i == 0) meta[0] = active ? 1 : 0;
            named_barrier(BAR_FACTOR, TS_FACTOR);
            if (i == 0) mbar_arrive(lfull);
            lap(5);
            if (g + gridDim.x < count) {
                tc_fence_after();
                fill(nz);
            }
            lap(6);
        }
    }
    if constexpr (PROF) {
        const int pt = static_cast<int>(opts);  // profiled factor thread
        pcy[7] = static_cast<uint32_t>(clock()) - tstart;
        pcy[11] = pcy[7];
        // constant indices only: pcy stays in registers
#pragma unroll
        for (int q = 0; q < TS_PROF_SLOTS; ++q) {
            const bool bs = q == 8 || q == 9;
            if ((i == pt && !bs) || (i == 32 * BS_WARP && bs)) prof[blockIdx.x * TS_PROF_SLOTS + q] = pcy[q];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<128>(tmem);
    }
}

void launch_solve(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                  cudaStream_t s) {
    const TsPlan P(f);
    // at least 46 KB of shared memory per CTA: never more than 4 CTAs (4 x 128 TMEM columns)
    // on an SM, so no CTA waits in tcgen05.alloc for another to finish
    const int smem = static_cast<int>(std::max<size_t>(P.total, 46 * 1024));
    static const int per_sm = [] {  // CTAs per SM (A/B switch for latency measurements; at most 4)
        const char* e = measure_env("ALSK_TS_CTAS");
        return e ? std::max(1, std::min(4, std::atoi(e))) : 4;
    }();
    static const bool want_prof = measure_env("ALSK_TS_PROF") != nullptr;
    // persistent CTAs with a static system assignment: never launch more than are resident
    // at once (large f: shared memory allows only 3 or 2 per SM), or the extra CTAs run as a
    // second wave after the others
    int resident = 0;
    ALSK_CUDA(cudaFuncSetAttribute(tc_solve_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // CTAs that fit an SM's shared memory (228 KB, 1 KB reserved per CTA + 1 KB static);
    // cudaOccupancyMaxActiveBlocksPerMultiprocessor reports 1 for this kernel, which is not
    // what the hardware runs
    resident = static_cast<int>((228 * 1024) / (smem + 2 * 1024));
    const int ctas_per_sm = std::max(1, std::min(per_sm, resident));
    static bool said = false;
    if (!said && measure_env("ALSK_TS_VERBOSE")) {
        std::fprintf(stderr, "[tc_solve] f=%d smem=%d resident=%d ctas_per_sm=%d\n", f, smem, resident, ctas_per_sm);
        said = true;
    }
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(count, ctas_per_sm * static_cast<int64_t>(num_sms())));
    // back-off of the factor threads' short waits (MMA completion, hand-off, loads)
    // ALSK_TS_WAITS=mma_first,backsub (ns): first sleep of the MMA wait, back-substitution poll
    static const std::array<uint32_t, 2> tun = [] {
        std::array<uint32_t, 2> v{200u, 1000u};
        if (const char* e = measure_env("ALSK_TS_WAITS")) {
            unsigned a = 0, b = 0;
            if (std::sscanf(e, "%u,%u", &a, &b) == 2) v = {a, b};
        }
        return v;
    }();
    static const uint32_t sleep_ns = [] {
        const char* e = measure_env("ALSK_TS_SLEEP");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 32u;  // parking (0) measured slower
    }();
    // ALSK_TS_PROF=<factor thread>: whose phases the profile reports
    const uint32_t opts = want_prof ? static_cast<uint32_t>(std::atoi(measure_env("ALSK_TS_PROF")) & 127) : 0u;
    if (!want_prof) {
        ALSK_CUDA(cudaFuncSetAttribute(tc_solve_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        tc_solve_kernel<false><<<grid, TS_THREADS, smem, s>>>(packed, count, f, x, st.min_row, st.column + status_off,
                                                              st.pivot + status_off, status_off, nullptr, sleep_ns, opts,
                                                              tun[0], tun[1]);
        ALSK_LAUNCHED();
        return;
    }
    ALSK_CUDA(cudaFuncSetAttribute(tc_solve_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    DevBuf prof;
    prof.alloc(sizeof(long long) * grid * TS_PROF_SLOTS, s);
    ALSK_CUDA(cudaMemsetAsync(prof.as<void>(), 0, sizeof(long long) * grid * TS_PROF_SLOTS, s));
    tc_solve_kernel<true><<<grid, TS_THREADS, smem, s>>>(packed, count, f, x, st.min_row, st.column + status_off,
                                                         st.pivot + status_off, status_off, prof.as<long long>(), sleep_ns, opts,
                                                         tun[0], tun[1]);
    ALSK_LAUNCHED();
    std::vector<long long> h(static_cast<size_t>(grid) * TS_PROF_SLOTS);
    ALSK_CUDA(cudaMemcpyAsync(h.data(), prof.as<void>(), h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s));
    ALSK_CUDA(cudaStreamSynchronize(s));
    double acc[TS_PROF_SLOTS] = {};
    for (unsigned c = 0; c < grid; ++c)
        for (int q = 0; q < TS_PROF_SLOTS; ++q) acc[q] += static_cast<double>(h[c * TS_PROF_SLOTS + q]);
    for (double& v : acc) v /= static_cast<double>(count) * 1e3;
    std::fprintf(stderr,
                 "[ts-prof f=%d rows=%lld grid=%u] kcyc/system: diag %.2f potrf %.2f trsm %.2f panel %.2f mma %.2f "
                 "handoff %.2f fill %.2f start %.2f | total %.2f | backsub %.2f bs-wait %.2f | flags %.2f trsm-math %.2f\n",
                 f, static_cast<long long>(count), grid, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], acc[6],
                 acc[10], acc[11], acc[8], acc[9], acc[12], acc[13]);
}

}  // namespace

bool packed_solve(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                  cudaStream_t s) {
    static const bool tiles = measure_env("ALSK_SOLVE_TILES") != nullptr;  // A/B switches for measurements
    static const bool tmem = measure_env("ALSK_SOLVE_TMEM") != nullptr;
    if (tiles) return packed_solve_tiles(packed, count, f, x, st, status_off, s);
    if (!tmem && warp_solve(packed, count, f, x, st, status_off, s)) return true;
    if (f < 8 || f > 127) return packed_solve_tiles(packed, count, f, x, st, status_off, s);
    if (count <= 0) return true;
    launch_solve(packed, count, f, x, st, status_off, s);
    return true;
}

}  // namespace alsk
