// Tensor-core get_hermitian + get_bias (ALSK_PREC_TF32X2): tcgen05 kind::tf32 with a two-term
// split, one persistent CTA per SM. Writes A_u (+ lambda n_u) and B_u either in the
// get_hermitian layout (MODE_FULL) or lower-packed for the batched TMEM Cholesky solve of
// tc_solve.cu (MODE_PACKED, the half-sweep path).
//
// Replaces, for this precision, assemble_mo_rows (solver.hpp:99-157) in the loop body of
// update_x (solver.hpp:336-344); batch_solve_into (solver.hpp:204-262) is tc_solve.cu.
//
// Arithmetic. The gathered rows are augmented with the rating, theta'_k = [theta_k, r_k]
// (f+1 features), and every entry is split x = h + l, h = rna_tf32(x), l = rna_tf32(x - h).
// Two MMAs per 8-rating k-step: D += H^T [H | L] (M = 128, N = 2*NF, NF = round16(f+1)) and
// D1 += L^T H (N = NF, into the second half), so with D = [D0 | D1]:
//   D0 + D1 = H^T H + H^T L + L^T H = sum_k theta'_k theta'_k^T
// up to the dropped L^T L term (2^-22 relative), both halves symmetric: the lane owning row
// i reads its lower-triangle cells directly, no transpose. Rows < f are A_u
// (solver.hpp:130-140), row f is B_u (the bias rides along, solver.hpp:137).
// The tensor core's FP32 accumulation truncates, which biases long sums; rows longer than
// SEG_CHUNKS x 32 ratings are therefore accumulated in segments, each drained from TMEM and
// added into a per-group shared-memory row (panel-blocked lower triangle) with
// round-to-nearest FP32 adds.
//
// Warp roles (576 threads, 1 CTA per SM, rows j = blockIdx.x + t*gridDim.x):
//   warps 0-3  : the epilogue group (NG = 1; the code supports NG groups taking rows
//                t % NG). Lane i reads row i's lower cells from TMEM (segment sums in shared
//                memory) and writes A_u + lambda n_u and B_u to HBM, 32 bytes per lane and
//                8-column block.
//   warps 4-15 : split warps: read the staged rating-major rows, split tf32 hi/lo and
//                write them transposed into the K-major operand tile (lane = rating), with
//                zero padding of partial k-groups.
//   warp 16    : MMA issuer (one thread), owns the TMEM allocation (2 buffers x 256 columns).
//   warp 17    : loader, the only reader of the CSR arrays (8-chunk register prefetch queue of
//                column indices and ratings); the factor rows arrive by TMA tile::gather4, four
//                rows per instruction, into a staging ring of 4-row groups, completion counted
//                as transaction bytes on the stage mbarrier. Padding rows of a partial k-group
//                gather a row past the tensor map and arrive as zeros.
// Pipelines: staging ring (raw_full / raw_empty, 8 deep), operand ring (hl_full / hl_empty,
// 2 deep, released by tcgen05.commit; deeper rings measured slower) and the TMEM double
// buffer (tfull / tempty), one TMEM job per row segment. Ring positions are kept as counters
// (a runtime `% stages` per chunk in every role cost ~10% of the issue slots).
// The gather is not the bound any more: with per-lane cp.async (lane = rating, 16 bytes per
// instruction, 32 rows touched by each) the L1 handled one 16-byte request per clock and the
// loaders were busy ~90% of the kernel; TMA gather4 moves a 400-byte row in ~6 cycles per SM
// in isolation (scripts/probes/l2bw_probe.cu mode 7). What remains is the tensor pipe (the
// MMA issuer is busy ~46% of the kernel: 2.75 MFLOP of tcgen05 work per 32-rating chunk at
// f = 100, 8x the algorithmic flops because of M = 128 padding and the three split
// products) and the split warps' shared-memory traffic (~49%), overlapping imperfectly.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <array>
#include <vector>

#include "kernels.cuh"
#include "measure.cuh"
#include "tc_common.cuh"

namespace alsk {
namespace {
using namespace tc;

constexpr int KC = 32;                   // ratings per stage (four k-groups of 8)
constexpr int HL_BYTES = 256 * KC * 4;      // 32 KB: H rows [0,NF) then L rows [NF,2NF), K-major
constexpr int HL_STAGES_MAX = 2;           // operand-ring depth (measured: 2 58.5, 3 59.8, 4 60.2 ms/iter)
constexpr int SEG_CHUNKS = 16;              // TMEM accumulation segment: 16 x 32 ratings
#ifndef TC_NSPLIT
#define TC_NSPLIT 12
#endif
constexpr int NSPLIT = TC_NSPLIT;                // split warps (8 and 16 measured ~1% slower)
constexpr int NG = 1;                     // epilogue groups (two measured 1% slower once the epilogue
                                          // lost its transpose; with it, one was 12% slower)
constexpr int W_SPLIT = 4 * NG, W_MMA = W_SPLIT + NSPLIT, W_LOAD = W_MMA + 1;
#ifndef TC_NLOAD
#define TC_NLOAD 1
#endif
constexpr int NLOAD = TC_NLOAD;           // loader warps (each issues its share of a chunk's TMA gathers)
#ifndef TC_QUEUE
#define TC_QUEUE 8                        // chunks of CSR indices/ratings in flight in the loader
#endif
constexpr int NWARPS = W_LOAD + NLOAD;
constexpr int NTHREADS = 32 * NWARPS;     // 4*NG epilogue + NSPLIT split + MMA + NLOAD loader warps
constexpr int TMEM_COLS = 512;           // two buffers x 256 columns (D0 @ +0, D1 @ +NF)

// ---- shared-memory plan (host and device agree) ----
// A stage holds KC gathered factor rows as KC/4 TMA gather4 groups: 4 rows of ldt floats
// back to back, each group padded to a 128-byte boundary (the TMA destination alignment).
__host__ __device__ inline int group_stride(int ldt) { return (16 * ldt + 127) & ~127; }

struct TcPlan {
    int f, stages, nb, hls, gs, raw_bytes;
    int s_floats, grp_floats;
    size_t hl_off, ring_bytes, grp_bytes, bar_off, info_off, total;
    __host__ __device__ TcPlan(int f_, int nb_, int stages_, int ldt, int hls_)
        : f(f_), stages(stages_), nb(nb_), hls(hls_) {
        gs = group_stride(ldt);
        raw_bytes = (KC / 4) * gs;
        s_floats = static_cast<int>(packed_stride(f));  // segment sums, panel-blocked (kernels.cuh)
        grp_floats = s_floats;
        hl_off = (static_cast<size_t>(stages) * raw_bytes + 1023) & ~static_cast<size_t>(1023);  // UMMA atoms: 1 KB
        ring_bytes = hl_off + static_cast<size_t>(hls) * HL_BYTES;
        grp_bytes = static_cast<size_t>(grp_floats) * 4;
        bar_off = (ring_bytes + NG * grp_bytes + 15) & ~static_cast<size_t>(15);
        info_off = bar_off + static_cast<size_t>(2 * stages + 2 * hls + 6) * 8 + 16;
        total = info_off + static_cast<size_t>(stages) * (KC * 4 + 16) + hls * 16 + 1024;  // + align slack
    }
};

// 4 factor rows (r0..r3, full width) into shared memory by one TMA gather, completion as
// transaction bytes on `bar`; rows at or past the map's row count arrive as zeros
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

// spin (ns == 0), park in try_wait with a suspend-time hint (ns == 1) or nanosleep back-off
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity, uint32_t ns) {
    if (ns == 0) mbar_wait(bar, parity);
    else if (ns == 1) mbar_wait_park(bar, parity);
    else mbar_wait_sleep(bar, parity, ns);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// Metadata the TMA warp forwards with every staged chunk (and the split warps with every
// operand stage): rating count (-1 = end of work) and segment flags for the MMA issuer.
struct ChunkInfo {
    int cnt;
    uint32_t flags;  // bit0: first chunk of a TMEM segment, bit1: last, bit2: owner group
    int pad0, pad1;
};
constexpr uint32_t CH_FIRST = 1u, CH_LAST = 2u, CH_OWNER1 = 4u;

// Walks the CTA's chunk sequence (rows j = blockIdx.x + t*gridDim.x, 32 ratings per chunk,
// empty rows skipped) for one warp. Row extents come in batches of 32 rows, one row per
// lane: the next batch's row_ptr loads are issued when the current batch starts, so a row
// change is a register shuffle, never a dependent global load.
struct ChunkWalker {
    const int64_t* row_ptr;
    int64_t rb, nrows;
    int64_t ck0, ck1, nk0, nk1;  // this lane's row of the current / next batch
    int64_t k0, n, c0;
    int batch, slot, t;
    bool live;
    __device__ void fetch(int b, int64_t& a0, int64_t& a1) const {
        const int64_t j = blockIdx.x + static_cast<int64_t>(gridDim.x) * (32 * b + (threadIdx.x & 31));
        a0 = a1 = 0;
        if (j < nrows) {
            a0 = row_ptr[rb + j];
            a1 = row_ptr[rb + j + 1];
        }
    }
    __device__ void seek() {  // from (batch, slot) to the first non-empty row, or the end
        for (;;) {
            const int64_t j = blockIdx.x + static_cast<int64_t>(gridDim.x) * (32 * batch + slot);
            if (j >= nrows) {
                live = false;
                return;
            }
            k0 = __shfl_sync(0xffffffffu, ck0, slot);
            n = __shfl_sync(0xffffffffu, ck1, slot) - k0;
            c0 = 0;
            t = 32 * batch + slot;
            if (n > 0) return;
            if (++slot == 32) next_batch();
        }
    }
    __device__ void next_batch() {
        ++batch;
        slot = 0;
        ck0 = nk0;
        ck1 = nk1;
        fetch(batch + 1, nk0, nk1);
    }
    __device__ ChunkWalker(const int64_t* rp, int64_t rb_, int64_t nrows_)
        : row_ptr(rp), rb(rb_), nrows(nrows_), batch(0), slot(0), t(0), live(true) {
        fetch(0, ck0, ck1);
        fetch(1, nk0, nk1);
        seek();
    }
    __device__ bool valid() const { return live; }
    __device__ ChunkInfo info() const {
        ChunkInfo ci{};
        if (!live) {
            ci.cnt = -1;
            return ci;
        }
        const int64_t left = n - c0;
        ci.cnt = left < KC ? static_cast<int>(left) : KC;
        const int64_t ch = c0 / KC;
        ci.flags = ((ch % SEG_CHUNKS) == 0 ? CH_FIRST : 0u) |
                   ((c0 + KC >= n || (ch % SEG_CHUNKS) == SEG_CHUNKS - 1) ? CH_LAST : 0u) | ((t % NG) ? CH_OWNER1 : 0u);
        return ci;
    }
    __device__ void advance() {
        c0 += KC;
        if (c0 >= n) {
            if (++slot == 32) next_batch();
            seek();
        }
    }
};

struct RowIter {  // the CTA's row sequence j = blockIdx.x + t * gridDim.x
    int64_t j, nrows;
    __device__ RowIter(int64_t nrows_) : j(blockIdx.x), nrows(nrows_) {}
    __device__ bool more() const { return j < nrows; }
    __device__ void next() { j += gridDim.x; }
};

__device__ __forceinline__ int64_t row_segments(int64_t n) {
    const int64_t nch = (n + KC - 1) / KC;
    return (nch + SEG_CHUNKS - 1) / SEG_CHUNKS;
}

// MODE_FULL: A (full, mirrored) + B rows (get_hermitian layout). MODE_PACKED: lower-packed A
// then B, panel-blocked (packed_stride(f) floats per row, kernels.cuh), for the batched solve
// (tc_solve.cu).
enum { MODE_FULL = 1, MODE_PACKED = 2 };

template <int NB, int MODE>
__global__ void __launch_bounds__(NTHREADS, 1)
tc_update_kernel(const __grid_constant__ CUtensorMap theta_map, int ldt, const int64_t* __restrict__ row_ptr,
                 const int32_t* __restrict__ col_idx, const float* __restrict__ values, int64_t col_lo, int theta_last, int f,
                 float lambda, int64_t rb, int64_t nrows, int stages, float* __restrict__ out_a,
                 float* __restrict__ out_b, long long* __restrict__ prof, int hls, uint32_t epi_sleep,
                 uint32_t load_sleep, uint32_t split_sleep, uint32_t mma_sleep, uint32_t dry) {
    // optional per-warp cycle accounting (ALSK_TC_PROF=1): pc[] slots per role, see launch_tc
    long long pc[6] = {0, 0, 0, 0, 0, 0};
    long long tp0 = 0;
#define TP(v) long long v = prof ? clock64() : 0
#define TA(v, slot) \
    if (prof) pc[slot] += clock64() - v
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* base = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    const TcPlan P(f, NB, stages, ldt, hls);
    const int RAW = P.raw_bytes;
    const int HL_STAGES = hls;
    // augmented features per operand half; a multiple of 16 keeps every 16-column TMEM load of
    // the second half aligned
    const int NF = (f + 1 + 15) & ~15;
    uint8_t* ring = base;                                    // stages x RAW: rating-major staging
    uint8_t* hl = base + P.hl_off;                           // HL_STAGES x HL_BYTES, 1 KB aligned
    float* grp0 = reinterpret_cast<float*>(base + P.ring_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + P.bar_off);
    uint64_t* raw_full = bars;
    uint64_t* raw_empty = bars + stages;
    uint64_t* hl_full = bars + 2 * stages;
    uint64_t* hl_empty = hl_full + HL_STAGES;
    // tfull[2*g + b]: a job for group g finished in TMEM buffer b. One barrier per (owner,
    // buffer) pair: jobs on a buffer drain in order, so each owner's barrier is at most one
    // phase ahead of it and parity waits cannot alias.
    uint64_t* tfull = hl_empty + HL_STAGES;
    uint64_t* tempty = tfull + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    ChunkInfo* raw_info = reinterpret_cast<ChunkInfo*>(base + P.info_off);  // [stages]
    float* raw_vals = reinterpret_cast<float*>(raw_info + stages);          // [stages][KC]
    ChunkInfo* hl_info = reinterpret_cast<ChunkInfo*>(raw_vals + stages * KC);  // [HL_STAGES]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&raw_full[s], NLOAD);  // one arrival per loader warp (+ the gathers' transaction bytes)
            mbar_init(&raw_empty[s], NSPLIT);
        }
        for (int s = 0; s < HL_STAGES; ++s) {
            mbar_init(&hl_full[s], NSPLIT);
            mbar_init(&hl_empty[s], 1);
        }
        for (int b = 0; b < 4; ++b) mbar_init(&tfull[b], 1);
        for (int b = 0; b < 2; ++b) mbar_init(&tempty[b], 4);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < static_cast<int>(P.ring_bytes / 16); i += NTHREADS)
        reinterpret_cast<float4*>(ring)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (warp == W_MMA) tmem_alloc<TMEM_COLS>(tmem_slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (prof) tp0 = clock64();

    if (warp >= W_LOAD) {
        // ---------------- loader (the only reader of the CSR arrays) ----------------
        // Walks the chunk sequence, lane = rating slot. A 4-deep register queue holds the
        // column indices and ratings of upcoming chunks, so their global loads are in flight
        // long before the chunk is staged. The factor rows are fetched by TMA: lanes 0..7
        // issue one tile::gather4 each (rows 4g..4g+3 of the chunk), completion counted as
        // transaction bytes on the stage's mbarrier; the padding slots of the last k-group
        // gather row `theta_rows` (past the map) and arrive as zeros. No per-lane copies:
        // the LSU/L1 stays free for the split warps.
        constexpr int D = TC_QUEUE;
        const int ldr = warp - W_LOAD;
        const int oob_row = theta_last + 1;
        const uint32_t row_bytes = static_cast<uint32_t>(ldt) * 4u;
        ChunkWalker w(row_ptr, rb, nrows);
        ChunkInfo qi[D];
        int qc[D];
        float qv[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            qi[d] = w.info();
            qc[d] = 0;
            qv[d] = 0.f;
            if (qi[d].cnt > 0 && lane < qi[d].cnt) {
                qc[d] = col_idx[w.k0 + w.c0 + lane];
                qv[d] = values[w.k0 + w.c0 + lane];
            }
            if (w.valid()) w.advance();
        }
        // Slot d of the queue is consumed and refilled in place (static register names): a
        // register holding an in-flight load is next read D chunks later, so the loads never
        // stall the loop.
        bool done = false;
        int ring_s = 0;  // stage and phase of the ring position (no runtime division per chunk)
        uint32_t ring_ph = 0;
        for (;;) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                if (done) break;
                const ChunkInfo ci = qi[d];
                // never gather outside Theta: an out-of-partition column is reported by the
                // caller's column check (solver.hpp:120-123), possibly after this launch
                const int v = lane < ci.cnt ? min(max(qc[d] - static_cast<int>(col_lo), 0), theta_last) : oob_row;
                const float rv = qv[d];
                qi[d] = w.info();
                qc[d] = 0;
                qv[d] = 0.f;
                if (qi[d].cnt > 0 && lane < qi[d].cnt) {
                    qc[d] = col_idx[w.k0 + w.c0 + lane];
                    qv[d] = values[w.k0 + w.c0 + lane];
                }
                if (w.valid()) w.advance();

                const int s = ring_s;
                const uint32_t ph = ring_ph;
                {
                    TP(t0);
                    tc_wait(&raw_empty[s], ph ^ 1u, load_sleep);
                    TA(t0, 0);
                }
                if (ldr == 0) {
                    raw_vals[s * KC + lane] = rv;
                    if (lane == 0) raw_info[s] = ci;
                }
                // loader ldr issues groups g = ldr, ldr + NLOAD, ... (lane q: g = ldr + NLOAD q)
                const int ngrp = ci.cnt > 0 ? ((ci.cnt + 7) & ~7) >> 2 : 0;
                const int mine = ngrp > ldr ? (ngrp - ldr + NLOAD - 1) / NLOAD : 0;
                const int g = (ldr + NLOAD * lane) & 7;
                const int r0 = __shfl_sync(0xffffffffu, v, 4 * g), r1 = __shfl_sync(0xffffffffu, v, 4 * g + 1);
                const int r2 = __shfl_sync(0xffffffffu, v, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, v, 4 * g + 3);
                __syncwarp();
                if (lane == 0) {
                    if (mine > 0) mbar_expect_tx(&raw_full[s], static_cast<uint32_t>(mine) * 4u * row_bytes);
                    else mbar_arrive(&raw_full[s]);
                }
                __syncwarp();
                if (lane < mine) tma_gather4(smem_u32(ring + s * RAW + g * P.gs), &theta_map, r0, r1, r2, r3, &raw_full[s]);
                if (ci.cnt < 0) done = true;
                if (++ring_s == stages) ring_s = 0, ring_ph ^= 1u;
            }
            if (done) break;
        }
    } else if (warp >= W_SPLIT && warp < W_MMA) {
        // ---------------- split warps ----------------
        // lane = rating slot k of the chunk; warp pw handles feature chunks c16 = pw + NSPLIT*t.
        // Every offset below is a per-thread constant plus a multiple of t.
        const int pw = warp - W_SPLIT;
        const int k = lane;
        const uint32_t raw_k = static_cast<uint32_t>((k >> 2) * P.gs + (k & 3) * ldt * 4 + pw * 16);
        uint32_t kq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r8 = 4 * (pw & 1) + q;  // feature & 7
            kq[q] = static_cast<uint32_t>((pw >> 1) * 1024 + r8 * 128 + ((((k >> 2) ^ r8)) << 4) + (k & 3) * 4);
        }
        const uint32_t l_off = static_cast<uint32_t>(NF * 128);
        // the rating slot (feature f) lives in chunk f>>2: warp (f>>2)%NSPLIT, step
        // (f>>2)/NSPLIT, element f&3
        const bool owns_r = pw == ((f >> 2) % NSPLIT);
        const int r8f = 4 * (pw & 1) + (f & 3);
        const uint32_t r_off = static_cast<uint32_t>((pw >> 1) * 1024 + r8f * 128 + ((((k >> 2) ^ r8f)) << 4) +
                                                     (k & 3) * 4 + ((f >> 2) / NSPLIT) * (NSPLIT * 512));
        constexpr int NC16 = 2 * NB;              // 16-byte feature chunks below 8*NB
        constexpr int TPW = (NC16 + NSPLIT - 1) / NSPLIT;  // chunks per split warp (upper bound)
        const int nc16 = NC16 < (NF >> 2) ? NC16 : (NF >> 2);  // never spill H rows into the L half
        int ring_s = 0, ring_hs = 0;
        uint32_t ring_ph = 0, ring_hph = 0;
        for (;; ring_s = ring_s + 1 == stages ? (ring_ph ^= 1u, 0) : ring_s + 1,
                ring_hs = ring_hs + 1 == HL_STAGES ? (ring_hph ^= 1u, 0) : ring_hs + 1) {
            const int s = ring_s;
            const int hs = ring_hs;
            TP(t0);
            tc_wait(&raw_full[s], ring_ph, split_sleep);
            TA(t0, 0);
            const ChunkInfo ci = raw_info[s];
            TP(t1);
            tc_wait(&hl_empty[hs], ring_hph ^ 1u, split_sleep);
            TA(t1, 1);
            TP(t2);
            if (ci.cnt >= 0 && !(dry & 1u)) {
                // Padding slots of the k-group were zeroed by the loader, so the split is
                // branch-free: h = rna_tf32(x), 2l = 2 rna_tf32(x - h) by bit ops.
                const uint8_t* __restrict__ raw = ring + s * RAW + raw_k;  // staging and operand
                uint8_t* __restrict__ H = hl + hs * HL_BYTES;                // tiles never alias
#pragma unroll
                for (int t = 0; t < TPW; ++t) {
                    if (pw + NSPLIT * t < nc16) {  // uniform per warp
                        const float4 x =
                            *reinterpret_cast<const float4*>(__builtin_assume_aligned(raw + t * (NSPLIT * 16), 16));
                        const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float h = __uint_as_float((__float_as_uint(xv[q]) + 0x1000u) & 0xFFFFE000u);
                            const float l = xv[q] - h;
                            const float lr = __uint_as_float((__float_as_uint(l) + 0x1000u) & 0xFFFFE000u);
                            uint8_t* dst = H + kq[q] + t * (NSPLIT * 512);
                            *reinterpret_cast<float*>(dst) = h;
                            *reinterpret_cast<float*>(dst + l_off) = lr;
                        }
                    }
                }
                if (owns_r) {  // overwrite feature f (zero column) with the rating
                    const float r = raw_vals[s * KC + k];
                    const float r_hi = tf32_rna(r), r_lo = tf32_rna(r - r_hi);
                    *reinterpret_cast<float*>(H + r_off) = r_hi;
                    *reinterpret_cast<float*>(H + r_off + l_off) = r_lo;
                }
                TA(t2, 2);
                TP(t3);
                fence_proxy_async_smem();
                TA(t3, 3);
            }
            if (pw == 0 && lane == 0) hl_info[hs] = ci;
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&raw_empty[s]);
                mbar_arrive(&hl_full[hs]);
            }
            if (ci.cnt < 0) break;
        }
    } else if (warp == W_MMA) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc = idesc_tf32(128, 2 * NF), idesc1 = idesc_tf32(128, NF);
        uint32_t job = 0;
        int ring_hs = 0;
        uint32_t ring_hph = 0;
        for (;; ring_hs = ring_hs + 1 == HL_STAGES ? (ring_hph ^= 1u, 0) : ring_hs + 1) {
            const int hs = ring_hs;
            // every lane waits (a lane-0-only wait followed by a warp shuffle measured ~700
            // cycles of reconvergence per chunk)
            TP(t0);
            tc_wait(&hl_full[hs], ring_hph, mma_sleep);
            TA(t0, 0);
            const ChunkInfo ci = hl_info[hs];
            if (ci.cnt < 0) break;
            const uint32_t b = job & 1u;
            const uint32_t dcol = tmem + b * 256u;
            TP(t1);
            if (ci.flags & CH_FIRST) tc_wait(&tempty[b], ((job >> 1) & 1u) ^ 1u, mma_sleep);
            TA(t1, 1);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t hb = smem_u32(hl + hs * HL_BYTES);
                const int ksteps = (ci.cnt + 7) >> 3;
                TP(t2);
                for (int kb = 0; kb < ((dry & 2u) ? 0 : ksteps); ++kb) {
                    const uint32_t acc = (!(ci.flags & CH_FIRST) || kb > 0) ? 1u : 0u;
                    const uint64_t dh = sdesc_sw128(hb + kb * 32, 16, 1024);               // H rows
                    const uint64_t dl = sdesc_sw128(hb + NF * 128 + kb * 32, 16, 1024);    // L rows
                    mma_tf32(dcol, dh, dh, idesc, acc);        // [D0 | D1] (+)= H^T [H | L]
                    mma_tf32(dcol + NF, dl, dh, idesc1, 1u);   // D1 += L^T H
                }
                TA(t2, 2);
                TP(t3);
                mma_commit(&hl_empty[hs]);
                if (ci.flags & CH_LAST) mma_commit(&tfull[2 * ((ci.flags & CH_OWNER1) ? 1 : 0) + b]);
                TA(t3, 3);
            }
            __syncwarp();
            if (ci.flags & CH_LAST) ++job;
        }
    } else {
        // ---------------- epilogue groups ----------------
        // Lane e of the group owns matrix row e (TMEM lane e): its lower cells j <= e (row f:
        // j < f) are D0 + D1 of its own lane, so each lane writes its row's 8-column blocks
        // (panel-blocked, kernels.cuh) straight to HBM, 32 bytes per block, consecutive lanes
        // at consecutive addresses. Rows of several segments keep the running sums in the
        // group's shared-memory row (same layout, conflict-free 16-byte accesses).
        const int g = warp >> 2;
        const int e = threadIdx.x & 127;
        float* acc_row = grp0 + g * P.grp_floats;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int wtop = 32 * (warp & 3) + 31;                // last row of my warp
        const int nc16 = (min(wtop, f) >> 4) + 1;             // 16-column chunks holding my warp's lower cells
        const int nb_mine = e < f ? (e >> 3) + 1 : (e == f ? ((f - 1) >> 3) + 1 : 0);  // my 8-column blocks
        const int64_t pkn = packed_stride(f);
        uint32_t job = 0, use[2] = {0u, 0u};
        int t = 0;
        for (RowIter it(nrows); it.more(); it.next(), ++t) {
            const int64_t u = rb + it.j;
            const int64_t n = row_ptr[u + 1] - row_ptr[u];
            const uint32_t nseg = static_cast<uint32_t>(row_segments(n));
            if ((t % NG) != g) {
                job += nseg;
                continue;
            }
            const int64_t row = it.j;
            const float reg = lambda * static_cast<float>(n);  // float arithmetic as solver.hpp:141,152
            float* pk = out_a + row * pkn;                                   // MODE_PACKED
            float* a_out = out_a + row * static_cast<int64_t>(f) * f;        // MODE_FULL
            float* b_out = out_b + row * static_cast<int64_t>(f);
            if (n == 0) {
                if constexpr (MODE == MODE_FULL) {
                    for (int idx = e; idx < f * f; idx += 128) a_out[idx] = 0.f;
                    for (int j = e; j < f; j += 128) b_out[j] = 0.f;
                } else {
                    for (int64_t idx = e; idx < pkn; idx += 128) pk[idx] = 0.f;
                }
                continue;
            }
            for (uint32_t sg = 0; sg < nseg; ++sg, ++job) {
                const uint32_t b = job & 1u;
                const uint32_t dcol = tmem + b * 256u + lane_base;
                const bool first = sg == 0, last = sg + 1 == nseg;
                TP(t0);
                // long, latency-tolerant wait (the group has the other group's row as slack):
                // back off so the spinning does not take issue slots from the split warps
                tc_wait(&tfull[2 * g + b], use[b] & 1u, epi_sleep);
                TA(t0, 4);
                ++use[b];
                tc_fence_after();
                TP(t1);
                for (int c = 0; c < nc16; ++c) {
                    float d0[16], d1[16];
                    tmem_ld16(dcol + c * 16, d0);
                    tmem_ld16(dcol + NF + c * 16, d1);
                    tmem_ld_wait();
                    if (dry & 4u) {  // measurement switch: D treated as zero
#pragma unroll
                        for (int q = 0; q < 16; ++q) d0[q] = d1[q] = 0.f;
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int bk = 2 * c + h;  // 8-column block
                        if (bk >= nb_mine) continue;
                        float v[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const int j = 8 * bk + q;
                            const bool cell = e < f ? j <= e : j < f;
                            v[q] = cell ? d0[8 * h + q] + d1[8 * h + q] : 0.f;
                        }
                        const int64_t off = pb_block(f, bk) + 8 * (e - 8 * bk);
                        float4* accp = reinterpret_cast<float4*>(acc_row + off);
                        if (!first) {  // running sum of the earlier segments, round-to-nearest adds
                            const float4 p0 = accp[0], p1 = accp[1];
                            v[0] += p0.x, v[1] += p0.y, v[2] += p0.z, v[3] += p0.w;
                            v[4] += p1.x, v[5] += p1.y, v[6] += p1.z, v[7] += p1.w;
                        }
                        if (!last) {
                            accp[0] = make_float4(v[0], v[1], v[2], v[3]);
                            accp[1] = make_float4(v[4], v[5], v[6], v[7]);
                            continue;
                        }
                        if (e < f && (e >> 3) == bk) v[e & 7] += reg;  // lambda n_u on the diagonal
                        if constexpr (MODE == MODE_PACKED) {
                            float4* dst = reinterpret_cast<float4*>(pk + off);
                            dst[0] = make_float4(v[0], v[1], v[2], v[3]);
                            dst[1] = make_float4(v[4], v[5], v[6], v[7]);
                        } else {
                            // A written full from the lower triangle (row and its mirror), so it
                            // mirrors bit-exactly; B = row f
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const int j = 8 * bk + q;
                                if (e < f && j <= e) {
                                    a_out[static_cast<int64_t>(e) * f + j] = v[q];
                                    a_out[static_cast<int64_t>(j) * f + e] = v[q];
                                } else if (e == f && j < f) {
                                    b_out[j] = v[q];
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if ((e & 31) == 0) mbar_arrive(&tempty[b]);
                TA(t1, 4);
            }
        }
    }
    if (prof) {
        pc[5] = clock64() - tp0;
        if (lane == 0)
            for (int i = 0; i < 6; ++i) prof[(static_cast<int64_t>(blockIdx.x) * NWARPS + warp) * 6 + i] = pc[i];
    }
#undef TP
#undef TA
    tc_fence_before();
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// ---- host side ----
// TMA map of the factor rows for the loader's gathers: rows x ldt floats, one row per box
// row, out-of-range rows read as zeros. A factor without rows maps a zeroed dummy row (only
// empty rows can then be valid; anything else fails the caller's column check).
CUtensorMap factor_rows_map(const float* theta, int64_t theta_rows, int ldt) {
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        ALSK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw Failure(ALSK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    const void* base = theta;
    int64_t rows = theta_rows;
    if (!theta || theta_rows < 1) {
        static std::mutex mu;
        static std::vector<void*> dummies;  // per device, process lifetime (512 zero bytes)
        int dev = 0;
        ALSK_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lock(mu);
        if (dummies.size() <= static_cast<size_t>(dev)) dummies.resize(dev + 1, nullptr);
        if (!dummies[dev]) {
            ALSK_CUDA(cudaMalloc(&dummies[dev], 512));
            ALSK_CUDA(cudaMemset(dummies[dev], 0, 512));
        }
        base = dummies[dev];
        rows = 1;
    }
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ldt), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldt) * 4};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(ldt), 1}, es[2] = {1, 1};
    // L2 promotion of the gathered rows: 64 B reads the fewest DRAM bytes (Netflix Theta half,
    // X gathered from HBM: 24.5 GB at 256 B, 23.0 at none or 128, 21.8 at 64; same time).
    // A/B: ALSK_TC_L2PROMO = 0 (none), 64, 128, 256
    static const CUtensorMapL2promotion promo = [] {
        const char* e = measure_env("ALSK_TC_L2PROMO");
        const int v = e ? std::atoi(e) : 64;
        return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                      : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }();
    const CUresult rc = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) throw Failure(ALSK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(rc)) + ")");
    return m;
}

template <int NB, int MODE>
void launch_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, int ldt, float lambda, int64_t rb,
               int64_t re, float* x, float* a, float* b, const SolveStatus* st, cudaStream_t s) {
    // deepest operand ring first (the MMA is fed by the split through it), then the staging ring
    static const int max_hls = [] {  // A/B switches for measurements
        const char* e = measure_env("ALSK_TC_HLS");
        return e ? std::max(2, std::min(HL_STAGES_MAX, std::atoi(e))) : HL_STAGES_MAX;
    }();
    static const int max_stages = [] {
        const char* e = measure_env("ALSK_TC_STAGES");
        return e ? std::max(2, std::min(8, std::atoi(e))) : 8;  // 8 vs 6: -0.3 ms per half with the TMA loader
    }();
    int hls = max_hls, stages = max_stages;
    for (;;) {
        while (stages > 2 && TcPlan(f, NB, stages, ldt, hls).total > 227 * 1024) --stages;
        if (stages >= 3 || hls == 2) break;
        --hls;
        stages = max_stages;
    }
    const TcPlan P(f, NB, stages, ldt, hls);
    // nanosleep back-off (ns, 0 = spin) of the waits of the epilogue, loader, split and MMA
    // warps (ALSK_TC_SLEEP=epi,load,split,mma)
    static const std::array<uint32_t, 4> sleeps = [] {
        std::array<uint32_t, 4> v{128u, 32u, 50u, 20u};
        if (const char* e = measure_env("ALSK_TC_SLEEP")) {
            unsigned a = 0, b = 0, c = 0, d = 0;
            if (std::sscanf(e, "%u,%u,%u,%u", &a, &b, &c, &d) == 4) v = {a, b, c, d};
        }
        return v;
    }();
    // ALSK_TC_DRY (measurements only, bit mask): 1 = split warps skip the split, 2 = no
    // MMAs, 4 = the epilogue treats D as zero
    static const uint32_t dry = [] {
        const char* e = measure_env("ALSK_TC_DRY");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
    }();
    auto k = tc_update_kernel<NB, MODE>;
    ALSK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(P.total)));
    const int64_t nrows = re - rb;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(nrows, num_sms()));
    static const bool want_prof = measure_env("ALSK_TC_PROF") != nullptr;
    DevBuf prof;
    if (want_prof) {
        prof.alloc(sizeof(long long) * grid * NWARPS * 6, s);
        ALSK_CUDA(cudaMemsetAsync(prof.as<void>(), 0, sizeof(long long) * grid * NWARPS * 6, s));
    }
    const CUtensorMap map = factor_rows_map(theta, theta_rows, ldt);
    k<<<grid, NTHREADS, P.total, s>>>(map, ldt, r.row_ptr, r.col_idx, r.values, r.col_offset,
                                       static_cast<int>(std::max<int64_t>(theta_rows, 1) - 1), f, lambda, rb, nrows, stages,
                                       a, b, want_prof ? prof.as<long long>() : nullptr, hls, sleeps[0], sleeps[1],
                                       sleeps[2], sleeps[3], dry);
    ALSK_LAUNCHED();
    if (want_prof) {
        std::vector<long long> h(static_cast<size_t>(grid) * NWARPS * 6);
        ALSK_CUDA(cudaMemcpyAsync(h.data(), prof.as<void>(), h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s));
        ALSK_CUDA(cudaStreamSynchronize(s));
        // per-role mean over CTAs (Mcycles): epilogue = warp 0, split = warp 8, mma = 12, tma = 13
        const char* names[4] = {"epi(w0): diag,panel,trail,backsub,pre,total",
                                "split: raw_full,hl_empty,work,fence,-,total",
                                "mma: hl_full,tempty,issue,commit,-,total", "load: raw_empty,-,-,-,-,total"};
        const int ws[4] = {0, W_SPLIT, W_MMA, W_LOAD};
        for (int r = 0; r < 4; ++r) {
            double acc[6] = {0, 0, 0, 0, 0, 0};
            for (unsigned c = 0; c < grid; ++c)
                for (int i = 0; i < 6; ++i) acc[i] += static_cast<double>(h[(static_cast<size_t>(c) * NWARPS + ws[r]) * 6 + i]);
            std::fprintf(stderr, "[tc-prof f=%d rows=%lld] %-46s", f, static_cast<long long>(nrows), names[r]);
            for (int i = 0; i < 6; ++i) std::fprintf(stderr, " %9.3f", acc[i] / grid / 1e6);
            std::fprintf(stderr, "\n");
        }
    }
}

struct Strided {
    const float* ptr;
    int ldt;
    DevBuf owned;
};
void strided(Strided& t, const float* theta, int64_t rows, int f, cudaStream_t s) {
    t.ptr = theta;
    t.ldt = f;
    if (f % 4 == 0 && (reinterpret_cast<uintptr_t>(theta) & 15) == 0) return;
    t.ldt = (f + 3) & ~3;
    const int64_t nr = std::max<int64_t>(rows, 1);
    t.owned.alloc(sizeof(float) * nr * t.ldt, s);
    ALSK_CUDA(cudaMemsetAsync(t.owned.as<void>(), 0, sizeof(float) * nr * t.ldt, s));
    if (rows > 0)
        ALSK_CUDA(cudaMemcpy2DAsync(t.owned.as<float>(), sizeof(float) * t.ldt, theta, sizeof(float) * f,
                                    sizeof(float) * f, rows, cudaMemcpyDeviceToDevice, s));
    t.ptr = t.owned.as<float>();
}

// get_hermitian on tensor cores (MODE_FULL), or the half-sweep as tensor-core Hermitian
// batches (MODE_PACKED into a device scratch) each followed by the batched packed solve.
template <int MODE>
bool dispatch_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb, int64_t re,
                 float* x, float* a, float* b, const SolveStatus* st, cudaStream_t s, const Scratch* ext = nullptr) {
    if (!tc_supported(f)) return false;
    if (re <= rb) return true;
    Strided th;
    strided(th, theta, theta_rows, f, s);
    const int nb = (f + 1 + 7) / 8;
    const int64_t pkn = packed_stride(f);
    // Packed-row scratch. A caller-owned workspace (sessions, alsk_workspace_*) is used as
    // is: stream-ordered, no lock, no host synchronisation. Otherwise the per-device default
    // scratch (ALSK_TC_SCRATCH_MB, default 4096 MB, grown on demand up to what the half
    // needs and halved on allocation failure) is shared by all callers of that device; they
    // are serialised on it until the stream has drained the batches that use it.
    static const int64_t scratch_mb = [] {
        const char* e = std::getenv("ALSK_TC_SCRATCH_MB");
        return e ? std::max<int64_t>(64, std::atoll(e)) : int64_t(4096);
    }();
    struct DefaultScratch {
        float* ptr = nullptr;
        size_t bytes = 0;
        std::mutex mu;
    };
    static DefaultScratch defaults[kMaxDevices];
    std::unique_lock<std::mutex> lock;
    float* scratch_p = nullptr;
    int64_t batch = re - rb;
    if (MODE == MODE_PACKED) {
        if (ext) {
            scratch_p = ext->ptr;
            batch = std::min<int64_t>(re - rb, std::max<int64_t>(1, static_cast<int64_t>(ext->bytes / (pkn * 4))));
        } else {
            int dev = 0;
            ALSK_CUDA(cudaGetDevice(&dev));
            DefaultScratch& d = defaults[dev % kMaxDevices];
            lock = std::unique_lock<std::mutex>(d.mu);
            int64_t want = std::min<int64_t>(re - rb, std::max<int64_t>(1, (scratch_mb << 20) / (pkn * 4)));
            if (d.bytes < sizeof(float) * want * pkn) {
                ALSK_CUDA(cudaStreamSynchronize(s));
                if (d.ptr) cudaFree(d.ptr);
                d.ptr = nullptr;
                d.bytes = 0;
                for (;;) {
                    const size_t need = sizeof(float) * want * pkn;
                    if (cudaMalloc(&d.ptr, need) == cudaSuccess) {
                        d.bytes = need;
                        break;
                    }
                    (void)cudaGetLastError();
                    if (want == 1) ALSK_CUDA(cudaErrorMemoryAllocation);
                    want = std::max<int64_t>(1, want / 2);  // retry with a smaller batch
                }
            }
            scratch_p = d.ptr;
            batch = std::min<int64_t>(re - rb, std::max<int64_t>(1, static_cast<int64_t>(d.bytes / (pkn * 4))));
        }
    }
    struct {
        float* p;
        float* as() const { return p; }
    } scratch{scratch_p};
#define ALSK_TC_CASE(NBV)                                                                              \
    if (nb <= NBV) {                                                                                   \
        if (MODE == MODE_FULL) {                                                                       \
            PhaseTimer pt(PHASE_HERMITIAN, s);                                                         \
            launch_tc<NBV, MODE_FULL>(r, th.ptr, theta_rows, f, th.ldt, lambda, rb, re, x, a, b, st, s); \
        } else {                                                                                       \
            for (int64_t b0 = rb; b0 < re; b0 += batch) {                                             \
                const int64_t b1 = std::min(re, b0 + batch);                                           \
                {                                                                                      \
                    PhaseTimer pt(PHASE_HERMITIAN, s);                                                 \
                    launch_tc<NBV, MODE_PACKED>(r, th.ptr, theta_rows, f, th.ldt, lambda, b0, b1, nullptr, \
                                                scratch.as(), nullptr, nullptr, s);              \
                }                                                                                      \
                PhaseTimer pt(PHASE_SOLVE, s);                                                         \
                packed_solve(scratch.as(), b1 - b0, f, x + (b0 - rb) * f, *st, b0 - rb, s);      \
            }                                                                                          \
            if (!ext) ALSK_CUDA(cudaStreamSynchronize(s)); /* the shared scratch is free again */    \
        }                                                                                              \
        return true;                                                                                   \
    }
    ALSK_TC_CASE(5)
    ALSK_TC_CASE(7)
    ALSK_TC_CASE(10)
    ALSK_TC_CASE(13)
    ALSK_TC_CASE(15)
#undef ALSK_TC_CASE
    return false;
}


}  // namespace

bool tc_supported(int f) { return f >= 16 && f <= 119; }  // 2*round16(f+1) <= 256, tiles <= 128

bool update_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb, int64_t re,
               float* x_out, const SolveStatus& st, cudaStream_t s, const Scratch* scratch) {
    return dispatch_tc<MODE_PACKED>(r, theta, theta_rows, f, lambda, rb, re, x_out, nullptr, nullptr, &st, s, scratch);
}

bool hermitian_packed_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
                         int64_t re, float* out_packed, cudaStream_t s) {
    if (!tc_supported(f)) return false;
    if (re <= rb) return true;
    Strided th;
    strided(th, theta, theta_rows, f, s);
    const int nb = (f + 1 + 7) / 8;
#define ALSK_TC_PK(NBV)                                                                                  \
    if (nb <= NBV) {                                                                                     \
        PhaseTimer pt(PHASE_HERMITIAN, s);                                                               \
        launch_tc<NBV, MODE_PACKED>(r, th.ptr, theta_rows, f, th.ldt, lambda, rb, re, nullptr, out_packed, nullptr, \
                                    nullptr, s);                                                         \
        return true;                                                                                     \
    }
    ALSK_TC_PK(5)
    ALSK_TC_PK(7)
    ALSK_TC_PK(10)
    ALSK_TC_PK(13)
    ALSK_TC_PK(15)
#undef ALSK_TC_PK
    return false;
}

bool hermitian_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb, int64_t re,
                  float* A, float* B, cudaStream_t s) {
    return dispatch_tc<MODE_FULL>(r, theta, theta_rows, f, lambda, rb, re, nullptr, A, B, nullptr, s);
}

}  // namespace alsk
