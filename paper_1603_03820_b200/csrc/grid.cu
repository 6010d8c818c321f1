// Scale-up (SU-ALS) plumbing on the device: grid partition indexing, the schedule-driven
// double reduction of partial Hermitians, the partitioned X update, and the packed
// partial-Hermitian / solve pair used by the data-parallel multi-GPU split.
//
//  grid_partition      sparse.hpp:250-314  per-row lower_bound of the column cuts; blocks
//                                          keep the parent's row-major order (bit-exact)
//  parallel_reduce     parallel.hpp:206-280, 436-477  any one-/two-phase schedule executed
//                                          per element with the reference's barrier
//                                          semantics and (dst, src)-sorted double adds
//  su_als_update_x     parallel.hpp:487-583  double partials -> reduce -> round once -> solve
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace alsk {

template <class T>
void exclusive_scan_ptr_i64(const T* in, int64_t n, int64_t* out, cudaStream_t s);

namespace {

// offs[u*(p+1)+i] = first position in row u (relative to row start) whose column >= cut[i]
__global__ void grid_offsets_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                    int64_t rows, const int64_t* __restrict__ cuts, int p,
                                    int64_t* __restrict__ offs, int64_t* __restrict__ counts) {
    for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < rows;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k0 = row_ptr[u], k1 = row_ptr[u + 1];
        int64_t prev = 0;
        for (int i = 0; i <= p; ++i) {
            int64_t lo = k0, hi = k1;
            const int64_t c = cuts[i];
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (col_idx[mid] < c) lo = mid + 1; else hi = mid;
            }
            const int64_t o = (i == p) ? (k1 - k0) : (lo - k0);
            offs[u * (p + 1) + i] = o;
            if (i > 0) counts[static_cast<int64_t>(i - 1) * rows + u] = o - prev;
            prev = o;
        }
    }
}

// copy the block (i, j) segments: warp per local row
__global__ void grid_fill_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                 const float* __restrict__ values, const int64_t* __restrict__ offs, int p, int i,
                                 int64_t r0, int64_t local_rows, const int64_t* __restrict__ brp,
                                 int32_t* __restrict__ bci, float* __restrict__ bv) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t lu = w0; lu < local_rows; lu += nw) {
        const int64_t u = r0 + lu;
        const int64_t src = row_ptr[u] + offs[u * (p + 1) + i];
        const int64_t len = offs[u * (p + 1) + i + 1] - offs[u * (p + 1) + i];
        const int64_t dst = brp[lu];
        for (int64_t e = lane; e < len; e += 32) {
            bci[dst + e] = col_idx[src + e];
            bv[dst + e] = values[src + e];
        }
    }
}

constexpr int kMaxWorkers = 32;

// One thread per element of one slice: replay the schedule (parallel.hpp:249-267).
// sched: for each phase, `n` transfers (src,dst) already filtered to this slice and sorted
// by (dst, src).
template <class In>
__global__ void reduce_schedule_kernel(const In* const* __restrict__ parts, int p, int64_t c0_elems,
                                       int64_t len, const int2* __restrict__ ph1, int n1,
                                       const int2* __restrict__ ph2, int n2, int slice,
                                       float* __restrict__ out_f, double* __restrict__ out_d) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < len;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double st[kMaxWorkers];
        double snap[kMaxWorkers];
        for (int w = 0; w < p; ++w) st[w] = static_cast<double>(parts[w][c0_elems + e]);
        for (int phase = 0; phase < 2; ++phase) {
            const int2* tr = phase == 0 ? ph1 : ph2;
            const int n = phase == 0 ? n1 : n2;
            for (int w = 0; w < p; ++w) snap[w] = st[w];
            for (int t = 0; t < n; ++t) st[tr[t].y] = st[tr[t].y] + snap[tr[t].x];
        }
        if (out_f) out_f[e] = static_cast<float>(st[slice]);
        if (out_d) out_d[e] = st[slice];
    }
}

__global__ void round_to_float_kernel(const double* __restrict__ in, int64_t n, float* __restrict__ out) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[e] = static_cast<float>(in[e]);
}

// packed lower (f(f+1)/2) + B (f) doubles -> full mirrored float A, float B
__global__ void unpack_packed_kernel(const double* __restrict__ packed, int64_t count, int f,
                                     float* __restrict__ A, float* __restrict__ B) {
    const int64_t per = static_cast<int64_t>(f) * (f + 1) / 2 + f;
    for (int64_t row = blockIdx.x; row < count; row += gridDim.x) {
        const double* src = packed + row * per;
        float* a = A + row * static_cast<int64_t>(f) * f;
        for (int e = threadIdx.x; e < f * f; e += blockDim.x) {
            const int i = e / f, j = e - i * f;
            const int hi = i > j ? i : j, lo = i > j ? j : i;
            a[e] = static_cast<float>(src[hi * (hi + 1) / 2 + lo]);
        }
        for (int i = threadIdx.x; i < f; i += blockDim.x)
            B[row * f + i] = static_cast<float>(src[f * (f + 1) / 2 + i]);
    }
}

int grid_blocks(int64_t n, int threads = 256) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148LL * 16)));
}

std::vector<int64_t> even_cuts(int64_t total, int parts) {  // sparse.hpp:95-100
    std::vector<int64_t> c(parts + 1);
    for (int k = 0; k <= parts; ++k) c[k] = total * k / parts;
    return c;
}

}  // namespace

// ------------------------------------------------------------------ grid partition ---
GridDevice grid_partition_device(const DevCsr& r, int p, int q, cudaStream_t s) {
    const int64_t qmax = std::max<int64_t>(r.rows, 1), pmax = std::max<int64_t>(r.cols, 1);
    if (q < 1 || q > qmax)
        fail_input("row partition count q=" + std::to_string(q) + " outside [1, " + std::to_string(qmax) + "]");
    if (p < 1 || p > pmax)
        fail_input("column partition count p=" + std::to_string(p) + " outside [1, " + std::to_string(pmax) + "]");
    GridDevice g;
    g.p = p;
    g.q = q;
    g.row_cuts = even_cuts(r.rows, q);
    g.col_cuts = even_cuts(r.cols, p);
    DevBuf cuts(sizeof(int64_t) * (p + 1), s);
    h2d(cuts.as<int64_t>(), g.col_cuts.data(), p + 1, s);
    g.offs.alloc(sizeof(int64_t) * std::max<int64_t>(r.rows, 1) * (p + 1), s);
    DevBuf counts(sizeof(int64_t) * std::max<int64_t>(r.rows, 1) * p, s);
    if (r.rows > 0) {
        grid_offsets_kernel<<<grid_blocks(r.rows), 256, 0, s>>>(r.row_ptr, r.col_idx, r.rows, cuts.as<int64_t>(), p,
                                                                 g.offs.as<int64_t>(), counts.as<int64_t>());
        ALSK_LAUNCHED();
    }
    g.block_row_ptr.resize(static_cast<size_t>(p) * q);
    g.block_nnz.assign(static_cast<size_t>(p) * q, 0);
    for (int j = 0; j < q; ++j) {
        const int64_t r0 = g.row_cuts[j], lr = g.row_cuts[j + 1] - r0;
        for (int i = 0; i < p; ++i) {
            DevBuf& brp = g.block_row_ptr[static_cast<size_t>(j) * p + i];
            brp.alloc(sizeof(int64_t) * (lr + 1), s);
            exclusive_scan_ptr_i64<int64_t>(counts.as<int64_t>() + static_cast<int64_t>(i) * r.rows + r0, lr,
                                            brp.as<int64_t>(), s);
            d2h(&g.block_nnz[static_cast<size_t>(j) * p + i], brp.as<int64_t>() + lr, 1, s);
        }
    }
    ALSK_CUDA(cudaStreamSynchronize(s));
    return g;
}

void grid_fill_block(const DevCsr& r, const GridDevice& g, int i, int j, int32_t* bci, float* bv,
                     cudaStream_t s) {
    const int64_t r0 = g.row_cuts[j], lr = g.row_cuts[j + 1] - r0;
    if (lr <= 0) return;
    grid_fill_kernel<<<grid_blocks(lr * 32), 256, 0, s>>>(r.row_ptr, r.col_idx, r.values, g.offs.as<int64_t>(), g.p,
                                                          i, r0, lr, g.block_row_ptr[static_cast<size_t>(j) * g.p + i].as<int64_t>(),
                                                          bci, bv);
    ALSK_LAUNCHED();
}

// ------------------------------------------------------------------ reduce schedule ---
ReduceSchedule build_reduce_schedule(int p, const int32_t* group_of, bool two_phase) {
    if (p < 1) fail_input("topology needs at least one worker");
    if (p > kMaxWorkers) fail_input("at most 32 workers are supported by the device reduction");
    ReduceSchedule sc;
    sc.p = p;
    std::vector<std::vector<int>> groups;
    if (!group_of) {
        groups.emplace_back();
        for (int w = 0; w < p; ++w) groups[0].push_back(w);
    } else {
        int ng = 0;
        for (int w = 0; w < p; ++w) {
            if (group_of[w] < 0) fail_input("group member " + std::to_string(w) + " outside worker range");
            ng = std::max(ng, group_of[w] + 1);
        }
        groups.assign(ng, {});
        for (int w = 0; w < p; ++w) groups[group_of[w]].push_back(w);
        for (const auto& g : groups)
            if (g.empty()) fail_input("empty worker group");
    }
    sc.phase1.assign(p, {});
    sc.phase2.assign(p, {});
    if (!two_phase) {  // parallel.hpp:443-447
        for (int slice = 0; slice < p; ++slice)
            for (int src = 0; src < p; ++src)
                if (src != slice) sc.phase1[slice].push_back({src, slice});
    } else {  // parallel.hpp:450-463
        if (groups.size() < 2) fail_input("two-phase reduction needs at least 2 worker groups");
        for (int slice = 0; slice < p; ++slice) {
            const int dst = slice;
            for (const auto& g : groups) {
                const bool home = std::find(g.begin(), g.end(), dst) != g.end();
                const int holder = home ? dst : g[static_cast<size_t>(slice) % g.size()];
                for (int w : g)
                    if (w != holder) sc.phase1[slice].push_back({w, holder});
                if (!home) sc.phase2[slice].push_back({holder, dst});
            }
        }
    }
    auto by_dst_src = [](const int2& a, const int2& b) { return a.y != b.y ? a.y < b.y : a.x < b.x; };
    for (int s2 = 0; s2 < p; ++s2) {
        std::sort(sc.phase1[s2].begin(), sc.phase1[s2].end(), by_dst_src);
        std::sort(sc.phase2[s2].begin(), sc.phase2[s2].end(), by_dst_src);
    }
    return sc;
}

std::vector<int64_t> slice_cuts(int64_t count, int p) {  // parallel.hpp:160-168
    const int64_t base = count / p, rem = count % p;
    std::vector<int64_t> c(p + 1, 0);
    for (int i = 0; i < p; ++i) c[i + 1] = c[i] + base + (i < rem ? 1 : 0);
    return c;
}

// parts: device pointers to p partial batches laid out [A (count*f*f) | B (count*f)].
// For slice i writes out_f[i] (float [A slice | B slice]) and/or out_d[i] (double).
template <class In>
void reduce_slices(const std::vector<const In*>& parts_a, const std::vector<const In*>& parts_b, int64_t count,
                   int f, const ReduceSchedule& sc, const std::vector<float*>& out_a,
                   const std::vector<float*>& out_b, cudaStream_t s) {
    const int p = sc.p;
    const auto cuts = slice_cuts(count, p);
    DevBuf pa(sizeof(void*) * p, s), pb(sizeof(void*) * p, s);
    h2d(reinterpret_cast<const In**>(pa.as<void>()), parts_a.data(), p, s);
    h2d(reinterpret_cast<const In**>(pb.as<void>()), parts_b.data(), p, s);
    const int64_t ff = static_cast<int64_t>(f) * f;
    for (int sl = 0; sl < p; ++sl) {
        const int64_t c0 = cuts[sl], n = cuts[sl + 1] - c0;
        if (n == 0) continue;
        const auto& t1 = sc.phase1[sl];
        const auto& t2 = sc.phase2[sl];
        DevBuf d1(sizeof(int2) * std::max<size_t>(t1.size(), 1), s), d2(sizeof(int2) * std::max<size_t>(t2.size(), 1), s);
        h2d(d1.as<int2>(), t1.data(), t1.size(), s);
        h2d(d2.as<int2>(), t2.data(), t2.size(), s);
        reduce_schedule_kernel<In><<<grid_blocks(n * ff), 256, 0, s>>>(
            reinterpret_cast<const In* const*>(pa.as<void>()), p, c0 * ff, n * ff, d1.as<int2>(),
            static_cast<int>(t1.size()), d2.as<int2>(), static_cast<int>(t2.size()), sl, out_a[sl], nullptr);
        ALSK_LAUNCHED();
        reduce_schedule_kernel<In><<<grid_blocks(n * f), 256, 0, s>>>(
            reinterpret_cast<const In* const*>(pb.as<void>()), p, c0 * f, n * f, d1.as<int2>(),
            static_cast<int>(t1.size()), d2.as<int2>(), static_cast<int>(t2.size()), sl, out_b[sl], nullptr);
        ALSK_LAUNCHED();
        ALSK_CUDA(cudaStreamSynchronize(s));  // d1/d2 are freed at scope exit
    }
}

template void reduce_slices<float>(const std::vector<const float*>&, const std::vector<const float*>&, int64_t,
                                   int, const ReduceSchedule&, const std::vector<float*>&,
                                   const std::vector<float*>&, cudaStream_t);
template void reduce_slices<double>(const std::vector<const double*>&, const std::vector<const double*>&, int64_t,
                                    int, const ReduceSchedule&, const std::vector<float*>&,
                                    const std::vector<float*>&, cudaStream_t);

void unpack_packed(const double* packed, int64_t count, int f, float* A, float* B, cudaStream_t s) {
    if (count <= 0) return;
    unpack_packed_kernel<<<static_cast<unsigned>(std::min<int64_t>(count, 148 * 64)), 128, 0, s>>>(packed, count, f, A, B);
    ALSK_LAUNCHED();
}

}  // namespace alsk
