// Synthetic ratings generated in HBM, row range by row range (SURVEY.md §8(d) generator;
// our own workload generator, not a reference routine). Bit-identical to the host generator
// alsk_synth_csr (host_data.cpp), so a rank can build exactly its own rows of the full
// matrix without the others: row u's degree, columns and values depend only on (seed, u).
//
//   synth_tstar_kernel  thread per column: the planted theta*_v (10 floats, SplitMix64 stream
//                       seeded mix_seed(seed_t, v))
//   synth_rows_kernel   warp per row: Floyd's sampling of d_u distinct columns from the row's
//                       SplitMix64 stream (the draws are uniform across the warp, the
//                       membership test is a 32-lane ballot over the chosen set in shared
//                       memory), rank sort (distinct keys: rank = number of smaller keys), then
//                       per entry the planted dot product + the row stream's noise draw of that
//                       rank. SplitMix64 is counter-based, so the k-th draw after Floyd is
//                       mix(state + (k+1) * gamma) and the lanes fill the row in parallel.
// Float arithmetic is the host's (no contraction: __fmul_rn / __fadd_rn, same order).
// Also here: the column-range filter the model-parallel Theta half uses to keep one rank's
// items of a row chunk (order-preserving ballot compaction, columns rebased to the range).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace alsk {
namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr int kPlanted = 10;
constexpr int kSynthWarps = 8;

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// common.hpp:70-75
__host__ __device__ inline uint64_t mix_seed_d(uint64_t seed, uint64_t salt) {
    return mix64(seed + kGamma * (salt + 1));
}
__device__ inline float unit_of(uint64_t v) { return static_cast<float>(v >> 40) * 0x1.0p-24f; }

__device__ inline int64_t row_start(int64_t nnz, int64_t m, int64_t u) {
    return static_cast<int64_t>((static_cast<unsigned __int128>(nnz) * static_cast<uint64_t>(u)) /
                                static_cast<uint64_t>(m));
}

__global__ void synth_tstar_kernel(uint64_t seed_t, int64_t n, float* __restrict__ tstar) {
    for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t s = mix_seed_d(seed_t, static_cast<uint64_t>(v));
#pragma unroll
        for (int i = 0; i < kPlanted; ++i) {
            s += kGamma;
            tstar[v * kPlanted + i] = __fmul_rn(unit_of(mix64(s)), 0.6f);
        }
    }
}

__global__ void __launch_bounds__(kSynthWarps * 32)
synth_rows_kernel(int64_t m, int64_t n, int64_t nnz, uint64_t seed, uint64_t seed_x, int64_t rb, int64_t re,
                  const float* __restrict__ tstar, int64_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx,
                  float* __restrict__ values) {
    __shared__ int32_t chosen_all[kSynthWarps][kSynthMaxDegree];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    int32_t* chosen = chosen_all[w];
    const int64_t base0 = row_start(nnz, m, rb);
    const int64_t warps = static_cast<int64_t>(gridDim.x) * kSynthWarps;
    for (int64_t u = rb + static_cast<int64_t>(blockIdx.x) * kSynthWarps + w; u < re; u += warps) {
        const int64_t b = row_start(nnz, m, u);
        const int d = static_cast<int>(row_start(nnz, m, u + 1) - b);
        if (lane == 0) row_ptr[u - rb] = b - base0;
        if (u == re - 1 && lane == 0) row_ptr[re - rb] = row_start(nnz, m, re) - base0;
        // Floyd's sampling (host_data.cpp alsk_synth_csr), every lane drawing the same values
        uint64_t s = mix_seed_d(seed, static_cast<uint64_t>(u));
        int cnt = 0;
        for (int64_t j = n - d; j < n; ++j) {
            const uint64_t range = static_cast<uint64_t>(j + 1);
            const uint64_t threshold = (0 - range) % range;
            uint64_t v;
            do {
                s += kGamma;
                v = mix64(s);
            } while (v < threshold);
            const int32_t t = static_cast<int32_t>(v % range);
            bool dup = false;
            for (int i = lane; i < cnt; i += 32) dup |= chosen[i] == t;
            dup = __any_sync(0xffffffffu, dup);
            if (lane == 0) chosen[cnt] = dup ? static_cast<int32_t>(j) : t;
            ++cnt;
            __syncwarp();
        }
        // planted x*_u (every lane keeps a copy)
        float xu[kPlanted];
        {
            uint64_t sx = mix_seed_d(seed_x, static_cast<uint64_t>(u));
#pragma unroll
            for (int i = 0; i < kPlanted; ++i) {
                sx += kGamma;
                xu[i] = __fmul_rn(unit_of(mix64(sx)), 0.6f);
            }
        }
        for (int i = lane; i < d; i += 32) {
            const int32_t c = chosen[i];
            int rank = 0;
            for (int k = 0; k < d; ++k) rank += chosen[k] < c;
            const float* tv = tstar + static_cast<int64_t>(c) * kPlanted;
            float dot = 0.f;
#pragma unroll
            for (int q = 0; q < kPlanted; ++q) dot = __fadd_rn(dot, __fmul_rn(xu[q], tv[q]));
            const float noise = __fsub_rn(unit_of(mix64(s + kGamma * static_cast<uint64_t>(rank + 1))), 0.5f);
            col_idx[b - base0 + rank] = c;
            values[b - base0 + rank] = __fadd_rn(dot, noise);
        }
        __syncwarp();
    }
}

// Column-range filter: entries of each row with lo <= col < hi, order preserved, columns
// rebased to col - lo. Pass 1 counts per row, pass 2 scatters (ballot ranks).
__global__ void filter_count_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t rows,
                                    int32_t lo, int32_t hi, int64_t* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < rows; u += warps) {
        int c = 0;
        for (int64_t k = rp[u] + lane; k < rp[u + 1]; k += 32) c += (ci[k] >= lo && ci[k] < hi) ? 1 : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) cnt[u] = c;
    }
}

__global__ void filter_scatter_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                      const float* __restrict__ vals, int64_t rows, int32_t lo, int32_t hi,
                                      const int64_t* __restrict__ orp, int32_t* __restrict__ oci,
                                      float* __restrict__ ov) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < rows; u += warps) {
        int64_t o = orp[u];
        for (int64_t k0 = rp[u]; k0 < rp[u + 1]; k0 += 32) {
            const int64_t k = k0 + lane;
            const bool valid = k < rp[u + 1];
            const int32_t c = valid ? ci[k] : 0;
            const bool keep = valid && c >= lo && c < hi;
            const uint32_t mk = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                oci[o + __popc(mk & lt)] = c - lo;
                ov[o + __popc(mk & lt)] = vals[k];
            }
            o += __popc(mk);
        }
    }
}

unsigned warp_grid(int64_t rows, int threads) {
    const int64_t want = (rows * 32 + threads - 1) / threads;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(num_sms()) * 16)));
}

}  // namespace

int64_t synth_row_start(int64_t nnz, int64_t m, int64_t u) {
    return static_cast<int64_t>((static_cast<unsigned __int128>(nnz) * static_cast<uint64_t>(u)) /
                                static_cast<uint64_t>(m));
}

void synth_rows_device(int64_t m, int64_t n, int64_t nnz, uint64_t seed, int64_t rb, int64_t re, int64_t* row_ptr,
                       int32_t* col_idx, float* values, cudaStream_t s) {
    if (m < 1 || n < 1 || nnz < 0) fail_input("invalid synthetic shape");
    if (n > 2147483647LL) fail_input("column count " + std::to_string(n) + " exceeds the 32-bit index range");
    if (rb < 0 || re > m || rb > re) fail_input("synthetic row range outside the matrix");
    const int64_t dmax = (nnz + m - 1) / m;  // degrees differ by at most one
    if (dmax > n) fail_input("invalid synthetic shape: a row would need more ratings than columns");
    if (dmax > kSynthMaxDegree)
        fail_input("synthetic row degree " + std::to_string(dmax) + " exceeds the device generator's " +
                   std::to_string(kSynthMaxDegree));
    if (re == rb) {
        const int64_t z = 0;
        h2d(row_ptr, &z, 1, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const uint64_t seed_x = mix_seed_d(seed, 1001), seed_t = mix_seed_d(seed, 1002);
    DevBuf tstar(sizeof(float) * n * kPlanted, s);
    synth_tstar_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, num_sms() * 8)), 256, 0, s>>>(
        seed_t, n, tstar.as<float>());
    ALSK_LAUNCHED();
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>((re - rb + kSynthWarps - 1) / kSynthWarps, int64_t(num_sms()) * 8)));
    synth_rows_kernel<<<grid, kSynthWarps * 32, 0, s>>>(m, n, nnz, seed, seed_x, rb, re, tstar.as<float>(), row_ptr,
                                                        col_idx, values);
    ALSK_LAUNCHED();
}

int64_t filter_columns_device(const DevCsr& r, int64_t lo, int64_t hi, int64_t* row_ptr_out, int32_t* col_idx_out,
                              float* values_out, cudaStream_t s) {
    if (lo < 0 || hi < lo || hi > r.cols) fail_input("column range outside the matrix");
    DevBuf cnt(sizeof(int64_t) * std::max<int64_t>(r.rows, 1), s);
    const unsigned grid = warp_grid(r.rows, 256);
    if (r.rows > 0) {
        filter_count_kernel<<<grid, 256, 0, s>>>(r.row_ptr, r.col_idx, r.rows, static_cast<int32_t>(lo),
                                                 static_cast<int32_t>(hi), cnt.as<int64_t>());
        ALSK_LAUNCHED();
    }
    exclusive_scan_ptr_i64<int64_t>(cnt.as<int64_t>(), r.rows, row_ptr_out, s);
    int64_t total = 0;
    d2h(&total, row_ptr_out + r.rows, 1, s);
    ALSK_CUDA(cudaStreamSynchronize(s));
    if (col_idx_out != nullptr && total > 0) {
        filter_scatter_kernel<<<grid, 256, 0, s>>>(r.row_ptr, r.col_idx, r.values, r.rows, static_cast<int32_t>(lo),
                                                   static_cast<int32_t>(hi), row_ptr_out, col_idx_out, values_out);
        ALSK_LAUNCHED();
    }
    return total;
}

}  // namespace alsk
