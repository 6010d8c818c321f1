// Train/test split on the device: split_train_test (dataio.hpp:251-290)
// with the host Fisher-Yates kept as the source of truth — the same mt19937_64 stream and
// rejection-bounded draws choose the held-out positions, which travel to the device as a
// bitmask (nnz / 8 bytes) — and the CSR compaction done in HBM:
//
//   split_count_kernel    warp per row: kept entries of the row (popcount of the mask)
//   exclusive scan        train row_ptr
//   split_scatter_kernel  warp per row, 32 entries per step: ballot-ranked, order-preserving
//                         scatter of kept entries into the train CSR and held ones into the
//                         test triplets (row-major order, like the reference)
//
// HBM traffic per rating: 4 (col) + 4 (value) read + 4 + 4 (train) or 24 (test) written, plus
// the mask bit; both kernels are HBM-bound streaming passes.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <memory>
#include <random>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace alsk {
namespace {

constexpr int kSplitThreads = 256;

// bit_offset: global position of the chunk's first entry in the mask (0 for a whole matrix)
__global__ void split_count_kernel(const int64_t* __restrict__ rp, int64_t rows, const uint32_t* __restrict__ held,
                                   int64_t bit_offset, int64_t* __restrict__ kept) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < rows; u += warps) {
        const int64_t b = rp[u], e = rp[u + 1];
        int cnt = 0;
        for (int64_t k = b + lane; k < e; k += 32) {
            const int64_t g = k - rp[0] + bit_offset;
            cnt += ((held[g >> 5] >> (g & 31)) & 1u) ? 0 : 1;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) kept[u] = cnt;
    }
}

__global__ void split_scatter_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                     const float* __restrict__ vals, int64_t rows, const uint32_t* __restrict__ held,
                                     int64_t bit_offset, int64_t row_base, const int64_t* __restrict__ trp,
                                     int32_t* __restrict__ tci, float* __restrict__ tv,
                                     alsk_triplet* __restrict__ test) {
    const int64_t rp0 = rp[0];
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < rows; u += warps) {
        const int64_t b = rp[u], e = rp[u + 1];
        int64_t otr = trp[u], ote = (b - rp0) - trp[u];
        for (int64_t k0 = b; k0 < e; k0 += 32) {
            const int64_t k = k0 + lane;
            const bool valid = k < e;
            const int64_t g = k - rp0 + bit_offset;
            const bool h = valid && ((held[g >> 5] >> (g & 31)) & 1u);
            const uint32_t mh = __ballot_sync(0xffffffffu, h);
            const uint32_t mk = __ballot_sync(0xffffffffu, valid && !h);
            if (valid) {
                const int32_t c = ci[k];
                const float v = vals[k];
                if (h) {  // three 8-byte stores, padding zeroed (the host layout's bytes)
                    uint64_t* t = reinterpret_cast<uint64_t*>(test + ote + __popc(mh & lt));
                    t[0] = static_cast<uint64_t>(u + row_base);
                    t[1] = static_cast<uint64_t>(static_cast<int64_t>(c));
                    t[2] = static_cast<uint64_t>(__float_as_uint(v));
                } else {
                    const int64_t o = otr + __popc(mk & lt);
                    tci[o] = c;
                    tv[o] = v;
                }
            }
            ote += __popc(mh);
            otr += __popc(mk);
        }
    }
}

uint64_t bounded(std::mt19937_64& rng, uint64_t range) {  // dataio.hpp:98-105
    const uint64_t threshold = (0 - range) % range;
    for (;;) {
        const uint64_t v = rng();
        if (v >= threshold) return v % range;
    }
}

// The reference's partial Fisher-Yates over positions (dataio.hpp:259-266), 32-bit
// positions when they fit (the swaps are the same), emitted as a bitmask.
// The draws do not depend on the array, so they are taken first and the swaps run with
// the partner slot prefetched a few dozen swaps ahead (the random partner reads are the
// cost: one cache miss each); the identity fill is split over threads.
template <class P>
void held_mask_impl(int64_t nnz, int64_t k, uint64_t seed, std::vector<uint32_t>& mask) {
    std::unique_ptr<P[]> pos(new P[static_cast<size_t>(nnz)]);  // not value-initialised: filled below
    {
        const int nt = nnz >= (int64_t(1) << 22) ? 8 : 1;
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                for (int64_t i = nnz * t / nt, e = nnz * (t + 1) / nt; i < e; ++i) pos[i] = static_cast<P>(i);
            });
        for (auto& x : th) x.join();
    }
    std::unique_ptr<P[]> js(new P[static_cast<size_t>(k)]);
    std::mt19937_64 rng(seed);
    for (int64_t t = 0; t < k; ++t) js[t] = static_cast<P>(t + static_cast<int64_t>(bounded(rng, static_cast<uint64_t>(nnz - t))));
    constexpr int64_t kAhead = 48;
    for (int64_t t = 0; t < k; ++t) {
        if (t + kAhead < k) __builtin_prefetch(&pos[js[t + kAhead]], 1, 0);
        std::swap(pos[t], pos[js[t]]);
    }
    mask.assign(static_cast<size_t>((nnz + 31) / 32), 0u);
    for (int64_t t = 0; t < k; ++t) {
        const uint64_t p = static_cast<uint64_t>(pos[t]);
        mask[p >> 5] |= 1u << (p & 31);
    }
}

template <class P>
void held_mask(int64_t nnz, int64_t k, uint64_t seed, std::vector<uint32_t>& mask) {
    held_mask_impl<P>(nnz, k, seed, mask);
}

}  // namespace

void holdout_mask_host(int64_t nnz, int64_t k, uint64_t seed, std::vector<uint32_t>& mask) {
    if (nnz < (int64_t(1) << 32)) held_mask<uint32_t>(nnz, k, seed, mask);
    else held_mask<int64_t>(nnz, k, seed, mask);
}

int64_t split_holdout_count(int64_t nnz, double holdout) {
    if (!(holdout > 0.0) || !(holdout < 1.0)) fail_input("holdout fraction must lie strictly between 0 and 1");
    return static_cast<int64_t>(std::floor(holdout * static_cast<double>(nnz)));
}

// Compaction of a CSR (or a row chunk of one) by a held-out bitmask already in HBM: entry k
// of `r` is held out when bit (k - row_ptr[0] + bit_offset) is set. Train row pointers start
// at 0; test triplets carry row ids shifted by row_base. Returns the train nnz (syncs s).
int64_t split_with_mask_device(const DevCsr& r, const uint32_t* dmask, int64_t bit_offset, int64_t row_base,
                               int64_t* train_row_ptr, int32_t* train_col_idx, float* train_values,
                               alsk_triplet* test, cudaStream_t s) {
    DevBuf kept(sizeof(int64_t) * std::max<int64_t>(r.rows, 1), s);
    const int64_t want = (r.rows * 32 + kSplitThreads - 1) / kSplitThreads;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(num_sms()) * 8)));
    if (r.rows > 0) {
        split_count_kernel<<<grid, kSplitThreads, 0, s>>>(r.row_ptr, r.rows, dmask, bit_offset, kept.as<int64_t>());
        ALSK_LAUNCHED();
    }
    exclusive_scan_ptr_i64<int64_t>(kept.as<int64_t>(), r.rows, train_row_ptr, s);
    if (r.rows > 0 && r.nnz > 0) {
        split_scatter_kernel<<<grid, kSplitThreads, 0, s>>>(r.row_ptr, r.col_idx, r.values, r.rows, dmask, bit_offset,
                                                            row_base, train_row_ptr, train_col_idx, train_values,
                                                            test);
        ALSK_LAUNCHED();
    }
    int64_t keep = 0;
    d2h(&keep, train_row_ptr + r.rows, 1, s);
    ALSK_CUDA(cudaStreamSynchronize(s));
    return keep;
}

void split_train_test_device(const DevCsr& r, double holdout, uint64_t seed, int64_t* train_row_ptr,
                             int32_t* train_col_idx, float* train_values, alsk_triplet* test, cudaStream_t s) {
    const int64_t k = split_holdout_count(r.nnz, holdout);
    std::vector<uint32_t> mask;
    holdout_mask_host(r.nnz, k, seed, mask);
    DevBuf dmask(sizeof(uint32_t) * std::max<size_t>(mask.size(), 1), s);
    if (!mask.empty())
        ALSK_CUDA(cudaMemcpyAsync(dmask.as<uint32_t>(), mask.data(), sizeof(uint32_t) * mask.size(),
                                  cudaMemcpyHostToDevice, s));
    split_with_mask_device(r, dmask.as<uint32_t>(), 0, 0, train_row_ptr, train_col_idx, train_values, test, s);
    // (split_with_mask_device synchronised s: the host mask may go)
}

}  // namespace alsk
