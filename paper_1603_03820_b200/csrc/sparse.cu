// Sparse index plumbing on the device, bit-exact with sparse.hpp:
//  * stable LSD radix sort (8-bit digits, upsweep histogram / scan / ranked scatter),
//  * exclusive scans over int64 counts (row_ptr / col_ptr construction),
//  * csr_to_csc / csc_to_csr (sparse.hpp:185-231): a stable sort of the nonzeros by column
//    with (row, value) payload reproduces the counting-sort transpose exactly, because the
//    input is row-major and stability keeps rows ascending within each column,
//  * csr_from_triplets (sparse.hpp:132-170): two stable passes (column, then row), range
//    and duplicate checks naming the same coordinate the reference names,
//  * grid_partition (sparse.hpp:250-314): per-row binary search of the column cuts.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "measure.cuh"

namespace alsk {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys per tile
constexpr int kWarps = kSortThreads / 32;

// ---------------------------------------------------------------- scans (int64) -----
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ int64_t block_inclusive_scan(int64_t v, int64_t* warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    if (lane == 31) warp_tot[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < (blockDim.x >> 5) ? warp_tot[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t n = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += n;
        }
        if (lane < (blockDim.x >> 5)) warp_tot[lane] = w;
    }
    __syncthreads();
    if (warp > 0) v += warp_tot[warp - 1];
    return v;
}

template <class T>
__global__ void scan_reduce_kernel(const T* __restrict__ in, int64_t n, int64_t* __restrict__ sums) {
    __shared__ int64_t wt[32];
    const int64_t base = blockIdx.x * static_cast<int64_t>(kScanTile);
    int64_t acc = 0;
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + threadIdx.x * static_cast<int64_t>(kScanItems) + i;
        if (idx < n) acc += static_cast<int64_t>(in[idx]);
    }
    const int64_t t = block_inclusive_scan<T>(acc, wt);
    if (threadIdx.x == blockDim.x - 1) sums[blockIdx.x] = t;
}

// Single-block exclusive scan of `n` int64 in place (sequential tiles with carry).
__global__ void scan_sums_kernel(int64_t* __restrict__ sums, int64_t n) {
    __shared__ int64_t wt[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t idx = base + threadIdx.x;
        const int64_t v = idx < n ? sums[idx] : 0;
        const int64_t inc = block_inclusive_scan<int64_t>(v, wt);
        const int64_t c = carry;
        if (idx < n) sums[idx] = c + inc - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = c + inc;
        __syncthreads();
    }
}

template <class T>
__global__ void scan_apply_kernel(const T* __restrict__ in, int64_t n, const int64_t* __restrict__ sums,
                                  int64_t* __restrict__ out, int64_t out_base) {
    __shared__ int64_t wt[32];
    const int64_t base = blockIdx.x * static_cast<int64_t>(kScanTile);
    int64_t vals[kScanItems];
    int64_t acc = 0;
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + threadIdx.x * static_cast<int64_t>(kScanItems) + i;
        vals[i] = idx < n ? static_cast<int64_t>(in[idx]) : 0;
        acc += vals[i];
    }
    const int64_t inc = block_inclusive_scan<T>(acc, wt);
    int64_t run = sums[blockIdx.x] + inc - acc + out_base;
    for (int i = 0; i < kScanItems; ++i) {
        const int64_t idx = base + threadIdx.x * static_cast<int64_t>(kScanItems) + i;
        if (idx < n) out[idx] = run;
        run += vals[i];
    }
}

// out[0..n] = exclusive scan of in[0..n) with out[n] = total (a CSR pointer array).
template <class T>
void exclusive_scan_ptr(const T* in, int64_t n, int64_t* out, cudaStream_t s) {
    if (n == 0) {
        ALSK_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
        return;
    }
    const int64_t nb = (n + kScanTile - 1) / kScanTile;
    DevBuf sums(sizeof(int64_t) * (nb + 1), s);
    scan_reduce_kernel<T><<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, sums.as<int64_t>());
    ALSK_LAUNCHED();
    ALSK_CUDA(cudaMemsetAsync(sums.as<int64_t>() + nb, 0, sizeof(int64_t), s));
    scan_sums_kernel<<<1, 1024, 0, s>>>(sums.as<int64_t>(), nb + 1);
    ALSK_LAUNCHED();
    scan_apply_kernel<T><<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, sums.as<int64_t>(), out, 0);
    ALSK_LAUNCHED();
    // total = exclusive prefix at position nb of the block sums
    ALSK_CUDA(cudaMemcpyAsync(out + n, sums.as<int64_t>() + nb, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
}

// --------------------------------------------------------------- radix sort ---------
// Digit histogram per tile, stored digit-major: hist[d * ntiles + tile].
__global__ void radix_upsweep_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                     int64_t ntiles, int64_t* __restrict__ hist) {
    __shared__ unsigned cnt[256];
    for (int d = threadIdx.x; d < 256; d += blockDim.x) cnt[d] = 0;
    __syncthreads();
    const int64_t base = blockIdx.x * static_cast<int64_t>(kSortTile);
    for (int i = threadIdx.x; i < kSortTile; i += blockDim.x) {
        const int64_t idx = base + i;
        if (idx < n) atomicAdd(&cnt[(keys[idx] >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[d * ntiles + blockIdx.x] = cnt[d];
}

// Stable ranked scatter. Warp w owns tile elements [w*512, (w+1)*512) processed item by
// item (lanes ascending inside an item), so warp-local ranks follow element order;
// warps are combined in order, tiles by the digit-major global scan.
template <class P>
__global__ void radix_scatter_kernel(const uint32_t* __restrict__ keys_in, const P* __restrict__ pay_in,
                                     int64_t n, int shift, int64_t ntiles,
                                     const int64_t* __restrict__ offsets, uint32_t* __restrict__ keys_out,
                                     P* __restrict__ pay_out) {
    __shared__ unsigned whist[kWarps][256];
    __shared__ int64_t tile_base[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < 256; d += blockDim.x) {
        for (int w = 0; w < kWarps; ++w) whist[w][d] = 0;
        tile_base[d] = offsets[d * ntiles + blockIdx.x];
    }
    __syncthreads();
    const int64_t base = blockIdx.x * static_cast<int64_t>(kSortTile) + warp * (32 * kSortItems);
    unsigned digit[kSortItems];
    unsigned local[kSortItems];
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int64_t idx = base + i * 32 + lane;
        const bool valid = idx < n;
        const unsigned d = valid ? ((keys_in[idx] >> shift) & 255u) : 256u + lane;  // invalid: unique
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned rank = __popc(peers & lt_mask);
        unsigned prior = 0;
        if (valid) prior = whist[warp][d];
        __syncwarp();
        const int leader = __ffs(peers) - 1;
        if (valid && lane == leader) whist[warp][d] = prior + __popc(peers);
        __syncwarp();
        digit[i] = d;
        local[i] = prior + rank;
    }
    __syncthreads();
    // exclusive scan across warps per digit
    for (int d = threadIdx.x; d < 256; d += blockDim.x) {
        unsigned run = 0;
        for (int w = 0; w < kWarps; ++w) {
            const unsigned c = whist[w][d];
            whist[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
        const int64_t idx = base + i * 32 + lane;
        if (idx < n) {
            const unsigned d = digit[i];
            const int64_t pos = tile_base[d] + whist[warp][d] + local[i];
            keys_out[pos] = keys_in[idx];
            pay_out[pos] = pay_in[idx];
        }
    }
}

// Stable sort of (key, payload) by key bits [0, bits). Result ends in (k0, p0); k1/p1 scratch.
template <class P>
void radix_sort_pairs(uint32_t* k0, P* p0, uint32_t* k1, P* p1, int64_t n, int bits, cudaStream_t s) {
    if (n <= 1 || bits <= 0) return;
    const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
    DevBuf hist(sizeof(int64_t) * (256 * ntiles + 1), s);
    uint32_t* kin = k0; P* pin = p0; uint32_t* kout = k1; P* pout = p1;
    for (int shift = 0; shift < bits; shift += 8) {
        radix_upsweep_kernel<<<static_cast<unsigned>(ntiles), kSortThreads, 0, s>>>(kin, n, shift, ntiles,
                                                                                   hist.as<int64_t>());
        ALSK_LAUNCHED();
        exclusive_scan_ptr<int64_t>(hist.as<int64_t>(), 256 * ntiles, hist.as<int64_t>(), s);
        radix_scatter_kernel<P><<<static_cast<unsigned>(ntiles), kSortThreads, 0, s>>>(
            kin, pin, n, shift, ntiles, hist.as<int64_t>(), kout, pout);
        ALSK_LAUNCHED();
        std::swap(kin, kout);
        std::swap(pin, pout);
    }
    if (kin != k0) {
        ALSK_CUDA(cudaMemcpyAsync(k0, kin, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
        ALSK_CUDA(cudaMemcpyAsync(p0, pin, sizeof(P) * n, cudaMemcpyDeviceToDevice, s));
    }
}

int bits_for(int64_t count) {  // bits to represent values in [0, count)
    int b = 0;
    while (b < 63 && (int64_t(1) << b) < count) ++b;
    return b;
}


// ------------------------------------------------ chunked counting-sort transpose ---
// csr_to_csc as a stable LSD sort of the nonzeros by column in 8-bit digits (one pass when
// n <= 256, two when n <= 65536), each pass a counting sort spread over C chunks of
// consecutive elements (one CTA each, one wave):
//  tr_tile_rows  row of the first nonzero of every tile (binary search), so pass 1 reads the
//                CSR arrays directly (no packed copy of the matrix);
//  tr_count      per-chunk digit histogram -> H[chunk][256] (pass 1 also counts the columns
//                for col_ptr, and derives the digit histogram from them);
//  tr_colscan    per digit, exclusive prefix of H over the chunks (in place) and the totals;
//  tr_scatter    per tile of 4096 nonzeros (warp w: elements 256w .. 256w+255, lane l every
//                32nd): every warp ranks its 8 rounds of digits in element order
//                (__match_any_sync, one counter read-modify-write per distinct digit), one
//                pass over the per-warp counters turns them into tile positions, the tile is
//                stably sorted by digit in shared memory and written out in sorted order, so
//                consecutive threads store consecutive positions of a digit's run. Stable in
//                every pass: the result is the reference's (rows ascending within a column).
//                Each (chunk, digit) pair writes one contiguous run, so at most C x 256
//                partially written lines are live in L2 (a full-column counting sort would
//                keep C x n of them and turn every write into a read-modify-write).
// Pass 1 writes (next key byte, row, value) = 9 bytes per nonzero; pass 2 the final arrays.
constexpr int kTrThreads = 512;
constexpr int kTrWarps = kTrThreads / 32;
constexpr int kTrSub = 8;                  // elements per thread per tile
constexpr int kTrTile = kTrThreads * kTrSub;
constexpr int kTrSpan = 1024;              // row_ptr entries staged per tile (else global search)
constexpr int kTrColHist = 44 * 1024;      // column histogram in shared memory up to this n
constexpr int kDig = 256;
constexpr int kTrMaxChunkTiles = 1024;     // tiles per chunk (one wave of chunks: >= 4M nonzeros per chunk)

__global__ void tr_tile_rows_kernel(const int64_t* __restrict__ row_ptr, int64_t rows, int64_t nnz,
                                    int64_t ntiles, int32_t* __restrict__ tile_row) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t <= ntiles;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t e = std::min<int64_t>(t * kTrTile, nnz - 1);
        int64_t lo = 0, hi = rows - 1;  // largest r with row_ptr[r] <= e
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (row_ptr[mid] <= e) lo = mid; else hi = mid - 1;
        }
        tile_row[t] = static_cast<int32_t>(t == ntiles ? rows - 1 : lo);
    }
}

// KEY8: keys are the u8 digits of a previous pass (per-warp private histograms); else int32
// columns: the column histogram (shared memory when n fits, else global atomics) gives both
// col_ptr's counts and, summed by low byte, the digit histogram
template <bool KEY8, bool COLS, bool PACKED = false>
__global__ void __launch_bounds__(kTrThreads)
tr_count_kernel(const void* __restrict__ keys, int64_t nnz, int64_t chunk, int n, uint32_t* __restrict__ H,
                unsigned long long* __restrict__ colcnt) {
    extern __shared__ uint32_t colhist[];
    __shared__ uint32_t dig[kTrWarps][kDig];
    const bool smem_cols = COLS && n <= kTrColHist;
    const int warp = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < kTrWarps * kDig; d += blockDim.x) (&dig[0][0])[d] = 0;
    if (smem_cols)
        for (int c = threadIdx.x; c < n; c += blockDim.x) colhist[c] = 0;
    __syncthreads();
    const int64_t e0 = blockIdx.x * chunk, e1 = std::min<int64_t>(nnz, e0 + chunk);
    if constexpr (PACKED) {  // the key byte is the top byte of each 32-bit word
        const uint32_t* kw = static_cast<const uint32_t*>(keys);
        const int64_t a0 = std::min<int64_t>(e1, (e0 + 3) & ~int64_t(3)), a1 = std::max<int64_t>(a0, e1 & ~int64_t(3));
        for (int64_t e = e0 + threadIdx.x; e < a0; e += kTrThreads) atomicAdd(&dig[warp][__ldcs(kw + e) >> 24], 1u);
        for (int64_t e = a1 + threadIdx.x; e < e1; e += kTrThreads) atomicAdd(&dig[warp][__ldcs(kw + e) >> 24], 1u);
        const uint4* k4 = reinterpret_cast<const uint4*>(kw + a0);
        for (int64_t q = threadIdx.x; q < (a1 - a0) >> 2; q += kTrThreads) {
            const uint4 w = __ldcs(k4 + q);
            atomicAdd(&dig[warp][w.x >> 24], 1u);
            atomicAdd(&dig[warp][w.y >> 24], 1u);
            atomicAdd(&dig[warp][w.z >> 24], 1u);
            atomicAdd(&dig[warp][w.w >> 24], 1u);
        }
    } else if constexpr (KEY8) {
        const uint8_t* k8 = static_cast<const uint8_t*>(keys);
        // 4 keys per 32-bit load where aligned
        const int64_t a0 = std::min<int64_t>(e1, (e0 + 3) & ~int64_t(3)), a1 = std::max<int64_t>(a0, e1 & ~int64_t(3));
        for (int64_t e = e0 + threadIdx.x; e < a0; e += kTrThreads) atomicAdd(&dig[warp][__ldcs(k8 + e)], 1u);
        for (int64_t e = a1 + threadIdx.x; e < e1; e += kTrThreads) atomicAdd(&dig[warp][__ldcs(k8 + e)], 1u);
        const uint32_t* k32 = reinterpret_cast<const uint32_t*>(k8 + a0);
        for (int64_t q = threadIdx.x; q < (a1 - a0) >> 2; q += kTrThreads) {
            const uint32_t w = __ldcs(k32 + q);
            atomicAdd(&dig[warp][w & 255u], 1u);
            atomicAdd(&dig[warp][(w >> 8) & 255u], 1u);
            atomicAdd(&dig[warp][(w >> 16) & 255u], 1u);
            atomicAdd(&dig[warp][w >> 24], 1u);
        }
    } else {
        const int32_t* cols = static_cast<const int32_t*>(keys);
        auto add = [&](int c) {
            if (smem_cols) {
                atomicAdd(colhist + c, 1u);
            } else {
                atomicAdd(&dig[warp][c & (kDig - 1)], 1u);
                if constexpr (COLS) atomicAdd(colcnt + c, 1ull);
            }
        };
        // 16-byte loads, four in flight per thread (chunks start at multiples of the tile)
        const int64_t a0 = std::min<int64_t>(e1, (e0 + 3) & ~int64_t(3)), a1 = std::max<int64_t>(a0, e1 & ~int64_t(3));
        for (int64_t e = e0 + threadIdx.x; e < a0; e += kTrThreads) add(__ldcs(cols + e));
        for (int64_t e = a1 + threadIdx.x; e < e1; e += kTrThreads) add(__ldcs(cols + e));
        const int4* c4 = reinterpret_cast<const int4*>(cols + a0);
        const int64_t nq = (a1 - a0) >> 2;
        int64_t q = threadIdx.x;
        for (; q + 3 * kTrThreads < nq; q += 4 * kTrThreads) {
            int4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) w[u] = __ldcs(c4 + q + u * kTrThreads);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                add(w[u].x);
                add(w[u].y);
                add(w[u].z);
                add(w[u].w);
            }
        }
        for (; q < nq; q += kTrThreads) {
            const int4 w = __ldcs(c4 + q);
            add(w.x);
            add(w.y);
            add(w.z);
            add(w.w);
        }
    }
    __syncthreads();
    uint32_t* out = H + static_cast<int64_t>(blockIdx.x) * kDig;
    for (int d = threadIdx.x; d < kDig; d += blockDim.x) {
        uint32_t v = 0;
        if (!KEY8 && smem_cols) {
            for (int c = d; c < n; c += kDig) v += colhist[c];
        } else {
#pragma unroll
            for (int w = 0; w < kTrWarps; ++w) v += dig[w][d];
        }
        out[d] = v;
    }
    if (smem_cols)
        for (int c = threadIdx.x; c < n; c += blockDim.x)
            if (colhist[c]) atomicAdd(colcnt + c, static_cast<unsigned long long>(colhist[c]));
}

// block (32 digits, 32 chunk groups): per digit, exclusive prefix over the chunks in place
// and the digit totals
__global__ void tr_colscan_kernel(uint32_t* __restrict__ H, int nchunks, int n,
                                  unsigned long long* __restrict__ totals) {
    __shared__ uint32_t part[32][33];
    const int col = blockIdx.x * 32 + threadIdx.x;
    const int g = threadIdx.y;
    const int per = (nchunks + 31) / 32;
    const int k0 = std::min(nchunks, g * per), k1 = std::min(nchunks, (g + 1) * per);
    uint32_t sum = 0;
    if (col < n)
        for (int k = k0; k < k1; ++k) sum += H[static_cast<int64_t>(k) * n + col];
    part[g][threadIdx.x] = sum;
    __syncthreads();
    if (g == 0) {
        uint32_t run = 0;
        for (int i = 0; i < 32; ++i) {
            const uint32_t v = part[i][threadIdx.x];
            part[i][threadIdx.x] = run;
            run += v;
        }
        if (col < n) totals[col] = run;
    }
    __syncthreads();
    if (col < n) {
        uint32_t run = part[g][threadIdx.x];
        for (int k = k0; k < k1; ++k) {
            const int64_t i = static_cast<int64_t>(k) * n + col;
            const uint32_t v = H[i];
            H[i] = run;
            run += v;
        }
    }
}

// exclusive scan of the 256 digit totals (one block)
__global__ void tr_digit_base_kernel(const unsigned long long* __restrict__ totals, uint32_t* __restrict__ base) {
    __shared__ unsigned long long v[kDig];
    v[threadIdx.x] = totals[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long run = 0;
        for (int d = 0; d < kDig; ++d) {
            const unsigned long long x = v[d];
            v[d] = run;
            run += x;
        }
    }
    __syncthreads();
    base[threadIdx.x] = static_cast<uint32_t>(v[threadIdx.x]);
}

__device__ __forceinline__ int tr_row_search(const int64_t* __restrict__ rp, int lo, int hi, int64_t e) {
    while (lo < hi) {  // largest r in [lo, hi] with rp[r] <= e
        const int mid = (lo + hi + 1) >> 1;
        if (rp[mid] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

struct TrSmem {
    uint32_t wcnt[kTrWarps][kDig];  // per-warp digit counters, then their exclusive prefix over warps
    uint32_t match[kTrWarps][kDig]; // per-warp peer masks of the current round (zero between rounds)
    uint32_t tstart[kDig];          // tile-local start of each digit
    uint32_t gbase[kDig];           // global position of tile-local sorted index 0 of each digit's run
    uint32_t off[kDig];             // the chunk's running global offset of each digit
    uint32_t wsum[kDig / 32];
    int32_t s_row[kTrTile];         // row (PACK: | next key byte << 24)
    float s_val[kTrTile];
    uint8_t s_dig[kTrTile];
    uint8_t s_key[kTrTile];
    int64_t s_rp[kTrSpan + 2];
    int32_t s_trow[kTrMaxChunkTiles + 1];  // first row of each tile of the chunk
};

// FROM_CSR: read (column, value) and the row (tile search) from the CSR arrays, digit = the
// column's low byte; else read (key byte, row, value) of the previous pass. TO_FINAL: write
// (row, value) to the CSC arrays; else (column's next byte, row, value) for the next pass.
// PACK (rows < 2^24): the intermediate carries the key byte in the row's top byte.
// The next tile's inputs are loaded into registers before the current tile's write-out.
template <bool FROM_CSR, bool TO_FINAL, bool PACK>
__global__ void __launch_bounds__(kTrThreads, 2)
tr_scatter_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                  const uint8_t* __restrict__ key_in, const int32_t* __restrict__ row_in,
                  const float* __restrict__ val_in, int64_t nnz, int64_t chunk, const uint32_t* __restrict__ H,
                  const uint32_t* __restrict__ digit_base, const int32_t* __restrict__ tile_row,
                  uint8_t* __restrict__ key_out, int32_t* __restrict__ row_out, float* __restrict__ val_out) {
    extern __shared__ __align__(16) uint8_t tr_smem_raw[];
    TrSmem& S = *reinterpret_cast<TrSmem*>(tr_smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t* Hrow = H + static_cast<int64_t>(blockIdx.x) * kDig;
    for (int d = threadIdx.x; d < kDig; d += blockDim.x) S.off[d] = digit_base[d] + Hrow[d];
    for (int d = lane; d < kDig; d += 32) S.match[warp][d] = 0u;
    const int64_t e0 = blockIdx.x * chunk, e1 = std::min<int64_t>(nnz, e0 + chunk);
    // this thread's elements of a tile: tb + 256 warp + 32 j + lane
    int dg[kTrSub], kk[kTrSub], rw[kTrSub];
    float v[kTrSub];
    auto load = [&](int64_t tb) {
        const int tcount = static_cast<int>(std::min<int64_t>(kTrTile, e1 - tb));
#pragma unroll
        for (int j = 0; j < kTrSub; ++j) {
            const int i = 256 * warp + 32 * j + lane;
            const int64_t e = tb + i;
            const bool ok = i < tcount;
            if constexpr (FROM_CSR) {
                const int c = ok ? __ldcs(col_idx + e) : 0;
                dg[j] = ok ? (c & (kDig - 1)) : -1 - lane;  // past the end: a digit of its own
                kk[j] = (c >> 8) & 255;
                v[j] = ok ? __ldcs(val_in + e) : 0.f;
                rw[j] = 0;
            } else if constexpr (PACK) {
                const int32_t x = ok ? __ldcs(row_in + e) : 0;
                dg[j] = ok ? static_cast<int>(static_cast<uint32_t>(x) >> 24) : -1 - lane;
                kk[j] = 0;
                rw[j] = x & 0xFFFFFF;
                v[j] = ok ? __ldcs(val_in + e) : 0.f;
            } else {
                dg[j] = ok ? static_cast<int>(__ldcs(key_in + e)) : -1 - lane;
                kk[j] = 0;
                rw[j] = ok ? __ldcs(row_in + e) : 0;
                v[j] = ok ? __ldcs(val_in + e) : 0.f;
            }
        }
    };
    // FROM_CSR: the tiles' first rows in shared memory, and each tile's row_ptr slice loaded
    // into registers with its elements (two per thread), stored to shared memory at its start
    constexpr int kRpPer = (kTrSpan + 2 + kTrThreads - 1) / kTrThreads;
    int64_t rpv[kRpPer];
    const int64_t t0 = e0 / kTrTile, nt = (e1 - e0 + kTrTile - 1) / kTrTile;
    if constexpr (FROM_CSR) {
        for (int64_t i = threadIdx.x; i <= nt; i += blockDim.x) S.s_trow[i] = tile_row[t0 + i];
        __syncthreads();
    }
    auto load_rp = [&](int64_t ti) {
        if constexpr (FROM_CSR) {
            const int ra = S.s_trow[ti], rb = S.s_trow[ti + 1];
#pragma unroll
            for (int k = 0; k < kRpPer; ++k) {
                const int i = threadIdx.x + k * kTrThreads;
                rpv[k] = (rb - ra <= kTrSpan && i <= rb - ra + 1) ? row_ptr[ra + i] : 0;
            }
        }
    };
    if (e0 < e1) {
        load(e0);
        load_rp(0);
    }
    for (int64_t tb = e0; tb < e1; tb += kTrTile) {
        const int tcount = static_cast<int>(std::min<int64_t>(kTrTile, e1 - tb));
        int ra = 0, rb = 0;
        bool staged = false;
        if constexpr (FROM_CSR) {
            const int64_t ti = (tb - e0) / kTrTile;
            ra = S.s_trow[ti];
            rb = S.s_trow[ti + 1];
            staged = rb - ra <= kTrSpan;
            if (staged) {
#pragma unroll
                for (int k = 0; k < kRpPer; ++k) {
                    const int i = threadIdx.x + k * kTrThreads;
                    if (i <= rb - ra + 1) S.s_rp[i] = rpv[k];
                }
            }
        }
#pragma unroll
        for (int d = lane; d < kDig; d += 32) S.wcnt[warp][d] = 0;
        __syncthreads();  // row_ptr staged, counters zeroed (and the previous tile fully written)
        // per-warp stable ranks, rounds in element order; peers = lanes with the same digit,
        // matched through a per-warp mask per digit in shared memory (atomic OR of the lane
        // bits, read back, reset by the leader): ~a dozen instructions per element, where
        // MATCH.ANY stalled on the MIO queue and 8 bit-ballots cost ~45
        uint32_t* mm = S.match[warp];
        int rank[kTrSub];
#pragma unroll
        for (int j = 0; j < kTrSub; ++j) {
            if (dg[j] >= 0) atomicOr(&mm[dg[j]], 1u << lane);
            __syncwarp();
            const unsigned peers = dg[j] >= 0 ? mm[dg[j]] : (1u << lane);
            __syncwarp();
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (lane == leader && dg[j] >= 0) {
                old = S.wcnt[warp][dg[j]];
                S.wcnt[warp][dg[j]] = old + __popc(peers);
                mm[dg[j]] = 0u;
            }
            old = __shfl_sync(0xffffffffu, old, leader);
            rank[j] = static_cast<int>(old) + __popc(peers & lt);
            __syncwarp();
        }
        __syncthreads();
        // digit d = thread: exclusive prefix of its counters over the warps, tile start of the
        // digit (block scan of the totals), global base of its run
        if (threadIdx.x < kDig) {
            const int d = threadIdx.x;
            uint32_t c[kTrWarps];
#pragma unroll
            for (int w = 0; w < kTrWarps; ++w) c[w] = S.wcnt[w][d];
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kTrWarps; ++w) {
                const uint32_t x = c[w];
                S.wcnt[w][d] = run;
                run += x;
            }
            uint32_t inc = run;  // inclusive scan of the totals over the digits
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, dd);
                if (lane >= dd) inc += y;
            }
            if (lane == 31) S.wsum[warp] = inc;
            S.tstart[d] = inc - run;  // within the warp's 32 digits for now
        }
        __syncthreads();
        if (threadIdx.x < kDig) {
            const int d = threadIdx.x;
            uint32_t pre = 0;
            for (int w = 0; w < warp; ++w) pre += S.wsum[w];
            const uint32_t st = S.tstart[d] + pre;
            S.tstart[d] = st;
            S.gbase[d] = S.off[d] - st;
        }
        __syncthreads();
        // stable sort of the tile by digit in shared memory; rows: the row of each element
        // follows its predecessor's (+32 elements), two probes then a binary search
        int r = ra;
        if constexpr (FROM_CSR) {
            const int64_t e = tb + 256 * warp + lane;
            if (256 * warp + lane < tcount)
                r = staged ? ra + tr_row_search(S.s_rp, 0, rb - ra, e) : tr_row_search(row_ptr, ra, rb, e);
        }
#pragma unroll
        for (int j = 0; j < kTrSub; ++j) {
            if (dg[j] >= 0) {
                const int i = 256 * warp + 32 * j + lane;
                if constexpr (FROM_CSR) {
                    const int64_t e = tb + i;
                    if (j > 0) {
                        if (staged) {
                            const int lr = r - ra;
                            if (S.s_rp[lr + 1] <= e)
                                r = S.s_rp[lr + 2] > e ? r + 1 : ra + tr_row_search(S.s_rp, lr + 2, rb - ra, e);
                        } else {
                            r = tr_row_search(row_ptr, r, rb, e);
                        }
                    }
                    rw[j] = r;
                }
                const int p = static_cast<int>(S.tstart[dg[j]] + S.wcnt[warp][dg[j]]) + rank[j];
                S.s_dig[p] = static_cast<uint8_t>(dg[j]);
                if constexpr (PACK && !TO_FINAL) {
                    S.s_row[p] = rw[j] | (kk[j] << 24);
                } else {
                    S.s_key[p] = static_cast<uint8_t>(kk[j]);
                    S.s_row[p] = rw[j];
                }
                S.s_val[p] = v[j];
            }
        }
        __syncthreads();
        if (tb + kTrTile < e1) {  // in flight during the write-out
            load(tb + kTrTile);
            load_rp((tb - e0) / kTrTile + 1);
        }
        // write-out in sorted order: consecutive threads, consecutive positions of a run
        for (int i = threadIdx.x; i < tcount; i += kTrThreads) {
            const int d = S.s_dig[i];
            const uint32_t pos = S.gbase[d] + static_cast<uint32_t>(i);
            if constexpr (!TO_FINAL && !PACK) key_out[pos] = S.s_key[i];
            row_out[pos] = S.s_row[i];
            val_out[pos] = S.s_val[i];
        }
        // the chunk's running offsets move past this tile (counts = next digit start - start)
        if (threadIdx.x < kDig) {
            const int d = threadIdx.x;
            const uint32_t nxt = d == kDig - 1 ? static_cast<uint32_t>(tcount) : S.tstart[d + 1];
            S.off[d] += nxt - S.tstart[d];
        }
        __syncthreads();
    }
}

// --------------------------------------------------------------- helpers -------------
// Per nonzero: key = column, payload = (row << 32) | value bits.
__global__ void csr_pack_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                const float* __restrict__ values, int64_t rows,
                                uint32_t* __restrict__ keys, uint64_t* __restrict__ pay) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t u = warp0; u < rows; u += nw) {
        for (int64_t k = row_ptr[u] + lane; k < row_ptr[u + 1]; k += 32) {
            keys[k] = static_cast<uint32_t>(col_idx[k]);
            pay[k] = (static_cast<uint64_t>(static_cast<uint32_t>(u)) << 32) | __float_as_uint(values[k]);
        }
    }
}

__global__ void count_keys_kernel(const uint32_t* __restrict__ keys, int64_t n, unsigned long long* __restrict__ cnt) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(cnt + keys[k], 1ull);
}

__global__ void unpack_kernel(const uint64_t* __restrict__ pay, int64_t n, int32_t* __restrict__ idx_out,
                              float* __restrict__ val_out) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t p = pay[k];
        idx_out[k] = static_cast<int32_t>(p >> 32);
        val_out[k] = __uint_as_float(static_cast<uint32_t>(p));
    }
}

int grid_for(int64_t n, int threads = 256) {
    const int64_t b = (n + threads - 1) / threads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 148LL * 16)));
}

__global__ void triplet_range_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                                     int64_t count, int64_t m, int64_t n, unsigned long long* __restrict__ bad) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < count;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = rows[k], c = cols[k];
        if (r < 0 || r >= m || c < 0 || c >= n) atomicMin(bad, static_cast<unsigned long long>(k));
    }
}

__global__ void iota_keys_kernel(const int64_t* __restrict__ src, int64_t n, uint32_t* __restrict__ keys,
                                 uint64_t* __restrict__ idx) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        keys[k] = static_cast<uint32_t>(src[k]);
        idx[k] = static_cast<uint64_t>(k);
    }
}

__global__ void gather_keys_kernel(const int64_t* __restrict__ src, const uint64_t* __restrict__ idx,
                                   int64_t n, uint32_t* __restrict__ keys) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        keys[k] = static_cast<uint32_t>(src[idx[k]]);
}

// After the (row, col) sort: emit col_idx/values, count rows, flag the first duplicate.
__global__ void emit_sorted_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                                   const float* __restrict__ vals, const uint64_t* __restrict__ idx,
                                   int64_t n, int32_t* __restrict__ col_out, float* __restrict__ val_out,
                                   unsigned long long* __restrict__ row_cnt,
                                   unsigned long long* __restrict__ first_dup) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t s = idx[k];
        const int64_t r = rows[s], c = cols[s];
        col_out[k] = static_cast<int32_t>(c);
        val_out[k] = vals[s];
        atomicAdd(row_cnt + r, 1ull);
        if (k > 0) {
            const uint64_t q = idx[k - 1];
            if (rows[q] == r && cols[q] == c) atomicMin(first_dup, static_cast<unsigned long long>(k));
        }
    }
}

}  // namespace

template <class T>
void exclusive_scan_ptr_i64(const T* in, int64_t n, int64_t* out, cudaStream_t s) {
    exclusive_scan_ptr<T>(in, n, out, s);
}
template void exclusive_scan_ptr_i64<int64_t>(const int64_t*, int64_t, int64_t*, cudaStream_t);
template void exclusive_scan_ptr_i64<unsigned long long>(const unsigned long long*, int64_t, int64_t*, cudaStream_t);

void csr_from_triplets_device(int64_t m, int64_t n, const int64_t* rows, const int64_t* cols,
                              const float* vals, int64_t count, int64_t* row_ptr, int32_t* col_idx,
                              float* values, cudaStream_t s) {
    if (m < 0 || n < 0) fail_input("matrix dimensions must be non-negative");
    if (n > 2147483647LL) fail_input("column count " + std::to_string(n) + " exceeds the 32-bit index range");
    if (m > 0xffffffffLL) fail_input("row count exceeds the device sort range");
    DevBuf bad(sizeof(unsigned long long), s);
    ALSK_CUDA(cudaMemsetAsync(bad.as<void>(), 0xff, sizeof(unsigned long long), s));
    if (count > 0) {
        triplet_range_kernel<<<grid_for(count), 256, 0, s>>>(rows, cols, count, m, n, bad.as<unsigned long long>());
        ALSK_LAUNCHED();
    }
    unsigned long long hbad = 0;
    d2h(&hbad, bad.as<unsigned long long>(), 1, s);
    ALSK_CUDA(cudaStreamSynchronize(s));
    if (hbad != ~0ull) {
        int64_t r = 0, c = 0;
        d2h(&r, rows + hbad, 1, s);
        d2h(&c, cols + hbad, 1, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
        fail_input("triplet (" + std::to_string(r) + ", " + std::to_string(c) + ") outside " +
                   std::to_string(m) + "x" + std::to_string(n));
    }
    DevBuf cnt(sizeof(unsigned long long) * std::max<int64_t>(m, 1), s);
    ALSK_CUDA(cudaMemsetAsync(cnt.as<void>(), 0, sizeof(unsigned long long) * std::max<int64_t>(m, 1), s));
    if (count == 0) {
        exclusive_scan_ptr<unsigned long long>(cnt.as<unsigned long long>(), m, row_ptr, s);
        return;
    }
    DevBuf k0(sizeof(uint32_t) * count, s), k1(sizeof(uint32_t) * count, s);
    DevBuf p0(sizeof(uint64_t) * count, s), p1(sizeof(uint64_t) * count, s);
    // LSD: stable by column, then stable by row => (row, col) order, ties in input order
    iota_keys_kernel<<<grid_for(count), 256, 0, s>>>(cols, count, k0.as<uint32_t>(), p0.as<uint64_t>());
    ALSK_LAUNCHED();
    radix_sort_pairs<uint64_t>(k0.as<uint32_t>(), p0.as<uint64_t>(), k1.as<uint32_t>(), p1.as<uint64_t>(),
                               count, bits_for(n), s);
    gather_keys_kernel<<<grid_for(count), 256, 0, s>>>(rows, p0.as<uint64_t>(), count, k0.as<uint32_t>());
    ALSK_LAUNCHED();
    radix_sort_pairs<uint64_t>(k0.as<uint32_t>(), p0.as<uint64_t>(), k1.as<uint32_t>(), p1.as<uint64_t>(),
                               count, bits_for(m), s);
    ALSK_CUDA(cudaMemsetAsync(bad.as<void>(), 0xff, sizeof(unsigned long long), s));
    emit_sorted_kernel<<<grid_for(count), 256, 0, s>>>(rows, cols, vals, p0.as<uint64_t>(), count, col_idx,
                                                       values, cnt.as<unsigned long long>(),
                                                       bad.as<unsigned long long>());
    ALSK_LAUNCHED();
    d2h(&hbad, bad.as<unsigned long long>(), 1, s);
    ALSK_CUDA(cudaStreamSynchronize(s));
    if (hbad != ~0ull) {
        uint64_t src = 0;
        d2h(&src, p0.as<uint64_t>() + hbad, 1, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
        int64_t r = 0, c = 0;
        d2h(&r, rows + src, 1, s);
        d2h(&c, cols + src, 1, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
        fail_input("duplicate coordinate (" + std::to_string(r) + ", " + std::to_string(c) + ")");
    }
    exclusive_scan_ptr<unsigned long long>(cnt.as<unsigned long long>(), m, row_ptr, s);
}

void csr_to_csc_radix(const DevCsr& a, int64_t* col_ptr, int32_t* row_idx, float* values,
                      cudaStream_t s) {
    const int64_t n = a.nnz;
    if (a.rows > 0xffffffffLL) fail_input("row count exceeds the device transpose range");
    DevBuf cnt(sizeof(unsigned long long) * std::max<int64_t>(a.cols, 1), s);
    ALSK_CUDA(cudaMemsetAsync(cnt.as<void>(), 0, sizeof(unsigned long long) * std::max<int64_t>(a.cols, 1), s));
    if (n == 0) {
        exclusive_scan_ptr<unsigned long long>(cnt.as<unsigned long long>(), a.cols, col_ptr, s);
        return;
    }
    DevBuf k0(sizeof(uint32_t) * n, s), k1(sizeof(uint32_t) * n, s);
    DevBuf p0(sizeof(uint64_t) * n, s), p1(sizeof(uint64_t) * n, s);
    csr_pack_kernel<<<grid_for(a.rows * 32), 256, 0, s>>>(a.row_ptr, a.col_idx, a.values, a.rows,
                                                          k0.as<uint32_t>(), p0.as<uint64_t>());
    ALSK_LAUNCHED();
    count_keys_kernel<<<grid_for(n), 256, 0, s>>>(k0.as<uint32_t>(), n, cnt.as<unsigned long long>());
    ALSK_LAUNCHED();
    exclusive_scan_ptr<unsigned long long>(cnt.as<unsigned long long>(), a.cols, col_ptr, s);
    radix_sort_pairs<uint64_t>(k0.as<uint32_t>(), p0.as<uint64_t>(), k1.as<uint32_t>(),
                               p1.as<uint64_t>(), n, bits_for(a.cols), s);
    unpack_kernel<<<grid_for(n), 256, 0, s>>>(p0.as<uint64_t>(), n, row_idx, values);
    ALSK_LAUNCHED();
}

// Counting-sort transpose for n <= 65536 columns and positions below 2^32 (every named
// shape's CSR -> CSC); the radix sort of (column; row, value) pairs otherwise.
bool csr_to_csc_counting(const DevCsr& a, int64_t* col_ptr, int32_t* row_idx, float* values, cudaStream_t s) {
    const int64_t n = a.cols, nnz = a.nnz;
    if (n < 1 || n > 65536 || nnz >= (int64_t(1) << 32) || a.rows >= (int64_t(1) << 31) || nnz == 0) return false;
    const bool two = n > kDig;
    const int64_t ntiles_total = (nnz + kTrTile - 1) / kTrTile;
    const int ssm = static_cast<int>(sizeof(TrSmem));
    const bool pack = a.rows < (int64_t(1) << 24);  // the pass-1 key byte rides in the row's top byte
    ALSK_CUDA(cudaFuncSetAttribute(tr_scatter_kernel<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
    ALSK_CUDA(cudaFuncSetAttribute(tr_scatter_kernel<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
    ALSK_CUDA(cudaFuncSetAttribute(tr_scatter_kernel<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
    ALSK_CUDA(cudaFuncSetAttribute(tr_scatter_kernel<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
    ALSK_CUDA(cudaFuncSetAttribute(tr_scatter_kernel<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
    int occ = 0;
    ALSK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tr_scatter_kernel<true, false, false>, kTrThreads, ssm));
    const int64_t want = static_cast<int64_t>(num_sms()) * std::max(occ, 1);
    const int64_t tiles_per_chunk = std::min<int64_t>(kTrMaxChunkTiles,
                                                      std::max<int64_t>(1, (ntiles_total + want - 1) / want));
    const int64_t chunk = tiles_per_chunk * kTrTile;
    const int nchunks = static_cast<int>((nnz + chunk - 1) / chunk);
    DevBuf tile_row(sizeof(int32_t) * (ntiles_total + 1), s);
    DevBuf H(sizeof(uint32_t) * static_cast<size_t>(nchunks) * kDig, s);
    DevBuf totals(sizeof(unsigned long long) * kDig, s), base(sizeof(uint32_t) * kDig, s);
    DevBuf colcnt(sizeof(unsigned long long) * n, s);
    ALSK_CUDA(cudaMemsetAsync(colcnt.as<void>(), 0, sizeof(unsigned long long) * n, s));
    tr_tile_rows_kernel<<<grid_for(ntiles_total + 1), 256, 0, s>>>(a.row_ptr, a.rows, nnz, ntiles_total,
                                                                   tile_row.as<int32_t>());
    ALSK_LAUNCHED();
    const size_t colsmem = n <= kTrColHist ? sizeof(uint32_t) * n : 0;
    ALSK_CUDA(cudaFuncSetAttribute(tr_count_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(colsmem)));
    auto digit_pass = [&](auto count_k, const void* keys, auto scatter_k, const uint8_t* key_in, const int32_t* row_in,
                          const float* val_in, uint8_t* key_out, int32_t* row_out, float* val_out, size_t csm) {
        count_k<<<nchunks, kTrThreads, csm, s>>>(keys, nnz, chunk, static_cast<int>(n), H.as<uint32_t>(),
                                                 colcnt.as<unsigned long long>());
        ALSK_LAUNCHED();
        tr_colscan_kernel<<<kDig / 32, dim3(32, 32), 0, s>>>(H.as<uint32_t>(), nchunks, kDig,
                                                              totals.as<unsigned long long>());
        ALSK_LAUNCHED();
        tr_digit_base_kernel<<<1, kDig, 0, s>>>(totals.as<unsigned long long>(), base.as<uint32_t>());
        ALSK_LAUNCHED();
        scatter_k<<<nchunks, kTrThreads, ssm, s>>>(a.row_ptr, a.col_idx, key_in, row_in, val_in, nnz, chunk,
                                                 H.as<uint32_t>(), base.as<uint32_t>(), tile_row.as<int32_t>(), key_out,
                                                 row_out, val_out);
        ALSK_LAUNCHED();
    };
    if (!two) {
        digit_pass(tr_count_kernel<false, true>, a.col_idx, tr_scatter_kernel<true, true, false>, nullptr, nullptr,
                   a.values, nullptr, row_idx, values, colsmem);
    } else if (pack) {
        DevBuf rw(sizeof(int32_t) * nnz, s), vl(sizeof(float) * nnz, s);
        digit_pass(tr_count_kernel<false, true>, a.col_idx, tr_scatter_kernel<true, false, true>, nullptr, nullptr,
                   a.values, nullptr, rw.as<int32_t>(), vl.as<float>(), colsmem);
        digit_pass(tr_count_kernel<true, false, true>, rw.as<int32_t>(), tr_scatter_kernel<false, true, true>, nullptr,
                   rw.as<int32_t>(), vl.as<float>(), nullptr, row_idx, values, 0);
    } else {
        DevBuf k8(static_cast<size_t>(nnz), s), rw(sizeof(int32_t) * nnz, s), vl(sizeof(float) * nnz, s);
        digit_pass(tr_count_kernel<false, true>, a.col_idx, tr_scatter_kernel<true, false, false>, nullptr, nullptr,
                   a.values, k8.as<uint8_t>(), rw.as<int32_t>(), vl.as<float>(), colsmem);
        digit_pass(tr_count_kernel<true, false>, k8.as<uint8_t>(), tr_scatter_kernel<false, true, false>,
                   k8.as<uint8_t>(), rw.as<int32_t>(), vl.as<float>(), nullptr, row_idx, values, 0);
    }
    exclusive_scan_ptr<unsigned long long>(colcnt.as<unsigned long long>(), n, col_ptr, s);
    return true;
}

void csr_to_csc_device(const DevCsr& a, int64_t* col_ptr, int32_t* row_idx, float* values,
                       cudaStream_t s) {
    static const bool radix_only = measure_env("ALSK_TRANSPOSE_RADIX") != nullptr;  // A/B switch
    if (!radix_only && csr_to_csc_counting(a, col_ptr, row_idx, values, s)) return;
    csr_to_csc_radix(a, col_ptr, row_idx, values, s);
}

}  // namespace alsk
