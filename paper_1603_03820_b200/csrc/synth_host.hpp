// Deterministic synthetic ratings on the host (our own generator, not a
// reference routine). Header-only and CUDA-free so that two programs share ONE definition:
// libalskit_cuda.so (alsk_synth_csr, host_data.cpp) and the bench's reference arm
// (oracle/ref_capi.cpp), which must not load the product library. The device generator
// (synth.cu) reproduces it bit for bit.
//
// Row u gets d_u = floor(nnz(u+1)/m) - floor(nnz u/m) distinct columns drawn by Floyd's
// algorithm from a SplitMix64 stream seeded with mix_seed(seed, u), sorted ascending. Values
// follow a planted rank-10 model r = <x*_u, theta*_v> + U[-0.5, 0.5) with x*_u / theta*_v
// drawn from their own per-id streams, so generation is row-parallel.
#pragma once

#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

namespace alsk_synth {

// splitmix64 finaliser (reference common.hpp:70-75)
inline uint64_t mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct SplitMix64 {
    uint64_t s;
    uint64_t operator()() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    uint64_t bounded(uint64_t range) {
        const uint64_t threshold = (0 - range) % range;
        for (;;) {
            const uint64_t v = (*this)();
            if (v >= threshold) return v % range;
        }
    }
    float unit() { return static_cast<float>((*this)() >> 40) * 0x1.0p-24f; }
};

constexpr int kPlanted = 10;

inline void planted_row(uint64_t s, int64_t id, float* out) {
    SplitMix64 g{mix_seed(s, static_cast<uint64_t>(id))};
    for (int i = 0; i < kPlanted; ++i) out[i] = g.unit() * 0.6f;
}

template <class Fn>
void parallel_rows(int64_t m, int threads, Fn&& fn) {
    std::vector<std::thread> pool;
    const int64_t per = (m + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t u0 = t * per, u1 = std::min<int64_t>(m, u0 + per);
        if (u0 >= u1) break;
        pool.emplace_back(fn, u0, u1);
    }
    for (auto& th : pool) th.join();
}

inline int64_t row_start(int64_t m, int64_t nnz, int64_t u) {
    return static_cast<int64_t>((static_cast<unsigned __int128>(nnz) * static_cast<uint64_t>(u)) /
                                static_cast<uint64_t>(m));
}

// Returns 0 on success, 1 for an invalid shape, 2 when a row needs more ratings than columns.
inline int synth_csr(int64_t m, int64_t n, int64_t nnz, uint64_t seed, int threads, int64_t* row_ptr,
                     int32_t* col_idx, float* values) {
    if (m < 1 || n < 1 || nnz < 0) return 1;
    const uint64_t seed_x = mix_seed(seed, 1001), seed_t = mix_seed(seed, 1002);
    for (int64_t u = 0; u <= m; ++u) row_ptr[u] = row_start(m, nnz, u);
    for (int64_t u = 0; u < m; ++u)
        if (row_ptr[u + 1] - row_ptr[u] > n) return 2;
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    std::vector<float> tstar(static_cast<size_t>(n) * kPlanted);
    parallel_rows(n, threads, [&](int64_t v0, int64_t v1) {
        for (int64_t v = v0; v < v1; ++v) planted_row(seed_t, v, tstar.data() + v * kPlanted);
    });
    parallel_rows(m, threads, [&](int64_t u0, int64_t u1) {
        std::vector<int64_t> chosen;
        float xu[kPlanted];
        for (int64_t u = u0; u < u1; ++u) {
            const int64_t d = row_ptr[u + 1] - row_ptr[u];
            SplitMix64 g{mix_seed(seed, static_cast<uint64_t>(u))};
            chosen.clear();
            for (int64_t j = n - d; j < n; ++j) {  // Floyd's sampling of d distinct columns
                const int64_t t = static_cast<int64_t>(g.bounded(static_cast<uint64_t>(j + 1)));
                bool dup = false;
                for (int64_t c : chosen)
                    if (c == t) { dup = true; break; }
                chosen.push_back(dup ? j : t);
            }
            std::sort(chosen.begin(), chosen.end());
            planted_row(seed_x, u, xu);
            int64_t k = row_ptr[u];
            for (int64_t c : chosen) {
                const float* tv = tstar.data() + c * kPlanted;
                float dot = 0.f;
                for (int i = 0; i < kPlanted; ++i) dot += xu[i] * tv[i];
                col_idx[k] = static_cast<int32_t>(c);
                values[k] = dot + (g.unit() - 0.5f);
                ++k;
            }
        }
    });
    return 0;
}

}  // namespace alsk_synth
