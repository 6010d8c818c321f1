// Host-side data helpers of libalskit_cuda.so: seeded factor init, the holdout split and
// the deterministic synthetic generator. These are the reference's host routines on
// either side of the hot path (factor.hpp, common.hpp, dataio.hpp); they are sequential
// RNG streams by specification, so they stay on the host and are restated bit-exactly.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "alskit_cuda.h"
#include "synth_host.hpp"

namespace alsk {
void set_last_error(const char* msg);  // capi.cu
}

namespace {

// splitmix64 finaliser (common.hpp:70-75)
inline uint64_t mix_seed(uint64_t seed, uint64_t salt) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// top 24 bits of one mt19937_64 draw scaled to [0,1) (factor.hpp:41-43)
inline float uniform_unit(std::mt19937_64& rng) {
    return static_cast<float>(rng() >> 40) * 0x1.0p-24f;
}

// rejection-sampled draw from [0, range) (dataio.hpp:103-109)
inline uint64_t bounded_u64(std::mt19937_64& rng, uint64_t range) {
    const uint64_t threshold = (0 - range) % range;
    for (;;) {
        const uint64_t v = rng();
        if (v >= threshold) return v % range;
    }
}

}  // namespace

extern "C" {

uint64_t alsk_mix_seed(uint64_t seed, uint64_t salt) { return mix_seed(seed, salt); }

// random_factor (factor.hpp:49-54)
void alsk_random_factor(int64_t rows, int f, uint64_t seed, float* out) {
    std::mt19937_64 rng(seed);
    const int64_t n = rows * static_cast<int64_t>(f);
    for (int64_t i = 0; i < n; ++i) out[i] = uniform_unit(rng);
}

// split_train_test (dataio.hpp:251-290). Called twice: with train_row_ptr == nullptr it
// only reports k (held-out count); the second call fills the caller's buffers.
alsk_status alsk_split_train_test(const alsk_csr* r, double holdout, uint64_t seed, int64_t* k_out,
                                  int64_t* train_row_ptr, int32_t* train_col_idx,
                                  float* train_values, alsk_triplet* test_out) {
    if (!(holdout > 0.0) || !(holdout < 1.0)) {  // dataio.hpp:253-254
        alsk::set_last_error("holdout fraction must lie strictly between 0 and 1");
        return ALSK_ERR_INPUT;
    }
    const int64_t nnz = r->nnz;
    const int64_t k = static_cast<int64_t>(std::floor(holdout * static_cast<double>(nnz)));
    *k_out = k;
    if (train_row_ptr == nullptr) return ALSK_OK;
    std::vector<int64_t> pos(static_cast<size_t>(nnz));
    for (int64_t i = 0; i < nnz; ++i) pos[i] = i;
    std::mt19937_64 rng(seed);
    for (int64_t t = 0; t < k; ++t) {
        const int64_t j = t + static_cast<int64_t>(bounded_u64(rng, static_cast<uint64_t>(nnz - t)));
        std::swap(pos[t], pos[j]);
    }
    std::vector<char> held(static_cast<size_t>(nnz), 0);
    for (int64_t t = 0; t < k; ++t) held[static_cast<size_t>(pos[t])] = 1;
    int64_t tr = 0, te = 0;
    train_row_ptr[0] = 0;
    for (int64_t u = 0; u < r->rows; ++u) {
        for (int64_t e = r->row_ptr[u]; e < r->row_ptr[u + 1]; ++e) {
            if (held[e]) {
                test_out[te].row = u;
                test_out[te].col = r->col_idx[e];
                test_out[te].value = r->values[e];
                ++te;
            } else {
                train_col_idx[tr] = r->col_idx[e];
                train_values[tr] = r->values[e];
                ++tr;
            }
        }
        train_row_ptr[u + 1] = tr;
    }
    return ALSK_OK;
}

}  // extern "C"

extern "C" {

// Deterministic synthetic ratings; the generator itself lives in
// synth_host.hpp, shared with the bench's reference arm.
alsk_status alsk_synth_csr(int64_t m, int64_t n, int64_t nnz, uint64_t seed, int threads,
                           int64_t* row_ptr, int32_t* col_idx, float* values) {
    const int rc = alsk_synth::synth_csr(m, n, nnz, seed, threads, row_ptr, col_idx, values);
    if (rc == 1) {
        alsk::set_last_error("invalid synthetic shape");
        return ALSK_ERR_INPUT;
    }
    if (rc == 2) {
        alsk::set_last_error("invalid synthetic shape: a row would need more ratings than columns");
        return ALSK_ERR_INPUT;
    }
    return ALSK_OK;
}

}  // extern "C"
