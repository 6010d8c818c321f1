// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into libalskit_cuda.so, never on the
// product path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load liboracle.so, and only as the checker.
//
// A plain-C++ CPU restatement of the reference ALS path (alskit, /root/reference/proj/
// include/alskit), written against the C ABI types of include/alskit_cuda.h so tests can
// feed identical buffers to the oracle and to the CUDA library. Each function cites the
// reference lines it restates. Parity of this restatement is pinned two ways:
//   * against the reference itself, compiled unmodified from /root/reference into
//     oracle/_ref/libalskit_ref.so (oracle/ref_capi.cpp; tests/test_oracle_pinning.py),
//   * against golden vectors generated from that build (tests/golden/, gen script
//     tests/golden/make_golden.py) and the reference's own KATs.
// Built with -O3 -ffp-contract=off, the x86-64 baseline arithmetic of the reference's
// Release build (CMakeLists.txt:8-10, no -march), so float mode matches bit for bit too.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "alskit_cuda.h"

namespace {

thread_local std::string g_err;
thread_local int64_t g_bad = -1;

alsk_status err(alsk_status s, const std::string& m) {
    g_err = m;
    return s;
}

// check_update_shapes (solver.hpp:76-81)
alsk_status shapes(const alsk_csr* r, int64_t theta_rows, int f) {
    if (r->col_offset == 0 && theta_rows != r->cols)
        return err(ALSK_ERR_INPUT, "factor rows " + std::to_string(theta_rows) +
                                       " do not match matrix columns " + std::to_string(r->cols));
    if (f < 1) return err(ALSK_ERR_INPUT, "rank must be >= 1");
    return ALSK_OK;
}

// assemble_mo_rows (solver.hpp:99-157): lower-triangle accumulation per row in ascending
// nonzero order, lambda*n on the diagonal after the sum, mirrored, rounded to float once.
template <class Acc>
alsk_status assemble(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                     double lambda, int64_t rb, int64_t re, float* A, float* B) {
    const int64_t lo = r->col_offset, hi = lo + theta_rows;
    std::vector<Acc> acc(static_cast<size_t>(f) * f), bacc(f);
    for (int64_t u = rb; u < re; ++u) {
        std::fill(acc.begin(), acc.end(), Acc(0));
        std::fill(bacc.begin(), bacc.end(), Acc(0));
        const int64_t k0 = r->row_ptr[u], k1 = r->row_ptr[u + 1];
        for (int64_t k = k0; k < k1; ++k) {
            const int64_t v = r->col_idx[k];
            if (v < lo || v >= hi)
                return err(ALSK_ERR_INPUT, "column " + std::to_string(v) + " outside partition [" +
                                               std::to_string(lo) + ", " + std::to_string(hi) + ")");
            const float* th = theta + (v - lo) * f;
            const Acc rv = static_cast<Acc>(r->values[k]);
            for (int i = 0; i < f; ++i) {
                const Acc ti = static_cast<Acc>(th[i]);
                for (int j = 0; j <= i; ++j) acc[static_cast<size_t>(i) * f + j] += ti * static_cast<Acc>(th[j]);
                bacc[i] += rv * ti;
            }
        }
        const Acc reg = static_cast<Acc>(lambda) * static_cast<Acc>(k1 - k0);
        float* a = A + (u - rb) * static_cast<int64_t>(f) * f;
        float* b = B + (u - rb) * f;
        for (int i = 0; i < f; ++i) {
            for (int j = 0; j < i; ++j) {
                const float val = static_cast<float>(acc[static_cast<size_t>(i) * f + j]);
                a[i * f + j] = val;
                a[j * f + i] = val;
            }
            a[i * f + i] = static_cast<float>(acc[static_cast<size_t>(i) * f + i] + reg);
            b[i] = static_cast<float>(bacc[i]);
        }
    }
    return ALSK_OK;
}

// batch_solve_into (solver.hpp:204-262): double Cholesky (left-looking), forward and
// backward substitution; zero A -> zero x; non-positive pivot per policy.
// Returns the first failing index (or -1); writes pivot/column of that failure.
int64_t solve(const float* A, const float* B, int64_t count, int f, bool zero_row, float* X,
              double* piv_out, int* col_out) {
    std::vector<double> l(static_cast<size_t>(f) * f), y(f);
    for (int64_t k = 0; k < count; ++k) {
        const float* a = A + k * static_cast<int64_t>(f) * f;
        const float* b = B + k * f;
        float* x = X + k * f;
        bool zero = true;
        for (int64_t i = 0; zero && i < static_cast<int64_t>(f) * f; ++i) zero = a[i] == 0.0f;
        if (zero) {
            std::fill(x, x + f, 0.0f);
            continue;
        }
        bool broke = false;
        for (int c = 0; c < f && !broke; ++c) {
            for (int rr = c; rr < f; ++rr) {
                double s = static_cast<double>(a[rr * f + c]);
                for (int t = 0; t < c; ++t) s -= l[rr * f + t] * l[c * f + t];
                if (rr == c) {
                    if (!(s > 0.0)) {
                        if (!zero_row) {
                            *piv_out = s;
                            *col_out = c;
                            return k;
                        }
                        std::fill(x, x + f, 0.0f);
                        broke = true;
                        break;
                    }
                    l[c * f + c] = std::sqrt(s);
                } else {
                    l[rr * f + c] = s / l[c * f + c];
                }
            }
        }
        if (broke) continue;
        for (int i = 0; i < f; ++i) {
            double s = static_cast<double>(b[i]);
            for (int j = 0; j < i; ++j) s -= l[i * f + j] * y[j];
            y[i] = s / l[i * f + i];
        }
        for (int i = f - 1; i >= 0; --i) {
            double s = y[i];
            for (int j = i + 1; j < f; ++j) s -= l[j * f + i] * static_cast<double>(x[j]);
            x[i] = static_cast<float>(s / l[i * f + i]);
        }
    }
    return -1;
}

alsk_status breakdown(int64_t k, double piv, int col) {
    g_bad = k;
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", piv);  // std::to_string(double) format
    return err(ALSK_ERR_NUMERICAL, "cholesky breakdown at batch index " + std::to_string(k) +
                                       " (pivot " + buf + " at column " + std::to_string(col) + ")");
}

double dot_rows(const float* a, const float* b, int f) {  // solver.hpp:265-270
    double s = 0.0;
    for (int i = 0; i < f; ++i) s += static_cast<double>(a[i]) * static_cast<double>(b[i]);
    return s;
}

uint64_t mix(uint64_t seed, uint64_t salt) {  // common.hpp:70-75
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int64_t orc_last_breakdown_index(void) { return g_bad; }

uint64_t orc_mix_seed(uint64_t seed, uint64_t salt) { return mix(seed, salt); }

// random_factor (factor.hpp:41-54)
void orc_random_factor(int64_t rows, int f, uint64_t seed, float* out) {
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < rows * f; ++i) out[i] = static_cast<float>(rng() >> 40) * 0x1.0p-24f;
}

// get_hermitian_mo_into (solver.hpp:292-304) / get_hermitian_base (277-287)
alsk_status orc_hermitian(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                          double lambda, int acc_double, int64_t rb, int64_t re, int check_shape,
                          float* A, float* B) {
    if (check_shape) {
        const alsk_status s = shapes(r, theta_rows, f);
        if (s != ALSK_OK) return s;
    }
    if (rb < 0 || re > r->rows || rb > re)
        return err(ALSK_ERR_INPUT, "row range [" + std::to_string(rb) + ", " + std::to_string(re) +
                                       ") outside matrix");
    return acc_double ? assemble<double>(r, theta, theta_rows, f, lambda, rb, re, A, B)
                      : assemble<float>(r, theta, theta_rows, f, lambda, rb, re, A, B);
}

// batch_solve (solver.hpp:320-325)
alsk_status orc_batch_solve(const float* A, const float* B, int64_t count, int f, int zero_row,
                            float* X) {
    double piv = 0;
    int col = 0;
    const int64_t bad = solve(A, B, count, f, zero_row != 0, X, &piv, &col);
    if (bad >= 0) return breakdown(bad, piv, col);
    return ALSK_OK;
}

// update_x (solver.hpp:330-345): batches of batch_rows rows, assemble then solve.
alsk_status orc_update_x(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                         double lambda, int acc_double, int64_t batch_rows, float* X) {
    const alsk_status s = shapes(r, theta_rows, f);
    if (s != ALSK_OK) return s;
    const int64_t step = batch_rows < 1 ? 1 : batch_rows;
    std::vector<float> A, B;
    for (int64_t b0 = 0; b0 < r->rows; b0 += step) {
        const int64_t b1 = std::min(r->rows, b0 + step);
        A.assign(static_cast<size_t>(b1 - b0) * f * f, 0.f);
        B.assign(static_cast<size_t>(b1 - b0) * f, 0.f);
        const alsk_status h = orc_hermitian(r, theta, theta_rows, f, lambda, acc_double, b0, b1, 1,
                                            A.data(), B.data());
        if (h != ALSK_OK) return h;
        double piv = 0;
        int col = 0;
        const int64_t bad = solve(A.data(), B.data(), b1 - b0, f, false, X + b0 * f, &piv, &col);
        if (bad >= 0) return breakdown(bad, piv, col);
    }
    return ALSK_OK;
}

// loss (solver.hpp:358-390)
alsk_status orc_loss(const alsk_csr* r, const float* x, int64_t x_rows, const float* theta,
                     int64_t theta_rows, int f, double lambda, double* out) {
    if (x_rows != r->rows) return err(ALSK_ERR_INPUT, "x rows do not match matrix rows");
    const alsk_status s = shapes(r, theta_rows, f);
    if (s != ALSK_OK) return s;
    double sq = 0.0;
    std::vector<int64_t> col_nnz(static_cast<size_t>(r->cols), 0);
    for (int64_t u = 0; u < r->rows; ++u)
        for (int64_t k = r->row_ptr[u]; k < r->row_ptr[u + 1]; ++k) {
            const int64_t v = r->col_idx[k];
            ++col_nnz[v];
            const double d = static_cast<double>(r->values[k]) - dot_rows(x + u * f, theta + v * f, f);
            sq += d * d;
        }
    double reg = 0.0;
    for (int64_t u = 0; u < r->rows; ++u) {
        const double n = static_cast<double>(r->row_ptr[u + 1] - r->row_ptr[u]);
        if (n == 0.0) continue;
        reg += n * dot_rows(x + u * f, x + u * f, f);
    }
    for (int64_t v = 0; v < r->cols; ++v) {
        const double n = static_cast<double>(col_nnz[v]);
        if (n == 0.0) continue;
        reg += n * dot_rows(theta + v * f, theta + v * f, f);
    }
    *out = sq + lambda * reg;
    return ALSK_OK;
}

// rmse (solver.hpp:393-406)
alsk_status orc_rmse(const alsk_triplet* t, int64_t count, const float* x, int64_t x_rows,
                     const float* theta, int64_t theta_rows, int f, double* out) {
    if (count <= 0) return err(ALSK_ERR_INPUT, "empty test set");
    double sq = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        if (t[i].row < 0 || t[i].row >= x_rows || t[i].col < 0 || t[i].col >= theta_rows)
            return err(ALSK_ERR_INPUT, "test pair (" + std::to_string(t[i].row) + ", " +
                                           std::to_string(t[i].col) + ") outside factor shapes");
        const double d = static_cast<double>(t[i].value) - dot_rows(x + t[i].row * f, theta + t[i].col * f, f);
        sq += d * d;
    }
    *out = std::sqrt(sq / static_cast<double>(count));
    return ALSK_OK;
}

// csr_to_csc (sparse.hpp:185-207): counting sort, rows ascending within each column.
alsk_status orc_csr_to_csc(const alsk_csr* a, int64_t* col_ptr, int32_t* row_idx, float* vals) {
    std::fill(col_ptr, col_ptr + a->cols + 1, 0);
    for (int64_t k = 0; k < a->nnz; ++k) ++col_ptr[a->col_idx[k] + 1];
    for (int64_t v = 0; v < a->cols; ++v) col_ptr[v + 1] += col_ptr[v];
    std::vector<int64_t> next(col_ptr, col_ptr + a->cols);
    for (int64_t u = 0; u < a->rows; ++u)
        for (int64_t k = a->row_ptr[u]; k < a->row_ptr[u + 1]; ++k) {
            const int64_t slot = next[a->col_idx[k]]++;
            row_idx[slot] = static_cast<int32_t>(u);
            vals[slot] = a->values[k];
        }
    return ALSK_OK;
}

// csr_from_triplets (sparse.hpp:132-170)
alsk_status orc_csr_from_triplets(int64_t m, int64_t n, const alsk_triplet* t, int64_t count,
                                  int64_t* row_ptr, int32_t* col_idx, float* vals) {
    if (m < 0 || n < 0) return err(ALSK_ERR_INPUT, "matrix dimensions must be non-negative");
    for (int64_t i = 0; i < count; ++i)
        if (t[i].row < 0 || t[i].row >= m || t[i].col < 0 || t[i].col >= n)
            return err(ALSK_ERR_INPUT, "triplet (" + std::to_string(t[i].row) + ", " +
                                           std::to_string(t[i].col) + ") outside " +
                                           std::to_string(m) + "x" + std::to_string(n));
    std::vector<int64_t> order(static_cast<size_t>(count));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        return t[a].row != t[b].row ? t[a].row < t[b].row : t[a].col < t[b].col;
    });
    std::fill(row_ptr, row_ptr + m + 1, 0);
    for (int64_t k = 0; k < count; ++k) {
        const alsk_triplet& e = t[order[k]];
        if (k > 0) {
            const alsk_triplet& p = t[order[k - 1]];
            if (p.row == e.row && p.col == e.col)
                return err(ALSK_ERR_INPUT, "duplicate coordinate (" + std::to_string(e.row) + ", " +
                                               std::to_string(e.col) + ")");
        }
        col_idx[k] = static_cast<int32_t>(e.col);
        vals[k] = e.value;
        ++row_ptr[e.row + 1];
    }
    for (int64_t u = 0; u < m; ++u) row_ptr[u + 1] += row_ptr[u];
    return ALSK_OK;
}

// even_cuts (sparse.hpp:95-100)
void orc_even_cuts(int64_t total, int parts, int64_t* cuts) {
    for (int k = 0; k <= parts; ++k) cuts[k] = total * k / parts;
}

// slice_cuts (parallel.hpp:160-168)
void orc_slice_cuts(int64_t count, int p, int64_t* cuts) {
    const int64_t base = count / p, rem = count % p;
    cuts[0] = 0;
    for (int i = 0; i < p; ++i) cuts[i + 1] = cuts[i] + base + (i < rem ? 1 : 0);
}

// grid_partition (sparse.hpp:250-314), counts: block (i,j) at j*p+i.
alsk_status orc_grid_partition_counts(const alsk_csr* r, int p, int q, int64_t* row_cuts,
                                      int64_t* col_cuts, int64_t* block_nnz) {
    const int64_t qmax = std::max<int64_t>(r->rows, 1), pmax = std::max<int64_t>(r->cols, 1);
    if (q < 1 || q > qmax)
        return err(ALSK_ERR_INPUT, "row partition count q=" + std::to_string(q) + " outside [1, " +
                                       std::to_string(qmax) + "]");
    if (p < 1 || p > pmax)
        return err(ALSK_ERR_INPUT, "column partition count p=" + std::to_string(p) + " outside [1, " +
                                       std::to_string(pmax) + "]");
    orc_even_cuts(r->rows, q, row_cuts);
    orc_even_cuts(r->cols, p, col_cuts);
    std::fill(block_nnz, block_nnz + static_cast<int64_t>(p) * q, 0);
    for (int j = 0; j < q; ++j)
        for (int64_t u = row_cuts[j]; u < row_cuts[j + 1]; ++u) {
            int i = 0;
            for (int64_t k = r->row_ptr[u]; k < r->row_ptr[u + 1]; ++k) {
                while (r->col_idx[k] >= col_cuts[i + 1]) ++i;
                ++block_nnz[static_cast<int64_t>(j) * p + i];
            }
        }
    return ALSK_OK;
}

alsk_status orc_grid_partition_fill(const alsk_csr* r, int p, int q, int64_t* const* brp,
                                    int32_t* const* bci, float* const* bv) {
    std::vector<int64_t> rc(q + 1), cc(p + 1), bn(static_cast<size_t>(p) * q);
    const alsk_status s = orc_grid_partition_counts(r, p, q, rc.data(), cc.data(), bn.data());
    if (s != ALSK_OK) return s;
    for (int j = 0; j < q; ++j) {
        const int64_t r0 = rc[j], r1 = rc[j + 1];
        for (int i = 0; i < p; ++i) std::fill(brp[j * p + i], brp[j * p + i] + (r1 - r0) + 1, 0);
        for (int64_t u = r0; u < r1; ++u) {
            int i = 0;
            for (int64_t k = r->row_ptr[u]; k < r->row_ptr[u + 1]; ++k) {
                while (r->col_idx[k] >= cc[i + 1]) ++i;
                ++brp[j * p + i][u - r0 + 1];
            }
        }
        for (int i = 0; i < p; ++i)
            for (int64_t u = 0; u < r1 - r0; ++u) brp[j * p + i][u + 1] += brp[j * p + i][u];
        std::vector<int64_t> cur(p);
        for (int64_t u = r0; u < r1; ++u) {
            std::fill(cur.begin(), cur.end(), 0);
            int i = 0;
            for (int64_t k = r->row_ptr[u]; k < r->row_ptr[u + 1]; ++k) {
                while (r->col_idx[k] >= cc[i + 1]) ++i;
                const int64_t slot = brp[j * p + i][u - r0] + cur[i]++;
                bci[j * p + i][slot] = r->col_idx[k];
                bv[j * p + i][slot] = r->values[k];
            }
        }
    }
    return ALSK_OK;
}

// split_train_test (dataio.hpp:251-290)
alsk_status orc_split_train_test(const alsk_csr* r, double holdout, uint64_t seed, int64_t* k_out,
                                 int64_t* trp, int32_t* tci, float* tv, alsk_triplet* test) {
    if (!(holdout > 0.0) || !(holdout < 1.0))
        return err(ALSK_ERR_INPUT, "holdout fraction must lie strictly between 0 and 1");
    const int64_t nnz = r->nnz;
    const int64_t k = static_cast<int64_t>(std::floor(holdout * static_cast<double>(nnz)));
    *k_out = k;
    if (!trp) return ALSK_OK;
    std::vector<int64_t> pos(static_cast<size_t>(nnz));
    std::iota(pos.begin(), pos.end(), 0);
    std::mt19937_64 rng(seed);
    for (int64_t t = 0; t < k; ++t) {
        const uint64_t range = static_cast<uint64_t>(nnz - t);
        const uint64_t thr = (0 - range) % range;
        uint64_t v;
        do v = rng(); while (v < thr);
        std::swap(pos[t], pos[t + static_cast<int64_t>(v % range)]);
    }
    std::vector<char> held(static_cast<size_t>(nnz), 0);
    for (int64_t t = 0; t < k; ++t) held[pos[t]] = 1;
    int64_t a = 0, b = 0;
    trp[0] = 0;
    for (int64_t u = 0; u < r->rows; ++u) {
        for (int64_t e = r->row_ptr[u]; e < r->row_ptr[u + 1]; ++e) {
            if (held[e]) test[b++] = alsk_triplet{u, r->col_idx[e], r->values[e]};
            else { tci[a] = r->col_idx[e]; tv[a] = r->values[e]; ++a; }
        }
        trp[u + 1] = a;
    }
    return ALSK_OK;
}

// reduce_batches one-phase (parallel.hpp:206-280): slice i of the double sum of all p
// partials, own partial first then the others in ascending source order, rounded once.
alsk_status orc_parallel_reduce(const float* const* pa, const float* const* pb, int p,
                                int64_t count, int f, float* const* oa, float* const* ob) {
    std::vector<int64_t> cuts(p + 1);
    orc_slice_cuts(count, p, cuts.data());
    const int64_t ff = static_cast<int64_t>(f) * f;
    for (int s = 0; s < p; ++s) {
        const int64_t c0 = cuts[s], c1 = cuts[s + 1];
        const int64_t la = (c1 - c0) * ff, lb = (c1 - c0) * f;
        std::vector<double> acc(static_cast<size_t>(la + lb));
        for (int64_t e = 0; e < la; ++e) acc[e] = pa[s][c0 * ff + e];
        for (int64_t e = 0; e < lb; ++e) acc[la + e] = pb[s][c0 * f + e];
        for (int src = 0; src < p; ++src) {
            if (src == s) continue;
            for (int64_t e = 0; e < la; ++e) acc[e] += static_cast<double>(pa[src][c0 * ff + e]);
            for (int64_t e = 0; e < lb; ++e) acc[la + e] += static_cast<double>(pb[src][c0 * f + e]);
        }
        for (int64_t e = 0; e < la; ++e) oa[s][e] = static_cast<float>(acc[e]);
        for (int64_t e = 0; e < lb; ++e) ob[s][e] = static_cast<float>(acc[la + e]);
    }
    return ALSK_OK;
}

// random_triplets (tests/test_util.hpp:36-48): nnz distinct coordinates from one
// mt19937_64 stream, ratings 0.5 + 4.5*unit with unit = (rng()>>11)*2^-53. Lets the
// Python tests rebuild the reference tests' instances seed for seed.
void orc_random_triplets(uint64_t seed, int64_t m, int64_t n, int64_t nnz, alsk_triplet* out) {
    std::mt19937_64 rng(seed);
    std::set<std::pair<int64_t, int64_t>> seen;
    int64_t k = 0;
    while (k < nnz) {
        const int64_t u = static_cast<int64_t>(rng() % static_cast<uint64_t>(m));
        const int64_t v = static_cast<int64_t>(rng() % static_cast<uint64_t>(n));
        if (!seen.insert({u, v}).second) continue;
        const double unit = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        out[k++] = alsk_triplet{u, v, static_cast<float>(0.5 + 4.5 * unit)};
    }
}

}  // extern "C"
