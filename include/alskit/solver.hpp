// alskit drop-in (B200): the ALS hot path (reference solver.hpp:30-452) on libalskit_cuda.
//
// Same names, signatures and error behaviour. With SolverConfig::accumulate_double = true
// (the reference default) the device runs the reference-order FP64 kernels and the
// results are bit-identical to the reference; with accumulate_double = false it runs the
// fused FP32 kernel (register-blocked Hermitian + in-register Cholesky), within 1e-3
// normwise per half-sweep. bin and threads never change results (solver.hpp:88-91).
#pragma once

#include <cmath>
#include <functional>
#include <limits>
#include <memory>
#include <span>
#include <vector>

#include "alskit/common.hpp"
#include "alskit/factor.hpp"
#include "alskit/sparse.hpp"

namespace alskit {

struct HermitianBatch {  // solver.hpp:30-58
    offset_t count = 0;
    int f = 0;
    std::vector<real_t> a;  // count * f * f
    std::vector<real_t> b;  // count * f
    void resize(offset_t count_, int f_) {
        count = count_;
        f = f_;
        a.resize(static_cast<std::size_t>(count_) * f_ * f_);
        b.resize(static_cast<std::size_t>(count_) * f_);
    }
    [[nodiscard]] real_t* a_at(offset_t k) noexcept { return a.data() + static_cast<std::size_t>(k) * f * f; }
    [[nodiscard]] const real_t* a_at(offset_t k) const noexcept { return a.data() + static_cast<std::size_t>(k) * f * f; }
    [[nodiscard]] real_t* b_at(offset_t k) noexcept { return b.data() + static_cast<std::size_t>(k) * f; }
    [[nodiscard]] const real_t* b_at(offset_t k) const noexcept { return b.data() + static_cast<std::size_t>(k) * f; }
};

struct SolverConfig {  // solver.hpp:61-69
    int f = 8;
    double lambda = 0.05;
    int bin = 16;
    offset_t batch_rows = 4096;
    bool accumulate_double = true;
    int threads = 0;
    std::uint64_t seed = 42;
};

enum class BreakdownPolicy { fail, zero_row };  // solver.hpp:72

namespace detail {
inline alsk_solver_config cfg_view(const SolverConfig& c) {
    return alsk_solver_config{c.f, c.lambda, c.bin, c.batch_rows, c.accumulate_double ? 1 : 0, c.threads, c.seed};
}
}  // namespace detail

inline HermitianBatch get_hermitian_base(const CsrMatrix& r, const FactorMatrix& theta, double lambda,
                                         bool accumulate_double = true) {  // solver.hpp:277-287
    HermitianBatch out;
    out.resize(r.rows, theta.f);
    const alsk_csr v = detail::view(r);
    detail::check(alsk_get_hermitian_base(&v, theta.entries.data(), theta.rows, theta.f, lambda,
                                          accumulate_double ? 1 : 0, out.a.data(), out.b.data()));
    return out;
}

inline void get_hermitian_mo_into(const CsrMatrix& r, const FactorMatrix& theta, const SolverConfig& cfg,
                                  offset_t row_begin, offset_t row_end, HermitianBatch& out) {  // solver.hpp:292-304
    if (row_begin >= 0 && row_end <= r.rows && row_begin <= row_end) out.resize(row_end - row_begin, theta.f);
    const alsk_csr v = detail::view(r);
    const alsk_solver_config c = detail::cfg_view(cfg);
    detail::check(alsk_get_hermitian_mo_into(&v, theta.entries.data(), theta.rows, theta.f, &c, row_begin, row_end,
                                             out.a.data(), out.b.data()));
}

inline HermitianBatch get_hermitian_mo(const CsrMatrix& r, const FactorMatrix& theta,
                                       const SolverConfig& cfg) {  // solver.hpp:309-314
    HermitianBatch out;
    get_hermitian_mo_into(r, theta, cfg, 0, r.rows, out);
    return out;
}

inline FactorMatrix batch_solve(const HermitianBatch& batch, BreakdownPolicy policy = BreakdownPolicy::fail,
                                int /*threads*/ = 1) {  // solver.hpp:320-325
    FactorMatrix x(batch.count, batch.f);
    detail::check(alsk_batch_solve(batch.a.data(), batch.b.data(), batch.count, batch.f,
                                   policy == BreakdownPolicy::fail ? ALSK_BREAKDOWN_FAIL : ALSK_BREAKDOWN_ZERO_ROW,
                                   x.entries.data()));
    return x;
}

inline FactorMatrix update_x(const CsrMatrix& r, const FactorMatrix& theta, const SolverConfig& cfg) {  // 330-345
    FactorMatrix x(r.rows, theta.f);
    const alsk_csr v = detail::view(r);
    const alsk_solver_config c = detail::cfg_view(cfg);
    detail::check(alsk_update_x(&v, theta.entries.data(), theta.rows, theta.f, &c, x.entries.data()));
    return x;
}

// update_theta (solver.hpp:349-352): the CSC is read in place as the CSR of R^T (the
// reference's transpose_of copy is not needed).
inline FactorMatrix update_theta(const CscMatrix& r_csc, const FactorMatrix& x, const SolverConfig& cfg) {
    FactorMatrix theta(r_csc.cols, x.f);
    const alsk_solver_config c = detail::cfg_view(cfg);
    detail::check(alsk_update_theta(r_csc.rows, r_csc.cols, r_csc.nnz(), r_csc.col_ptr.data(), r_csc.row_idx.data(),
                                    r_csc.values.data(), x.entries.data(), x.rows, x.f, &c, theta.entries.data()));
    return theta;
}

inline double loss(const CsrMatrix& r, const FactorMatrix& x, const FactorMatrix& theta, double lambda) {  // 358-390
    double out = 0.0;
    const alsk_csr v = detail::view(r);
    detail::check(alsk_loss(&v, x.entries.data(), x.rows, theta.entries.data(), theta.rows, theta.f, lambda, &out));
    return out;
}

inline double rmse(std::span<const Triplet> test, const FactorMatrix& x, const FactorMatrix& theta) {  // 393-406
    double out = 0.0;
    detail::check(alsk_rmse(reinterpret_cast<const alsk_triplet*>(test.data()), static_cast<int64_t>(test.size()),
                            x.entries.data(), x.rows, theta.entries.data(), theta.rows, theta.f, &out));
    return out;
}

struct IterationMetrics {  // solver.hpp:409-413
    int iteration = 0;
    double train_j = 0.0;
    double test_rmse = std::numeric_limits<double>::quiet_NaN();
};

struct AlsResult {  // solver.hpp:415-419
    FactorMatrix x;
    FactorMatrix theta;
    std::vector<IterationMetrics> history;
};

using IterationCallback = std::function<bool(int iteration, const FactorMatrix& x, const FactorMatrix& theta)>;

// als_train (solver.hpp:432-452) on a device-resident session: R and R^T are uploaded once
// and the factors stay in HBM; they are copied back only for the callback and the result.
inline AlsResult als_train(const CsrMatrix& r, const CscMatrix& r_csc, std::span<const Triplet> test,
                           const SolverConfig& cfg, int iterations, const IterationCallback& callback = {}) {
    if (iterations < 0) throw InputError("iterations must be >= 0");
    if (r_csc.rows != r.rows || r_csc.cols != r.cols || r_csc.nnz() != r.nnz())
        throw InputError("csr and csc inputs describe different matrices");
    AlsResult res;
    res.x = random_factor(r.rows, cfg.f, cfg.seed);
    res.theta = random_factor(r.cols, cfg.f, detail::mix_seed(cfg.seed, 1));
    if (iterations == 0) return res;
    const alsk_csr v = detail::view(r);
    alsk_session* raw = nullptr;
    detail::check(alsk_session_create(&v, r_csc.col_ptr.data(), r_csc.row_idx.data(), r_csc.values.data(),
                                      reinterpret_cast<const alsk_triplet*>(test.data()),
                                      static_cast<int64_t>(test.size()), cfg.f, cfg.lambda,
                                      cfg.accumulate_double ? ALSK_PREC_FP64_EXACT : ALSK_PREC_FP32, cfg.batch_rows,
                                      res.x.entries.data(), res.theta.entries.data(), &raw));
    std::unique_ptr<alsk_session, void (*)(alsk_session*)> sess(raw, alsk_session_destroy);
    for (int t = 1; t <= iterations; ++t) {
        detail::check(alsk_session_half_x(sess.get()));
        detail::check(alsk_session_half_theta(sess.get()));
        IterationMetrics row;
        row.iteration = t;
        detail::check(alsk_session_loss(sess.get(), &row.train_j));
        if (!test.empty()) detail::check(alsk_session_rmse(sess.get(), &row.test_rmse));
        res.history.push_back(row);
        if (callback) {
            detail::check(alsk_session_factors(sess.get(), res.x.entries.data(), res.theta.entries.data()));
            if (!callback(t, res.x, res.theta)) break;
        }
    }
    detail::check(alsk_session_factors(sess.get(), res.x.entries.data(), res.theta.entries.data()));
    return res;
}

}  // namespace alskit
