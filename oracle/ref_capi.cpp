// ORACLE — TEST INFRASTRUCTURE ONLY (checker and CPU baseline, never the product).
//
// Compiles the UNMODIFIED reference headers from /root/reference/proj/include (path via
// -I, namespace renamed with -Dalskit=alskit_ref) into oracle/_ref/libalskit_ref.so and
// exposes them through plain-C entry points with the same buffer conventions as
// include/alskit_cuda.h. No reference source is copied into this repository; the build
// recipe is oracle/Makefile, outputs land only in oracle/_ref/ (git-ignored).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "alskit/alskit.hpp"  // from /root/reference/proj/include, namespace alskit_ref
#include "../include/alskit_cuda.h"  // our C ABI types only (by path: -I points at the reference)
#include "../paper_1603_03820_b200/csrc/synth_host.hpp"  // the bench's data generator (CUDA-free, shared)

namespace R = alskit_ref;

namespace {

thread_local std::string g_err;

R::CsrMatrix to_csr(const alsk_csr* a) {
    R::CsrMatrix m;
    m.rows = a->rows;
    m.cols = a->cols;
    m.col_offset = a->col_offset;
    m.row_ptr.assign(a->row_ptr, a->row_ptr + a->rows + 1);
    m.col_idx.assign(a->col_idx, a->col_idx + a->nnz);
    m.values.assign(a->values, a->values + a->nnz);
    return m;
}

R::FactorMatrix to_factor(const float* p, int64_t rows, int f) {
    R::FactorMatrix m(rows, f);
    std::memcpy(m.entries.data(), p, sizeof(float) * rows * f);
    return m;
}

R::SolverConfig to_cfg(double lambda, int acc_double, int64_t batch_rows, int threads) {
    R::SolverConfig c;
    c.lambda = lambda;
    c.accumulate_double = acc_double != 0;
    c.batch_rows = batch_rows;
    c.threads = threads;
    return c;
}

template <class Fn>
alsk_status guarded(Fn&& fn) {
    try {
        fn();
        return ALSK_OK;
    } catch (const R::Error& e) {
        g_err = e.what();
        switch (e.category()) {
            case R::Error::Category::input: return ALSK_ERR_INPUT;
            case R::Error::Category::capacity: return ALSK_ERR_CAPACITY;
            case R::Error::Category::numerical: return ALSK_ERR_NUMERICAL;
            case R::Error::Category::io: return ALSK_ERR_IO;
        }
        return ALSK_ERR_INPUT;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_hardware_threads(void) { return R::resolve_threads(0); }

alsk_status ref_hermitian_mo(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                             double lambda, int acc_double, int bin, int64_t rb, int64_t re,
                             float* A, float* B) {
    return guarded([&] {
        R::SolverConfig cfg = to_cfg(lambda, acc_double, 4096, 1);
        cfg.bin = bin;
        R::HermitianBatch out;
        R::get_hermitian_mo_into(to_csr(r), to_factor(theta, theta_rows, f), cfg, rb, re, out);
        std::memcpy(A, out.a.data(), sizeof(float) * out.a.size());
        std::memcpy(B, out.b.data(), sizeof(float) * out.b.size());
    });
}

alsk_status ref_local_hermitian(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                                double lambda, int acc_double, float* A, float* B) {
    return guarded([&] {
        const R::HermitianBatch out = R::local_hermitian(to_csr(r), to_factor(theta, theta_rows, f),
                                                         to_cfg(lambda, acc_double, 4096, 1));
        std::memcpy(A, out.a.data(), sizeof(float) * out.a.size());
        std::memcpy(B, out.b.data(), sizeof(float) * out.b.size());
    });
}

alsk_status ref_batch_solve(const float* A, const float* B, int64_t count, int f, int zero_row,
                            float* X) {
    return guarded([&] {
        R::HermitianBatch batch;
        batch.resize(count, f);
        std::memcpy(batch.a.data(), A, sizeof(float) * batch.a.size());
        std::memcpy(batch.b.data(), B, sizeof(float) * batch.b.size());
        const R::FactorMatrix x =
            R::batch_solve(batch, zero_row ? R::BreakdownPolicy::zero_row : R::BreakdownPolicy::fail, 1);
        std::memcpy(X, x.entries.data(), sizeof(float) * x.entries.size());
    });
}

// update_x with the reference's own threading: threads=0 means hardware_concurrency
// (thread_pool.hpp:20-24). This is also the CPU baseline arm of bench.py.
alsk_status ref_update_x(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                         double lambda, int acc_double, int64_t batch_rows, int threads, float* X) {
    return guarded([&] {
        const R::FactorMatrix x = R::update_x(to_csr(r), to_factor(theta, theta_rows, f),
                                              to_cfg(lambda, acc_double, batch_rows, threads));
        std::memcpy(X, x.entries.data(), sizeof(float) * x.entries.size());
    });
}

alsk_status ref_loss(const alsk_csr* r, const float* x, int64_t x_rows, const float* theta,
                     int64_t theta_rows, int f, double lambda, double* out) {
    return guarded([&] {
        *out = R::loss(to_csr(r), to_factor(x, x_rows, f), to_factor(theta, theta_rows, f), lambda);
    });
}

alsk_status ref_rmse(const alsk_triplet* t, int64_t count, const float* x, int64_t x_rows,
                     const float* theta, int64_t theta_rows, int f, double* out) {
    return guarded([&] {
        std::vector<R::Triplet> test(static_cast<size_t>(count));
        for (int64_t i = 0; i < count; ++i) test[i] = R::Triplet{t[i].row, t[i].col, t[i].value};
        *out = R::rmse(test, to_factor(x, x_rows, f), to_factor(theta, theta_rows, f));
    });
}

alsk_status ref_csr_to_csc(const alsk_csr* a, int64_t* col_ptr, int32_t* row_idx, float* vals) {
    return guarded([&] {
        const R::CscMatrix c = R::csr_to_csc(to_csr(a));
        std::memcpy(col_ptr, c.col_ptr.data(), sizeof(int64_t) * c.col_ptr.size());
        std::memcpy(row_idx, c.row_idx.data(), sizeof(int32_t) * c.row_idx.size());
        std::memcpy(vals, c.values.data(), sizeof(float) * c.values.size());
    });
}

alsk_status ref_csr_from_triplets(int64_t m, int64_t n, const alsk_triplet* t, int64_t count,
                                  int64_t* row_ptr, int32_t* col_idx, float* vals) {
    return guarded([&] {
        std::vector<R::Triplet> tr(static_cast<size_t>(count));
        for (int64_t i = 0; i < count; ++i) tr[i] = R::Triplet{t[i].row, t[i].col, t[i].value};
        const R::CsrMatrix a = R::csr_from_triplets(m, n, tr);
        std::memcpy(row_ptr, a.row_ptr.data(), sizeof(int64_t) * a.row_ptr.size());
        std::memcpy(col_idx, a.col_idx.data(), sizeof(int32_t) * a.col_idx.size());
        std::memcpy(vals, a.values.data(), sizeof(float) * a.values.size());
    });
}

void ref_random_factor(int64_t rows, int f, uint64_t seed, float* out) {
    const R::FactorMatrix x = R::random_factor(rows, f, seed);
    std::memcpy(out, x.entries.data(), sizeof(float) * x.entries.size());
}

uint64_t ref_mix_seed(uint64_t seed, uint64_t salt) { return R::detail::mix_seed(seed, salt); }

alsk_status ref_split_train_test(const alsk_csr* r, double holdout, uint64_t seed, int64_t* k_out,
                                 int64_t* trp, int32_t* tci, float* tv, alsk_triplet* test) {
    return guarded([&] {
        const R::SplitResult s = R::split_train_test(to_csr(r), holdout, seed);
        *k_out = static_cast<int64_t>(s.test.size());
        if (!trp) return;
        std::memcpy(trp, s.train.row_ptr.data(), sizeof(int64_t) * s.train.row_ptr.size());
        std::memcpy(tci, s.train.col_idx.data(), sizeof(int32_t) * s.train.col_idx.size());
        std::memcpy(tv, s.train.values.data(), sizeof(float) * s.train.values.size());
        for (size_t i = 0; i < s.test.size(); ++i)
            test[i] = alsk_triplet{s.test[i].row, s.test[i].col, s.test[i].value};
    });
}

alsk_status ref_grid_partition_counts(const alsk_csr* r, int p, int q, int64_t* row_cuts,
                                      int64_t* col_cuts, int64_t* block_nnz) {
    return guarded([&] {
        const R::GridPartition g = R::grid_partition(to_csr(r), p, q);
        std::memcpy(row_cuts, g.row_cuts.data(), sizeof(int64_t) * g.row_cuts.size());
        std::memcpy(col_cuts, g.col_cuts.data(), sizeof(int64_t) * g.col_cuts.size());
        for (size_t b = 0; b < g.blocks.size(); ++b) block_nnz[b] = g.blocks[b].nnz();
    });
}

alsk_status ref_grid_partition_fill(const alsk_csr* r, int p, int q, int64_t* const* brp,
                                    int32_t* const* bci, float* const* bv) {
    return guarded([&] {
        const R::GridPartition g = R::grid_partition(to_csr(r), p, q);
        for (size_t b = 0; b < g.blocks.size(); ++b) {
            const R::CsrMatrix& blk = g.blocks[b];
            std::memcpy(brp[b], blk.row_ptr.data(), sizeof(int64_t) * blk.row_ptr.size());
            std::memcpy(bci[b], blk.col_idx.data(), sizeof(int32_t) * blk.col_idx.size());
            std::memcpy(bv[b], blk.values.data(), sizeof(float) * blk.values.size());
        }
    });
}

// parallel_reduce over the reference's one-phase or two-phase schedule.
alsk_status ref_parallel_reduce(const float* const* pa, const float* const* pb, int p,
                                int64_t count, int f, const int32_t* group_of, int two_phase,
                                float* const* oa, float* const* ob) {
    return guarded([&] {
        std::vector<R::HermitianBatch> parts(p);
        for (int i = 0; i < p; ++i) {
            parts[i].resize(count, f);
            std::memcpy(parts[i].a.data(), pa[i], sizeof(float) * parts[i].a.size());
            std::memcpy(parts[i].b.data(), pb[i], sizeof(float) * parts[i].b.size());
        }
        R::Topology topo;
        topo.workers = p;
        if (group_of) {
            int ng = 0;
            for (int i = 0; i < p; ++i) ng = std::max(ng, group_of[i] + 1);
            topo.groups.assign(ng, {});
            for (int i = 0; i < p; ++i) topo.groups[group_of[i]].push_back(i);
        }
        const R::ReduceSchedule sched = R::build_reduce_schedule(
            topo, two_phase ? R::ReduceScheme::two_phase : R::ReduceScheme::one_phase);
        const auto out = R::parallel_reduce(parts, sched, 1);
        for (int i = 0; i < p; ++i) {
            std::memcpy(oa[i], out[i].a.data(), sizeof(float) * out[i].a.size());
            std::memcpy(ob[i], out[i].b.data(), sizeof(float) * out[i].b.size());
        }
    });
}

// su_als_update_x over a grid built by the reference itself from `r`.
alsk_status ref_su_als_update_x(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                                int p, int q, double lambda, int acc_double, int two_phase,
                                float* X) {
    return guarded([&] {
        const R::CsrMatrix rr = to_csr(r);
        const R::GridPartition g = R::grid_partition(rr, p, q);
        const auto parts = R::split_factor(to_factor(theta, theta_rows, f), g.col_cuts);
        R::Topology topo;
        topo.workers = p;
        if (two_phase) {
            topo.groups.assign(2, {});
            for (int i = 0; i < p; ++i) topo.groups[i < p / 2 ? 0 : 1].push_back(i);
        }
        const R::FactorMatrix x = R::su_als_update_x(
            g, parts, topo, two_phase ? R::ReduceScheme::two_phase : R::ReduceScheme::one_phase,
            to_cfg(lambda, acc_double, 4096, 1));
        std::memcpy(X, x.entries.data(), sizeof(float) * x.entries.size());
    });
}

// Planner KAT (parallel.hpp:287-386)
alsk_status ref_plan_partition(int64_t m, int64_t n, int64_t nnz, int f, int workers,
                               int64_t capacity, int64_t headroom, int* p_out, int* q_out,
                               int64_t* footprint_out) {
    return guarded([&] {
        R::Topology topo;
        topo.workers = workers;
        topo.capacity = capacity;
        const R::PartitionPlan plan = R::plan_partition(m, n, nnz, f, topo, headroom);
        *p_out = plan.p;
        *q_out = plan.q;
        *footprint_out = plan.per_worker_footprint;
    });
}

// binary ratings cache, the reference's own writer/reader (dataio.hpp:116-163), for
// cross-checking the repo's implementation file for file
alsk_status ref_save_cache(const alsk_csr* a, const char* path) {
    return guarded([&] { R::save_binary_cache(to_csr(a), path); });
}
alsk_status ref_load_cache(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz, int64_t* row_ptr,
                           int32_t* col_idx, float* vals, int64_t cap_rows, int64_t cap_nnz) {
    return guarded([&] {
        const R::CsrMatrix a = R::load_binary_cache(path);
        *rows = a.rows;
        *cols = a.cols;
        *nnz = a.nnz();
        if (a.rows <= cap_rows && a.nnz() <= cap_nnz) {
            std::memcpy(row_ptr, a.row_ptr.data(), sizeof(int64_t) * a.row_ptr.size());
            std::memcpy(col_idx, a.col_idx.data(), sizeof(int32_t) * a.col_idx.size());
            std::memcpy(vals, a.values.data(), sizeof(float) * a.values.size());
        }
    });
}

// checkpoints, the reference's own writer/reader (dataio.hpp:600-651) and restore_latest
// (dataio.hpp:659-686), for cross-checking file for file
alsk_status ref_write_checkpoint(const char* dir, int iteration, int which, int64_t rows, int f, uint64_t digest,
                                 const float* entries) {
    return guarded([&] {
        R::Checkpoint cp;
        cp.iteration = iteration;
        cp.which = static_cast<R::FactorKind>(which);
        cp.factor = R::FactorMatrix(rows, f);
        std::memcpy(cp.factor.entries.data(), entries, sizeof(float) * rows * f);
        cp.digest = digest;
        R::write_checkpoint(cp, dir);
    });
}
alsk_status ref_read_checkpoint(const char* path, int* iteration, int* which, int64_t* rows, int* f,
                                uint64_t* digest, float* entries, int64_t cap) {
    return guarded([&] {
        const R::Checkpoint cp = R::read_checkpoint(path);
        *iteration = cp.iteration;
        *which = static_cast<int>(cp.which);
        *rows = cp.factor.rows;
        *f = cp.factor.f;
        *digest = cp.digest;
        if (static_cast<int64_t>(cp.factor.entries.size()) <= cap)
            std::memcpy(entries, cp.factor.entries.data(), sizeof(float) * cp.factor.entries.size());
    });
}
alsk_status ref_restore_latest_iteration(const char* dir, int* iteration, int* which, int* found) {
    return guarded([&] {
        const auto cp = R::restore_latest(dir);
        *found = cp ? 1 : 0;
        if (cp) {
            *iteration = cp->iteration;
            *which = static_cast<int>(cp->which);
        }
    });
}

}  // extern "C"

// ---- bench.py's reference arm -------------------------------------------------------------
// The reference's own train_run iteration (driver.hpp:113-115, 178-181, 256-258), run in a
// process that never loads libalskit_cuda.so:
//   load_binary_cache -> split_train_test(R, holdout, mix_seed(seed, 2)) ->
//   rt = transpose_of(csr_to_csc(train)); x = random_factor(m, f, seed),
//   theta = random_factor(n, f, mix_seed(seed, 1)); per iteration
//   x = update_x(train, theta, cfg); theta = update_x(rt, x, cfg)   (threads = 0).
// The cache is written once by ref_bench_write_cache (the shared synthetic generator,
// synth_host.hpp, through the reference's own save_binary_cache).
namespace {
struct BenchState {
    R::CsrMatrix train, rt;
    std::vector<R::Triplet> test;
    R::FactorMatrix x, theta;
    R::SolverConfig cfg;
};
BenchState* g_bench = nullptr;

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

R::CsrMatrix prefix_rows(const R::CsrMatrix& a, int64_t k) {
    R::CsrMatrix s;
    s.rows = k;
    s.cols = a.cols;
    s.col_offset = a.col_offset;
    s.row_ptr.assign(a.row_ptr.begin(), a.row_ptr.begin() + k + 1);
    const int64_t nz = s.row_ptr.back();
    s.col_idx.assign(a.col_idx.begin(), a.col_idx.begin() + nz);
    s.values.assign(a.values.begin(), a.values.begin() + nz);
    return s;
}
}  // namespace

extern "C" {

alsk_status ref_bench_write_cache(int64_t m, int64_t n, int64_t nnz, uint64_t seed, const char* path) {
    return guarded([&] {
        R::CsrMatrix a;
        a.rows = m;
        a.cols = n;
        a.row_ptr.resize(static_cast<size_t>(m) + 1);
        a.col_idx.resize(static_cast<size_t>(nnz));
        a.values.resize(static_cast<size_t>(nnz));
        if (alsk_synth::synth_csr(m, n, nnz, seed, 0, a.row_ptr.data(), a.col_idx.data(), a.values.data()) != 0)
            throw R::InputError("invalid synthetic shape");
        R::save_binary_cache(a, path);
    });
}

// Load + split + transpose + init; seconds of each setup stage into setup_s[0..3].
alsk_status ref_bench_prepare(const char* cache, double holdout, uint64_t seed, int f, double lambda,
                              int64_t* train_nnz, int64_t* test_count, double* setup_s) {
    return guarded([&] {
        delete g_bench;
        g_bench = new BenchState();
        auto t0 = std::chrono::steady_clock::now();
        const R::CsrMatrix r = R::load_binary_cache(cache);
        setup_s[0] = seconds_since(t0);
        t0 = std::chrono::steady_clock::now();
        R::SplitResult split = R::split_train_test(r, holdout, R::detail::mix_seed(seed, 2));
        setup_s[1] = seconds_since(t0);
        t0 = std::chrono::steady_clock::now();
        g_bench->rt = R::transpose_of(R::csr_to_csc(split.train));
        setup_s[2] = seconds_since(t0);
        g_bench->train = std::move(split.train);
        g_bench->test = std::move(split.test);
        t0 = std::chrono::steady_clock::now();
        g_bench->x = R::random_factor(g_bench->train.rows, f, seed);
        g_bench->theta = R::random_factor(g_bench->train.cols, f, R::detail::mix_seed(seed, 1));
        setup_s[3] = seconds_since(t0);
        g_bench->cfg.f = f;
        g_bench->cfg.lambda = lambda;
        g_bench->cfg.threads = 0;  // hardware_concurrency (thread_pool.hpp:20-24)
        *train_nnz = g_bench->train.nnz();
        *test_count = static_cast<int64_t>(g_bench->test.size());
    });
}

// One full ALS iteration exactly as train_run does it (driver.hpp:256-258).
alsk_status ref_bench_iteration(double* x_half_s, double* theta_half_s) {
    return guarded([&] {
        if (!g_bench) throw R::InputError("ref_bench_prepare first");
        auto t0 = std::chrono::steady_clock::now();
        g_bench->x = R::update_x(g_bench->train, g_bench->theta, g_bench->cfg);
        *x_half_s = seconds_since(t0);
        t0 = std::chrono::steady_clock::now();
        g_bench->theta = R::update_x(g_bench->rt, g_bench->x, g_bench->cfg);
        *theta_half_s = seconds_since(t0);
    });
}

// A bounded sample: update_x on the first kx rows of train and the first kt rows of rt,
// timed separately, plus their nonzero counts (for extrapolation by nnz).
alsk_status ref_bench_sample(int64_t kx, int64_t kt, double* x_s, double* t_s, int64_t* nzx, int64_t* nzt) {
    return guarded([&] {
        if (!g_bench) throw R::InputError("ref_bench_prepare first");
        kx = std::min<int64_t>(kx, g_bench->train.rows);
        kt = std::min<int64_t>(kt, g_bench->rt.rows);
        const R::CsrMatrix sx = prefix_rows(g_bench->train, kx), st = prefix_rows(g_bench->rt, kt);
        *nzx = sx.nnz();
        *nzt = st.nnz();
        auto t0 = std::chrono::steady_clock::now();
        (void)R::update_x(sx, g_bench->theta, g_bench->cfg);
        *x_s = seconds_since(t0);
        t0 = std::chrono::steady_clock::now();
        (void)R::update_x(st, g_bench->x, g_bench->cfg);
        *t_s = seconds_since(t0);
    });
}

// train_J and test RMSE of the current factors (the reference's serial eval, timed apart).
alsk_status ref_bench_eval(double* loss_out, double* rmse_out, double* loss_s, double* rmse_s) {
    return guarded([&] {
        if (!g_bench) throw R::InputError("ref_bench_prepare first");
        auto t0 = std::chrono::steady_clock::now();
        *loss_out = R::loss(g_bench->train, g_bench->x, g_bench->theta, g_bench->cfg.lambda);
        *loss_s = seconds_since(t0);
        t0 = std::chrono::steady_clock::now();
        *rmse_out = g_bench->test.empty() ? 0.0 : R::rmse(g_bench->test, g_bench->x, g_bench->theta);
        *rmse_s = seconds_since(t0);
    });
}

// Copies of the current factors (x: rows*f, theta: cols*f).
alsk_status ref_bench_factors(float* x, float* theta) {
    return guarded([&] {
        if (!g_bench) throw R::InputError("ref_bench_prepare first");
        std::memcpy(x, g_bench->x.entries.data(), sizeof(float) * g_bench->x.entries.size());
        std::memcpy(theta, g_bench->theta.entries.data(), sizeof(float) * g_bench->theta.entries.size());
    });
}

void ref_bench_release(void) {
    delete g_bench;
    g_bench = nullptr;
}

}  // extern "C"

// The reference's own train_run (driver.hpp:107-268) on a binary cache, for the C++ driver
// parity test (tests/test_train_run.py): factors out, metrics / checkpoints on disk.
// stop_after > 0: the callback stops the run after that iteration (a killed run).
// The same with the planner fields (config.hpp:54-60): capacity (scalars, 0 = unlimited),
// force_p/force_q (0 = plan), one worker -- the run tests/test_train_run.py compares with our
// train_run's out-of-core sides.
extern "C" alsk_status ref_train_run_plan(const char* cache, int f, double lambda, int iterations, uint64_t seed,
                                          int acc_double, const char* metrics, int64_t capacity, int force_p,
                                          int force_q, float* x_out, float* theta_out) {
    return guarded([&] {
        R::RunConfig cfg;
        cfg.data = cache;
        cfg.format = R::RatingsFormat::binary_cache;
        cfg.f = f;
        cfg.lambda = lambda;
        cfg.iterations = iterations;
        cfg.seed = seed;
        cfg.accumulate_double = acc_double != 0;
        cfg.metrics = metrics ? metrics : "";
        cfg.capacity = capacity;
        cfg.force_p = force_p;
        cfg.force_q = force_q;
        const R::TrainResult r = R::train_run(cfg);
        std::memcpy(x_out, r.x.entries.data(), sizeof(float) * r.x.entries.size());
        std::memcpy(theta_out, r.theta.entries.data(), sizeof(float) * r.theta.entries.size());
    });
}

extern "C" alsk_status ref_train_run(const char* cache, int f, double lambda, int iterations, uint64_t seed,
                                     int acc_double, const char* ckpt_dir, const char* metrics, int resume,
                                     int stop_after, float* x_out, float* theta_out, int* start_iteration,
                                     uint64_t* digest) {
    return guarded([&] {
        R::RunConfig cfg;
        cfg.data = cache;
        cfg.format = R::RatingsFormat::binary_cache;
        cfg.f = f;
        cfg.lambda = lambda;
        cfg.iterations = iterations;
        cfg.seed = seed;
        cfg.accumulate_double = acc_double != 0;
        cfg.checkpoint_dir = ckpt_dir ? ckpt_dir : "";
        cfg.metrics = metrics ? metrics : "";
        cfg.resume = resume != 0;
        R::IterationCallback cb;
        if (stop_after > 0) cb = [&](int t, const R::FactorMatrix&, const R::FactorMatrix&) { return t < stop_after; };
        const R::TrainResult r = R::train_run(cfg, cb);
        std::memcpy(x_out, r.x.entries.data(), sizeof(float) * r.x.entries.size());
        std::memcpy(theta_out, r.theta.entries.data(), sizeof(float) * r.theta.entries.size());
        *start_iteration = r.start_iteration;
        *digest = r.digest;
    });
}
