// alskit drop-in (B200): train_run, the production training loop of the reference's
// proj/include/alskit/driver.hpp:107-268, on a device-resident
// session of libalskit_cuda.so.
//
// Same iteration order, checkpoints, resume rules and metrics CSV as the reference:
//   split_train_test(R, holdout, mix_seed(seed, 2)); rt = R^T; x = random_factor(m, f, seed),
//   theta = random_factor(n, f, mix_seed(seed, 1)); resume adopts the newest compatible
//   checkpoint (theta@t: also read x@t; a dangling x@t: recompute theta@t first);
//   per iteration X half, snapshot x@t, Theta half, snapshot theta@t, metrics row.
// The factors never leave HBM between halves: snapshots are device-to-device copies taken
// on the session's stream and drained by the CheckpointWriter's background thread, and the
// metrics row's train_J / test RMSE are computed on the device. Config-file parsing, the
// text loaders, the CLI and the multi-worker grid planner stay out of scope:
// the run is given the ratings matrix (or a binary cache path) and the math-defining knobs.
// With accumulate_double = true the run is the reference's bit for bit (factors, metrics
// values, checkpoint bytes).
#pragma once

#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <limits>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "alskit/dataio.hpp"
#include "alskit/parallel.hpp"
#include "alskit/solver.hpp"
#include "alskit/sparse.hpp"

namespace alskit {

/// The math-defining and artifact fields of the reference's RunConfig (config.hpp:37-67).
struct RunConfig {
    std::string data;  // binary ratings cache (the text formats are out of scope)
    double holdout = 0.1;
    int f = 8;
    double lambda = 0.05;
    int iterations = 10;
    int bin = 16;
    offset_t batch_rows = 4096;
    std::uint64_t seed = 42;
    bool accumulate_double = true;
    int threads = 0;
    std::string checkpoint_dir;
    std::string metrics;
    bool resume = false;
    // the planner fields (config.hpp:54-60) with one worker -- the GPU: capacity in scalars
    // (0 = unlimited), headroom -1 = capacity / 24, force_p/force_q 0 = plan. A side whose plan
    // splits (p > 1 or q > 1) runs its half-sweeps out of core over its persisted grid
    // (alsk_ooc_update); workers, groups and the two-phase reduce are out of scope (one GPU,
    // one-phase reduce).
    offset_t capacity = 0;
    offset_t headroom = -1;
    int force_p = 0;
    int force_q = 0;
};

namespace detail {
/// A private scratch directory (persisted grids of a split side), removed with its contents.
class ScratchDir {
  public:
    const std::filesystem::path& path() {
        if (path_.empty()) {
            static std::atomic<unsigned> counter{0};
            path_ = std::filesystem::temp_directory_path() /
                    ("alskit-grids-" + std::to_string(static_cast<long long>(::getpid())) + "-" +
                     std::to_string(counter.fetch_add(1)));
            std::filesystem::create_directories(path_);
        }
        return path_;
    }
    ~ScratchDir() {
        std::error_code ec;
        if (!path_.empty()) std::filesystem::remove_all(path_, ec);
    }

  private:
    std::filesystem::path path_;
};

inline std::string format_real(double v) {  // config.hpp:105-109
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}
inline std::uint64_t fnv1a64(const std::string& s) noexcept {  // common.hpp:78-85
    std::uint64_t h = 1469598103934665603ULL;
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ULL;
    }
    return h;
}
/// driver.hpp:86-97: RMSE of predicting the train mean.
inline double baseline_rmse_of(const CsrMatrix& train, std::span<const Triplet> test) {
    if (test.empty()) return std::numeric_limits<double>::quiet_NaN();
    double mean = 0.0;
    for (real_t v : train.values) mean += static_cast<double>(v);
    if (train.nnz() > 0) mean /= static_cast<double>(train.nnz());
    double sq = 0.0;
    for (const Triplet& t : test) {
        const double d = static_cast<double>(t.value) - mean;
        sq += d * d;
    }
    return std::sqrt(sq / static_cast<double>(test.size()));
}
}  // namespace detail

/// config.hpp:297-307: binds checkpoints to the run (shape + math-defining fields).
inline std::uint64_t run_digest(const RunConfig& cfg, offset_t m, offset_t n, offset_t nnz) {
    std::ostringstream canon;
    canon << "alskit-run;m=" << m << ";n=" << n << ";nnz=" << nnz << ";f=" << cfg.f
          << ";lambda=" << detail::format_real(cfg.lambda) << ";bin=" << cfg.bin << ";batch_rows=" << cfg.batch_rows
          << ";seed=" << cfg.seed << ";holdout=" << detail::format_real(cfg.holdout)
          << ";accumulate_double=" << (cfg.accumulate_double ? 1 : 0);
    return detail::fnv1a64(canon.str());
}

struct IterationRow {  // driver.hpp:50-55
    int iteration = 0;
    double wall_seconds = 0.0;
    double train_j = 0.0;
    double test_rmse = std::numeric_limits<double>::quiet_NaN();
};

struct TrainResult {  // driver.hpp:57-66
    FactorMatrix x;
    FactorMatrix theta;
    std::vector<IterationRow> rows;
    double baseline_rmse = std::numeric_limits<double>::quiet_NaN();
    std::uint64_t digest = 0;
    int start_iteration = 1;
    int p = 1;
    int q = 1;
};

/// driver.hpp:107-268 on the device; `r` is the whole ratings matrix (before the split).
inline TrainResult train_run(const CsrMatrix& r, const RunConfig& cfg, const IterationCallback& after_iteration = {}) {
    if (cfg.f < 1) throw InputError("f must be >= 1");
    if (cfg.iterations < 0) throw InputError("iterations must be >= 0");
    if (cfg.capacity < 0) throw InputError("capacity must be non-negative");  // config.hpp:280-285
    if (cfg.headroom < -1) throw InputError("headroom must be -1 (auto) or non-negative");
    if (cfg.force_p < 0 || cfg.force_q < 0) throw InputError("force_p and force_q must be non-negative");
    if ((cfg.force_p > 0) != (cfg.force_q > 0)) throw InputError("force_p and force_q must be set together");
    if (r.rows < 1 || r.cols < 1) throw InputError("dataset " + cfg.data + " is empty");
    const std::uint64_t digest = run_digest(cfg, r.rows, r.cols, r.nnz());
    const SplitResult split = split_train_test(r, cfg.holdout, detail::mix_seed(cfg.seed, 2));
    const CsrMatrix& train = split.train;
    const CscMatrix rt = csr_to_csc(train);  // the Theta-side view, built once (driver.hpp:115)

    // per-side plan (driver.hpp:121-161) with one worker; a split side's grid is persisted once
    // into a private scratch directory and its half-sweeps stream it
    struct Side {
        int p = 1, q = 1;
        bool split = false;
        std::filesystem::path grid;
    };
    detail::ScratchDir scratch;
    auto make_side = [&](const CsrMatrix& mat, const char* name) {
        Side sd;
        if (cfg.force_p > 0) {
            sd.p = cfg.force_p;
            sd.q = cfg.force_q;
        } else if (cfg.capacity > 0) {
            Topology topo;
            topo.workers = 1;
            topo.capacity = cfg.capacity;
            const PartitionPlan plan = plan_partition(mat.rows, mat.cols, mat.nnz(), cfg.f, topo,
                                                      cfg.headroom >= 0 ? cfg.headroom : cfg.capacity / 24);
            sd.p = plan.p;
            sd.q = plan.q;
        }
        sd.split = sd.p > 1 || sd.q > 1;
        if (sd.split) {
            sd.grid = scratch.path() / name;
            persist_grid(grid_partition(mat, sd.p, sd.q), sd.grid);
        }
        return sd;
    };
    const Side side_x = make_side(train, "grid_x");
    const Side side_t = make_side(transpose_of(rt), "grid_theta");

    TrainResult result;
    result.digest = digest;
    result.p = side_x.p;
    result.q = side_x.q;
    result.baseline_rmse = detail::baseline_rmse_of(train, split.test);
    FactorMatrix x = random_factor(train.rows, cfg.f, cfg.seed);
    FactorMatrix theta = random_factor(train.cols, cfg.f, detail::mix_seed(cfg.seed, 1));

    // resume: adopt the newest compatible checkpoint state (driver.hpp:183-201)
    const bool use_ckpt = !cfg.checkpoint_dir.empty();
    const std::filesystem::path ckpt_dir = cfg.checkpoint_dir;
    int completed = 0;
    bool dangling_x = false;
    if (cfg.resume && use_ckpt) {
        if (auto latest = restore_latest(ckpt_dir, digest)) {
            completed = latest->iteration;
            if (latest->which == FactorKind::theta) {
                theta = std::move(latest->factor);
                Checkpoint cx = read_checkpoint(checkpoint_path(ckpt_dir, completed, FactorKind::x));
                if (cx.digest != digest)
                    throw InputError("checkpoint config digest mismatch at iteration " + std::to_string(completed));
                x = std::move(cx.factor);
            } else {
                x = std::move(latest->factor);
                dangling_x = true;  // Theta@completed must be recomputed
            }
        }
    }
    result.start_iteration = dangling_x ? completed : completed + 1;

    // metrics CSV (driver.hpp:205-218): appended to on resume, %.17g values
    std::ofstream metrics;
    if (!cfg.metrics.empty()) {
        std::error_code ec;
        const bool append = cfg.resume && std::filesystem::exists(cfg.metrics, ec) &&
                            std::filesystem::file_size(cfg.metrics, ec) > 0;
        metrics.open(cfg.metrics, append ? std::ios::app : std::ios::trunc);
        if (!metrics) throw IoError("cannot open metrics file " + cfg.metrics);
        if (!append) {
            metrics << "iteration,wall_seconds,train_J,test_RMSE\n";
            if (cfg.iterations > 0) metrics << "# baseline_rmse=" << detail::format_real(result.baseline_rmse) << '\n';
            metrics.flush();
        }
    }

    // the device session: train and R^T uploaded once, factors resident in HBM
    const alsk_csr v = detail::view(train);
    alsk_session* raw = nullptr;
    detail::check(alsk_session_create(&v, rt.col_ptr.data(), rt.row_idx.data(), rt.values.data(),
                                      reinterpret_cast<const alsk_triplet*>(split.test.data()),
                                      static_cast<int64_t>(split.test.size()), cfg.f, cfg.lambda,
                                      cfg.accumulate_double ? ALSK_PREC_FP64_EXACT : ALSK_PREC_FP32, cfg.batch_rows,
                                      x.entries.data(), theta.entries.data(), &raw));
    std::unique_ptr<alsk_session, void (*)(alsk_session*)> sess(raw, alsk_session_destroy);
    float* dx = nullptr;
    float* dtheta = nullptr;
    void* stream = nullptr;
    detail::check(alsk_session_device(sess.get(), &dx, &dtheta, &stream));

    std::optional<CheckpointWriter> writer;
    if (use_ckpt) writer.emplace(ckpt_dir);
    auto snapshot = [&](int iteration, FactorKind which) {
        if (!writer) return;
        if (which == FactorKind::x)
            writer->submit_device(iteration, which, dx, train.rows, cfg.f, digest, stream);
        else
            writer->submit_device(iteration, which, dtheta, train.cols, cfg.f, digest, stream);
    };
    auto host_factors = [&] {
        detail::check(alsk_session_factors(sess.get(), x.entries.data(), theta.entries.data()));
    };

    const auto run_start = std::chrono::steady_clock::now();
    auto emit_row = [&](int iteration) {  // driver.hpp:230-246
        IterationRow row;
        row.iteration = iteration;
        row.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - run_start).count();
        detail::check(alsk_session_loss(sess.get(), &row.train_j));
        if (split.test.empty())
            row.test_rmse = std::numeric_limits<double>::quiet_NaN();
        else
            detail::check(alsk_session_rmse(sess.get(), &row.test_rmse));
        result.rows.push_back(row);
        if (metrics.is_open()) {
            char head[64];
            std::snprintf(head, sizeof head, "%d,%.3f,", row.iteration, row.wall_seconds);
            metrics << head << detail::format_real(row.train_j) << ',' << detail::format_real(row.test_rmse) << '\n';
            metrics.flush();
        }
    };
    auto callback = [&](int t) {
        if (!after_iteration) return true;
        host_factors();
        return after_iteration(t, x, theta);
    };

    const alsk_solver_config scfg{cfg.f, cfg.lambda, cfg.bin, cfg.batch_rows, cfg.accumulate_double ? 1 : 0,
                                  cfg.threads, cfg.seed};
    auto half_x = [&] {  // driver.hpp:163-167: update_x, or the SU-ALS side out of core
        if (side_x.split)
            detail::check(alsk_ooc_update(side_x.grid.c_str(), dtheta, train.cols, cfg.f, &scfg, dx, stream));
        else
            detail::check(alsk_session_half_x(sess.get()));
    };
    auto half_theta = [&] {
        if (side_t.split)
            detail::check(alsk_ooc_update(side_t.grid.c_str(), dx, train.rows, cfg.f, &scfg, dtheta, stream));
        else
            detail::check(alsk_session_half_theta(sess.get()));
    };

    bool stopped = false;
    if (dangling_x) {  // finish the interrupted iteration first (driver.hpp:249-254)
        half_theta();
        snapshot(completed, FactorKind::theta);
        emit_row(completed);
        if (!callback(completed)) stopped = true;
    }
    for (int t = completed + 1; !stopped && t <= cfg.iterations; ++t) {  // driver.hpp:255-262
        half_x();
        snapshot(t, FactorKind::x);
        half_theta();
        snapshot(t, FactorKind::theta);
        emit_row(t);
        if (!callback(t)) break;
    }
    if (writer) writer->flush();
    host_factors();
    result.x = std::move(x);
    result.theta = std::move(theta);
    return result;
}

/// train_run on cfg.data, a binary ratings cache (dataio.hpp:133-163).
inline TrainResult train_run(const RunConfig& cfg, const IterationCallback& after_iteration = {}) {
    if (cfg.data.empty()) throw InputError("no dataset configured (set data=PATH)");
    return train_run(load_binary_cache(cfg.data), cfg, after_iteration);
}

}  // namespace alskit
