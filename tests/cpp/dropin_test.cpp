// C++ drop-in test: the reference's own unit-test expectations (proj/tests/test_*.cpp),
// restated as plain asserts against include/alskit/*.hpp, i.e. the reference API served by
// libalskit_cuda.so. Exit code 0 = all passed; prints one line per failure.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <unistd.h>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "alskit/alskit.hpp"

using namespace alskit;

static int g_fail = 0;
#define CHECK(cond)                                                         \
    do {                                                                    \
        if (!(cond)) {                                                      \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
            ++g_fail;                                                       \
        }                                                                   \
    } while (0)

template <class E, class F>
static bool throws_with(F&& f, const std::string& needle) {
    try {
        f();
    } catch (const E& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

// random_triplets (tests/test_util.hpp:36-48)
static std::vector<Triplet> random_triplets(std::mt19937_64& rng, offset_t m, offset_t n, offset_t nnz) {
    std::set<std::pair<offset_t, offset_t>> seen;
    std::vector<Triplet> out;
    while (static_cast<offset_t>(out.size()) < nnz) {
        const offset_t u = static_cast<offset_t>(rng() % static_cast<std::uint64_t>(m));
        const offset_t v = static_cast<offset_t>(rng() % static_cast<std::uint64_t>(n));
        if (!seen.insert({u, v}).second) continue;
        out.push_back({u, v, static_cast<real_t>(0.5 + 4.5 * (static_cast<double>(rng() >> 11) * 0x1.0p-53))});
    }
    return out;
}

static double normwise(const std::vector<real_t>& a, const std::vector<real_t>& b) {
    double d = 0, s = 1e-30;
    for (std::size_t i = 0; i < a.size(); ++i) {
        d = std::max(d, std::abs(double(a[i]) - double(b[i])));
        s = std::max(s, std::abs(double(b[i])));
    }
    return d / s;
}

int main() {
    // ---- sparse (test_sparse.cpp) ----
    {
        const CsrMatrix a = csr_from_triplets(2, 2, std::vector<Triplet>{{0, 0, 1.0f}, {1, 1, 2.0f}});
        CHECK((a.row_ptr == std::vector<offset_t>{0, 1, 2}) && (a.col_idx == std::vector<index_t>{0, 1}));
        const CsrMatrix b = csr_from_triplets(1, 3, std::vector<Triplet>{{0, 2, 5.0f}, {0, 0, 3.0f}});
        CHECK((b.col_idx == std::vector<index_t>{0, 2}) && (b.values == std::vector<real_t>{3.0f, 5.0f}));
        CHECK(throws_with<InputError>([] { csr_from_triplets(3, 3, std::vector<Triplet>{{0, 1, 1}, {1, 2, 2}, {1, 2, 3}}); }, "(1, 2)"));
        CHECK(throws_with<InputError>([] { csr_from_triplets(2, 2, std::vector<Triplet>{{0, 2, 1}}); }, "outside"));
        std::mt19937_64 rng(11);
        const CsrMatrix r = csr_from_triplets(10, 10, random_triplets(rng, 10, 10, 100));
        const CsrMatrix back = csc_to_csr(csr_to_csc(r));
        CHECK(back.row_ptr == r.row_ptr && back.col_idx == r.col_idx && back.values == r.values);
        const CsrMatrix id = csr_from_triplets(4, 4, std::vector<Triplet>{{0, 0, 1}, {1, 1, 2}, {2, 2, 3}, {3, 3, 4}});
        const GridPartition g = grid_partition(id, 2, 2);
        CHECK(g.block(0, 0).nnz() == 2 && g.block(1, 1).nnz() == 2 && g.block(1, 0).nnz() == 0);
        CHECK(g.block(1, 1).col_offset == 2 && (g.block(1, 1).col_idx == std::vector<index_t>{2, 3}));
    }
    // ---- binary cache (test_dataio.cpp:112-146) ----
    {
        std::mt19937_64 rng(17);
        const CsrMatrix a = csr_from_triplets(11, 23, random_triplets(rng, 11, 23, 140));
        const auto dir = std::filesystem::temp_directory_path() / ("alsk_dropin_" + std::to_string(::getpid()));
        std::filesystem::create_directories(dir);
        const auto path = dir / "r.cache";
        save_binary_cache(a, path);
        const CsrMatrix b = load_binary_cache(path);
        CHECK(a.rows == b.rows && a.cols == b.cols && a.row_ptr == b.row_ptr && a.col_idx == b.col_idx &&
              a.values == b.values);
        std::filesystem::resize_file(path, std::filesystem::file_size(path) - 5);
        CHECK(throws_with<IoError>([&] { load_binary_cache(path); }, "cache size does not match its header"));
        const auto junk = dir / "junk.cache";
        std::FILE* fj = std::fopen(junk.c_str(), "wb");
        std::fputs("this is not a cache file at all, but long enough to read", fj);
        std::fclose(fj);
        CHECK(throws_with<IoError>([&] { load_binary_cache(junk); }, "bad magic"));
        // grid persistence and streaming (dataio.hpp:352-540)
        {
            std::mt19937_64 rg(23);
            const CsrMatrix big = csr_from_triplets(40, 30, random_triplets(rg, 40, 30, 300));
            const GridPartition g = grid_partition(big, 3, 2);
            const auto gd = dir / "grid";
            persist_grid(g, gd);
            const GridMeta meta = load_grid_meta(gd);
            CHECK(meta.p == 3 && meta.q == 2 && meta.row_cuts == g.row_cuts && meta.col_cuts == g.col_cuts);
            const CsrMatrix b = load_block(gd, meta, 1, 1);
            CHECK(b.col_offset == g.block(1, 1).col_offset && b.col_idx == g.block(1, 1).col_idx &&
                  b.values == g.block(1, 1).values);
            CHECK(throws_with<InputError>([&] { load_block(gd, meta, 3, 0); }, "lies outside the 3x2 grid"));
            int n = 0;
            offset_t nnz = 0;
            DeviceBlockStream bs(gd, row_major_order(meta));
            while (auto blk = bs.next()) {
                CHECK(blk->ref == row_major_order(meta)[static_cast<std::size_t>(n)]);
                CHECK(blk->device.nnz == g.block(blk->ref.i, blk->ref.j).nnz());
                nnz += blk->device.nnz;
                ++n;
            }
            CHECK(n == 6 && nnz == big.nnz());
        }
        // checkpoints (dataio.hpp:546-786)
        const FactorMatrix fx = random_factor(9, 4, 5);
        const auto ck = dir / "ck";
        write_checkpoint({3, FactorKind::x, fx, 42}, ck);
        const Checkpoint back = read_checkpoint(checkpoint_path(ck, 3, FactorKind::x));
        CHECK(back.iteration == 3 && back.which == FactorKind::x && back.digest == 42 && back.factor.entries == fx.entries);
        {
            CheckpointWriter w(ck);
            w.submit({3, FactorKind::theta, fx, 42});
            w.flush();
        }
        const auto latest = restore_latest(ck, 42);
        CHECK(latest && latest->iteration == 3 && latest->which == FactorKind::theta);
        CHECK(throws_with<InputError>([&] { restore_latest(ck, 7); }, "digest mismatch"));
        CHECK(!restore_latest(dir / "none"));
        std::filesystem::remove_all(dir);
    }
    // ---- solver (test_solver.cpp) ----
    {
        const CsrMatrix r = csr_from_triplets(1, 1, std::vector<Triplet>{{0, 0, 2.0f}});
        FactorMatrix theta(1, 1);
        theta.entries[0] = 3.0f;
        const HermitianBatch base = get_hermitian_base(r, theta, 0.1);
        CHECK(base.a[0] == 9.1f && base.b[0] == 6.0f);
        SolverConfig cfg;
        cfg.lambda = 0.1;
        const HermitianBatch mo = get_hermitian_mo(r, theta, cfg);
        CHECK(mo.a[0] == base.a[0] && mo.b[0] == base.b[0]);
    }
    {
        HermitianBatch batch;
        batch.resize(2, 2);
        batch.a_at(0)[0] = 2.0f; batch.a_at(0)[3] = 2.0f; batch.b_at(0)[0] = 4.0f; batch.b_at(0)[1] = 2.0f;
        batch.a_at(1)[0] = 1.0f; batch.a_at(1)[3] = -1.0f; batch.b_at(1)[0] = 1.0f;
        CHECK(throws_with<NumericalError>([&] { batch_solve(batch); }, "batch index 1"));
        const FactorMatrix x = batch_solve(batch, BreakdownPolicy::zero_row);
        CHECK(x.row(0)[0] == 2.0f && x.row(0)[1] == 1.0f && x.row(1)[0] == 0.0f && x.row(1)[1] == 0.0f);
    }
    {
        std::mt19937_64 rng(113);
        const CsrMatrix r = csr_from_triplets(40, 30, random_triplets(rng, 40, 30, 250));
        const FactorMatrix theta = random_factor(30, 5, 114);
        for (bool dbl : {true, false}) {
            SolverConfig one, all;
            one.lambda = all.lambda = 0.05;
            one.accumulate_double = all.accumulate_double = dbl;
            one.batch_rows = 1;
            all.batch_rows = 40;
            CHECK(update_x(r, theta, one).entries == update_x(r, theta, all).entries);
            const CscMatrix csc = csr_to_csc(r);
            const FactorMatrix x = random_factor(40, 5, 115);
            CHECK(update_theta(csc, x, one).entries == update_x(transpose_of(csc), x, one).entries);
        }
        SolverConfig c;
        c.lambda = 0.1;
        const FactorMatrix x0 = random_factor(40, 5, 112);
        CHECK(loss(r, update_x(r, theta, c), theta, 0.1) <= loss(r, x0, theta, 0.1) * (1 + 1e-6));
        CHECK(throws_with<InputError>([&] { get_hermitian_mo(r, random_factor(7, 5, 1), c); }, "do not match"));
        CHECK(throws_with<InputError>([&] { rmse(std::vector<Triplet>{}, x0, theta); }, "empty test set"));
    }
    // ---- scale-up (test_parallel.cpp / acceptance_02) ----
    {
        std::mt19937_64 rng(133);
        const CsrMatrix r = csr_from_triplets(60, 48, random_triplets(rng, 60, 48, 900));
        const FactorMatrix theta = random_factor(48, 6, 134);
        SolverConfig cfg;
        cfg.lambda = 0.05;
        const FactorMatrix whole = update_x(r, theta, cfg);
        const GridPartition g = grid_partition(r, 2, 2);
        Topology topo;
        topo.workers = 2;
        const FactorMatrix su = su_als_update_x(g, split_factor(theta, g.col_cuts), topo, ReduceScheme::one_phase, cfg);
        CHECK(normwise(su.entries, whole.entries) <= 1e-6);
        Topology t4;
        t4.workers = 4;
        t4.groups = {{0, 1}, {2, 3}};
        CHECK(build_reduce_schedule(t4, ReduceScheme::one_phase).total_transfers() == 12);
        CHECK(build_reduce_schedule(t4, ReduceScheme::two_phase).cross_group_transfers() == 4);
        Topology big;
        big.workers = 1;
        big.capacity = 4'000'000'000;
        const PartitionPlan plan = plan_partition(480189, 17770, 99072112, 100, big, 0);
        CHECK(plan.p == 1 && plan.q == 2);
    }
    // ---- als_train on the device session (test_solver.cpp:358-367, acceptance_03) ----
    {
        std::mt19937_64 rng(122);
        const CsrMatrix r = csr_from_triplets(30, 25, random_triplets(rng, 30, 25, 200));
        SolverConfig cfg;
        cfg.f = 3;
        cfg.seed = 9001;
        cfg.lambda = 0.1;
        const AlsResult zero = als_train(r, csr_to_csc(r), {}, cfg, 0);
        CHECK(zero.history.empty() && zero.x.entries == random_factor(30, 3, 9001).entries);
        const AlsResult res = als_train(r, csr_to_csc(r), {}, cfg, 8);
        bool mono = true;
        for (std::size_t t = 1; t < res.history.size(); ++t)
            mono &= res.history[t].train_j <= res.history[t - 1].train_j * (1 + 1e-6);
        CHECK(res.history.size() == 8 && mono);
        // FP64 session reproduces the host-buffer half-steps bit for bit
        FactorMatrix x = random_factor(30, 3, 9001), th = random_factor(25, 3, detail::mix_seed(9001, 1));
        const CscMatrix csc = csr_to_csc(r);
        for (int t = 0; t < 8; ++t) {
            x = update_x(r, th, cfg);
            th = update_theta(csc, x, cfg);
        }
        CHECK(x.entries == res.x.entries && th.entries == res.theta.entries);
    }
    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
    return g_fail ? 1 : 0;
}
