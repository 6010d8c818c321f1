// train_run (include/alskit/driver.hpp) as a small program, for tests/test_train_run.py:
//   train_run_cli <cache> <f> <lambda> <iterations> <seed> <accumulate_double> <ckpt_dir|-> <metrics|-> <resume>
//                 <out_prefix> [stop_after] [capacity force_p force_q]
// Writes <out_prefix>_x.f32 / _theta.f32 (raw float32) and prints one summary line. With
// stop_after = k the callback stops the run after iteration k (a "killed" run).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "alskit/driver.hpp"

int main(int argc, char** argv) {
    if (argc < 11) {
        std::fprintf(stderr, "usage: see the header comment\n");
        return 2;
    }
    alskit::RunConfig cfg;
    cfg.data = argv[1];
    cfg.f = std::atoi(argv[2]);
    cfg.lambda = std::atof(argv[3]);
    cfg.iterations = std::atoi(argv[4]);
    cfg.seed = std::strtoull(argv[5], nullptr, 10);
    cfg.accumulate_double = std::atoi(argv[6]) != 0;
    cfg.checkpoint_dir = std::string(argv[7]) == "-" ? "" : argv[7];
    cfg.metrics = std::string(argv[8]) == "-" ? "" : argv[8];
    cfg.resume = std::atoi(argv[9]) != 0;
    const std::string out = argv[10];
    const int stop_after = argc > 11 ? std::atoi(argv[11]) : -1;
    if (argc > 14) {  // the planner fields (config.hpp:54-60)
        cfg.capacity = std::atoll(argv[12]);
        cfg.force_p = std::atoi(argv[13]);
        cfg.force_q = std::atoi(argv[14]);
    }
    try {
        alskit::IterationCallback cb;
        if (stop_after > 0) cb = [&](int t, const alskit::FactorMatrix&, const alskit::FactorMatrix&) { return t < stop_after; };
        const alskit::TrainResult r = alskit::train_run(cfg, cb);
        std::ofstream(out + "_x.f32", std::ios::binary)
            .write(reinterpret_cast<const char*>(r.x.entries.data()), static_cast<std::streamsize>(r.x.entries.size() * 4));
        std::ofstream(out + "_theta.f32", std::ios::binary)
            .write(reinterpret_cast<const char*>(r.theta.entries.data()),
                   static_cast<std::streamsize>(r.theta.entries.size() * 4));
        std::printf("ok start=%d rows=%zu digest=%llu baseline=%.17g p=%d q=%d\n", r.start_iteration, r.rows.size(),
                    static_cast<unsigned long long>(r.digest), r.baseline_rmse, r.p, r.q);
        return 0;
    } catch (const alskit::Error& e) {
        std::printf("error %s\n", e.what());
        return 3;
    }
}
