// C ABI of libalskit_cuda.so (include/alskit_cuda.h). Host-buffer entry points stage
// inputs to the device, run the kernels and copy results back, mirroring the synchronous
// reference API; `_dev` entry points work on device pointers and a caller stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "alskit_cuda.h"
#include "measure.cuh"
#include "kernels.cuh"
#include "cache_io.cuh"
#include "checkpoint_io.cuh"
#include "grid_io.cuh"

namespace alsk {

std::atomic<uint64_t> g_launches{0};

namespace {

thread_local std::string t_error;
thread_local int64_t t_breakdown = -1;

// Kernel-only timing of the fused half-sweep kernel (CUDA events on the launching stream),
// enabled by alsk_profile_begin; read by bench.py for the roofline figure.
struct Profile {
    bool on = false;
    double ms = 0.0;
    uint64_t launches = 0;
    double phase_ms[PHASE_COUNT] = {};
    uint64_t phase_n[PHASE_COUNT] = {};
} g_prof;

}  // namespace

// For the host-only entry points (host_data.cpp), which return a status without a guard.
void set_last_error(const char* msg) { t_error = msg; }
void set_breakdown_index(int64_t k) { t_breakdown = k; }

bool prof_on() { return g_prof.on; }
void prof_add(int phase, float ms) {
    g_prof.phase_ms[phase] += ms;
    g_prof.phase_n[phase] += 1;
}
namespace {
struct Deferred {
    int phase;
    cudaEvent_t e0, e1;
};
std::mutex g_defer_mu;
std::vector<Deferred> g_deferred;
void resolve_deferred() {
    std::vector<Deferred> d;
    {
        std::lock_guard<std::mutex> lk(g_defer_mu);
        d.swap(g_deferred);
    }
    for (auto& e : d) {
        cudaEventSynchronize(e.e1);
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, e.e0, e.e1) == cudaSuccess) prof_add(e.phase, ms);
        cudaEventDestroy(e.e0);
        cudaEventDestroy(e.e1);
    }
}
}  // namespace
void prof_defer(int phase, cudaEvent_t e0, cudaEvent_t e1) {
    std::lock_guard<std::mutex> lk(g_defer_mu);
    g_deferred.push_back({phase, e0, e1});
}

namespace {

// check_update_shapes (solver.hpp:76-81)
void check_update_shapes(const alsk_csr* r, int64_t theta_rows, int f) {
    if (r->col_offset == 0 && theta_rows != r->cols)
        fail_input("factor rows " + std::to_string(theta_rows) + " do not match matrix columns " +
                   std::to_string(r->cols));
    if (f < 1) fail_input("rank must be >= 1");
}

// Device copy of a host CSR.
struct StagedCsr {
    DevBuf row_ptr, col_idx, values;
    DevCsr view;
    StagedCsr(const alsk_csr* h, cudaStream_t s) {
        row_ptr.alloc(sizeof(int64_t) * (h->rows + 1), s);
        col_idx.alloc(sizeof(int32_t) * std::max<int64_t>(h->nnz, 1), s);
        values.alloc(sizeof(float) * std::max<int64_t>(h->nnz, 1), s);
        h2d(row_ptr.as<int64_t>(), h->row_ptr, h->rows + 1, s);
        h2d(col_idx.as<int32_t>(), h->col_idx, h->nnz, s);
        h2d(values.as<float>(), h->values, h->nnz, s);
        view.rows = h->rows;
        view.cols = h->cols;
        view.col_offset = h->col_offset;
        view.nnz = h->nnz;
        view.row_ptr = row_ptr.as<int64_t>();
        view.col_idx = col_idx.as<int32_t>();
        view.values = values.as<float>();
    }
};

DevCsr dev_view(const alsk_csr* r) {
    DevCsr v;
    v.rows = r->rows;
    v.cols = r->cols;
    v.col_offset = r->col_offset;
    v.nnz = r->nnz;
    v.row_ptr = r->row_ptr;
    v.col_idx = r->col_idx;
    v.values = r->values;
    return v;
}

struct StatusBufs {
    DevBuf min_row, column, pivot;
    SolveStatus st{};
    StatusBufs(int64_t count, cudaStream_t s) {
        min_row.alloc(sizeof(unsigned long long), s);
        column.alloc(sizeof(int32_t) * std::max<int64_t>(count, 1), s);
        pivot.alloc(sizeof(double) * std::max<int64_t>(count, 1), s);
        ALSK_CUDA(cudaMemsetAsync(min_row.as<void>(), 0xff, sizeof(unsigned long long), s));
        st.min_row = min_row.as<unsigned long long>();
        st.column = column.as<int32_t>();
        st.pivot = pivot.as<double>();
    }
    // Raise the reference's NumericalError (solver.hpp:232-235) if any row broke down.
    // `index_base` is subtracted from the failing launch-relative row to get the batch
    // index; batch_rows > 0 folds a global row into update_x's batch numbering.
    void raise_if_broken(cudaStream_t s, int64_t batch_rows, int64_t first_row = 0) {
        unsigned long long bad = 0;
        d2h(&bad, st.min_row, 1, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
        if (bad == ~0ull) return;
        int32_t col = 0;
        double piv = 0.0;
        d2h(&col, st.column + bad, 1, s);
        d2h(&piv, st.pivot + bad, 1, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
        const int64_t g = first_row + static_cast<int64_t>(bad);  // matrix row of the failure
        const int64_t k = batch_rows > 0 ? g % batch_rows : g;
        t_breakdown = k;
        fail_numerical("cholesky breakdown at batch index " + std::to_string(k) + " (pivot " +
                       std::to_string(piv) + " at column " + std::to_string(col - 1) + ")");
    }
};

// Rows per materialised batch so A stays within ~2 GiB of device memory.
int64_t device_batch_rows(int f, int64_t rows) {
    const int64_t per = static_cast<int64_t>(f) * f * 4 + static_cast<int64_t>(f) * 4 + 16;
    return std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t(2) << 30) / per));
}

// FP32-mode engine: 0 = auto (tensor cores where the shape allows), 1 = CUDA-core FFMA
// kernel, 2 = tensor cores. ALSK_PREC_TF32X2 always asks for the tensor cores.
std::atomic<int> g_fp32_engine{0};
bool use_tensor_cores(alsk_precision prec, int f) {
    if (prec == ALSK_PREC_FP64_EXACT || !tc_supported(f)) return false;
    if (prec == ALSK_PREC_TF32X2) return true;
    return g_fp32_engine.load() != 1;  // auto -> tensor cores
}

// Core of update_x on device data: rows [rb,re) -> x_out (rows-local).
void update_rows_device(const DevCsr& r, const float* theta, int64_t theta_rows, int f,
                        double lambda, alsk_precision prec, int64_t batch_rows, int64_t rb, int64_t re,
                        float* x_out, cudaStream_t s) {
    if (re <= rb) return;
    const bool exact = prec == ALSK_PREC_FP64_EXACT;
    check_columns(r, rb, re, r.col_offset, r.col_offset + theta_rows, s);
    StatusBufs sb(re - rb, s);
    const int64_t br = batch_rows < 1 ? 1 : batch_rows;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (g_prof.on) {
        ALSK_CUDA(cudaEventCreate(&e0));
        ALSK_CUDA(cudaEventCreate(&e1));
        ALSK_CUDA(cudaEventRecord(e0, s));
    }
    const bool fused = !exact && (use_tensor_cores(prec, f)
                                      ? update_tc(r, theta, theta_rows, f, static_cast<float>(lambda), rb, re, x_out,
                                                  sb.st, s)
                                      : update_fused_fp32(r, theta, theta_rows, f, static_cast<float>(lambda), rb,
                                                          re, x_out, sb.st, s));
    if (fused) {
        if (e0) {
            ALSK_CUDA(cudaEventRecord(e1, s));
            prof_defer(PHASE_FUSED, e0, e1);
        }
        sb.raise_if_broken(s, br, rb);
        return;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    const int64_t chunk = device_batch_rows(f, re - rb);
    DevBuf A(sizeof(float) * chunk * f * f, s), B(sizeof(float) * chunk * f, s);
    for (int64_t b0 = rb; b0 < re; b0 += chunk) {
        const int64_t b1 = std::min(re, b0 + chunk);
        {
            PhaseTimer pt(PHASE_HERMITIAN, s);
            hermitian_materialize(r, theta, f, lambda, exact, b0, b1, A.as<float>(), B.as<float>(), s);
        }
        SolveStatus st = sb.st;
        st.column += (b0 - rb);
        st.pivot += (b0 - rb);
        // solve_exact reports launch-relative rows; shift by the batch offset
        {
            PhaseTimer pt(PHASE_SOLVE, s);
            solve_exact(A.as<float>(), B.as<float>(), b1 - b0, f, false, x_out + (b0 - rb) * f, st, s);
        }
        unsigned long long bad = 0;
        d2h(&bad, sb.st.min_row, 1, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
        if (bad != ~0ull) {
            const int64_t global = (b0 - rb) + static_cast<int64_t>(bad);
            int32_t col = 0;
            double piv = 0.0;
            d2h(&col, st.column + bad, 1, s);
            d2h(&piv, st.pivot + bad, 1, s);
            ALSK_CUDA(cudaStreamSynchronize(s));
            const int64_t k = (rb + global) % br;
            t_breakdown = k;
            fail_numerical("cholesky breakdown at batch index " + std::to_string(k) + " (pivot " +
                           std::to_string(piv) + " at column " + std::to_string(col - 1) + ")");
        }
    }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

// The synchronous half-sweep (column check, breakdown raised with the reference's text) for
// the other translation units (multigpu.cu's FP64-exact path).
void update_rows_sync(const DevCsr& r, const float* theta, int64_t theta_rows, int f, double lambda,
                      alsk_precision prec, int64_t batch_rows, int64_t rb, int64_t re, float* x_out, cudaStream_t s) {
    update_rows_device(r, theta, theta_rows, f, lambda, prec, batch_rows, rb, re, x_out, s);
}
bool fp32_uses_tensor_cores(alsk_precision prec, int f) { return use_tensor_cores(prec, f); }
}  // namespace alsk

using namespace alsk;

extern "C" {

const char* alsk_last_error(void) { return t_error.c_str(); }
int64_t alsk_last_breakdown_index(void) { return t_breakdown; }
int alsk_device_available(void) {
    int n = 0;
    return (cudaGetDeviceCount(&n) == cudaSuccess && n > 0) ? 1 : 0;
}
uint64_t alsk_kernel_launch_count(void) { return g_launches.load(); }
void alsk_set_fp32_engine(int engine) { g_fp32_engine.store(engine); }
int alsk_fp32_engine(void) { return g_fp32_engine.load(); }
void alsk_profile_begin(void) {
    resolve_deferred();  // events recorded before this window are not counted in it
    g_prof = Profile{true, 0.0, 0};
}
void alsk_profile_phase(int phase, double* ms, uint64_t* launches) {
    resolve_deferred();
    const bool ok = phase >= 0 && phase < PHASE_COUNT;
    *ms = ok ? g_prof.phase_ms[phase] : 0.0;
    *launches = ok ? g_prof.phase_n[phase] : 0;
}
void alsk_profile_phases(double* herm_ms, uint64_t* herm_launches, double* solve_ms, uint64_t* solve_launches) {
    resolve_deferred();
    *herm_ms = g_prof.phase_ms[PHASE_HERMITIAN];
    *herm_launches = g_prof.phase_n[PHASE_HERMITIAN];
    *solve_ms = g_prof.phase_ms[PHASE_SOLVE];
    *solve_launches = g_prof.phase_n[PHASE_SOLVE];
}
void alsk_profile_end(double* total_ms, uint64_t* launches) {
    resolve_deferred();
    *total_ms = g_prof.phase_ms[PHASE_FUSED];
    *launches = g_prof.phase_n[PHASE_FUSED];
    g_prof.on = false;
}
const char* alsk_build_info(void) {
    return "libalskit_cuda (sm_100a; fused fp32 hermitian+cholesky, reference-order fp64 path, "
           "radix-sort transposes)";
}

alsk_status alsk_get_hermitian_mo_into(const alsk_csr* r, const float* theta, int64_t theta_rows,
                                       int f, const alsk_solver_config* cfg, int64_t row_begin,
                                       int64_t row_end, float* a_out, float* b_out) {
    return guard([&] {
        check_update_shapes(r, theta_rows, f);
        if (row_begin < 0 || row_end > r->rows || row_begin > row_end)
            fail_input("row range [" + std::to_string(row_begin) + ", " + std::to_string(row_end) +
                       ") outside matrix");
        const int64_t count = row_end - row_begin;
        if (count == 0) return;
        require_device();
        cudaStream_t s = nullptr;
        StagedCsr R(r, s);
        DevBuf T(sizeof(float) * std::max<int64_t>(theta_rows * f, 1), s);
        h2d(T.as<float>(), theta, theta_rows * f, s);
        check_columns(R.view, row_begin, row_end, r->col_offset, r->col_offset + theta_rows, s);
        DevBuf A(sizeof(float) * count * f * f, s), B(sizeof(float) * count * f, s);
        hermitian_materialize(R.view, T.as<float>(), f, cfg->lambda, cfg->accumulate_double != 0,
                              row_begin, row_end, A.as<float>(), B.as<float>(), s);
        d2h(a_out, A.as<float>(), count * f * f, s);
        d2h(b_out, B.as<float>(), count * f, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

alsk_status alsk_get_hermitian_base(const alsk_csr* r, const float* theta, int64_t theta_rows,
                                    int f, double lambda, int accumulate_double, float* a_out,
                                    float* b_out) {
    alsk_solver_config cfg{};
    cfg.lambda = lambda;
    cfg.accumulate_double = accumulate_double;
    return alsk_get_hermitian_mo_into(r, theta, theta_rows, f, &cfg, 0, r->rows, a_out, b_out);
}

alsk_status alsk_local_hermitian(const alsk_csr* block, const float* theta_part,
                                 int64_t theta_rows, int f, const alsk_solver_config* cfg,
                                 float* a_out, float* b_out) {
    return guard([&] {
        const int64_t count = block->rows;
        if (count == 0) return;
        require_device();
        cudaStream_t s = nullptr;
        StagedCsr R(block, s);
        DevBuf T(sizeof(float) * std::max<int64_t>(theta_rows * f, 1), s);
        h2d(T.as<float>(), theta_part, theta_rows * f, s);
        check_columns(R.view, 0, count, block->col_offset, block->col_offset + theta_rows, s);
        DevBuf A(sizeof(float) * count * f * f, s), B(sizeof(float) * count * f, s);
        hermitian_materialize(R.view, T.as<float>(), f, cfg->lambda, cfg->accumulate_double != 0, 0,
                              count, A.as<float>(), B.as<float>(), s);
        d2h(a_out, A.as<float>(), count * f * f, s);
        d2h(b_out, B.as<float>(), count * f, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

alsk_status alsk_batch_solve(const float* a, const float* b, int64_t count, int f,
                             alsk_breakdown policy, float* x_out) {
    return guard([&] {
        if (count == 0) return;
        if (f < 1) fail_input("rank must be >= 1");
        require_device();
        cudaStream_t s = nullptr;
        DevBuf A(sizeof(float) * count * f * f, s), B(sizeof(float) * count * f, s),
            X(sizeof(float) * count * f, s);
        h2d(A.as<float>(), a, count * f * f, s);
        h2d(B.as<float>(), b, count * f, s);
        StatusBufs sb(count, s);
        solve_exact(A.as<float>(), B.as<float>(), count, f, policy == ALSK_BREAKDOWN_ZERO_ROW,
                    X.as<float>(), sb.st, s);
        if (policy == ALSK_BREAKDOWN_FAIL) sb.raise_if_broken(s, 0);
        d2h(x_out, X.as<float>(), count * f, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

// update_x on host buffers (solver.hpp:330-345), pipelined: the rows are split into
// ranges (kPipeCuts); each range's col_idx/values go host->device on a copy stream while the
// previous range computes, and each solved range of X goes back while the next computes.
// Only row_ptr and the gathered factor must be resident before the first range starts.
alsk_status alsk_update_x(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                          const alsk_solver_config* cfg, float* x_out) {
    return guard([&] {
        check_update_shapes(r, theta_rows, f);
        if (r->rows == 0) return;
        require_device();
        static cudaStream_t s = nullptr, c = nullptr;  // compute / copy streams (process lifetime)
        if (!s) {
            ALSK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            ALSK_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
        }
        const int64_t m = r->rows, nnz = r->nnz;
        DevBuf RP(sizeof(int64_t) * (m + 1), s), CI(sizeof(int32_t) * std::max<int64_t>(nnz, 1), s),
            V(sizeof(float) * std::max<int64_t>(nnz, 1), s), T(sizeof(float) * std::max<int64_t>(theta_rows * f, 1), s),
            X(sizeof(float) * m * f, s);
        struct Events {
            std::vector<cudaEvent_t> ev;
            cudaEvent_t make() {
                cudaEvent_t e;
                ALSK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                ev.push_back(e);
                return e;
            }
            ~Events() {
                for (auto e : ev) cudaEventDestroy(e);
            }
        } evs;
        struct Drain {  // destroyed before the buffers: no copy may outlive them (errors included)
            cudaStream_t c, s;
            ~Drain() {
                cudaStreamSynchronize(c);
                cudaStreamSynchronize(s);
            }
        } drain{c, s};
#ifdef ALSK_MEASURE
        // ALSK_E2E_PROF=1: timeline of this call's copy and compute streams (stderr)
        static const bool e2e_prof = measure_env("ALSK_E2E_PROF") != nullptr;
        std::vector<std::pair<const char*, cudaEvent_t>> tl;
        auto mark = [&](const char* what, cudaStream_t on) {
            if (!e2e_prof) return;
            cudaEvent_t e;
            ALSK_CUDA(cudaEventCreate(&e));
            ALSK_CUDA(cudaEventRecord(e, on));
            tl.emplace_back(what, e);
        };
        mark("start", s);
        auto dump = [&] {
            if (!e2e_prof || tl.empty()) return;
            std::fprintf(stderr, "[e2e-prof m=%lld nnz=%lld]", static_cast<long long>(m), static_cast<long long>(nnz));
            for (auto& [w, e] : tl) {
                float ms = 0.f;
                ALSK_CUDA(cudaEventElapsedTime(&ms, tl[0].second, e));
                std::fprintf(stderr, " %s@%.2f", w, ms);
            }
            for (auto& [w, e] : tl) ALSK_CUDA(cudaEventDestroy(e));
            tl.clear();
            std::fprintf(stderr, "\n");
        };
#else
        auto mark = [](const char*, cudaStream_t) {};
        auto dump = [] {};
#endif
        cudaEvent_t allocated = evs.make();
        ALSK_CUDA(cudaEventRecord(allocated, s));
        ALSK_CUDA(cudaStreamWaitEvent(c, allocated, 0));
        h2d(RP.as<int64_t>(), r->row_ptr, m + 1, c);
        h2d(T.as<float>(), theta, theta_rows * f, c);
        cudaEvent_t base = evs.make();
        ALSK_CUDA(cudaEventRecord(base, c));
        // Ranges cut at these fractions of the nonzeros (sizes 1,2,3,5,8,12,12,10,6,3,2 / 64):
        // H2D (~56 GB/s) outruns the compute (~1.7x), so once a range computes the next one is
        // staged as long as sizes grow by less than that; only the first range's upload and
        // the last range's download are exposed, and both are small.
        static constexpr double kPipeCuts[] = {0.0, 1.0 / 64, 3.0 / 64, 6.0 / 64, 11.0 / 64, 19.0 / 64, 31.0 / 64,
                                               43.0 / 64, 53.0 / 64, 59.0 / 64, 62.0 / 64, 1.0};
        std::vector<double> fr(std::begin(kPipeCuts), std::end(kPipeCuts));
        if (const char* e = measure_env("ALSK_PIPE_CUTS")) {  // A/B: "n1,n2,...,64" in 64ths
            fr.assign(1, 0.0);
            for (const char* q = e; *q;) {
                char* end = nullptr;
                const double v = std::strtod(q, &end);
                if (end == q) break;
                fr.push_back(v / 64.0);
                q = *end ? end + 1 : end;
            }
        }
        const int kPipeRanges = static_cast<int>(fr.size()) - 1;
        std::vector<int64_t> cut{0};
        for (int k = 1; k < kPipeRanges; ++k) {
            const int64_t want = static_cast<int64_t>(fr[k] * static_cast<double>(nnz));
            const int64_t row = std::lower_bound(r->row_ptr, r->row_ptr + m + 1, want) - r->row_ptr;
            if (row > cut.back() && row < m) cut.push_back(row);
        }
        cut.push_back(m);
        const int64_t nb = static_cast<int64_t>(cut.size()) - 1;
        std::vector<cudaEvent_t> staged(nb);
        for (int64_t k = 0; k < nb; ++k) {
            const int64_t b0 = cut[k], b1 = cut[k + 1];
            const int64_t k0 = r->row_ptr[b0], k1 = r->row_ptr[b1];
            h2d(CI.as<int32_t>() + k0, r->col_idx + k0, k1 - k0, c);
            h2d(V.as<float>() + k0, r->values + k0, k1 - k0, c);
            staged[k] = evs.make();
            ALSK_CUDA(cudaEventRecord(staged[k], c));
            mark("c:staged", c);
        }
        DevCsr view;
        view.rows = m;
        view.cols = r->cols;
        view.col_offset = r->col_offset;
        view.nnz = nnz;
        view.row_ptr = RP.as<int64_t>();
        view.col_idx = CI.as<int32_t>();
        view.values = V.as<float>();
        ALSK_CUDA(cudaStreamWaitEvent(s, base, 0));
        const alsk_precision prec = cfg->accumulate_double != 0 ? ALSK_PREC_FP64_EXACT : ALSK_PREC_FP32;
        if (prec == ALSK_PREC_FP32 && use_tensor_cores(prec, f)) {
            // Tensor-core path without host synchronisation between ranges: a packed-row
            // scratch owned by this call (stream-ordered pool), the column check running
            // asynchronously ahead of each range (the Hermitian clamps its gather index, so a
            // bad column never reads outside Theta), breakdown status per range; errors are
            // resolved once at the end in the reference's order (batch by batch: a batch's
            // column check precedes its solve, solver.hpp:120-123 and 230-235).
            const int64_t br = cfg->batch_rows < 1 ? 1 : cfg->batch_rows;
            int64_t maxr = 1;
            for (int64_t k = 0; k < nb; ++k) maxr = std::max(maxr, cut[k + 1] - cut[k]);
            const size_t pkn = static_cast<size_t>(packed_stride(f)) * 4;
            const int64_t cap = std::max<int64_t>(1, static_cast<int64_t>((size_t(4096) << 20) / pkn));
            DevBuf SC(pkn * static_cast<size_t>(std::min(maxr, cap)), s);
            const Scratch ext{SC.as<float>(), SC.bytes()};
            DevBuf flag(sizeof(unsigned long long), s), mins(sizeof(unsigned long long) * nb, s);
            DevBuf col(sizeof(int32_t) * m, s), piv(sizeof(double) * m, s);
            ALSK_CUDA(cudaMemsetAsync(flag.as<void>(), 0xff, sizeof(unsigned long long), s));
            ALSK_CUDA(cudaMemsetAsync(mins.as<void>(), 0xff, sizeof(unsigned long long) * nb, s));
            const int64_t col_lo = r->col_offset, col_hi = r->col_offset + theta_rows;
            for (int64_t k = 0; k < nb; ++k) {
                const int64_t b0 = cut[k], b1 = cut[k + 1];
                ALSK_CUDA(cudaStreamWaitEvent(s, staged[k], 0));
                mark("s:range-start", s);
                check_columns_async(view, r->row_ptr[b0], r->row_ptr[b1], col_lo, col_hi,
                                    flag.as<unsigned long long>(), s);
                SolveStatus st{mins.as<unsigned long long>() + k, col.as<int32_t>() + b0, piv.as<double>() + b0};
                update_tc(view, T.as<float>(), theta_rows, f, static_cast<float>(cfg->lambda), b0, b1,
                          X.as<float>() + b0 * f, st, s, &ext);
                mark("s:range-end", s);
                cudaEvent_t solved = evs.make();
                ALSK_CUDA(cudaEventRecord(solved, s));
                ALSK_CUDA(cudaStreamWaitEvent(c, solved, 0));
                d2h(x_out + b0 * f, X.as<float>() + b0 * f, (b1 - b0) * f, c);
            }
            unsigned long long bad = 0;
            std::vector<unsigned long long> mh(nb);
            d2h(&bad, flag.as<unsigned long long>(), 1, s);
            d2h(mh.data(), mins.as<unsigned long long>(), nb, s);
            mark("c:end", c);
            ALSK_CUDA(cudaStreamSynchronize(c));
            ALSK_CUDA(cudaStreamSynchronize(s));
            dump();
            int64_t rc = -1, rbk = -1;
            if (bad != ~0ull)  // the row holding the first bad nonzero
                rc = std::upper_bound(r->row_ptr, r->row_ptr + m + 1, static_cast<int64_t>(bad)) - r->row_ptr - 1;
            for (int64_t k = 0; k < nb && rbk < 0; ++k)
                if (mh[k] != ~0ull) rbk = cut[k] + static_cast<int64_t>(mh[k]);
            if (rc >= 0 && (rbk < 0 || rc / br <= rbk / br)) fail_bad_column(view, bad, col_lo, col_hi, s);
            if (rbk >= 0) {
                int32_t cc = 0;
                double pv = 0.0;
                d2h(&cc, col.as<int32_t>() + rbk, 1, s);
                d2h(&pv, piv.as<double>() + rbk, 1, s);
                ALSK_CUDA(cudaStreamSynchronize(s));
                t_breakdown = rbk % br;
                fail_numerical("cholesky breakdown at batch index " + std::to_string(rbk % br) + " (pivot " +
                               std::to_string(pv) + " at column " + std::to_string(cc - 1) + ")");
            }
            return;
        }
        for (int64_t k = 0; k < nb; ++k) {
            const int64_t b0 = cut[k], b1 = cut[k + 1];
            ALSK_CUDA(cudaStreamWaitEvent(s, staged[k], 0));
            mark("s:range-start", s);
            update_rows_device(view, T.as<float>(), theta_rows, f, cfg->lambda, prec, cfg->batch_rows, b0, b1,
                               X.as<float>() + b0 * f, s);
            mark("s:range-end", s);
            cudaEvent_t solved = evs.make();
            ALSK_CUDA(cudaEventRecord(solved, s));
            ALSK_CUDA(cudaStreamWaitEvent(c, solved, 0));
            d2h(x_out + b0 * f, X.as<float>() + b0 * f, (b1 - b0) * f, c);
        }
        mark("c:end", c);
        ALSK_CUDA(cudaStreamSynchronize(c));
        ALSK_CUDA(cudaStreamSynchronize(s));  // the buffers are freed (stream-ordered) on s
        dump();
    });
}

alsk_status alsk_update_theta(int64_t rows, int64_t cols, int64_t nnz, const int64_t* col_ptr,
                              const int32_t* row_idx, const float* values, const float* x,
                              int64_t x_rows, int f, const alsk_solver_config* cfg,
                              float* theta_out) {
    alsk_csr rt{};
    rt.rows = cols;
    rt.cols = rows;
    rt.col_offset = 0;
    rt.nnz = nnz;
    rt.row_ptr = col_ptr;
    rt.col_idx = row_idx;
    rt.values = values;
    return alsk_update_x(&rt, x, x_rows, f, cfg, theta_out);
}

alsk_status alsk_loss(const alsk_csr* r, const float* x, int64_t x_rows, const float* theta,
                      int64_t theta_rows, int f, double lambda, double* out) {
    return guard([&] {
        if (x_rows != r->rows) fail_input("x rows do not match matrix rows");
        check_update_shapes(r, theta_rows, f);
        require_device();
        cudaStream_t s = nullptr;
        StagedCsr R(r, s);
        DevBuf X(sizeof(float) * std::max<int64_t>(x_rows * f, 1), s);
        DevBuf T(sizeof(float) * std::max<int64_t>(theta_rows * f, 1), s);
        h2d(X.as<float>(), x, x_rows * f, s);
        h2d(T.as<float>(), theta, theta_rows * f, s);
        DevBuf cn(sizeof(int64_t) * std::max<int64_t>(r->cols, 1), s);
        column_counts(R.view, cn.as<int64_t>(), s);
        *out = loss_device(R.view, cn.as<int64_t>(), X.as<float>(), T.as<float>(), f, lambda, s);
    });
}

alsk_status alsk_rmse(const alsk_triplet* test, int64_t count, const float* x, int64_t x_rows,
                      const float* theta, int64_t theta_rows, int f, double* out) {
    return guard([&] {
        if (count <= 0) fail_input("empty test set");
        require_device();
        cudaStream_t s = nullptr;
        std::vector<int64_t> hr(count), hc(count);
        std::vector<float> hv(count);
        for (int64_t i = 0; i < count; ++i) {
            hr[i] = test[i].row;
            hc[i] = test[i].col;
            hv[i] = test[i].value;
        }
        DevBuf R(sizeof(int64_t) * count, s), C(sizeof(int64_t) * count, s), V(sizeof(float) * count, s);
        h2d(R.as<int64_t>(), hr.data(), count, s);
        h2d(C.as<int64_t>(), hc.data(), count, s);
        h2d(V.as<float>(), hv.data(), count, s);
        DevBuf X(sizeof(float) * std::max<int64_t>(x_rows * f, 1), s);
        DevBuf T(sizeof(float) * std::max<int64_t>(theta_rows * f, 1), s);
        h2d(X.as<float>(), x, x_rows * f, s);
        h2d(T.as<float>(), theta, theta_rows * f, s);
        *out = rmse_device(R.as<int64_t>(), C.as<int64_t>(), V.as<float>(), count, X.as<float>(),
                           x_rows, T.as<float>(), theta_rows, f, s);
    });
}

alsk_status alsk_csr_to_csc(const alsk_csr* a, int64_t* col_ptr_out, int32_t* row_idx_out,
                            float* values_out) {
    return guard([&] {
        require_device();
        cudaStream_t s = nullptr;
        StagedCsr R(a, s);
        DevBuf cp(sizeof(int64_t) * (a->cols + 1), s);
        DevBuf ri(sizeof(int32_t) * std::max<int64_t>(a->nnz, 1), s);
        DevBuf vv(sizeof(float) * std::max<int64_t>(a->nnz, 1), s);
        csr_to_csc_device(R.view, cp.as<int64_t>(), ri.as<int32_t>(), vv.as<float>(), s);
        d2h(col_ptr_out, cp.as<int64_t>(), a->cols + 1, s);
        d2h(row_idx_out, ri.as<int32_t>(), a->nnz, s);
        d2h(values_out, vv.as<float>(), a->nnz, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

alsk_status alsk_csc_to_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* col_ptr,
                            const int32_t* row_idx, const float* values, int64_t* row_ptr_out,
                            int32_t* col_idx_out, float* values_out) {
    // The CSC of R is the CSR of R^T; its stable transpose is the CSR of R.
    alsk_csr t{};
    t.rows = cols;
    t.cols = rows;
    t.nnz = nnz;
    t.row_ptr = col_ptr;
    t.col_idx = row_idx;
    t.values = values;
    return alsk_csr_to_csc(&t, row_ptr_out, col_idx_out, values_out);
}

alsk_status alsk_csr_from_triplets(int64_t m, int64_t n, const alsk_triplet* t, int64_t count,
                                   int64_t* row_ptr_out, int32_t* col_idx_out, float* values_out) {
    return guard([&] {
        if (m < 0 || n < 0) fail_input("matrix dimensions must be non-negative");
        require_device();
        cudaStream_t s = nullptr;
        std::vector<int64_t> hr(std::max<int64_t>(count, 1)), hc(std::max<int64_t>(count, 1));
        std::vector<float> hv(std::max<int64_t>(count, 1));
        for (int64_t i = 0; i < count; ++i) {
            hr[i] = t[i].row;
            hc[i] = t[i].col;
            hv[i] = t[i].value;
        }
        const int64_t cn = std::max<int64_t>(count, 1);
        DevBuf R(sizeof(int64_t) * cn, s), C(sizeof(int64_t) * cn, s), V(sizeof(float) * cn, s);
        h2d(R.as<int64_t>(), hr.data(), count, s);
        h2d(C.as<int64_t>(), hc.data(), count, s);
        h2d(V.as<float>(), hv.data(), count, s);
        DevBuf rp(sizeof(int64_t) * (m + 1), s), ci(sizeof(int32_t) * cn, s), vv(sizeof(float) * cn, s);
        csr_from_triplets_device(m, n, R.as<int64_t>(), C.as<int64_t>(), V.as<float>(), count,
                                 rp.as<int64_t>(), ci.as<int32_t>(), vv.as<float>(), s);
        d2h(row_ptr_out, rp.as<int64_t>(), m + 1, s);
        d2h(col_idx_out, ci.as<int32_t>(), count, s);
        d2h(values_out, vv.as<float>(), count, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

alsk_status alsk_grid_partition_counts(const alsk_csr* r, int p, int q, int64_t* row_cuts_out,
                                       int64_t* col_cuts_out, int64_t* block_nnz_out) {
    return guard([&] {
        require_device();
        cudaStream_t s = nullptr;
        StagedCsr R(r, s);
        GridDevice g = grid_partition_device(R.view, p, q, s);
        std::copy(g.row_cuts.begin(), g.row_cuts.end(), row_cuts_out);
        std::copy(g.col_cuts.begin(), g.col_cuts.end(), col_cuts_out);
        std::copy(g.block_nnz.begin(), g.block_nnz.end(), block_nnz_out);
    });
}

alsk_status alsk_grid_partition_fill(const alsk_csr* r, int p, int q, int64_t* const* block_row_ptr,
                                     int32_t* const* block_col_idx, float* const* block_values) {
    return guard([&] {
        require_device();
        cudaStream_t s = nullptr;
        StagedCsr R(r, s);
        GridDevice g = grid_partition_device(R.view, p, q, s);
        for (int j = 0; j < q; ++j)
            for (int i = 0; i < p; ++i) {
                const size_t b = static_cast<size_t>(j) * p + i;
                const int64_t lr = g.row_cuts[j + 1] - g.row_cuts[j], nz = g.block_nnz[b];
                DevBuf ci(sizeof(int32_t) * std::max<int64_t>(nz, 1), s), vv(sizeof(float) * std::max<int64_t>(nz, 1), s);
                grid_fill_block(R.view, g, i, j, ci.as<int32_t>(), vv.as<float>(), s);
                d2h(block_row_ptr[b], g.block_row_ptr[b].as<int64_t>(), lr + 1, s);
                d2h(block_col_idx[b], ci.as<int32_t>(), nz, s);
                d2h(block_values[b], vv.as<float>(), nz, s);
                ALSK_CUDA(cudaStreamSynchronize(s));
            }
    });
}

alsk_status alsk_parallel_reduce(const float* const* parts_a, const float* const* parts_b, int p,
                                 int64_t count, int f, const int32_t* group_of, int two_phase,
                                 float* const* out_a, float* const* out_b) {
    return guard([&] {
        const ReduceSchedule sc = build_reduce_schedule(p, group_of, two_phase != 0);
        require_device();
        cudaStream_t s = nullptr;
        const int64_t ff = static_cast<int64_t>(f) * f;
        std::vector<DevBuf> da, db;
        std::vector<const float*> pa, pb;
        for (int w = 0; w < p; ++w) {
            da.emplace_back(sizeof(float) * std::max<int64_t>(count * ff, 1), s);
            db.emplace_back(sizeof(float) * std::max<int64_t>(count * f, 1), s);
            h2d(da.back().as<float>(), parts_a[w], count * ff, s);
            h2d(db.back().as<float>(), parts_b[w], count * f, s);
            pa.push_back(da.back().as<float>());
            pb.push_back(db.back().as<float>());
        }
        const auto cuts = slice_cuts(count, p);
        std::vector<DevBuf> oa, ob;
        std::vector<float*> poa, pob;
        for (int w = 0; w < p; ++w) {
            const int64_t n = cuts[w + 1] - cuts[w];
            oa.emplace_back(sizeof(float) * std::max<int64_t>(n * ff, 1), s);
            ob.emplace_back(sizeof(float) * std::max<int64_t>(n * f, 1), s);
            poa.push_back(oa.back().as<float>());
            pob.push_back(ob.back().as<float>());
        }
        reduce_slices<float>(pa, pb, count, f, sc, poa, pob, s);
        for (int w = 0; w < p; ++w) {
            const int64_t n = cuts[w + 1] - cuts[w];
            d2h(out_a[w], poa[w], n * ff, s);
            d2h(out_b[w], pob[w], n * f, s);
        }
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

alsk_status alsk_su_als_update_x(const alsk_csr* blocks, int p, int q, const int64_t* row_cuts,
                                 const int64_t* col_cuts, const float* const* theta_parts, int f,
                                 const alsk_solver_config* cfg, const int32_t* group_of,
                                 int two_phase, float* x_out) {
    return guard([&] {
        if (f < 1) fail_input("rank must be >= 1");
        const ReduceSchedule sc = build_reduce_schedule(p, group_of, two_phase != 0);
        require_device();
        cudaStream_t s = nullptr;
        const bool dbl = cfg->accumulate_double != 0;
        const int64_t ff = static_cast<int64_t>(f) * f;
        std::vector<DevBuf> theta(p);
        for (int i = 0; i < p; ++i) {
            const int64_t rows = col_cuts[i + 1] - col_cuts[i];
            theta[i].alloc(sizeof(float) * std::max<int64_t>(rows * f, 1), s);
            h2d(theta[i].as<float>(), theta_parts[i], rows * f, s);
        }
        const int64_t total_rows = row_cuts[q];
        DevBuf X(sizeof(float) * std::max<int64_t>(total_rows * f, 1), s);
        for (int j = 0; j < q; ++j) {  // sequential model-parallel loop (parallel.hpp:532)
            const int64_t lr = row_cuts[j + 1] - row_cuts[j];
            if (lr == 0) continue;
            const size_t esz = dbl ? sizeof(double) : sizeof(float);
            std::vector<DevBuf> pa(p), pb(p);
            for (int i = 0; i < p; ++i) {
                const alsk_csr* b = &blocks[static_cast<size_t>(j) * p + i];
                StagedCsr Bk(b, s);
                const int64_t want = col_cuts[i + 1] - col_cuts[i];
                check_columns(Bk.view, 0, lr, b->col_offset, b->col_offset + want, s);
                pa[i].alloc(esz * lr * ff, s);
                pb[i].alloc(esz * lr * f, s);
                if (dbl)
                    hermitian_materialize_d(Bk.view, theta[i].as<float>(), f, cfg->lambda, true, 0, lr,
                                            pa[i].as<double>(), pb[i].as<double>(), false, s);
                else
                    hermitian_materialize(Bk.view, theta[i].as<float>(), f, cfg->lambda, false, 0, lr,
                                          pa[i].as<float>(), pb[i].as<float>(), s);
                ALSK_CUDA(cudaStreamSynchronize(s));  // block staging freed at scope exit
            }
            const auto cuts = slice_cuts(lr, p);
            std::vector<DevBuf> oa(p), ob(p);
            std::vector<float*> poa, pob;
            for (int i = 0; i < p; ++i) {
                const int64_t n = cuts[i + 1] - cuts[i];
                oa[i].alloc(sizeof(float) * std::max<int64_t>(n * ff, 1), s);
                ob[i].alloc(sizeof(float) * std::max<int64_t>(n * f, 1), s);
                poa.push_back(oa[i].as<float>());
                pob.push_back(ob[i].as<float>());
            }
            if (dbl) {
                std::vector<const double*> a, b;
                for (int i = 0; i < p; ++i) { a.push_back(pa[i].as<double>()); b.push_back(pb[i].as<double>()); }
                reduce_slices<double>(a, b, lr, f, sc, poa, pob, s);
            } else {
                std::vector<const float*> a, b;
                for (int i = 0; i < p; ++i) { a.push_back(pa[i].as<float>()); b.push_back(pb[i].as<float>()); }
                reduce_slices<float>(a, b, lr, f, sc, poa, pob, s);
            }
            for (int i = 0; i < p; ++i) {
                const int64_t n = cuts[i + 1] - cuts[i];
                if (n == 0) continue;
                StatusBufs sb(n, s);
                solve_exact(poa[i], pob[i], n, f, false, X.as<float>() + (row_cuts[j] + cuts[i]) * f, sb.st, s);
                sb.raise_if_broken(s, 0);
            }
        }
        d2h(x_out, X.as<float>(), total_rows * f, s);
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

// ---- device entry points ----------------------------------------------------------

alsk_status alsk_dev_update(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                            double lambda, alsk_precision precision, int64_t batch_rows,
                            int64_t row_begin, int64_t row_end, float* x_out, void* stream) {
    return guard([&] {
        check_update_shapes(r, theta_rows, f);
        require_device();
        update_rows_device(dev_view(r), theta, theta_rows, f, lambda, precision,
                           batch_rows, row_begin, row_end, x_out, as_stream(stream));
    });
}

alsk_status alsk_dev_hermitian(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                               double lambda, alsk_precision precision, int64_t row_begin,
                               int64_t row_end, float* a_out, float* b_out, void* stream) {
    return guard([&] {
        check_update_shapes(r, theta_rows, f);
        require_device();
        const DevCsr v = dev_view(r);
        if (precision != ALSK_PREC_FP64_EXACT) {
            check_columns(v, row_begin, row_end, r->col_offset, r->col_offset + theta_rows, as_stream(stream));
            const bool done = use_tensor_cores(precision, f)
                                  ? hermitian_tc(v, theta, theta_rows, f, static_cast<float>(lambda), row_begin,
                                                 row_end, a_out, b_out, as_stream(stream))
                                  : hermitian_fused_fp32(v, theta, theta_rows, f, static_cast<float>(lambda),
                                                         row_begin, row_end, a_out, b_out, as_stream(stream));
            if (done) return;
        }
        hermitian_materialize(v, theta, f, lambda, precision == ALSK_PREC_FP64_EXACT, row_begin,
                              row_end, a_out, b_out, as_stream(stream));
    });
}

alsk_status alsk_dev_loss(const alsk_csr* r, const int64_t* col_nnz, const float* x,
                          const float* theta, int64_t theta_rows, int f, double lambda,
                          double* out, void* stream) {
    return guard([&] {
        check_update_shapes(r, theta_rows, f);
        require_device();
        *out = loss_device(dev_view(r), col_nnz, x, theta, f, lambda, as_stream(stream));
    });
}

alsk_status alsk_dev_rmse(const int64_t* rows, const int64_t* cols, const float* values,
                          int64_t count, const float* x, int64_t x_rows, const float* theta,
                          int64_t theta_rows, int f, double* out, void* stream) {
    return guard([&] {
        if (count <= 0) fail_input("empty test set");
        require_device();
        *out = rmse_device(rows, cols, values, count, x, x_rows, theta, theta_rows, f, as_stream(stream));
    });
}

alsk_status alsk_dev_csr_to_csc(const alsk_csr* a, int64_t* col_ptr_out, int32_t* row_idx_out,
                                float* values_out, void* stream) {
    return guard([&] {
        require_device();
        csr_to_csc_device(dev_view(a), col_ptr_out, row_idx_out, values_out, as_stream(stream));
    });
}

// split_train_test (dataio.hpp:251-290) on device arrays: host Fisher-Yates picks the
// held-out positions (bit-exact with the reference), the device compacts the CSR. With
// train_row_ptr == NULL only *k_out is set (two-call sizing, like alsk_split_train_test).
alsk_status alsk_dev_split_train_test(const alsk_csr* r, double holdout, uint64_t seed, int64_t* k_out,
                                      int64_t* train_row_ptr, int32_t* train_col_idx, float* train_values,
                                      alsk_triplet* test_out, void* stream) {
    return guard([&] {
        *k_out = split_holdout_count(r->nnz, holdout);
        if (train_row_ptr == nullptr) return;
        require_device();
        split_train_test_device(dev_view(r), holdout, seed, train_row_ptr, train_col_idx, train_values, test_out,
                                as_stream(stream));
    });
}

// ---- per-rank synthetic data (bench / multi-GPU setup) ------------------------------
alsk_status alsk_dev_synth_rows(int64_t m, int64_t n, int64_t nnz, uint64_t seed, int64_t row_begin, int64_t row_end,
                                int64_t* row_ptr, int32_t* col_idx, float* values, void* stream) {
    return guard([&] {
        require_device();
        synth_rows_device(m, n, nnz, seed, row_begin, row_end, row_ptr, col_idx, values, as_stream(stream));
    });
}

int64_t alsk_synth_row_start(int64_t m, int64_t nnz, int64_t u) { return synth_row_start(nnz, m, u); }

alsk_status alsk_holdout_mask(int64_t nnz, double holdout, uint64_t seed, uint32_t* mask_out, int64_t* k_out) {
    return guard([&] {
        const int64_t k = split_holdout_count(nnz, holdout);
        *k_out = k;
        if (mask_out == nullptr) return;
        std::vector<uint32_t> mask;
        holdout_mask_host(nnz, k, seed, mask);
        std::memcpy(mask_out, mask.data(), sizeof(uint32_t) * mask.size());
    });
}

int64_t alsk_mask_count(const uint32_t* mask, int64_t bit_begin, int64_t bit_end) {
    int64_t c = 0;
    for (int64_t b = bit_begin; b < bit_end;) {
        if ((b & 31) == 0 && b + 32 <= bit_end) {
            c += __builtin_popcount(mask[b >> 5]);
            b += 32;
        } else {
            c += (mask[b >> 5] >> (b & 31)) & 1u;
            ++b;
        }
    }
    return c;
}

alsk_status alsk_dev_split_mask(const alsk_csr* r, const uint32_t* d_mask, int64_t bit_offset, int64_t row_base,
                                int64_t* train_row_ptr, int32_t* train_col_idx, float* train_values,
                                alsk_triplet* test_out, int64_t* train_nnz, void* stream) {
    return guard([&] {
        require_device();
        *train_nnz = split_with_mask_device(dev_view(r), d_mask, bit_offset, row_base, train_row_ptr, train_col_idx,
                                            train_values, test_out, as_stream(stream));
    });
}

alsk_status alsk_dev_filter_columns(const alsk_csr* r, int64_t col_begin, int64_t col_end, int64_t* row_ptr_out,
                                    int32_t* col_idx_out, float* values_out, int64_t* nnz_out, void* stream) {
    return guard([&] {
        require_device();
        *nnz_out = filter_columns_device(dev_view(r), col_begin, col_end, row_ptr_out, col_idx_out, values_out,
                                         as_stream(stream));
    });
}

alsk_status alsk_dev_partial_hermitian(const alsk_csr* r, const float* theta, int64_t theta_rows,
                                       int f, double lambda, int64_t row_begin, int64_t row_end,
                                       double* out_packed, void* stream) {
    return guard([&] {
        if (f < 1) fail_input("rank must be >= 1");
        require_device();
        const DevCsr v = dev_view(r);
        check_columns(v, row_begin, row_end, r->col_offset, r->col_offset + theta_rows, as_stream(stream));
        hermitian_materialize_d(v, theta, f, lambda, true, row_begin, row_end, out_packed, nullptr, true,
                                as_stream(stream));
    });
}

int64_t alsk_packed_stride(int f) {
    if (f < 1) return 0;
    return f <= 15 ? static_cast<int64_t>(f) * (f + 1) / 2 + f : packed_stride(f);
}

alsk_status alsk_dev_partial_hermitian_f32(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                                           double lambda, int64_t row_begin, int64_t row_end, float* out_packed,
                                           void* stream) {
    return guard([&] {
        if (f < 1) fail_input("rank must be >= 1");
        if (f > 15 && !tc_supported(f))
            fail_input("FP32 partial Hermitians need f <= 15 (register kernel) or 16 <= f <= 119 (tensor cores)");
        require_device();
        const DevCsr v = dev_view(r);
        check_columns(v, row_begin, row_end, r->col_offset, r->col_offset + theta_rows, as_stream(stream));
        if (f <= 15) {
            partial_small_fp32(v, theta, theta_rows, f, static_cast<float>(lambda), row_begin, row_end, out_packed,
                               as_stream(stream));
            return;
        }
        if (!hermitian_packed_tc(v, theta, theta_rows, f, static_cast<float>(lambda), row_begin, row_end, out_packed,
                                 as_stream(stream)))
            fail_input("tensor-core Hermitian unavailable for this rank");
    });
}

alsk_status alsk_dev_solve_packed_f32(const float* packed, int64_t count, int f, float* x_out, void* stream) {
    return guard([&] {
        if (count <= 0) return;
        if (f < 1) fail_input("rank must be >= 1");
        require_device();
        cudaStream_t s = as_stream(stream);
        StatusBufs sb(count, s);
        if (f <= 15)
            solve_small_packed(packed, count, f, x_out, sb.st, s);
        else
            packed_solve(packed, count, f, x_out, sb.st, 0, s);
        sb.raise_if_broken(s, 0);
    });
}

alsk_status alsk_dev_solve_packed(const double* packed, int64_t count, int f, float* x_out, void* stream) {
    return guard([&] {
        if (count <= 0) return;
        require_device();
        cudaStream_t s = as_stream(stream);
        DevBuf A(sizeof(float) * count * f * f, s), B(sizeof(float) * count * f, s);
        unpack_packed(packed, count, f, A.as<float>(), B.as<float>(), s);
        StatusBufs sb(count, s);
        solve_exact(A.as<float>(), B.as<float>(), count, f, false, x_out, sb.st, s);
        sb.raise_if_broken(s, 0);
    });
}

// ---- device-resident session ------------------------------------------------------
struct alsk_session {
    int64_t m = 0, n = 0, nnz = 0, test_count = 0;
    int f = 0;
    double lambda = 0.0;
    alsk_precision precision = ALSK_PREC_FP32;
    int64_t batch_rows = 4096;
    cudaStream_t stream = nullptr;
    DevBuf rp, ci, rv, cp, ri, cv, col_nnz, X, T, tr, tc, tv;
    DevCsr R, RT;
};

alsk_status alsk_session_create(const alsk_csr* r, const int64_t* col_ptr, const int32_t* row_idx,
                                const float* csc_values, const alsk_triplet* test, int64_t test_count,
                                int f, double lambda, alsk_precision precision, int64_t batch_rows,
                                const float* x0, const float* theta0, alsk_session** out) {
    return guard([&] {
        if (f < 1) fail_input("rank must be >= 1");
        require_device();
        auto* S = new alsk_session();
        try {
            S->m = r->rows;
            S->n = r->cols;
            S->nnz = r->nnz;
            S->f = f;
            S->lambda = lambda;
            S->precision = precision;
            S->batch_rows = batch_rows;
            ALSK_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
            cudaStream_t s = S->stream;
            const int64_t nz = std::max<int64_t>(r->nnz, 1);
            S->rp.alloc(sizeof(int64_t) * (S->m + 1), s);
            S->ci.alloc(sizeof(int32_t) * nz, s);
            S->rv.alloc(sizeof(float) * nz, s);
            h2d(S->rp.as<int64_t>(), r->row_ptr, S->m + 1, s);
            h2d(S->ci.as<int32_t>(), r->col_idx, r->nnz, s);
            h2d(S->rv.as<float>(), r->values, r->nnz, s);
            S->R = DevCsr{S->m, S->n, 0, r->nnz, S->rp.as<int64_t>(), S->ci.as<int32_t>(), S->rv.as<float>()};
            S->cp.alloc(sizeof(int64_t) * (S->n + 1), s);
            S->ri.alloc(sizeof(int32_t) * nz, s);
            S->cv.alloc(sizeof(float) * nz, s);
            if (col_ptr) {
                h2d(S->cp.as<int64_t>(), col_ptr, S->n + 1, s);
                h2d(S->ri.as<int32_t>(), row_idx, r->nnz, s);
                h2d(S->cv.as<float>(), csc_values, r->nnz, s);
            } else {
                csr_to_csc_device(S->R, S->cp.as<int64_t>(), S->ri.as<int32_t>(), S->cv.as<float>(), s);
            }
            S->RT = DevCsr{S->n, S->m, 0, r->nnz, S->cp.as<int64_t>(), S->ri.as<int32_t>(), S->cv.as<float>()};
            S->col_nnz.alloc(sizeof(int64_t) * std::max<int64_t>(S->n, 1), s);
            column_counts(S->R, S->col_nnz.as<int64_t>(), s);
            S->X.alloc(sizeof(float) * std::max<int64_t>(S->m * f, 1), s);
            S->T.alloc(sizeof(float) * std::max<int64_t>(S->n * f, 1), s);
            h2d(S->X.as<float>(), x0, S->m * f, s);
            h2d(S->T.as<float>(), theta0, S->n * f, s);
            S->test_count = test_count;
            if (test_count > 0) {
                std::vector<int64_t> hr(test_count), hc(test_count);
                std::vector<float> hv(test_count);
                for (int64_t i = 0; i < test_count; ++i) {
                    hr[i] = test[i].row;
                    hc[i] = test[i].col;
                    hv[i] = test[i].value;
                }
                S->tr.alloc(sizeof(int64_t) * test_count, s);
                S->tc.alloc(sizeof(int64_t) * test_count, s);
                S->tv.alloc(sizeof(float) * test_count, s);
                h2d(S->tr.as<int64_t>(), hr.data(), test_count, s);
                h2d(S->tc.as<int64_t>(), hc.data(), test_count, s);
                h2d(S->tv.as<float>(), hv.data(), test_count, s);
                ALSK_CUDA(cudaStreamSynchronize(s));
            }
            ALSK_CUDA(cudaStreamSynchronize(s));
        } catch (...) {
            delete S;
            throw;
        }
        *out = S;
    });
}

alsk_status alsk_session_half_x(alsk_session* S) {
    return guard([&] {
        update_rows_device(S->R, S->T.as<float>(), S->n, S->f, S->lambda, S->precision,
                           S->batch_rows, 0, S->m, S->X.as<float>(), S->stream);
    });
}

alsk_status alsk_session_half_theta(alsk_session* S) {
    return guard([&] {
        update_rows_device(S->RT, S->X.as<float>(), S->m, S->f, S->lambda, S->precision,
                           S->batch_rows, 0, S->n, S->T.as<float>(), S->stream);
    });
}

alsk_status alsk_session_loss(alsk_session* S, double* out) {
    return guard([&] {
        *out = loss_device(S->R, S->col_nnz.as<int64_t>(), S->X.as<float>(), S->T.as<float>(), S->f, S->lambda,
                           S->stream);
    });
}

alsk_status alsk_session_rmse(alsk_session* S, double* out) {
    return guard([&] {
        if (S->test_count <= 0) {
            *out = std::numeric_limits<double>::quiet_NaN();
            return;
        }
        *out = rmse_device(S->tr.as<int64_t>(), S->tc.as<int64_t>(), S->tv.as<float>(), S->test_count,
                           S->X.as<float>(), S->m, S->T.as<float>(), S->n, S->f, S->stream);
    });
}

alsk_status alsk_session_factors(alsk_session* S, float* x_out, float* theta_out) {
    return guard([&] {
        if (x_out) d2h(x_out, S->X.as<float>(), S->m * S->f, S->stream);
        if (theta_out) d2h(theta_out, S->T.as<float>(), S->n * S->f, S->stream);
        ALSK_CUDA(cudaStreamSynchronize(S->stream));
    });
}

alsk_status alsk_session_device(alsk_session* S, float** x, float** theta, void** stream) {
    return guard([&] {
        if (x) *x = S->X.as<float>();
        if (theta) *theta = S->T.as<float>();
        if (stream) *stream = S->stream;
    });
}

void alsk_session_destroy(alsk_session* S) {
    if (!S) return;
    cudaStream_t s = S->stream;
    if (s) cudaStreamSynchronize(s);
    delete S;  // DevBufs free on their stream
    if (s) {
        cudaDeviceSynchronize();
        cudaStreamDestroy(s);
    }
}

// ---- binary ratings cache (dataio.hpp:108-163; helpers in cache_io.cuh) ----

alsk_status alsk_cache_header(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz) {
    return guard([&] {
        File in(path, "rb");
        const Header h = read_header(in);
        *rows = static_cast<int64_t>(h.rows);
        *cols = static_cast<int64_t>(h.cols);
        *nnz = static_cast<int64_t>(h.nnz);
    });
}

alsk_status alsk_save_cache(const alsk_csr* r, const char* path) {
    return guard([&] {
        File out(path, "wb");
        const uint64_t h[5] = {kMagic, kVersion, static_cast<uint64_t>(r->rows), static_cast<uint64_t>(r->cols),
                               static_cast<uint64_t>(r->nnz)};
        out.write(h, sizeof(h));
        out.write(r->row_ptr, sizeof(int64_t) * (r->rows + 1));
        out.write(r->col_idx, sizeof(int32_t) * r->nnz);
        out.write(r->values, sizeof(float) * r->nnz);
        if (std::fflush(out.f) != 0) fail_io(std::string("write failed for ") + path);
    });
}

namespace alsk {
// The caller sized its buffers from an earlier header read; a file replaced since then (a
// re-persisted grid, a new cache) must not be loaded past them.
inline void check_capacity(const char* path, int64_t have_rows, int64_t have_nnz, int64_t cap_rows, int64_t cap_nnz) {
    if (have_rows > cap_rows || have_nnz > cap_nnz)
        fail_io(std::string(path) + ": file changed since its header was read (" + std::to_string(have_rows) +
                " rows / " + std::to_string(have_nnz) + " entries exceed the caller's " + std::to_string(cap_rows) +
                " / " + std::to_string(cap_nnz) + ")");
}
}  // namespace alsk

// Host buffers of capacity cap_rows+1 / cap_nnz (sizes from alsk_cache_header).
alsk_status alsk_load_cache(const char* path, int64_t cap_rows, int64_t cap_nnz, int64_t* row_ptr, int32_t* col_idx,
                            float* values) {
    return guard([&] {
        File in(path, "rb");
        const Header h = read_header(in);
        const int64_t rows = static_cast<int64_t>(h.rows), nnz = static_cast<int64_t>(h.nnz);
        check_capacity(path, rows, nnz, cap_rows, cap_nnz);
        in.read(row_ptr, sizeof(int64_t) * (rows + 1), "row_ptr");
        in.read(col_idx, sizeof(int32_t) * nnz, "col_idx");
        in.read(values, sizeof(float) * nnz, "values");
        Validator val{row_ptr, rows, static_cast<int64_t>(h.cols), nnz, in.path};
        val.ends();
        val.feed(col_idx, 0, nnz);
    });
}

// Device buffers: row_ptr[rows+1], col_idx[nnz], values[nnz] (sizes from alsk_cache_header).
alsk_status alsk_dev_load_cache(const char* path, int64_t cap_rows, int64_t cap_nnz, int64_t* row_ptr,
                                int32_t* col_idx, float* values, void* stream) {
    return guard([&] {
        require_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        File in(path, "rb");
        const Header h = read_header(in);
        const int64_t rows = static_cast<int64_t>(h.rows), nnz = static_cast<int64_t>(h.nnz);
        check_capacity(path, rows, nnz, cap_rows, cap_nnz);
        std::vector<int64_t> rp(static_cast<size_t>(rows) + 1);
        in.read(rp.data(), sizeof(int64_t) * rp.size(), "row_ptr");
        Validator val{rp.data(), rows, static_cast<int64_t>(h.cols), nnz, in.path};
        val.ends();
        ALSK_CUDA(cudaMemcpyAsync(row_ptr, rp.data(), sizeof(int64_t) * rp.size(), cudaMemcpyHostToDevice, s));
        // process-wide pinned staging (allocated once): read chunk k+1 while chunk k uploads
        PinnedStage& ps = pinned_stage();
        std::lock_guard<std::mutex> hold(ps.mu);
        ps.ensure();
        void* const* stage = ps.buf;
        cudaEvent_t* done = ps.ev;
        constexpr size_t kChunk = PinnedStage::kChunk;
        struct Drain {
            cudaStream_t s;
            ~Drain() { cudaStreamSynchronize(s); }  // the buffers are reused by the next load
        } drain{s};
        int buf = 0;
        // positional, multi-threaded reads of each chunk (the size matched the header, so a
        // short read is a truncation)
        auto stream_array = [&](void* dst, size_t elem, int64_t count, const char* what, size_t file_off) {
            const int64_t per = static_cast<int64_t>(kChunk / elem);
            for (int64_t k0 = 0; k0 < count; k0 += per, buf ^= 1) {
                const int64_t k1 = std::min(count, k0 + per);
                ALSK_CUDA(cudaEventSynchronize(done[buf]));  // the previous upload from this buffer is done
                if (!parallel_pio(fileno(in.f), static_cast<char*>(stage[buf]), elem * (k1 - k0), file_off + elem * k0,
                                  false))
                    fail_io(in.path + ": truncated while reading " + what);
                ALSK_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + elem * k0, stage[buf], elem * (k1 - k0),
                                          cudaMemcpyHostToDevice, s));
                ALSK_CUDA(cudaEventRecord(done[buf], s));
            }
        };
        const size_t ci_off = 40 + sizeof(int64_t) * static_cast<size_t>(rows + 1);
        stream_array(col_idx, sizeof(int32_t), nnz, "col_idx", ci_off);
        stream_array(values, sizeof(float), nnz, "values", ci_off + sizeof(int32_t) * static_cast<size_t>(nnz));
        // the CSR invariants are checked in HBM (validate.cu), the host only reads and copies
        const int64_t bad = csr_first_bad_row(row_ptr, col_idx, rows, static_cast<int64_t>(h.cols), nnz, s);
        if (bad >= 0) report_bad_row(rp.data(), rows, static_cast<int64_t>(h.cols), nnz, in.path, bad, col_idx, s);
    });
}

// ---- factor checkpoints (dataio.hpp:546-786) ----

alsk_status alsk_checkpoint_write(const char* dir, int iteration, int which, int64_t rows, int f, uint64_t digest,
                                  const float* entries) {
    return guard([&] {
        if (which != 0 && which != 1) fail_input("factor kind must be 0 (x) or 1 (theta)");
        write_checkpoint_file(dir, iteration, which, rows, f, digest, entries);
    });
}

alsk_status alsk_checkpoint_path(const char* dir, int iteration, int which, char* out, size_t cap) {
    return guard([&] {
        const std::string p = (fs::path(dir) / checkpoint_name(iteration, which)).string();
        if (p.size() + 1 > cap) fail_input("path buffer too small");
        std::memcpy(out, p.c_str(), p.size() + 1);
    });
}

alsk_status alsk_checkpoint_header(const char* path, int* iteration, int* which, int64_t* rows, int* f,
                                   uint64_t* digest) {
    return guard([&] {
        File in(path, "rb");
        const CkptHeader h = read_checkpoint_header(in);
        *iteration = h.iteration;
        *which = h.which;
        *rows = h.rows;
        *f = h.f;
        *digest = h.digest;
    });
}

alsk_status alsk_checkpoint_read(const char* path, int64_t cap_entries, float* entries) {
    return guard([&] {
        File in(path, "rb");
        const CkptHeader h = read_checkpoint_header(in);
        check_capacity(path, 0, static_cast<int64_t>(h.rows) * h.f, 0, cap_entries);
        in.read(entries, sizeof(float) * static_cast<size_t>(h.rows) * h.f, "payload");
    });
}

// Restore a factor straight into HBM (rows*f floats at d_entries), through pinned staging.
alsk_status alsk_dev_checkpoint_read(const char* path, int64_t cap_entries, float* d_entries, void* stream) {
    return guard([&] {
        require_device();
        File in(path, "rb");
        const CkptHeader h = read_checkpoint_header(in);
        check_capacity(path, 0, static_cast<int64_t>(h.rows) * h.f, 0, cap_entries);
        const size_t bytes = sizeof(float) * static_cast<size_t>(h.rows) * h.f;
        if (!bytes) return;
        void* stage = nullptr;
        ALSK_CUDA(cudaMallocHost(&stage, bytes));
        struct Free {
            void* p;
            ~Free() { cudaFreeHost(p); }
        } free_stage{stage};
        in.read(stage, bytes, "payload");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        ALSK_CUDA(cudaMemcpyAsync(d_entries, stage, bytes, cudaMemcpyHostToDevice, s));
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

// Newest checkpoint under dir (which = -1: either kind, theta outranking x at the same
// iteration; 0 / 1: that kind only). *found = 0 and out = "" when there is none.
alsk_status alsk_checkpoint_latest(const char* dir, int which, char* out, size_t cap, int* found) {
    return guard([&] {
        const std::string p = latest_checkpoint(dir, which);
        if (p.size() + 1 > cap) fail_input("path buffer too small");
        std::memcpy(out, p.c_str(), p.size() + 1);
        *found = p.empty() ? 0 : 1;
    });
}

alsk_status alsk_ckpt_writer_create(const char* dir, void** writer) {
    return guard([&] {
        *writer = new DeviceWriter(dir);  // CUDA state is created on the first device submit
    });
}

alsk_status alsk_ckpt_writer_submit_device(void* writer, int iteration, int which, int64_t rows, int f,
                                           uint64_t digest, const float* d_factor, void* stream) {
    return guard([&] {
        require_device();
        static_cast<DeviceWriter*>(writer)->submit_device(iteration, which, rows, f, digest, d_factor,
                                                          static_cast<cudaStream_t>(stream));
    });
}

alsk_status alsk_ckpt_writer_submit_host(void* writer, int iteration, int which, int64_t rows, int f,
                                         uint64_t digest, const float* entries) {
    return guard([&] {
        static_cast<DeviceWriter*>(writer)->submit_host(iteration, which, rows, f, digest, entries);
    });
}

alsk_status alsk_ckpt_writer_flush(void* writer) {
    return guard([&] { static_cast<DeviceWriter*>(writer)->flush(); });
}

void alsk_ckpt_writer_destroy(void* writer) { delete static_cast<DeviceWriter*>(writer); }

// ---- persisted grids and the out-of-core block stream (dataio.hpp:352-540) ----

alsk_status alsk_persist_grid_meta(const char* dir, int p, int q, int64_t rows, int64_t cols, const int64_t* row_cuts,
                                   const int64_t* col_cuts) {
    return guard([&] {
        GridMetaH g;
        g.p = p;
        g.q = q;
        g.rows = rows;
        g.cols = cols;
        g.row_cuts.assign(row_cuts, row_cuts + q + 1);
        g.col_cuts.assign(col_cuts, col_cuts + p + 1);
        write_grid_meta(dir, g);
    });
}

alsk_status alsk_block_path(const char* dir, int i, int j, char* out, size_t cap) {
    return guard([&] {
        const std::string p = block_path(dir, i, j);
        if (p.size() + 1 > cap) fail_input("path buffer too small");
        std::memcpy(out, p.c_str(), p.size() + 1);
    });
}

alsk_status alsk_grid_meta(const char* dir, int* p, int* q, int64_t* rows, int64_t* cols, int64_t* row_cuts,
                           int64_t* col_cuts) {
    return guard([&] {
        const GridMetaH g = read_grid_meta(dir);
        *p = g.p;
        *q = g.q;
        *rows = g.rows;
        *cols = g.cols;
        if (row_cuts) std::copy(g.row_cuts.begin(), g.row_cuts.end(), row_cuts);
        if (col_cuts) std::copy(g.col_cuts.begin(), g.col_cuts.end(), col_cuts);
    });
}

alsk_status alsk_block_stream_open(const char* dir, const int* order_ij, int count, void** stream_out) {
    return guard([&] {
        require_device();
        if (count < 0) fail_input("block count must be >= 0");
        *stream_out = new DeviceBlockStream(dir, std::vector<int>(order_ij, order_ij + 2 * count));
    });
}

alsk_status alsk_block_stream_next(void* bs, void* stream, int* has_block, int* i, int* j, alsk_csr* out) {
    return guard([&] {
        DeviceBlockStream::Out o{};
        *has_block = static_cast<DeviceBlockStream*>(bs)->next(as_stream(stream), o) ? 1 : 0;
        if (!*has_block) return;
        *i = o.i;
        *j = o.j;
        *out = alsk_csr{o.rows, o.cols, o.col_offset, o.nnz, o.row_ptr, o.col_idx, o.values};
    });
}

void alsk_block_stream_close(void* bs) { delete static_cast<DeviceBlockStream*>(bs); }

// ---- out-of-core half-sweep -----------------------------------
namespace alsk {
__global__ void ooc_add_rows_kernel(float* __restrict__ acc, const float* __restrict__ part, int64_t n4) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n4;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float4 a = reinterpret_cast<float4*>(acc)[k];
        const float4 b = reinterpret_cast<const float4*>(part)[k];
        a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
        reinterpret_cast<float4*>(acc)[k] = a;
    }
}
// flag[0] = first out-of-slab entry of a block (~0 if none); copies that entry's column into
// flag[1] while the block is still resident, so the error can be raised after it is released
__global__ void ooc_bad_column_kernel(const int32_t* __restrict__ col_idx, unsigned long long* flag) {
    if (flag[0] != ~0ull) flag[1] = static_cast<unsigned long long>(static_cast<int64_t>(col_idx[flag[0]]));
}
}  // namespace alsk

// One half-sweep over a persisted p x q grid (persist_grid, dataio.hpp:381-400) whose blocks
// need not fit in HBM together -- the scale-up of su_als_update_x (parallel.hpp:487-583) on
// one GPU: the device block stream uploads block (i, j) while the previous one computes; per
// row partition j the partial Hermitians of its blocks against the factor's column slabs are
// reduced and solved slice by slice (slice_cuts, parallel.hpp:160-168), as su_als's workers
// do. FP64-exact: double partials, the reference's one-phase reduce order, rounded once to
// float, the reference-order solve -- bit-identical to su_als_update_x on the same grid.
// FP32: the tensor-core packed partials (16 <= f <= 119) summed in block order, else float
// partials through the same reduce. Block columns outside their slab raise the reference's
// InputError (checked asynchronously; the tensor-core gather clamps meanwhile).
alsk_status alsk_ooc_update(const char* grid_dir, const float* factor, int64_t factor_rows, int f,
                            const alsk_solver_config* cfg, float* x_out, void* stream) {
    return guard([&] {
        if (f < 1) fail_input("rank must be >= 1");
        require_device();
        cudaStream_t s = as_stream(stream);
        const GridMetaH g = read_grid_meta(grid_dir);
        if (factor_rows != g.cols)
            fail_input("factor rows " + std::to_string(factor_rows) + " do not match matrix columns " +
                       std::to_string(g.cols));
        const int p = g.p, q = g.q;
        const bool exact = cfg->accumulate_double != 0;
        const bool tc = !exact && use_tensor_cores(ALSK_PREC_FP32, f);
        std::vector<int> order;
        for (int j = 0; j < q; ++j)
            for (int i = 0; i < p; ++i) order.insert(order.end(), {i, j});
        const ReduceSchedule sc = build_reduce_schedule(p, nullptr, false);
        int64_t lr_max = 1;
        for (int j = 0; j < q; ++j) lr_max = std::max(lr_max, g.row_cuts[j + 1] - g.row_cuts[j]);
        const int64_t ff = static_cast<int64_t>(f) * f;
        const size_t pkn = static_cast<size_t>(packed_stride(f));
        DevBuf acc, part;
        if (tc) {
            acc.alloc(sizeof(float) * pkn * lr_max, s);
            part.alloc(sizeof(float) * pkn * lr_max, s);
        }
        DeviceBlockStream bs(grid_dir, order);
        // per block of a partition: first out-of-slab entry and its column, checked on the
        // device; read back once per partition (no host round trip per block)
        DevBuf flags(sizeof(unsigned long long) * 2 * static_cast<size_t>(p), s);
        std::vector<unsigned long long> hflags(2 * static_cast<size_t>(p));
        for (int j = 0; j < q; ++j) {
            ALSK_CUDA(cudaMemsetAsync(flags.as<void>(), 0xff, sizeof(unsigned long long) * 2 * p, s));
            const int64_t r0 = g.row_cuts[j], lr = g.row_cuts[j + 1] - r0;
            const auto cuts = slice_cuts(lr, p);
            std::vector<DevBuf> pa, pb;
            if (!tc)
                for (int i = 0; i < p; ++i) {
                    const size_t esz = exact ? sizeof(double) : sizeof(float);
                    pa.emplace_back(esz * std::max<int64_t>(lr * ff, 1), s);
                    pb.emplace_back(esz * std::max<int64_t>(lr * f, 1), s);
                }
            for (int i = 0; i < p; ++i) {
                DeviceBlockStream::Out o{};
                if (!bs.next(s, o))
                    fail_io(std::string(grid_dir) + ": block stream ended before block (" + std::to_string(i) + ", " +
                            std::to_string(j) + ")");
                const DevCsr v{o.rows, o.cols, o.col_offset, o.nnz, o.row_ptr, o.col_idx, o.values};
                const int64_t lo = g.col_cuts[i], width = g.col_cuts[i + 1] - lo;
                if (lr == 0) continue;
                // the block's columns against its slab, resolved with the partition's statuses
                unsigned long long* fl = flags.as<unsigned long long>() + 2 * i;
                check_columns_async(v, 0, o.nnz, lo, lo + width, fl, s);
                ooc_bad_column_kernel<<<1, 1, 0, s>>>(v.col_idx, fl);
                ALSK_LAUNCHED();
                const float* slab = factor + lo * f;
                if (tc) {
                    // block i's packed partial rows, added into the partition's running rows by a
                    // streaming kernel (FP32, the blocks in order; adding in the Hermitian's
                    // epilogue instead measured 1.5x slower: a dependent load per packed block)
                    hermitian_packed_tc(v, slab, width, f, static_cast<float>(cfg->lambda), 0, lr,
                                        i == 0 ? acc.as<float>() : part.as<float>(), s);
                    if (i > 0) {
                        const int64_t n4 = static_cast<int64_t>(lr * pkn / 4);
                        ooc_add_rows_kernel<<<static_cast<unsigned>(std::min<int64_t>((n4 + 255) / 256, num_sms() * 8)), 256, 0, s>>>(acc.as<float>(), part.as<float>(), n4);
                        ALSK_LAUNCHED();
                    }
                } else if (exact) {
                    hermitian_materialize_d(v, slab, f, cfg->lambda, true, 0, lr, pa[i].as<double>(),
                                            pb[i].as<double>(), false, s);
                } else {
                    hermitian_materialize(v, slab, f, cfg->lambda, false, 0, lr, pa[i].as<float>(),
                                          pb[i].as<float>(), s);
                }
            }
            if (lr == 0) continue;
            // the partition's column errors in block order, before anything of it is solved
            // (the reference's worker assembles partition j block by block, then solves it)
            d2h(hflags.data(), flags.as<unsigned long long>(), 2 * static_cast<size_t>(p), s);
            ALSK_CUDA(cudaStreamSynchronize(s));
            for (int i = 0; i < p; ++i)
                if (hflags[2 * i] != ~0ull)
                    fail_input("column " + std::to_string(static_cast<int64_t>(hflags[2 * i + 1])) +
                               " outside partition [" + std::to_string(g.col_cuts[i]) + ", " +
                               std::to_string(g.col_cuts[i + 1]) + ")");
            std::vector<StatusBufs> status;
            status.reserve(p);
            if (tc) {
                for (int k = 0; k < p; ++k) {
                    const int64_t c0 = cuts[k], n = cuts[k + 1] - c0;
                    status.emplace_back(std::max<int64_t>(n, 1), s);
                    if (n) packed_solve(acc.as<float>() + c0 * pkn, n, f, x_out + (r0 + c0) * f, status.back().st, 0, s);
                }
            } else {
                std::vector<DevBuf> oa(p), ob(p);
                std::vector<float*> poa, pob;
                for (int k = 0; k < p; ++k) {
                    const int64_t n = cuts[k + 1] - cuts[k];
                    oa[k].alloc(sizeof(float) * std::max<int64_t>(n * ff, 1), s);
                    ob[k].alloc(sizeof(float) * std::max<int64_t>(n * f, 1), s);
                    poa.push_back(oa[k].as<float>());
                    pob.push_back(ob[k].as<float>());
                }
                if (exact) {
                    std::vector<const double*> a, b;
                    for (int i = 0; i < p; ++i) a.push_back(pa[i].as<double>()), b.push_back(pb[i].as<double>());
                    reduce_slices<double>(a, b, lr, f, sc, poa, pob, s);
                } else {
                    std::vector<const float*> a, b;
                    for (int i = 0; i < p; ++i) a.push_back(pa[i].as<float>()), b.push_back(pb[i].as<float>());
                    reduce_slices<float>(a, b, lr, f, sc, poa, pob, s);
                }
                for (int k = 0; k < p; ++k) {
                    const int64_t n = cuts[k + 1] - cuts[k];
                    status.emplace_back(std::max<int64_t>(n, 1), s);
                    if (n) solve_exact(poa[k], pob[k], n, f, false, x_out + (r0 + cuts[k]) * f, status.back().st, s);
                }
            }
            // this partition's breakdowns before the next partition's column checks (the
            // reference's worker loop solves partition j before assembling j+1)
            for (auto& sb : status) sb.raise_if_broken(s, 0);
        }
        ALSK_CUDA(cudaStreamSynchronize(s));
    });
}

alsk_status alsk_dev_to_host(void* dst, const void* src, size_t bytes, void* stream) {
    return guard([&] {
        require_device();
        ALSK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
        ALSK_CUDA(cudaStreamSynchronize(as_stream(stream)));
    });
}

alsk_status alsk_host_to_dev(void* dst, const void* src, size_t bytes, void* stream) {
    return guard([&] {
        require_device();
        ALSK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
        ALSK_CUDA(cudaStreamSynchronize(as_stream(stream)));
    });
}

}  // extern "C"
