// Multi-GPU ALS inside libalskit_cuda.so (reference su_als_update_x,
// parallel.hpp:487-583, and train_run's half_update, driver.hpp:168-172):
//
//  * alsk_comm_*      NCCL communicators. NCCL is resolved at run time (dlopen of
//                     libnccl.so.2, which is the already-loaded copy when PyTorch brought its
//                     own), so the library loads on hosts without NCCL and only the
//                     multi-GPU entry points report its absence. One communicator per GPU:
//                     one process per GPU (alsk_comm_init_rank with an id exchanged by the
//                     caller) or one process driving several GPUs (alsk_comm_init_all).
//  * alsk_workspace_* caller-owned packed-row scratch for the tensor-core half-sweep, so
//                     concurrent sessions never serialise on the per-device default.
//  * alsk_mp_*        one rank's share of a model-parallel ALS run. MODEL: rows of X, then of
//                     Theta, cut into P equal (padded) slices; each rank solves its slice and
//                     an in-place ncclAllGather refreshes the factor (per row the arithmetic is
//                     the one-GPU kernel's, so results are bit-identical for any P). HYBRID
//                     (the paper's SU-ALS data-parallel Theta half): X stays in per-rank slabs;
//                     per-item partial Hermitians over the local users (lambda n_v^local,
//                     parallel.hpp:408-411) are summed by ncclReduceScatter, each rank solves
//                     its item slice, and ncclAllGather refreshes Theta.
//                     Half-sweeps are asynchronous on the caller's stream: columns are
//                     validated once at creation, breakdowns are recorded on the device and
//                     raised by alsk_mp_check, so nothing blocks the host between halves.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "alskit_cuda.h"
#include "kernels.cuh"

namespace alsk {

void update_rows_sync(const DevCsr& r, const float* theta, int64_t theta_rows, int f, double lambda,
                      alsk_precision prec, int64_t batch_rows, int64_t rb, int64_t re, float* x_out, cudaStream_t s);
bool fp32_uses_tensor_cores(alsk_precision prec, int f);

namespace {

// ---- NCCL, resolved at run time -----------------------------------------------------------
struct Nccl {
    bool ok = false;
    std::string why;
    int version = 0;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl x;
        // RTLD_NOLOAD first: reuse a copy PyTorch (or the caller) already loaded
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            x.why = std::string("NCCL is not available: ") + (e ? e : "libnccl.so.2 not found");
            return x;
        }
        bool all = true;
        auto get = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) all = false;
        };
        get(x.GetUniqueId, "ncclGetUniqueId");
        get(x.CommInitRank, "ncclCommInitRank");
        get(x.CommInitAll, "ncclCommInitAll");
        get(x.CommDestroy, "ncclCommDestroy");
        get(x.CommAbort, "ncclCommAbort");
        get(x.CommGetAsyncError, "ncclCommGetAsyncError");
        get(x.AllGather, "ncclAllGather");
        get(x.ReduceScatter, "ncclReduceScatter");
        get(x.AllReduce, "ncclAllReduce");
        get(x.GroupStart, "ncclGroupStart");
        get(x.GroupEnd, "ncclGroupEnd");
        get(x.GetErrorString, "ncclGetErrorString");
        get(x.GetVersion, "ncclGetVersion");
        if (!all) {
            x.why = "NCCL library lacks required entry points";
            return x;
        }
        x.GetVersion(&x.version);
        x.ok = true;
        return x;
    }();
    return n;
}

const Nccl& need_nccl() {
    const Nccl& n = nccl();
    if (!n.ok) throw Failure(ALSK_ERR_CUDA, n.why);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress)
        throw Failure(ALSK_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

ncclDataType_t nccl_type(int dtype) {
    switch (dtype) {
        case ALSK_DTYPE_F32: return ncclFloat32;
        case ALSK_DTYPE_F64: return ncclFloat64;
        default: fail_input("unknown collective dtype " + std::to_string(dtype));
    }
}

size_t dtype_bytes(int dtype) { return dtype == ALSK_DTYPE_F64 ? 8 : 4; }

}  // namespace
}  // namespace alsk

struct alsk_comm {
    ncclComm_t nc = nullptr;
    int rank = 0, nranks = 1, device = 0;
    bool custom = false;  // collectives through caller-supplied transport (tests)
    alsk_comm_ops ops{};
};

struct alsk_workspace {
    int device = 0;
    float* scratch = nullptr;
    size_t bytes = 0;
};

using namespace alsk;

namespace {

void collective_allgather(alsk_comm* c, void* buf, int64_t chunk, int dtype, cudaStream_t s) {
    if (!c || c->nranks <= 1 || chunk <= 0) return;
    if (c->custom) {
        if (c->ops.allgather(c->ops.user, buf, chunk, dtype, s) != 0)
            throw Failure(ALSK_ERR_CUDA, "custom all-gather transport failed");
        return;
    }
    const Nccl& n = need_nccl();
    char* base = static_cast<char*>(buf);
    nccl_check(n.AllGather(base + static_cast<size_t>(c->rank) * chunk * dtype_bytes(dtype), buf,
                           static_cast<size_t>(chunk), nccl_type(dtype), c->nc, s),
               "ncclAllGather");
}

void collective_reduce_scatter(alsk_comm* c, const void* in, void* out, int64_t chunk, int dtype, cudaStream_t s) {
    if (!c || c->nranks <= 1) {
        if (chunk > 0 && in != out)
            ALSK_CUDA(cudaMemcpyAsync(out, in, static_cast<size_t>(chunk) * dtype_bytes(dtype),
                                      cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (chunk <= 0) return;
    if (c->custom) {
        if (c->ops.reduce_scatter(c->ops.user, in, out, chunk, dtype, s) != 0)
            throw Failure(ALSK_ERR_CUDA, "custom reduce-scatter transport failed");
        return;
    }
    const Nccl& n = need_nccl();
    nccl_check(n.ReduceScatter(in, out, static_cast<size_t>(chunk), nccl_type(dtype), ncclSum, c->nc, s),
               "ncclReduceScatter");
}

// Asynchronous NCCL errors (a peer died, a network fault) surface here instead of as a hang.
void comm_poll(alsk_comm* c) {
    if (!c || !c->nc) return;
    ncclResult_t e = ncclSuccess;
    nccl_check(need_nccl().CommGetAsyncError(c->nc, &e), "ncclCommGetAsyncError");
    if (e != ncclSuccess && e != ncclInProgress)
        throw Failure(ALSK_ERR_CUDA, std::string("NCCL asynchronous error: ") + nccl().GetErrorString(e));
}

// Wait for the stream while polling the communicator; abort it on an error or timeout so
// the other ranks fail instead of hanging.
void comm_wait(alsk_comm* c, cudaStream_t s, double timeout_s) {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) ALSK_CUDA(q);
        try {
            comm_poll(c);
        } catch (...) {
            if (c && c->nc) need_nccl().CommAbort(c->nc), c->nc = nullptr;
            throw;
        }
        if (timeout_s > 0 &&
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
            if (c && c->nc) need_nccl().CommAbort(c->nc), c->nc = nullptr;
            throw Failure(ALSK_ERR_CUDA, "collective timed out after " + std::to_string(timeout_s) +
                                             " s; communicator aborted");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

}  // namespace

// ---- model-parallel session ---------------------------------------------------------------
struct alsk_mp {
    alsk_comm* comm = nullptr;
    int rank = 0, world = 1;
    int mode = ALSK_MP_MODEL;
    int64_t m = 0, n = 0;
    int f = 0;
    double lambda = 0.0;
    alsk_precision prec = ALSK_PREC_FP32;
    DevCsr x, t;
    int64_t cx = 0, ct = 0;          // rows per slice (padded)
    int64_t xb = 0, xe = 0, tb = 0, te = 0;
    float* X = nullptr;              // MODEL: world*cx rows; HYBRID: the cx-row slab
    float* T = nullptr;              // world*ct rows
    void* partial = nullptr;         // HYBRID: world*ct packed rows (f32, or f64 in FP64 mode)
    void* mine = nullptr;            // HYBRID: ct reduced packed rows
    int64_t per = 0;                 // packed row length (elements)
    alsk_workspace* ws = nullptr;    // not owned when supplied by the caller
    bool own_ws = false;
    // breakdown status of the two halves, checked by alsk_mp_check
    unsigned long long* min_row[2] = {nullptr, nullptr};
    int32_t* column[2] = {nullptr, nullptr};
    double* pivot[2] = {nullptr, nullptr};
    int64_t status_base[2] = {0, 0};
    bool armed[2] = {false, false};
    // collective accounting (bytes per rank sent+received, and launches)
    int64_t coll_bytes = 0;
    int64_t coll_calls = 0;
};

namespace {

template <class T>
T* dalloc(int64_t count) {
    void* p = nullptr;
    ALSK_CUDA(cudaMalloc(&p, sizeof(T) * std::max<int64_t>(count, 1)));
    return static_cast<T*>(p);
}

DevCsr view_of(const alsk_csr* r) {
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

void free_mp(alsk_mp* S) {
    if (!S) return;
    cudaFree(S->X);
    cudaFree(S->T);
    cudaFree(S->partial);
    cudaFree(S->mine);
    for (int h = 0; h < 2; ++h) {
        cudaFree(S->min_row[h]);
        cudaFree(S->column[h]);
        cudaFree(S->pivot[h]);
    }
    if (S->own_ws && S->ws) {
        cudaFree(S->ws->scratch);
        delete S->ws;
    }
    delete S;
}

// One half-sweep's update of `rows` rows of r into out, asynchronously (FP32), or through the
// synchronous reference-order path (FP64 exact).
void half_update(alsk_mp* S, int h, const DevCsr& r, const float* theta, int64_t theta_rows, int64_t rows,
                 float* out, cudaStream_t s) {
    if (rows <= 0) return;
    if (S->prec == ALSK_PREC_FP64_EXACT) {
        update_rows_sync(r, theta, theta_rows, S->f, S->lambda, S->prec, 4096, 0, rows, out, s);
        return;
    }
    SolveStatus st{S->min_row[h], S->column[h], S->pivot[h]};
    ALSK_CUDA(cudaMemsetAsync(st.min_row, 0xff, sizeof(unsigned long long), s));
    S->armed[h] = true;
    bool done = false;
    if (fp32_uses_tensor_cores(S->prec, S->f)) {
        Scratch sc{S->ws->scratch, S->ws->bytes};
        done = update_tc(r, theta, theta_rows, S->f, static_cast<float>(S->lambda), 0, rows, out, st, s, &sc);
    }
    if (!done) {
        PhaseTimer pt(PHASE_FUSED, s);
        done = update_fused_fp32(r, theta, theta_rows, S->f, static_cast<float>(S->lambda), 0, rows, out, st, s);
    }
    if (!done) fail_input("no FP32 engine supports rank " + std::to_string(S->f));
}

void allgather_timed(alsk_mp* S, void* buf, int64_t chunk, int dtype, cudaStream_t s) {
    if (!S->comm || S->world <= 1) return;
    PhaseTimer pt(PHASE_COLLECTIVE, s);
    collective_allgather(S->comm, buf, chunk, dtype, s);
    S->coll_bytes += static_cast<int64_t>(S->world - 1) * chunk * static_cast<int64_t>(dtype_bytes(dtype));
    S->coll_calls += 1;
}

}  // namespace

extern "C" {

int alsk_comm_available(void) { return nccl().ok ? 1 : 0; }

int alsk_nccl_version(void) { return nccl().ok ? nccl().version : 0; }

alsk_status alsk_comm_unique_id(uint8_t* id_out) {
    return guard([&] {
        ncclUniqueId id;
        nccl_check(need_nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

alsk_status alsk_comm_init_rank(const uint8_t* id, int nranks, int rank, int device, alsk_comm** out) {
    return guard([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) fail_input("invalid rank " + std::to_string(rank) + " of " +
                                                                 std::to_string(nranks));
        require_device();
        auto* c = new alsk_comm();
        c->rank = rank;
        c->nranks = nranks;
        c->device = device;
        ALSK_CUDA(cudaSetDevice(device));
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
        const ncclResult_t r = need_nccl().CommInitRank(&c->nc, nranks, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

alsk_status alsk_comm_init_all(int ndev, const int* devices, alsk_comm** comms_out) {
    return guard([&] {
        if (ndev < 1) fail_input("need at least one device");
        require_device();
        int have = 0;
        ALSK_CUDA(cudaGetDeviceCount(&have));
        for (int i = 0; i < ndev; ++i)
            if (devices[i] < 0 || devices[i] >= have)
                fail_input("device " + std::to_string(devices[i]) + " does not exist (" + std::to_string(have) +
                           " visible)");
        std::vector<ncclComm_t> nc(static_cast<size_t>(ndev));
        nccl_check(need_nccl().CommInitAll(nc.data(), ndev, devices), "ncclCommInitAll");
        for (int i = 0; i < ndev; ++i) {
            auto* c = new alsk_comm();
            c->nc = nc[static_cast<size_t>(i)];
            c->rank = i;
            c->nranks = ndev;
            c->device = devices[i];
            comms_out[i] = c;
        }
    });
}

void alsk_comm_destroy(alsk_comm* c) {
    if (!c) return;
    if (c->nc && nccl().ok) nccl().CommDestroy(c->nc);
    delete c;
}

alsk_status alsk_comm_init_custom(int nranks, int rank, const alsk_comm_ops* ops, alsk_comm** out) {
    return guard([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) fail_input("invalid rank " + std::to_string(rank) + " of " +
                                                                 std::to_string(nranks));
        if (!ops || !ops->allgather || !ops->reduce_scatter) fail_input("custom transport needs both collectives");
        auto* c = new alsk_comm();
        c->rank = rank;
        c->nranks = nranks;
        cudaGetDevice(&c->device);
        c->custom = true;
        c->ops = *ops;
        *out = c;
    });
}

int alsk_comm_rank(const alsk_comm* c) { return c ? c->rank : 0; }
int alsk_comm_size(const alsk_comm* c) { return c ? c->nranks : 1; }

alsk_status alsk_comm_allgather(alsk_comm* c, void* buf, int64_t chunk_elems, int dtype, void* stream) {
    return guard([&] { collective_allgather(c, buf, chunk_elems, dtype, static_cast<cudaStream_t>(stream)); });
}

alsk_status alsk_comm_reduce_scatter(alsk_comm* c, const void* in, void* out, int64_t chunk_elems, int dtype,
                                     void* stream) {
    return guard([&] {
        collective_reduce_scatter(c, in, out, chunk_elems, dtype, static_cast<cudaStream_t>(stream));
    });
}

alsk_status alsk_comm_allreduce_max(alsk_comm* c, double* buf, int64_t count, void* stream) {
    return guard([&] {
        if (!c || c->nranks <= 1 || count <= 0) return;
        nccl_check(need_nccl().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclMax, c->nc,
                                         static_cast<cudaStream_t>(stream)),
                   "ncclAllReduce");
    });
}

alsk_status alsk_comm_wait(alsk_comm* c, void* stream, double timeout_s) {
    return guard([&] { comm_wait(c, static_cast<cudaStream_t>(stream), timeout_s); });
}

// ---- workspace ----------------------------------------------------------------------------
alsk_status alsk_workspace_create(size_t scratch_bytes, alsk_workspace** out) {
    return guard([&] {
        require_device();
        auto* w = new alsk_workspace();
        ALSK_CUDA(cudaGetDevice(&w->device));
        size_t want = std::max<size_t>(scratch_bytes, 1 << 20);
        for (;;) {  // halve on allocation failure: a smaller batch only costs more launches
            if (cudaMalloc(&w->scratch, want) == cudaSuccess) break;
            (void)cudaGetLastError();
            if (want <= (size_t(64) << 20)) {
                delete w;
                fail_capacity("cannot allocate a " + std::to_string(want) + "-byte packed-row workspace");
            }
            want /= 2;
        }
        w->bytes = want;
        *out = w;
    });
}

size_t alsk_workspace_bytes(const alsk_workspace* w) { return w ? w->bytes : 0; }

void alsk_workspace_destroy(alsk_workspace* w) {
    if (!w) return;
    cudaFree(w->scratch);
    delete w;
}

// ---- model-parallel session ---------------------------------------------------------------
alsk_status alsk_mp_create(alsk_comm* comm, int mode, int64_t m, int64_t n, int f, double lambda,
                           alsk_precision precision, const alsk_csr* x_local, const alsk_csr* t_local,
                           const float* x0, const float* theta0, alsk_workspace* ws, void* stream, alsk_mp** out) {
    return guard([&] {
        if (f < 1) fail_input("rank must be >= 1");
        if (mode != ALSK_MP_MODEL && mode != ALSK_MP_HYBRID) fail_input("unknown model-parallel mode");
        require_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        auto* S = new alsk_mp();
        try {
            S->comm = comm;
            S->rank = comm ? comm->rank : 0;
            S->world = comm ? comm->nranks : 1;
            S->mode = mode;
            S->m = m;
            S->n = n;
            S->f = f;
            S->lambda = lambda;
            S->prec = precision;
            S->x = view_of(x_local);
            S->t = view_of(t_local);
            S->cx = (m + S->world - 1) / S->world;
            S->ct = (n + S->world - 1) / S->world;
            S->xb = std::min(m, S->rank * S->cx);
            S->xe = std::min(m, (S->rank + 1) * S->cx);
            S->tb = std::min(n, S->rank * S->ct);
            S->te = std::min(n, (S->rank + 1) * S->ct);
            if (S->x.rows != S->xe - S->xb)
                fail_input("x_local has " + std::to_string(S->x.rows) + " rows; this rank's user slice has " +
                           std::to_string(S->xe - S->xb));
            if (mode == ALSK_MP_MODEL && S->t.rows != S->te - S->tb)
                fail_input("t_local has " + std::to_string(S->t.rows) + " rows; this rank's item slice has " +
                           std::to_string(S->te - S->tb));
            if (mode == ALSK_MP_HYBRID && S->t.rows != n)
                fail_input("hybrid t_local must hold every item (" + std::to_string(n) + " rows)");
            // columns validated once here, so the half-sweeps need no host round trip
            check_columns(S->x, 0, S->x.rows, 0, n, s);
            if (mode == ALSK_MP_MODEL)
                check_columns(S->t, 0, S->t.rows, 0, m, s);
            else
                check_columns(S->t, 0, S->t.rows, 0, S->xe - S->xb, s);
            const int64_t xrows = mode == ALSK_MP_MODEL ? S->cx * S->world : S->cx;
            S->X = dalloc<float>(xrows * f);
            S->T = dalloc<float>(S->ct * S->world * f);
            ALSK_CUDA(cudaMemsetAsync(S->X, 0, sizeof(float) * std::max<int64_t>(xrows * f, 1), s));
            ALSK_CUDA(cudaMemsetAsync(S->T, 0, sizeof(float) * std::max<int64_t>(S->ct * S->world * f, 1), s));
            if (x0) {
                const float* src = mode == ALSK_MP_MODEL ? x0 : x0 + S->xb * f;
                float* dst = S->X;
                const int64_t rows = mode == ALSK_MP_MODEL ? m : S->xe - S->xb;
                if (rows > 0)
                    ALSK_CUDA(cudaMemcpyAsync(dst, src, sizeof(float) * rows * f, cudaMemcpyDeviceToDevice, s));
            }
            if (theta0 && n > 0)
                ALSK_CUDA(cudaMemcpyAsync(S->T, theta0, sizeof(float) * n * f, cudaMemcpyDeviceToDevice, s));
            for (int h = 0; h < 2; ++h) {
                const int64_t rows = h == 0 ? S->cx : (mode == ALSK_MP_MODEL ? S->ct : S->ct);
                S->min_row[h] = dalloc<unsigned long long>(1);
                S->column[h] = dalloc<int32_t>(rows);
                S->pivot[h] = dalloc<double>(rows);
                ALSK_CUDA(cudaMemsetAsync(S->min_row[h], 0xff, sizeof(unsigned long long), s));
            }
            S->status_base[0] = S->xb;
            S->status_base[1] = S->tb;
            if (mode == ALSK_MP_HYBRID) {
                const bool f64 = precision == ALSK_PREC_FP64_EXACT;
                S->per = f64 ? static_cast<int64_t>(f) * (f + 1) / 2 + f : alsk_packed_stride(f);
                const size_t esz = f64 ? 8 : 4;
                ALSK_CUDA(cudaMalloc(&S->partial, esz * std::max<int64_t>(S->ct * S->world * S->per, 1)));
                if (S->world > 1)  // one rank: the partials are the reduced rows
                    ALSK_CUDA(cudaMalloc(&S->mine, esz * std::max<int64_t>(S->ct * S->per, 1)));
                ALSK_CUDA(cudaMemsetAsync(S->partial, 0, esz * std::max<int64_t>(S->ct * S->world * S->per, 1), s));
            }
            if (ws) {
                S->ws = ws;
            } else if (precision != ALSK_PREC_FP64_EXACT && fp32_uses_tensor_cores(precision, f)) {
                // packed rows for the larger half, up to 11 GiB (one batch at the Netflix shape)
                const int64_t rows = std::max(S->xe - S->xb, mode == ALSK_MP_MODEL ? S->te - S->tb : int64_t(0));
                const size_t need = sizeof(float) * static_cast<size_t>(std::max<int64_t>(rows, 1)) *
                                    static_cast<size_t>(packed_stride(f));
                alsk_workspace* w = nullptr;
                const alsk_status st = alsk_workspace_create(std::min(need, size_t(11) << 30), &w);
                if (st != ALSK_OK) throw Failure(st, alsk_last_error());
                S->ws = w;
                S->own_ws = true;
            }
            ALSK_CUDA(cudaStreamSynchronize(s));
        } catch (...) {
            free_mp(S);
            throw;
        }
        *out = S;
    });
}

alsk_status alsk_mp_half_x(alsk_mp* S, void* stream) {
    return guard([&] {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        float* out = S->mode == ALSK_MP_MODEL ? S->X + S->xb * S->f : S->X;
        half_update(S, 0, S->x, S->T, S->n, S->xe - S->xb, out, s);
        if (S->mode == ALSK_MP_MODEL) allgather_timed(S, S->X, S->cx * S->f, ALSK_DTYPE_F32, s);
    });
}

alsk_status alsk_mp_half_theta(alsk_mp* S, void* stream) {
    return guard([&] {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int f = S->f;
        if (S->mode == ALSK_MP_MODEL) {
            half_update(S, 1, S->t, S->X, S->m, S->te - S->tb, S->T + S->tb * f, s);
        } else {
            // data-parallel: partials of every item from the local users, summed across ranks
            const int64_t rows = S->te - S->tb;
            const bool f64 = S->prec == ALSK_PREC_FP64_EXACT;
            const int64_t xs = S->xe - S->xb;
            {
                PhaseTimer pt(PHASE_HERMITIAN, s);
                if (f64)
                    hermitian_materialize_d(S->t, S->X, f, S->lambda, true, 0, S->n, static_cast<double*>(S->partial),
                                            nullptr, true, s);
                else if (f <= 15)
                    partial_small_fp32(S->t, S->X, xs, f, static_cast<float>(S->lambda), 0, S->n,
                                       static_cast<float*>(S->partial), s);
                else if (!hermitian_packed_tc(S->t, S->X, xs, f, static_cast<float>(S->lambda), 0, S->n,
                                              static_cast<float*>(S->partial), s))
                    fail_input("FP32 partial Hermitians need f <= 15 or 16 <= f <= 119");
            }
            {
                PhaseTimer pt(PHASE_COLLECTIVE, s);
                const int dt = f64 ? ALSK_DTYPE_F64 : ALSK_DTYPE_F32;
                if (S->world > 1) collective_reduce_scatter(S->comm, S->partial, S->mine, S->ct * S->per, dt, s);
                if (S->world > 1) {
                    S->coll_bytes += static_cast<int64_t>(S->world - 1) * S->ct * S->per * (f64 ? 8 : 4);
                    S->coll_calls += 1;
                }
            }
            const void* red = S->world > 1 ? S->mine : S->partial;
            if (rows > 0) {
                SolveStatus st{S->min_row[1], S->column[1], S->pivot[1]};
                ALSK_CUDA(cudaMemsetAsync(st.min_row, 0xff, sizeof(unsigned long long), s));
                S->armed[1] = true;
                PhaseTimer pt(PHASE_SOLVE, s);
                if (f64) {  // round the reduced double sums to float once, then the reference-order solve
                    DevBuf A(sizeof(float) * rows * f * f, s), B(sizeof(float) * rows * f, s);
                    unpack_packed(static_cast<const double*>(red), rows, f, A.as<float>(), B.as<float>(), s);
                    solve_exact(A.as<float>(), B.as<float>(), rows, f, false, S->T + S->tb * f, st, s);
                }
                else if (f <= 15)
                    solve_small_packed(static_cast<const float*>(red), rows, f, S->T + S->tb * f, st, s);
                else
                    packed_solve(static_cast<const float*>(red), rows, f, S->T + S->tb * f, st, 0, s);
            }
        }
        allgather_timed(S, S->T, S->ct * f, ALSK_DTYPE_F32, s);
    });
}

// Synchronise the stream (polling NCCL for asynchronous errors) and raise a recorded
// Cholesky breakdown with the reference's text (solver.hpp:232-235; batch index relative to
// update_x's batch_rows = 4096 over the global row).
alsk_status alsk_mp_check(alsk_mp* S, void* stream) {
    return guard([&] {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        comm_wait(S->comm, s, 0.0);
        for (int h = 0; h < 2; ++h) {
            if (!S->armed[h]) continue;
            unsigned long long bad = ~0ull;
            ALSK_CUDA(cudaMemcpy(&bad, S->min_row[h], sizeof(bad), cudaMemcpyDeviceToHost));
            S->armed[h] = false;
            if (bad == ~0ull) continue;
            int32_t col = 0;
            double piv = 0.0;
            ALSK_CUDA(cudaMemcpy(&col, S->column[h] + bad, sizeof(col), cudaMemcpyDeviceToHost));
            ALSK_CUDA(cudaMemcpy(&piv, S->pivot[h] + bad, sizeof(piv), cudaMemcpyDeviceToHost));
            const int64_t g = S->status_base[h] + static_cast<int64_t>(bad);
            const int64_t k = g % 4096;
            set_breakdown_index(k);
            fail_numerical("cholesky breakdown at batch index " + std::to_string(k) + " (pivot " +
                           std::to_string(piv) + " at column " + std::to_string(col - 1) + ")" +
                           (h == 0 ? " in the X half" : " in the Theta half"));
        }
    });
}

alsk_status alsk_mp_factors(alsk_mp* S, float** x, int64_t* x_row_begin, float** theta) {
    return guard([&] {
        if (x) *x = S->X;
        if (x_row_begin) *x_row_begin = S->mode == ALSK_MP_MODEL ? 0 : S->xb;
        if (theta) *theta = S->T;
    });
}

void alsk_mp_slices(const alsk_mp* S, int64_t* x_begin, int64_t* x_end, int64_t* t_begin, int64_t* t_end) {
    *x_begin = S->xb;
    *x_end = S->xe;
    *t_begin = S->tb;
    *t_end = S->te;
}

void alsk_mp_collective_stats(const alsk_mp* S, int64_t* bytes, int64_t* calls) {
    *bytes = S->coll_bytes;
    *calls = S->coll_calls;
}

void alsk_mp_destroy(alsk_mp* S) {
    if (!S) return;
    cudaDeviceSynchronize();
    free_mp(S);
}

}  // extern "C"
