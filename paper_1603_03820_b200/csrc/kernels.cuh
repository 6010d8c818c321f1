// Internal launcher API between the .cu translation units of libalskit_cuda.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace alsk {

// Device view of a CsrMatrix (sparse.hpp:38-48); all pointers are device pointers.
struct DevCsr {
    int64_t rows = 0, cols = 0, col_offset = 0, nnz = 0;
    const int64_t* row_ptr = nullptr;
    const int32_t* col_idx = nullptr;
    const float* values = nullptr;
};

// Breakdown bookkeeping written by the solve kernels: first failing row (atomicMin) plus
// per-row column/pivot so the host can rebuild the reference's message
// (solver.hpp:230-235).
struct SolveStatus {
    unsigned long long* min_row;  // 1 value, init ~0ull
    int32_t* column;              // per row in launch (column+1, 0 = ok)
    double* pivot;                // per row in launch
};

// Columns of rows [rb,re) must lie in [col_lo, col_hi); throws InputError with the
// reference's message (solver.hpp:120-123) naming the first offending entry.
void check_columns(const DevCsr& r, int64_t rb, int64_t re, int64_t col_lo, int64_t col_hi,
                   cudaStream_t s);
// The same check of nonzeros [kb, ke) without host synchronisation: the first offending
// nonzero is atomicMin'ed into *first_bad (init ~0); fail_bad_column raises its message.
void check_columns_async(const DevCsr& r, int64_t kb, int64_t ke, int64_t col_lo, int64_t col_hi,
                         unsigned long long* first_bad, cudaStream_t s);
[[noreturn]] void fail_bad_column(const DevCsr& r, unsigned long long entry, int64_t col_lo, int64_t col_hi,
                                  cudaStream_t s);

// Materialised assembly (A full mirrored f*f floats + B f floats per row), rows [rb,re).
// acc_double: reference-order double accumulation (bit-exact with assemble_mo_rows<double>).
void hermitian_materialize(const DevCsr& r, const float* theta, int f, double lambda,
                           bool acc_double, int64_t rb, int64_t re, float* A, float* B,
                           cudaStream_t s);

// Double-output variant (BatchD, parallel.hpp:174-202): partial Hermitians kept in
// double until the cross-worker reduction. packed=false: full mirrored A + B per row;
// packed=true: lower-packed A then B, f(f+1)/2+f doubles per row, into A only.
void hermitian_materialize_d(const DevCsr& r, const float* theta, int f, double lambda, bool acc_double,
                             int64_t rb, int64_t re, double* A, double* B, bool packed, cudaStream_t s);

// Reference-order double Cholesky of float systems (batch_solve_into, solver.hpp:204-262).
void solve_exact(const float* A, const float* B, int64_t count, int f, bool zero_row_policy,
                 float* X, const SolveStatus& st, cudaStream_t s);

// FP32 fused assembly + in-register Cholesky for rows [rb,re) -> X rows (x_out[(u-rb)*f]).
// Returns false if f is outside the fused kernel's range (caller falls back to the
// materialised FP32 path).
bool update_fused_fp32(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda,
                       int64_t rb, int64_t re, float* x_out, const SolveStatus& st, cudaStream_t s);

// FP32 register-blocked assembly only (materialised output) — the hermitian timed alone.
bool partial_small_fp32(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
                        int64_t re, float* out, cudaStream_t s);
bool solve_small_packed(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, cudaStream_t s);
bool hermitian_fused_fp32(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda,
                          int64_t rb, int64_t re, float* A, float* B, cudaStream_t s);

// Tensor-core (tcgen05 kind::tf32, two-term split) Hermitian assembly, one persistent CTA per
// SM (tc_update.cu), followed by the batched TMEM Cholesky (tc_solve.cu).
// tc_supported: 16 <= f <= 119.
bool tc_supported(int f);
// Caller-owned packed-row scratch (a workspace): used stream-ordered, without locking or
// host synchronisation; nullptr selects the per-device default scratch.
struct Scratch {
    float* ptr = nullptr;
    size_t bytes = 0;
};
constexpr int kMaxDevices = 64;
bool update_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
               int64_t re, float* x_out, const SolveStatus& st, cudaStream_t s, const Scratch* scratch = nullptr);
// Packed (panel-blocked) rows [rb, re) of A_u + lambda n_u I and B_u on the tensor cores into
// out_packed (packed_stride(f) floats per row): the data-parallel split's FP32 partials.
bool hermitian_packed_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
                         int64_t re, float* out_packed, cudaStream_t s);
bool hermitian_tc(const DevCsr& r, const float* theta, int64_t theta_rows, int f, float lambda, int64_t rb,
                  int64_t re, float* A, float* B, cudaStream_t s);

// Packed Hermitian rows (panel-blocked): the lower triangle of the augmented matrix
// [A (lambda n_u included) ; b^T] stored by 8-column block b = 0 .. ceil(f/8)-1 as rows
// 8b .. f (row f = b^T) of 8 floats each (columns 8b .. 8b+7; cells above the diagonal or at
// columns >= f hold 0). A lane owning matrix row i reads its 8 entries of block b as two
// 16-byte vectors at pb_block(f, b) + 8 (i - 8b); every row is 32-byte aligned.
__host__ __device__ inline int64_t pb_block(int f, int b) {
    return 8 * (static_cast<int64_t>(b) * (f + 1) - 4 * static_cast<int64_t>(b) * (b - 1));
}
__host__ __device__ inline int64_t packed_stride(int f) { return pb_block(f, (f + 7) / 8); }
// element (i, j), j <= i (or i == f, j < f) of a packed row
__host__ __device__ inline int64_t pb_index(int f, int i, int j) {
    return pb_block(f, j >> 3) + 8 * static_cast<int64_t>(i - (j & ~7)) + (j & 7);
}

// Batched FP32 solves of packed rows (status rows reported at status_off + i):
//  packed_solve       - tensor-core Cholesky, matrix resident in TMEM (tc_solve.cu);
//  packed_solve_tiles - CUDA-core 8x8 register-tile Cholesky (chol_solve.cu).
bool packed_solve(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                  cudaStream_t s);
bool packed_solve_tiles(const float* packed, int64_t count, int f, float* x, const SolveStatus& st,
                        int64_t status_off, cudaStream_t s);
//  warp_solve         - one system per warp in shared memory, mma.sync Schur updates
//                       (warp_solve.cu; the default); false if f is outside 1..128.
bool warp_solve(const float* packed, int64_t count, int f, float* x, const SolveStatus& st, int64_t status_off,
                cudaStream_t s);


// Evaluation (solver.hpp:358-406). Deterministic two-level double reductions.
double loss_device(const DevCsr& r, const int64_t* col_nnz, const float* x, const float* theta,
                   int f, double lambda, cudaStream_t s);
double rmse_device(const int64_t* rows, const int64_t* cols, const float* values, int64_t count,
                   const float* x, int64_t x_rows, const float* theta, int64_t theta_rows, int f,
                   cudaStream_t s);
void column_counts(const DevCsr& r, int64_t* col_nnz, cudaStream_t s);

// Sparse index plumbing (sparse.hpp:132-314), bit-exact.
void csr_to_csc_device(const DevCsr& a, int64_t* col_ptr, int32_t* row_idx, float* values,
                       cudaStream_t s);
void csr_from_triplets_device(int64_t m, int64_t n, const int64_t* rows, const int64_t* cols,
                              const float* vals, int64_t count, int64_t* row_ptr, int32_t* col_idx,
                              float* values, cudaStream_t s);

template <class T>
void exclusive_scan_ptr_i64(const T* in, int64_t n, int64_t* out, cudaStream_t s);

// CSR invariant check after a raw upload (validate.cu): first failing row or -1; syncs s
int64_t csr_first_bad_row(const int64_t* rp, const int32_t* ci, int64_t rows, int64_t cols, int64_t nnz,
                          cudaStream_t s);

// split_train_test on the device (split.cu; dataio.hpp:251-290)
void holdout_mask_host(int64_t nnz, int64_t k, uint64_t seed, std::vector<uint32_t>& mask);
int64_t split_with_mask_device(const DevCsr& r, const uint32_t* dmask, int64_t bit_offset, int64_t row_base,
                               int64_t* train_row_ptr, int32_t* train_col_idx, float* train_values,
                               alsk_triplet* test, cudaStream_t s);

// Device synthetic generator (synth.cu), bit-identical to alsk_synth_csr: rows [rb, re)
// with row pointers rebased to 0. Row degrees are at most kSynthMaxDegree.
constexpr int kSynthMaxDegree = 1024;
int64_t synth_row_start(int64_t nnz, int64_t m, int64_t u);
void synth_rows_device(int64_t m, int64_t n, int64_t nnz, uint64_t seed, int64_t rb, int64_t re, int64_t* row_ptr,
                       int32_t* col_idx, float* values, cudaStream_t s);
// Entries with lo <= col < hi of every row, order kept, columns rebased to col - lo; with
// col_idx_out == NULL only row_ptr_out (rows+1) and the returned total are produced.
int64_t filter_columns_device(const DevCsr& r, int64_t lo, int64_t hi, int64_t* row_ptr_out, int32_t* col_idx_out,
                              float* values_out, cudaStream_t s);
int64_t split_holdout_count(int64_t nnz, double holdout);
void split_train_test_device(const DevCsr& r, double holdout, uint64_t seed, int64_t* train_row_ptr,
                             int32_t* train_col_idx, float* train_values, alsk_triplet* test, cudaStream_t s);

// Grid partition state on the device (sparse.hpp:71-84): cuts on the host, per-row split
// offsets and per-block row pointers on the device.
struct GridDevice {
    int p = 1, q = 1;
    std::vector<int64_t> row_cuts, col_cuts, block_nnz;
    DevBuf offs;
    std::vector<DevBuf> block_row_ptr;  // j*p+i
};
GridDevice grid_partition_device(const DevCsr& r, int p, int q, cudaStream_t s);
void grid_fill_block(const DevCsr& r, const GridDevice& g, int i, int j, int32_t* bci, float* bv,
                     cudaStream_t s);

// Reduction plan (parallel.hpp:84-124): per slice, phase-1 and phase-2 transfers
// (x = src, y = dst) sorted by (dst, src).
struct ReduceSchedule {
    int p = 1;
    std::vector<std::vector<int2>> phase1, phase2;
};
ReduceSchedule build_reduce_schedule(int p, const int32_t* group_of, bool two_phase);
std::vector<int64_t> slice_cuts(int64_t count, int p);
template <class In>
void reduce_slices(const std::vector<const In*>& parts_a, const std::vector<const In*>& parts_b, int64_t count,
                   int f, const ReduceSchedule& sc, const std::vector<float*>& out_a,
                   const std::vector<float*>& out_b, cudaStream_t s);
void unpack_packed(const double* packed, int64_t count, int f, float* A, float* B, cudaStream_t s);

}  // namespace alsk
