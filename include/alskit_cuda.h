/*
 * alskit_cuda.h — C ABI of the B200-native ALS hot path (libalskit_cuda.so).
 *
 * This is the drop-in boundary: plain C types, plain pointers and sizes, no torch and
 * no C++ types. Every entry point replaces one function of the reference's header-only
 * C++ API in /root/reference/proj/include/alskit (cited per entry as file:line). The
 * C++ drop-in headers in include/alskit/*.hpp re-expose these under the reference's own
 * names and signatures; ctypes/cffi bindings call them directly.
 *
 * Conventions
 *  - Every function returns an alsk_status. On failure a thread-local message is
 *    available from alsk_last_error(); the message text follows the reference's
 *    exception text (tests match substrings such as "cholesky breakdown at batch index 1").
 *  - Functions without the `_dev` suffix take HOST pointers and are synchronous
 *    (H2D -> kernels -> D2H), exactly like the synchronous reference API.
 *  - `_dev` functions take DEVICE pointers and a cudaStream_t (passed as void*; NULL =
 *    legacy default stream). They enqueue work and synchronise only where a status must
 *    be read back (input validation, Cholesky breakdown).
 *  - Types follow common.hpp:14-20: index_t = int32_t, offset_t = int64_t, real_t = float.
 *  - There is no CPU fallback: with no usable CUDA device every compute entry point
 *    returns ALSK_ERR_CUDA.
 */
#ifndef ALSKIT_CUDA_H_
#define ALSKIT_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error categories mirror alskit::Error::Category (common.hpp:24-64); the CLI exit codes
 * for input/capacity/numerical/io are 2/3/4/5 (tools/alskit.cpp:23-31). */
typedef enum alsk_status {
    ALSK_OK = 0,
    ALSK_ERR_INPUT = 1,     /* InputError     */
    ALSK_ERR_CAPACITY = 2,  /* CapacityError  */
    ALSK_ERR_NUMERICAL = 3, /* NumericalError */
    ALSK_ERR_IO = 4,        /* IoError        */
    ALSK_ERR_CUDA = 5       /* device / driver failure (no reference counterpart) */
} alsk_status;

/* BreakdownPolicy (solver.hpp:72). */
typedef enum alsk_breakdown { ALSK_BREAKDOWN_FAIL = 0, ALSK_BREAKDOWN_ZERO_ROW = 1 } alsk_breakdown;

/* Arithmetic of the Hermitian assembly + solve.
 *  FP64_EXACT: reference order, double accumulators, double Cholesky with separately
 *              rounded multiply/subtract — bit-identical to the reference's default
 *              accumulate_double=true path (solver.hpp:99-157, 204-262).
 *  FP32:       FP32-level arithmetic, tolerance-checked (normwise <= 1e-3 per
 *              half-sweep). The engine is chosen by alsk_set_fp32_engine: by default the
 *              tensor-core kernel (TF32X2 below) where 16 <= f <= 119, else the
 *              register-blocked FFMA kernel; both fuse the in-register Cholesky.
 *  TF32X2:     Hermitian and bias on tcgen05 tensor cores with the two-term TF32 split
 *              x = hi + lo (A = Hi^T Hi + Hi^T Lo + (Hi^T Lo)^T), FP32 accumulation in TMEM,
 *              FP32 Cholesky; falls back to the FFMA kernel outside 16 <= f <= 119. */
typedef enum alsk_precision {
    ALSK_PREC_FP64_EXACT = 0,
    ALSK_PREC_FP32 = 1,
    ALSK_PREC_TF32X2 = 2
} alsk_precision;

/* CsrMatrix (sparse.hpp:38-48). Pointers are host or device per function family. */
typedef struct alsk_csr {
    int64_t rows;
    int64_t cols;
    int64_t col_offset; /* first global column of a grid block (sparse.hpp:34-37) */
    int64_t nnz;
    const int64_t* row_ptr; /* rows+1 */
    const int32_t* col_idx; /* nnz, GLOBAL column ids */
    const float* values;    /* nnz */
} alsk_csr;

/* Triplet (sparse.hpp:17-23): {int64 row, int64 col, float value}, 24 bytes with padding. */
typedef struct alsk_triplet {
    int64_t row;
    int64_t col;
    float value;
} alsk_triplet;

/* SolverConfig (solver.hpp:61-69). `bin` and `threads` are accepted for API parity; the
 * result never depends on them (solver.hpp:88-91). accumulate_double selects
 * ALSK_PREC_FP64_EXACT (1) or ALSK_PREC_FP32 (0). */
typedef struct alsk_solver_config {
    int f;
    double lambda;
    int bin;
    int64_t batch_rows;
    int accumulate_double;
    int threads;
    uint64_t seed;
} alsk_solver_config;

/* ---- diagnostics ------------------------------------------------------------------- */
const char* alsk_last_error(void);
/* Batch index of the last Cholesky breakdown reported as ALSK_ERR_NUMERICAL (-1 if none). */
int64_t alsk_last_breakdown_index(void);
/* 1 when a CUDA device is usable in this process, else 0. */
int alsk_device_available(void);
/* Number of kernels this library has launched in this process (bench evidence). */
uint64_t alsk_kernel_launch_count(void);
const char* alsk_build_info(void);
/* Kernel-only timing of the fused half-sweep kernel: between begin and end, every fused
 * launch is bracketed by CUDA events on its stream; end returns the summed milliseconds
 * and the number of launches timed. */
void alsk_profile_begin(void);
/* Engine behind ALSK_PREC_FP32 (process-wide): 0 = auto (tensor cores where 16 <= f <= 119),
 * 1 = CUDA-core FFMA kernel, 2 = tensor cores. */
void alsk_set_fp32_engine(int engine);
int alsk_fp32_engine(void);
void alsk_profile_end(double* total_ms, uint64_t* launches);
/* Per-phase kernel time of the tensor-core engine since alsk_profile_begin: the
 * tensor-core Hermitian launches and the batched Cholesky launches. */
void alsk_profile_phases(double* herm_ms, uint64_t* herm_launches, double* solve_ms, uint64_t* solve_launches);
/* Any phase: 0 Hermitian, 1 batched solve, 2 fused half-sweep kernel, 3 collectives
 * (all-gather / reduce-scatter of a model-parallel session). Events are resolved here, so
 * profiling adds no host synchronisation to the timed calls. */
void alsk_profile_phase(int phase, double* ms, uint64_t* launches);
/* Measured FP32 FFMA throughput of the current device in TFLOP/s (roofline denominator). */
double alsk_fp32_peak_probe(void);
/* TFLOP/s of the Hermitian register-blocked inner loop alone (operands resident in shared
 * memory, no gather, no barriers) at `ctas_per_sm` 96-thread CTAs per SM. */
double alsk_herm_loop_probe(int ctas_per_sm, int variant);

/* ---- host-buffer drop-in entry points (synchronous) ------------------------------- */

/* get_hermitian_mo_into (solver.hpp:292-304): rows [row_begin,row_end) of r against
 * theta (theta_rows x f) into a_out[(row_end-row_begin)*f*f], b_out[(..)*f].
 * Also serves local_hermitian (parallel.hpp:412-421) when r->col_offset != 0. */
alsk_status alsk_get_hermitian_mo_into(const alsk_csr* r, const float* theta, int64_t theta_rows,
                                       int f, const alsk_solver_config* cfg, int64_t row_begin,
                                       int64_t row_end, float* a_out, float* b_out);

/* get_hermitian_base (solver.hpp:277-287): full batch, untiled reference entry point. */
alsk_status alsk_get_hermitian_base(const alsk_csr* r, const float* theta, int64_t theta_rows,
                                    int f, double lambda, int accumulate_double, float* a_out,
                                    float* b_out);

/* local_hermitian (parallel.hpp:412-421): no full-shape check, column range from
 * r->col_offset .. col_offset+theta_rows. */
alsk_status alsk_local_hermitian(const alsk_csr* block, const float* theta_part,
                                 int64_t theta_rows, int f, const alsk_solver_config* cfg,
                                 float* a_out, float* b_out);

/* batch_solve (solver.hpp:320-325 -> batch_solve_into 204-262): double Cholesky in the
 * reference's operation order (bit-identical). x_out[count*f]. */
alsk_status alsk_batch_solve(const float* a, const float* b, int64_t count, int f,
                             alsk_breakdown policy, float* x_out);

/* update_x (solver.hpp:330-345). precision from cfg->accumulate_double. x_out[rows*f]. */
alsk_status alsk_update_x(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                          const alsk_solver_config* cfg, float* x_out);

/* update_theta (solver.hpp:349-352): CSC arrays (col_ptr, row_idx, values) of R
 * (rows x cols) reinterpreted as the CSR of R^T without the copy transpose_of makes. */
alsk_status alsk_update_theta(int64_t rows, int64_t cols, int64_t nnz, const int64_t* col_ptr,
                              const int32_t* row_idx, const float* values, const float* x,
                              int64_t x_rows, int f, const alsk_solver_config* cfg,
                              float* theta_out);

/* loss (solver.hpp:358-390) and rmse (solver.hpp:393-406); double accumulation. */
alsk_status alsk_loss(const alsk_csr* r, const float* x, int64_t x_rows, const float* theta,
                      int64_t theta_rows, int f, double lambda, double* out);
alsk_status alsk_rmse(const alsk_triplet* test, int64_t count, const float* x, int64_t x_rows,
                      const float* theta, int64_t theta_rows, int f, double* out);

/* csr_to_csc (sparse.hpp:185-207) / csc_to_csr (209-231): stable transposes, bit-exact.
 * Outputs are caller-allocated: col_ptr_out[cols+1], row_idx_out[nnz], values_out[nnz]. */
alsk_status alsk_csr_to_csc(const alsk_csr* a, int64_t* col_ptr_out, int32_t* row_idx_out,
                            float* values_out);
alsk_status alsk_csc_to_csr(int64_t rows, int64_t cols, int64_t nnz, const int64_t* col_ptr,
                            const int32_t* row_idx, const float* values, int64_t* row_ptr_out,
                            int32_t* col_idx_out, float* values_out);

/* csr_from_triplets (sparse.hpp:132-170): range check, (row,col) sort, duplicate check.
 * row_ptr_out[m+1], col_idx_out[count], values_out[count]. */
alsk_status alsk_csr_from_triplets(int64_t m, int64_t n, const alsk_triplet* t, int64_t count,
                                   int64_t* row_ptr_out, int32_t* col_idx_out, float* values_out);

/* grid_partition (sparse.hpp:250-314), two calls:
 *  1) alsk_grid_partition_counts: row_cuts_out[q+1], col_cuts_out[p+1], block_nnz_out[p*q]
 *     (block (i,j) at j*p+i) so the caller can size the blocks;
 *  2) alsk_grid_partition_fill: block_row_ptr[b] (local_rows_j+1), block_col_idx[b],
 *     block_values[b] — arrays of p*q caller-allocated host pointers. */
alsk_status alsk_grid_partition_counts(const alsk_csr* r, int p, int q, int64_t* row_cuts_out,
                                       int64_t* col_cuts_out, int64_t* block_nnz_out);
alsk_status alsk_grid_partition_fill(const alsk_csr* r, int p, int q, int64_t* const* block_row_ptr,
                                     int32_t* const* block_col_idx, float* const* block_values);

/* parallel_reduce (parallel.hpp:474-477 -> reduce_batches 206-280) for the one-phase and
 * two-phase schedules: slice i of the elementwise double sum of p partial batches
 * (each count*(f*f) A + count*f B floats). parts_a/parts_b: p host pointers; the result
 * for slice i goes to out_a[i]/out_b[i] sized per slice_cuts(count,p) (parallel.hpp:160-168).
 * Summation order: own partial first, then sources ascending — the reference's order for
 * the one-phase schedule; the two-phase schedule sums within groups first (same values up
 * to double reassociation, rounded once to float). */
alsk_status alsk_parallel_reduce(const float* const* parts_a, const float* const* parts_b, int p,
                                 int64_t count, int f, const int32_t* group_of, int two_phase,
                                 float* const* out_a, float* const* out_b);

/* su_als_update_x (parallel.hpp:487-583): grid of p x q blocks (block (i,j) at j*p+i,
 * host CSR with col_offset), theta partitions (partition i has col_cuts[i+1]-col_cuts[i]
 * rows), reduce schedule from group_of/two_phase as in alsk_parallel_reduce. The capacity
 * check (parallel.hpp:512-519) is the host planner's job. With accumulate_double the
 * partial Hermitians stay double until the reduction and are rounded to float once.
 * x_out[row_cuts[q]*f]. */
alsk_status alsk_su_als_update_x(const alsk_csr* blocks, int p, int q, const int64_t* row_cuts,
                                 const int64_t* col_cuts, const float* const* theta_parts, int f,
                                 const alsk_solver_config* cfg, const int32_t* group_of,
                                 int two_phase, float* x_out);

/* ---- device-resident entry points (session / multi-GPU path) ---------------------- */

/* Fused update of rows [row_begin,row_end) of r (device CSR) against theta (device),
 * writing x rows into x_out + (row_begin-x_row_base)*f. The half-sweep of update_x.
 * Returns ALSK_ERR_NUMERICAL on breakdown (after a stream sync of one 16-byte status). */
alsk_status alsk_dev_update(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                            double lambda, alsk_precision precision, int64_t batch_rows,
                            int64_t row_begin, int64_t row_end, float* x_out, void* stream);

/* Partial Hermitian of rows [row_begin,row_end) in packed-lower double form for the
 * data-parallel split: out[(row-row_begin)*(f*(f+1)/2 + f)] with lambda*n_local on the
 * diagonal (parallel.hpp:408-411). */
alsk_status alsk_dev_partial_hermitian(const alsk_csr* r, const float* theta, int64_t theta_rows,
                                       int f, double lambda, int64_t row_begin, int64_t row_end,
                                       double* out_packed, void* stream);
/* Solve packed double systems (count of them) into x_out[count*f]. */
alsk_status alsk_dev_solve_packed(const double* packed, int64_t count, int f, float* x_out,
                                  void* stream);

/* FP32 variant of the data-parallel split (replaces local_hermitian + the double
 * reduce_batches, parallel.hpp:412-421, 206-280, at the FP32 tolerance): packed rows of
 * A_u + lambda n_u I and B_u for rows [row_begin,row_end) from the tensor cores
 * (16 <= f <= 119), panel-blocked, alsk_packed_stride(f) floats per row (layout in
 * INTEGRATION.md); partials of several slabs add entry-wise (lambda uses the local n_u,
 * so the sum carries lambda n_u of the whole row). */
int64_t alsk_packed_stride(int f);
alsk_status alsk_dev_partial_hermitian_f32(const alsk_csr* r, const float* theta, int64_t theta_rows,
                                           int f, double lambda, int64_t row_begin, int64_t row_end,
                                           float* out_packed, void* stream);
/* Solve packed FP32 systems (the layout above) with the batched TMEM Cholesky into
 * x_out[count*f]; a non-positive pivot raises NumericalError naming the row. */
alsk_status alsk_dev_solve_packed_f32(const float* packed, int64_t count, int f, float* x_out,
                                      void* stream);

/* Binary ratings cache (replaces save_binary_cache / load_binary_cache, dataio.hpp:116-163):
 * header of five little-endian u64 (magic "ALSKCACH", version 1, rows, cols, nnz), then
 * row_ptr int64[rows+1], col_idx int32[nnz], values f32[nnz]. Loads validate the CSR like
 * the reference (IoError "<path>: corrupt cache (<validate message>)"). alsk_dev_load_cache
 * streams the file into device buffers through pinned staging (read overlapped with the
 * upload). */
alsk_status alsk_cache_header(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz);
alsk_status alsk_save_cache(const alsk_csr* r, const char* path);
/* cap_rows / cap_nnz: the capacity of the caller's buffers (row_ptr holds cap_rows+1); a file
 * whose header grew since the caller read it is an IoError, never an overrun. */
alsk_status alsk_load_cache(const char* path, int64_t cap_rows, int64_t cap_nnz, int64_t* row_ptr, int32_t* col_idx,
                            float* values);
alsk_status alsk_dev_load_cache(const char* path, int64_t cap_rows, int64_t cap_nnz, int64_t* row_ptr,
                                int32_t* col_idx, float* values, void* stream);

/* Factor checkpoints (replace write_checkpoint / read_checkpoint / restore_latest /
 * CheckpointWriter, dataio.hpp:546-786): same file format (56-byte header: magic "ALSKCPKT",
 * version, iteration, which (0 = x, 1 = theta), rows, f, digest; then rows*f f32), same
 * ckpt_%06d_{x,theta}.bin names, atomic temp+rename, same IoError texts. */
alsk_status alsk_checkpoint_write(const char* dir, int iteration, int which, int64_t rows, int f, uint64_t digest,
                                  const float* entries);
alsk_status alsk_checkpoint_path(const char* dir, int iteration, int which, char* out, size_t cap);
alsk_status alsk_checkpoint_header(const char* path, int* iteration, int* which, int64_t* rows, int* f,
                                   uint64_t* digest);
alsk_status alsk_checkpoint_read(const char* path, int64_t cap_entries, float* entries);
alsk_status alsk_dev_checkpoint_read(const char* path, int64_t cap_entries, float* d_entries, void* stream);
/* which = -1: newest of either kind (theta outranks x at the same iteration); 0 / 1: that
 * kind only. *found = 0 when the directory holds none. */
alsk_status alsk_checkpoint_latest(const char* dir, int which, char* out, size_t cap, int* found);
/* Background writer: submit_device orders a D2H copy of the factor after `stream` on a
 * private copy stream into pinned memory and returns; one worker thread writes the file.
 * At most one snapshot in flight (submit waits for the previous write); write errors are
 * sticky and returned by the next submit or flush. */
alsk_status alsk_ckpt_writer_create(const char* dir, void** writer);
alsk_status alsk_ckpt_writer_submit_device(void* writer, int iteration, int which, int64_t rows, int f,
                                           uint64_t digest, const float* d_factor, void* stream);
alsk_status alsk_ckpt_writer_submit_host(void* writer, int iteration, int which, int64_t rows, int f,
                                         uint64_t digest, const float* entries);
alsk_status alsk_ckpt_writer_flush(void* writer);
void alsk_ckpt_writer_destroy(void* writer);

/* Persisted grids (persist_grid / load_grid_meta / load_block, dataio.hpp:352-439): a
 * grid.meta text file plus block_<i>_<j>.bin binary caches (alsk_save_cache per block). */
alsk_status alsk_persist_grid_meta(const char* dir, int p, int q, int64_t rows, int64_t cols, const int64_t* row_cuts,
                                   const int64_t* col_cuts);
alsk_status alsk_block_path(const char* dir, int i, int j, char* out, size_t cap);
/* row_cuts[q+1] / col_cuts[p+1] may be NULL (first call: sizes only). */
alsk_status alsk_grid_meta(const char* dir, int* p, int* q, int64_t* rows, int64_t* cols, int64_t* row_cuts,
                           int64_t* col_cuts);
/* Out-of-core block stream (BlockStream, dataio.hpp:447-524) into HBM: a loader thread
 * reads, validates and uploads blocks in the given order (pairs i0,j0,i1,j1,...) two ahead.
 * next() fills *out with device pointers (col_offset restored from grid.meta) and orders
 * `stream` after the upload; they stay valid until the following next() call, whose
 * position on `stream` gates the slot's reuse. *has_block = 0 once the plan is exhausted;
 * a loader error ("block (i, j): ...") surfaces on the next() that would return it. */
alsk_status alsk_block_stream_open(const char* dir, const int* order_ij, int count, void** stream_out);
/* Out-of-core half-sweep (the scale-up of su_als_update_x, parallel.hpp:487-583, for
 * matrices beyond HBM): one update of all rows of the grid persisted at
 * grid_dir, against `factor` (device, factor_rows = the grid's columns), into x_out (device,
 * grid rows x f) on `stream`. Blocks stream into HBM (alsk_block_stream_*) while the previous
 * one computes; per row partition the block partials are reduced slice by slice and solved.
 * accumulate_double: double partials, the one-phase reduce order, the reference-order solve
 * -- bit-identical to su_als_update_x on the same grid; else the FP32 tensor-core path
 * (16 <= f <= 119) or float partials. Errors as su_als_update_x: a block column outside its
 * slab (InputError "column v outside partition [lo, hi)"), a breakdown (NumericalError). */
alsk_status alsk_ooc_update(const char* grid_dir, const float* factor, int64_t factor_rows, int f,
                            const alsk_solver_config* cfg, float* x_out, void* stream);
alsk_status alsk_block_stream_next(void* block_stream, void* stream, int* has_block, int* i, int* j, alsk_csr* out);
void alsk_block_stream_close(void* block_stream);
/* Utility: synchronous device-to-host copy on `stream`. */
alsk_status alsk_dev_to_host(void* dst, const void* src, size_t bytes, void* stream);
alsk_status alsk_host_to_dev(void* dst, const void* src, size_t bytes, void* stream);

/* Device loss/rmse; result written to *out (host) after a stream sync. */
alsk_status alsk_dev_loss(const alsk_csr* r, const int64_t* col_nnz, const float* x,
                          const float* theta, int64_t theta_rows, int f, double lambda,
                          double* out, void* stream);
alsk_status alsk_dev_rmse(const int64_t* rows, const int64_t* cols, const float* values,
                          int64_t count, const float* x, int64_t x_rows, const float* theta,
                          int64_t theta_rows, int f, double* out, void* stream);

/* Device stable transpose: CSR (device) -> CSC (device, caller-allocated). */
alsk_status alsk_dev_csr_to_csc(const alsk_csr* a, int64_t* col_ptr_out, int32_t* row_idx_out,
                                float* values_out, void* stream);

/* Hermitian FP32 kernel alone (materialised A/B, device) — used to time the assembly
 * against the FP32 roofline separately from the solve. */
alsk_status alsk_dev_hermitian(const alsk_csr* r, const float* theta, int64_t theta_rows, int f,
                               double lambda, alsk_precision precision, int64_t row_begin,
                               int64_t row_end, float* a_out, float* b_out, void* stream);

/* ---- device-resident session (als_train / train_run caller) ---- */
/* R (CSR) and R^T (the CSC arrays of R, read as the CSR of R^T) are uploaded once; X and
 * Theta stay in HBM across half-sweeps. Host copies are made only on request. */
typedef struct alsk_session alsk_session;
alsk_status alsk_session_create(const alsk_csr* r, const int64_t* col_ptr, const int32_t* row_idx,
                                const float* csc_values, const alsk_triplet* test, int64_t test_count,
                                int f, double lambda, alsk_precision precision, int64_t batch_rows,
                                const float* x0, const float* theta0, alsk_session** out);
alsk_status alsk_session_half_x(alsk_session* s);      /* X = update_x(R, Theta)   */
alsk_status alsk_session_half_theta(alsk_session* s);  /* Theta = update_x(R^T, X) */
alsk_status alsk_session_loss(alsk_session* s, double* out);
alsk_status alsk_session_rmse(alsk_session* s, double* out); /* NaN when there is no test set */
alsk_status alsk_session_factors(alsk_session* s, float* x_out, float* theta_out);
/* The session's device factors and its stream (for device-side snapshots). */
alsk_status alsk_session_device(alsk_session* s, float** x, float** theta, void** stream);
void alsk_session_destroy(alsk_session* s);

/* ---- host data helpers (dataio/factor restatements used by the drivers) ------------ */

/* random_factor (factor.hpp:49-54) and mix_seed (common.hpp:70-75), bit-exact. */
void alsk_random_factor(int64_t rows, int f, uint64_t seed, float* out);
uint64_t alsk_mix_seed(uint64_t seed, uint64_t salt);

/* split_train_test (dataio.hpp:251-290), bit-exact: two calls — the first returns the
 * held-out count k and train nnz; the second fills caller buffers. */
alsk_status alsk_split_train_test(const alsk_csr* r, double holdout, uint64_t seed,
                                  int64_t* k_out, int64_t* train_row_ptr, int32_t* train_col_idx,
                                  float* train_values, alsk_triplet* test_out);

/* The same split with the CSR on the device (all pointers device memory): the held-out
 * positions come from the same host Fisher-Yates (bit-exact), the compaction into the train
 * CSR and the row-major test triplets runs in HBM. Two calls as above (train_row_ptr NULL:
 * only k). */
alsk_status alsk_dev_split_train_test(const alsk_csr* r, double holdout, uint64_t seed, int64_t* k_out,
                                      int64_t* train_row_ptr, int32_t* train_col_idx, float* train_values,
                                      alsk_triplet* test_out, void* stream);

/* Deterministic synthetic generator: row degree
 * floor(nnz(u+1)/m)-floor(nnz u/m), columns by Floyd sampling from mt19937_64(mix_seed(seed,u)),
 * values from a planted rank-10 model + U[-0.5,0.5) noise. Row-parallel on host threads.
 * Fills a CSR with exactly nnz entries. */
alsk_status alsk_synth_csr(int64_t m, int64_t n, int64_t nnz, uint64_t seed, int threads,
                           int64_t* row_ptr, int32_t* col_idx, float* values);

/* ---- per-rank synthetic data (the bench's multi-GPU setup) ------------------------- */
/* Rows [row_begin,row_end) of alsk_synth_csr's matrix generated in HBM, bit-identical to the
 * host generator; row_ptr (row_end-row_begin+1) starts at 0. Row degrees must be <= 1024. */
alsk_status alsk_dev_synth_rows(int64_t m, int64_t n, int64_t nnz, uint64_t seed, int64_t row_begin, int64_t row_end,
                                int64_t* row_ptr, int32_t* col_idx, float* values, void* stream);
/* Global offset of row u in that matrix: floor(nnz * u / m). */
int64_t alsk_synth_row_start(int64_t m, int64_t nnz, int64_t u);
/* The held-out positions of split_train_test (dataio.hpp:251-290; same Fisher-Yates draws)
 * as a bitmask of ceil(nnz/32) words (bit k set = entry k held out); mask_out NULL: only
 * *k_out. */
alsk_status alsk_holdout_mask(int64_t nnz, double holdout, uint64_t seed, uint32_t* mask_out, int64_t* k_out);
/* Set bits of a host mask in [bit_begin, bit_end). */
int64_t alsk_mask_count(const uint32_t* mask, int64_t bit_begin, int64_t bit_end);
/* Split a device CSR (or a row chunk of a larger one) by a device bitmask: entry k is held
 * out when bit (k - row_ptr[0] + bit_offset) is set. Train arrays sized for r->nnz, test
 * triplets for the held count (row ids + row_base); *train_nnz set on return. */
alsk_status alsk_dev_split_mask(const alsk_csr* r, const uint32_t* d_mask, int64_t bit_offset, int64_t row_base,
                                int64_t* train_row_ptr, int32_t* train_col_idx, float* train_values,
                                alsk_triplet* test_out, int64_t* train_nnz, void* stream);
/* Entries with col_begin <= col < col_end of every row, order kept, columns rebased to
 * col - col_begin (a model-parallel rank's item slice). col_idx_out NULL: row_ptr_out
 * (rows+1) and *nnz_out only. */
alsk_status alsk_dev_filter_columns(const alsk_csr* r, int64_t col_begin, int64_t col_end, int64_t* row_ptr_out,
                                    int32_t* col_idx_out, float* values_out, int64_t* nnz_out, void* stream);

/* ---- multi-GPU (replaces su_als_update_x's worker loop, parallel.hpp:487-583,
 * with one GPU per worker) ------------------------------------------------------------------ */
/* NCCL communicators. NCCL is loaded at run time; alsk_comm_available() is 0 when it is not
 * installed (the single-GPU entry points do not need it). One process per GPU: rank 0 makes a
 * 128-byte id (alsk_comm_unique_id), the caller ships it to every rank, and each rank calls
 * alsk_comm_init_rank. One process driving several GPUs: alsk_comm_init_all. */
typedef struct alsk_comm alsk_comm;
#define ALSK_COMM_ID_BYTES 128
enum { ALSK_DTYPE_F32 = 0, ALSK_DTYPE_F64 = 1 };
int alsk_comm_available(void);
int alsk_nccl_version(void);
alsk_status alsk_comm_unique_id(uint8_t* id_out /* ALSK_COMM_ID_BYTES */);
alsk_status alsk_comm_init_rank(const uint8_t* id, int nranks, int rank, int device, alsk_comm** out);
alsk_status alsk_comm_init_all(int ndev, const int* devices, alsk_comm** comms_out /* ndev */);
/* A communicator whose collectives go through caller-supplied functions (same semantics as
 * alsk_comm_allgather / alsk_comm_reduce_scatter, return 0 on success). Used by the tests to
 * run several ranks' sessions on one GPU over a host transport; NCCL is the product path. */
typedef struct alsk_comm_ops {
    int (*allgather)(void* user, void* buf, int64_t chunk_elems, int dtype, void* stream);
    int (*reduce_scatter)(void* user, const void* in, void* out, int64_t chunk_elems, int dtype, void* stream);
    void* user;
} alsk_comm_ops;
alsk_status alsk_comm_init_custom(int nranks, int rank, const alsk_comm_ops* ops, alsk_comm** out);
void alsk_comm_destroy(alsk_comm* comm);
int alsk_comm_rank(const alsk_comm* comm);
int alsk_comm_size(const alsk_comm* comm);
/* In-place all-gather: rank r's chunk sits at buf + r*chunk_elems; afterwards buf holds all. */
alsk_status alsk_comm_allgather(alsk_comm* comm, void* buf, int64_t chunk_elems, int dtype, void* stream);
/* Sum-reduce-scatter: in holds nranks*chunk_elems, out receives this rank's summed chunk. */
alsk_status alsk_comm_reduce_scatter(alsk_comm* comm, const void* in, void* out, int64_t chunk_elems, int dtype,
                                     void* stream);
alsk_status alsk_comm_allreduce_max(alsk_comm* comm, double* buf, int64_t count, void* stream);
/* Wait for the stream while polling NCCL's asynchronous error state; on an error or after
 * timeout_s (> 0) the communicator is aborted and ALSK_ERR_CUDA returned instead of a hang. */
alsk_status alsk_comm_wait(alsk_comm* comm, void* stream, double timeout_s);

/* Packed-row scratch of the tensor-core half-sweep, owned by the caller (halved on
 * allocation failure down to 64 MB). Sessions that own one never lock or synchronise. */
typedef struct alsk_workspace alsk_workspace;
alsk_status alsk_workspace_create(size_t scratch_bytes, alsk_workspace** out);
size_t alsk_workspace_bytes(const alsk_workspace* ws);
void alsk_workspace_destroy(alsk_workspace* ws);

/* One rank's share of a multi-GPU ALS run (a single-GPU run is comm = NULL).
 *  ALSK_MP_MODEL : x_local = CSR rows [xb, xe) of R (global item ids), t_local = CSR rows
 *                  [tb, te) of R^T (global user ids); slices are equal-count:
 *                  xb = rank*ceil(m/P), tb = rank*ceil(n/P). Each half solves the rank's slice
 *                  and all-gathers the factor in place (bit-identical to one GPU for any P).
 *  ALSK_MP_HYBRID: x_local as above; t_local = every item's ratings from this rank's users
 *                  (n rows, user ids local to the slab). The Theta half reduce-scatters
 *                  per-item partial Hermitians (lambda n_v^local, parallel.hpp:408-411), solves
 *                  the item slice and all-gathers Theta; X stays in per-rank slabs.
 * x0 (m*f) / theta0 (n*f) are device pointers (NULL = zeros). ws = NULL allocates a private
 * workspace. Half-sweeps are asynchronous on `stream`: columns are validated once here and
 * breakdowns are raised by alsk_mp_check (which also polls NCCL errors). */
typedef struct alsk_mp alsk_mp;
enum { ALSK_MP_MODEL = 0, ALSK_MP_HYBRID = 1 };
alsk_status alsk_mp_create(alsk_comm* comm, int mode, int64_t m, int64_t n, int f, double lambda,
                           alsk_precision precision, const alsk_csr* x_local, const alsk_csr* t_local,
                           const float* x0, const float* theta0, alsk_workspace* ws, void* stream, alsk_mp** out);
alsk_status alsk_mp_half_x(alsk_mp* mp, void* stream);
alsk_status alsk_mp_half_theta(alsk_mp* mp, void* stream);
alsk_status alsk_mp_check(alsk_mp* mp, void* stream);
/* Device factors: X (MODEL: all m rows after the all-gather; HYBRID: the slab starting at
 * global row *x_row_begin) and Theta (all n rows). Padded rows follow the real ones. */
alsk_status alsk_mp_factors(alsk_mp* mp, float** x, int64_t* x_row_begin, float** theta);
void alsk_mp_slices(const alsk_mp* mp, int64_t* x_begin, int64_t* x_end, int64_t* t_begin, int64_t* t_end);
/* Bytes this rank moved through collectives ((P-1)/P of each buffer) and the call count. */
void alsk_mp_collective_stats(const alsk_mp* mp, int64_t* bytes, int64_t* calls);
void alsk_mp_destroy(alsk_mp* mp);

#ifdef __cplusplus
}
#endif

#endif /* ALSKIT_CUDA_H_ */
