"""ctypes binding of libalskit_cuda.so (the C ABI in include/alskit_cuda.h).

The library is loaded from the package directory (built in-tree by build.py). There is no
fallback: if the shared object is missing the import fails loudly, and every compute entry
point reports ALSK_ERR_CUDA when no device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# ALSK_MEASURE_LIB=1 loads the measurement build (build.py with ALSK_MEASURE=1: profiling
# counters and A/B switches) instead of the product library.
_LIB_PATH = Path(__file__).resolve().parent / (
    "libalskit_cuda_measure.so" if os.environ.get("ALSK_MEASURE_LIB") == "1" else "libalskit_cuda.so")

i64 = C.c_int64
i32 = C.c_int32
u64 = C.c_uint64
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
vp = C.c_void_p


class CsrT(C.Structure):
    _fields_ = [("rows", i64), ("cols", i64), ("col_offset", i64), ("nnz", i64),
                ("row_ptr", vp), ("col_idx", vp), ("values", vp)]


class TripletT(C.Structure):
    _fields_ = [("row", i64), ("col", i64), ("value", C.c_float)]


class SolverConfigT(C.Structure):
    _fields_ = [("f", C.c_int), ("lambda_", C.c_double), ("bin", C.c_int), ("batch_rows", i64),
                ("accumulate_double", C.c_int), ("threads", C.c_int), ("seed", u64)]


assert C.sizeof(TripletT) == 24
CsrP = C.POINTER(CsrT)
CfgP = C.POINTER(SolverConfigT)

# name -> (restype, argtypes)
_SIGS = {
    "alsk_last_error": (C.c_char_p, []),
    "alsk_last_breakdown_index": (i64, []),
    "alsk_device_available": (C.c_int, []),
    "alsk_kernel_launch_count": (u64, []),
    "alsk_build_info": (C.c_char_p, []),
    "alsk_profile_begin": (None, []),
    "alsk_set_fp32_engine": (None, [C.c_int]),
    "alsk_profile_phases": (None, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "alsk_fp32_engine": (C.c_int, []),
    "alsk_profile_end": (None, [f64p, C.POINTER(u64)]),
    "alsk_fp32_peak_probe": (C.c_double, []),
    "alsk_herm_loop_probe": (C.c_double, [C.c_int, C.c_int]),
    "alsk_get_hermitian_mo_into": (C.c_int, [CsrP, vp, i64, C.c_int, CfgP, i64, i64, vp, vp]),
    "alsk_get_hermitian_base": (C.c_int, [CsrP, vp, i64, C.c_int, C.c_double, C.c_int, vp, vp]),
    "alsk_local_hermitian": (C.c_int, [CsrP, vp, i64, C.c_int, CfgP, vp, vp]),
    "alsk_batch_solve": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, vp]),
    "alsk_update_x": (C.c_int, [CsrP, vp, i64, C.c_int, CfgP, vp]),
    "alsk_update_theta": (C.c_int, [i64, i64, i64, vp, vp, vp, vp, i64, C.c_int, CfgP, vp]),
    "alsk_loss": (C.c_int, [CsrP, vp, i64, vp, i64, C.c_int, C.c_double, f64p]),
    "alsk_rmse": (C.c_int, [vp, i64, vp, i64, vp, i64, C.c_int, f64p]),
    "alsk_csr_to_csc": (C.c_int, [CsrP, vp, vp, vp]),
    "alsk_csc_to_csr": (C.c_int, [i64, i64, i64, vp, vp, vp, vp, vp, vp]),
    "alsk_csr_from_triplets": (C.c_int, [i64, i64, vp, i64, vp, vp, vp]),
    "alsk_grid_partition_counts": (C.c_int, [CsrP, C.c_int, C.c_int, vp, vp, vp]),
    "alsk_grid_partition_fill": (C.c_int, [CsrP, C.c_int, C.c_int, vp, vp, vp]),
    "alsk_parallel_reduce": (C.c_int, [vp, vp, C.c_int, i64, C.c_int, vp, C.c_int, vp, vp]),
    "alsk_su_als_update_x": (C.c_int, [CsrP, C.c_int, C.c_int, vp, vp, vp, C.c_int, CfgP, vp, C.c_int, vp]),
    "alsk_dev_update": (C.c_int, [CsrP, vp, i64, C.c_int, C.c_double, C.c_int, i64, i64, i64, vp, vp]),
    "alsk_dev_hermitian": (C.c_int, [CsrP, vp, i64, C.c_int, C.c_double, C.c_int, i64, i64, vp, vp, vp]),
    "alsk_dev_partial_hermitian": (C.c_int, [CsrP, vp, i64, C.c_int, C.c_double, i64, i64, vp, vp]),
    "alsk_dev_solve_packed": (C.c_int, [vp, i64, C.c_int, vp, vp]),
    "alsk_packed_stride": (i64, [C.c_int]),
    "alsk_cache_header": (C.c_int, [C.c_char_p, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
    "alsk_save_cache": (C.c_int, [CsrP, C.c_char_p]),
    "alsk_load_cache": (C.c_int, [C.c_char_p, i64, i64, vp, vp, vp]),
    "alsk_dev_load_cache": (C.c_int, [C.c_char_p, i64, i64, vp, vp, vp, vp]),
    "alsk_persist_grid_meta": (C.c_int, [C.c_char_p, C.c_int, C.c_int, i64, i64, vp, vp]),
    "alsk_block_path": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    "alsk_grid_meta": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(i64),
                                 vp, vp]),
    "alsk_block_stream_open": (C.c_int, [C.c_char_p, vp, C.c_int, C.POINTER(vp)]),
    "alsk_block_stream_next": (C.c_int, [vp, vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), CsrP]),
    "alsk_block_stream_close": (None, [vp]),
    "alsk_ooc_update": (C.c_int, [C.c_char_p, vp, i64, C.c_int, CfgP, vp, vp]),
    "alsk_dev_to_host": (C.c_int, [vp, vp, C.c_size_t, vp]),
    "alsk_host_to_dev": (C.c_int, [vp, vp, C.c_size_t, vp]),
    "alsk_dev_split_train_test": (C.c_int, [CsrP, C.c_double, C.c_uint64, C.POINTER(i64), vp, vp, vp, vp, vp]),
    "alsk_checkpoint_write": (C.c_int, [C.c_char_p, C.c_int, C.c_int, i64, C.c_int, C.c_uint64, vp]),
    "alsk_checkpoint_path": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    "alsk_checkpoint_header": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(i64),
                                         C.POINTER(C.c_int), C.POINTER(C.c_uint64)]),
    "alsk_checkpoint_read": (C.c_int, [C.c_char_p, i64, vp]),
    "alsk_dev_checkpoint_read": (C.c_int, [C.c_char_p, i64, vp, vp]),
    "alsk_checkpoint_latest": (C.c_int, [C.c_char_p, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_int)]),
    "alsk_ckpt_writer_create": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "alsk_ckpt_writer_submit_device": (C.c_int, [vp, C.c_int, C.c_int, i64, C.c_int, C.c_uint64, vp, vp]),
    "alsk_ckpt_writer_submit_host": (C.c_int, [vp, C.c_int, C.c_int, i64, C.c_int, C.c_uint64, vp]),
    "alsk_ckpt_writer_flush": (C.c_int, [vp]),
    "alsk_ckpt_writer_destroy": (None, [vp]),
    "alsk_dev_partial_hermitian_f32": (C.c_int, [CsrP, vp, i64, C.c_int, C.c_double, i64, i64, vp, vp]),
    "alsk_dev_solve_packed_f32": (C.c_int, [vp, i64, C.c_int, vp, vp]),
    "alsk_dev_loss": (C.c_int, [CsrP, vp, vp, vp, i64, C.c_int, C.c_double, f64p, vp]),
    "alsk_dev_rmse": (C.c_int, [vp, vp, vp, i64, vp, i64, vp, i64, C.c_int, f64p, vp]),
    "alsk_dev_csr_to_csc": (C.c_int, [CsrP, vp, vp, vp, vp]),
    "alsk_random_factor": (None, [i64, C.c_int, u64, vp]),
    "alsk_mix_seed": (u64, [u64, u64]),
    "alsk_split_train_test": (C.c_int, [CsrP, C.c_double, u64, i64p, vp, vp, vp, vp]),
    "alsk_synth_csr": (C.c_int, [i64, i64, i64, u64, C.c_int, vp, vp, vp]),
    "alsk_dev_synth_rows": (C.c_int, [i64, i64, i64, u64, i64, i64, vp, vp, vp, vp]),
    "alsk_synth_row_start": (i64, [i64, i64, i64]),
    "alsk_holdout_mask": (C.c_int, [i64, C.c_double, u64, vp, i64p]),
    "alsk_mask_count": (i64, [vp, i64, i64]),
    "alsk_dev_split_mask": (C.c_int, [CsrP, vp, i64, i64, vp, vp, vp, vp, i64p, vp]),
    "alsk_dev_filter_columns": (C.c_int, [CsrP, i64, i64, vp, vp, vp, i64p, vp]),
    "alsk_profile_phase": (None, [C.c_int, f64p, C.POINTER(u64)]),
    "alsk_session_device": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    # multi-GPU (multigpu.cu)
    "alsk_comm_available": (C.c_int, []),
    "alsk_nccl_version": (C.c_int, []),
    "alsk_comm_unique_id": (C.c_int, [vp]),
    "alsk_comm_init_rank": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "alsk_comm_init_all": (C.c_int, [C.c_int, vp, vp]),
    "alsk_comm_init_custom": (C.c_int, [C.c_int, C.c_int, vp, C.POINTER(vp)]),
    "alsk_comm_destroy": (None, [vp]),
    "alsk_comm_rank": (C.c_int, [vp]),
    "alsk_comm_size": (C.c_int, [vp]),
    "alsk_comm_allgather": (C.c_int, [vp, vp, i64, C.c_int, vp]),
    "alsk_comm_reduce_scatter": (C.c_int, [vp, vp, vp, i64, C.c_int, vp]),
    "alsk_comm_allreduce_max": (C.c_int, [vp, vp, i64, vp]),
    "alsk_comm_wait": (C.c_int, [vp, vp, C.c_double]),
    "alsk_workspace_create": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
    "alsk_workspace_bytes": (C.c_size_t, [vp]),
    "alsk_workspace_destroy": (None, [vp]),
    "alsk_mp_create": (C.c_int, [vp, C.c_int, i64, i64, C.c_int, C.c_double, C.c_int, CsrP, CsrP, vp, vp, vp, vp,
                                 C.POINTER(vp)]),
    "alsk_mp_half_x": (C.c_int, [vp, vp]),
    "alsk_mp_half_theta": (C.c_int, [vp, vp]),
    "alsk_mp_check": (C.c_int, [vp, vp]),
    "alsk_mp_factors": (C.c_int, [vp, C.POINTER(vp), C.POINTER(i64), C.POINTER(vp)]),
    "alsk_mp_slices": (None, [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
    "alsk_mp_collective_stats": (None, [vp, C.POINTER(i64), C.POINTER(i64)]),
    "alsk_mp_destroy": (None, [vp]),
}

# transport callbacks of alsk_comm_init_custom (alsk_comm_ops)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, vp, vp, i64, C.c_int, vp)
REDUCE_SCATTER_FN = C.CFUNCTYPE(C.c_int, vp, vp, vp, i64, C.c_int, vp)


class CommOpsT(C.Structure):
    _fields_ = [("allgather", ALLGATHER_FN), ("reduce_scatter", REDUCE_SCATTER_FN), ("user", vp)]


def _load() -> C.CDLL:
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue  # declared in the header but not yet exported: callers get AttributeError
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()
LIB_PATH = _LIB_PATH


def exported_symbols() -> list[str]:
    return [n for n in _SIGS if getattr(LIB, n, None) is not None]
