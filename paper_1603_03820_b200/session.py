"""Device-resident ALS session: R (CSR) and R^T (CSR of the transpose, i.e. the CSC arrays)
uploaded once, X and Theta kept in HBM across half-sweeps.

This is the caller of the hot path that train_run/als_train need:
the reference rebuilds nothing between halves either (driver.hpp:115, 255-262), but keeps
factors in host memory; here they never leave the device unless asked for. PyTorch is used
only for device allocation and the current stream; every kernel is libalskit_cuda's.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .alskit import (TRIPLET_DTYPE, CscMatrix, CsrMatrix, FactorMatrix, SolverConfig, _check,
                     cache_header, checkpoint_header, checkpoint_path, restore_latest,
                     FactorKind, InputError, IterationMetrics, BlockRef)

LIB = N.LIB
PREC_FP64_EXACT = 0
PREC_FP32 = 1
PREC_TF32X2 = 2


def _dev(a: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(device, non_blocking=False)


class DeviceCsr:
    """CSR arrays in HBM plus the C-ABI view of them."""

    def __init__(self, rows: int, cols: int, row_ptr, col_idx, values, device, col_offset: int = 0):
        self.rows, self.cols, self.col_offset = rows, cols, col_offset
        t = lambda a, dt: a if isinstance(a, torch.Tensor) else _dev(np.asarray(a, dt), device)  # noqa: E731
        self.row_ptr = t(row_ptr, np.int64)
        self.col_idx = t(col_idx, np.int32)
        self.values = t(values, np.float32)
        self.nnz = int(self.values.numel())
        self.c = N.CsrT(rows, cols, col_offset, self.nnz, self.row_ptr.data_ptr(),
                        self.col_idx.data_ptr(), self.values.data_ptr())

    @staticmethod
    def from_host(r: CsrMatrix, device) -> "DeviceCsr":
        return DeviceCsr(r.rows, r.cols, r.row_ptr, r.col_idx, r.values, device, r.col_offset)

    @staticmethod
    def from_cache(path, device) -> "DeviceCsr":
        """Load a binary ratings cache (dataio.hpp:133-163) straight into HBM: the file is
        streamed through pinned staging and validated on the host as it passes."""
        rows, cols, nnz = cache_header(path)
        rp = torch.empty(rows + 1, dtype=torch.int64, device=device)
        ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
        va = torch.empty(max(nnz, 1), dtype=torch.float32, device=device)
        _check(LIB.alsk_dev_load_cache(os.fsencode(path), rows, nnz, rp.data_ptr(), ci.data_ptr(), va.data_ptr(),
                                       stream_handle()))
        return DeviceCsr(rows, cols, rp, ci[:nnz], va[:nnz], device)

    def split_train_test(self, holdout_fraction: float, seed: int):
        """split_train_test (dataio.hpp:251-290) in HBM: returns (train DeviceCsr, test triplets
        as a (k, 24-byte) uint8 device tensor in TRIPLET_DTYPE layout), bit-identical to the
        host split."""
        k = C.c_int64()
        _check(LIB.alsk_dev_split_train_test(C.byref(self.c), holdout_fraction, seed & (2**64 - 1), C.byref(k),
                                             None, None, None, None, None))
        dev = self.values.device
        kk, keep = k.value, self.nnz - k.value
        rp = torch.empty(self.rows + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(max(keep, 1), dtype=torch.int32, device=dev)
        va = torch.empty(max(keep, 1), dtype=torch.float32, device=dev)
        te = torch.empty((max(kk, 1), TRIPLET_DTYPE.itemsize), dtype=torch.uint8, device=dev)
        _check(LIB.alsk_dev_split_train_test(C.byref(self.c), holdout_fraction, seed & (2**64 - 1), C.byref(k),
                                             rp.data_ptr(), ci.data_ptr(), va.data_ptr(), te.data_ptr(),
                                             stream_handle()))
        return DeviceCsr(self.rows, self.cols, rp, ci[:keep], va[:keep], dev), te[:kk]

    def transpose(self) -> "DeviceCsr":
        """Stable device transpose (csr_to_csc, sparse.hpp:185-207) viewed as the CSR of R^T."""
        dev = self.values.device
        col_ptr = torch.empty(self.cols + 1, dtype=torch.int64, device=dev)
        row_idx = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(self.nnz, 1), dtype=torch.float32, device=dev)
        _check(LIB.alsk_dev_csr_to_csc(C.byref(self.c), col_ptr.data_ptr(), row_idx.data_ptr(),
                                       vals.data_ptr(), stream_handle()))
        return DeviceCsr(self.cols, self.rows, col_ptr, row_idx[: self.nnz], vals[: self.nnz], dev)


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def dev_update(r: DeviceCsr, theta: torch.Tensor, theta_rows: int, f: int, lam: float, precision: int,
               out: torch.Tensor, row_begin: int = 0, row_end: Optional[int] = None,
               batch_rows: int = 4096) -> None:
    """One half-sweep (update_x, solver.hpp:330-345) of rows [row_begin,row_end) into
    out[(row-row_begin)*f ...]."""
    re = r.rows if row_end is None else row_end
    _check(LIB.alsk_dev_update(C.byref(r.c), theta.data_ptr(), theta_rows, f, lam, precision,
                               batch_rows, row_begin, re, out.data_ptr(), stream_handle()))


def dev_hermitian(r: DeviceCsr, theta: torch.Tensor, theta_rows: int, f: int, lam: float, precision: int,
                  a_out: torch.Tensor, b_out: torch.Tensor, row_begin: int = 0,
                  row_end: Optional[int] = None) -> None:
    """get_hermitian_mo_into (solver.hpp:292-304) on device buffers: A full mirrored f*f and
    B f floats per row of [row_begin,row_end)."""
    re = r.rows if row_end is None else row_end
    _check(LIB.alsk_dev_hermitian(C.byref(r.c), theta.data_ptr(), theta_rows, f, lam, precision, row_begin,
                                  re, a_out.data_ptr(), b_out.data_ptr(), stream_handle()))


class AlsSession:
    def __init__(self, r: CsrMatrix, r_csc: Optional[CscMatrix], test: Optional[np.ndarray],
                 cfg: SolverConfig, x0: FactorMatrix, theta0: FactorMatrix, device: str = "cuda"):
        if not torch.cuda.is_available():
            raise RuntimeError("AlsSession needs a CUDA device (libalskit_cuda has no CPU path)")
        self.device = torch.device(device)
        self.cfg = cfg
        self.f = x0.f
        self.m, self.n = r.rows, r.cols
        self.precision = PREC_FP64_EXACT if cfg.accumulate_double else PREC_FP32
        self.R = DeviceCsr.from_host(r, self.device)
        if r_csc is not None:
            self.RT = DeviceCsr(r_csc.cols, r_csc.rows, r_csc.col_ptr, r_csc.row_idx, r_csc.values,
                                self.device)
        else:
            self.RT = self.R.transpose()
        self.col_nnz = (self.RT.row_ptr[1:] - self.RT.row_ptr[:-1]).contiguous()
        self.X = _dev(x0.entries, self.device)
        self.T = _dev(theta0.entries, self.device)
        self.test = None
        if test is not None and len(test):
            t = np.ascontiguousarray(test, TRIPLET_DTYPE)
            self.test_rows = _dev(t["row"].copy(), self.device)
            self.test_cols = _dev(t["col"].copy(), self.device)
            self.test_vals = _dev(t["value"].copy(), self.device)
            self.test = len(t)

    def half_x(self) -> None:
        dev_update(self.R, self.T, self.n, self.f, self.cfg.lambda_, self.precision, self.X,
                   batch_rows=self.cfg.batch_rows)

    def half_theta(self) -> None:
        dev_update(self.RT, self.X, self.m, self.f, self.cfg.lambda_, self.precision, self.T,
                   batch_rows=self.cfg.batch_rows)

    def loss(self) -> float:
        out = C.c_double()
        _check(LIB.alsk_dev_loss(C.byref(self.R.c), self.col_nnz.data_ptr(), self.X.data_ptr(),
                                 self.T.data_ptr(), self.n, self.f, self.cfg.lambda_, C.byref(out),
                                 stream_handle()))
        return out.value

    def rmse(self) -> float:
        if not self.test:
            return float("nan")
        out = C.c_double()
        _check(LIB.alsk_dev_rmse(self.test_rows.data_ptr(), self.test_cols.data_ptr(),
                                 self.test_vals.data_ptr(), self.test, self.X.data_ptr(), self.m,
                                 self.T.data_ptr(), self.n, self.f, C.byref(out), stream_handle()))
        return out.value

    def factors(self):
        x = FactorMatrix(self.m, self.f, self.X.cpu().numpy().copy())
        t = FactorMatrix(self.n, self.f, self.T.cpu().numpy().copy())
        return x, t

    def load_factor(self, which: FactorKind, path) -> None:
        """Restore X or Theta from a checkpoint file straight into HBM."""
        _, _, rows, f, _ = checkpoint_header(path)
        want = (self.m if which == FactorKind.x else self.n, self.f)
        if (rows, f) != want:
            raise InputError(f"{path}: checkpoint holds a {rows}x{f} factor, the run needs {want[0]}x{want[1]}")
        dst = self.X if which == FactorKind.x else self.T
        _check(LIB.alsk_dev_checkpoint_read(os.fsencode(path), rows * f, dst.data_ptr(), stream_handle()))


class DeviceCheckpointWriter:
    """CheckpointWriter (dataio.hpp:717-786) fed from HBM: submit() queues a D2H copy of the
    factor behind the current stream into pinned memory and returns; one native worker
    thread writes the file (atomic temp + rename). At most one snapshot in flight; write
    errors are sticky and raised by the next submit() or flush()."""

    def __init__(self, dir):
        self.h = C.c_void_p()
        _check(LIB.alsk_ckpt_writer_create(os.fsencode(dir), C.byref(self.h)))

    def submit(self, iteration: int, which: FactorKind, factor: torch.Tensor, rows: int, f: int, digest: int):
        _check(LIB.alsk_ckpt_writer_submit_device(self.h, iteration, int(which), rows, f, digest & (2**64 - 1),
                                                  factor.data_ptr(), stream_handle()))

    def flush(self) -> None:
        _check(LIB.alsk_ckpt_writer_flush(self.h))

    def close(self) -> None:
        if self.h:
            LIB.alsk_ckpt_writer_destroy(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        self.close()


def train_resumable(sess: AlsSession, iterations: int, checkpoint_dir, digest: int, resume: bool = True,
                    after_iteration=None) -> tuple:
    """The iteration loop of train_run (driver.hpp:183-262) on a device session: resume
    from the newest compatible checkpoint (Theta@t also loads X@t; a lone X@t finishes
    iteration t's Theta half first), snapshot after every half through the device writer,
    flush at the end. Returns (start_iteration, [IterationMetrics])."""
    completed, dangling_x = 0, False
    if resume:
        latest = restore_latest(checkpoint_dir, digest)
        if latest is not None:
            completed = latest.iteration
            if latest.which == FactorKind.theta:
                sess.load_factor(FactorKind.theta, checkpoint_path(checkpoint_dir, completed, FactorKind.theta))
                px = checkpoint_path(checkpoint_dir, completed, FactorKind.x)
                if checkpoint_header(px)[4] != digest:
                    raise InputError(f"checkpoint config digest mismatch at iteration {completed}")
                sess.load_factor(FactorKind.x, px)
            else:
                sess.load_factor(FactorKind.x, checkpoint_path(checkpoint_dir, completed, FactorKind.x))
                dangling_x = True
    start = completed if dangling_x else completed + 1
    rows = []
    with DeviceCheckpointWriter(checkpoint_dir) as w:
        def row(t):
            m = IterationMetrics(t, sess.loss(), sess.rmse())
            rows.append(m)
            return after_iteration is None or after_iteration(t, sess)

        go = True
        if dangling_x:
            sess.half_theta()
            w.submit(completed, FactorKind.theta, sess.T, sess.n, sess.f, digest)
            go = row(completed)
        t = completed + 1
        while go and t <= iterations:
            sess.half_x()
            w.submit(t, FactorKind.x, sess.X, sess.m, sess.f, digest)
            sess.half_theta()
            w.submit(t, FactorKind.theta, sess.T, sess.n, sess.f, digest)
            go = row(t)
            t += 1
        w.flush()
    return start, rows


class DeviceBlock:
    """A streamed grid block in HBM (the C-ABI view of the stream's slot); valid until the
    stream's next next()."""

    def __init__(self, c: N.CsrT):
        self.c = c
        self.rows, self.cols, self.col_offset, self.nnz = c.rows, c.cols, c.col_offset, c.nnz

    def to_host(self) -> CsrMatrix:
        rp = np.empty(self.rows + 1, np.int64)
        ci = np.empty(self.nnz, np.int32)
        va = np.empty(self.nnz, np.float32)
        s = stream_handle()
        for dst, src in ((rp, self.c.row_ptr), (ci, self.c.col_idx), (va, self.c.values)):
            if dst.nbytes:
                _check(LIB.alsk_dev_to_host(dst.ctypes.data, src, dst.nbytes, s))
        return CsrMatrix(self.rows, self.cols, self.col_offset, rp, ci, va)


class DeviceBlockStream:
    """BlockStream (dataio.hpp:447-524) into HBM: iterate to get (BlockRef, DeviceBlock) in
    plan order, each upload overlapped with the work on the previous blocks."""

    def __init__(self, dir, order):
        flat = np.array([v for b in order for v in (b.i, b.j)] or [0], np.int32)
        self.h = C.c_void_p()
        _check(LIB.alsk_block_stream_open(os.fsencode(dir), flat.ctypes.data, len(order), C.byref(self.h)))

    def __iter__(self):
        return self

    def __next__(self):
        has, i, j = C.c_int(), C.c_int(), C.c_int()
        c = N.CsrT()
        _check(LIB.alsk_block_stream_next(self.h, stream_handle(), C.byref(has), C.byref(i), C.byref(j), C.byref(c)))
        if not has.value:
            raise StopIteration
        return BlockRef(i.value, j.value), DeviceBlock(c)

    def close(self) -> None:
        if self.h:
            LIB.alsk_block_stream_close(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        self.close()


def out_of_core_update_x(dir, theta: torch.Tensor, f: int, lam: float, out: torch.Tensor,
                         precision: int = PREC_FP32) -> None:
    """One half-sweep over a persisted grid that need not fit in HBM (the
    scale-up of su_als_update_x, parallel.hpp:487-583): alsk_ooc_update streams the blocks
    into HBM (block (i, j) uploads while the previous one computes), reduces each row
    partition's partial Hermitians slice by slice and solves them. PREC_FP64_EXACT is
    bit-identical to the reference's su_als_update_x on the same grid; PREC_FP32 uses the
    tensor-core partials. `theta` holds the factor of the grid's columns, `out` receives the
    grid's rows (both on the device). The Theta half is the same call on the persisted grid
    of R^T with X as the factor."""
    cfg = N.SolverConfigT(f, lam, 16, 4096, 1 if precision == PREC_FP64_EXACT else 0, 0, 0)
    _check(LIB.alsk_ooc_update(str(dir).encode(), theta.data_ptr(), theta.numel() // f, f, C.byref(cfg),
                               out.data_ptr(), stream_handle()))
