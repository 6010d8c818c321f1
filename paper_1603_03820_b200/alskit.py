"""Python mirror of the reference's ALS API (alskit, proj/include/alskit/*.hpp) on the
B200 C ABI.

Same names, argument meaning and error behaviour as the reference's C++ surface
(SURVEY.md §8(b)); every compute call goes to libalskit_cuda.so. Matrices are numpy-backed
dataclasses with the reference's field names; errors are the reference's four categories.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native as N

LIB = N.LIB

TRIPLET_DTYPE = np.dtype([("row", "<i8"), ("col", "<i8"), ("value", "<f4")], align=True)
assert TRIPLET_DTYPE.itemsize == 24


# ---------------------------------------------------------------- errors (common.hpp:24-64)
class Error(RuntimeError):
    category = "unknown"


class InputError(Error):
    category = "input"


class CapacityError(Error):
    category = "capacity"


class NumericalError(Error):
    category = "numerical"


class IoError(Error):
    category = "io"


class DeviceError(Error):
    category = "device"


_ERR = {1: InputError, 2: CapacityError, 3: NumericalError, 4: IoError, 5: DeviceError}


def _check(status: int) -> None:
    if status != 0:
        msg = LIB.alsk_last_error().decode(errors="replace")
        raise _ERR.get(status, Error)(msg)


def _p(a: Optional[np.ndarray]) -> Optional[int]:
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------- data structures
@dataclass
class CsrMatrix:
    """sparse.hpp:38-48"""
    rows: int = 0
    cols: int = 0
    col_offset: int = 0
    row_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    col_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def nnz(self) -> int:
        return int(self.values.size)

    def row_nnz(self, u: int) -> int:
        return int(self.row_ptr[u + 1] - self.row_ptr[u])

    def _c(self) -> N.CsrT:
        self.row_ptr = np.ascontiguousarray(self.row_ptr, np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, np.int32)
        self.values = np.ascontiguousarray(self.values, np.float32)
        return N.CsrT(self.rows, self.cols, self.col_offset, self.values.size,
                      _p(self.row_ptr), _p(self.col_idx), _p(self.values))


@dataclass
class CscMatrix:
    """sparse.hpp:52-61"""
    rows: int = 0
    cols: int = 0
    col_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    row_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def nnz(self) -> int:
        return int(self.values.size)

    def col_nnz(self, v: int) -> int:
        return int(self.col_ptr[v + 1] - self.col_ptr[v])


@dataclass
class FactorMatrix:
    """factor.hpp:16-34 — row-major rows x f float32 (entries is the flat view)."""
    rows: int = 0
    f: int = 0
    entries: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def __post_init__(self):
        if self.entries.size == 0 and self.rows * self.f > 0:
            self.entries = np.zeros(self.rows * self.f, np.float32)
        self.entries = np.ascontiguousarray(self.entries, np.float32).reshape(-1)

    def row(self, u: int) -> np.ndarray:
        return self.entries[u * self.f:(u + 1) * self.f]

    def as2d(self) -> np.ndarray:
        return self.entries.reshape(self.rows, self.f)


@dataclass
class HermitianBatch:
    """solver.hpp:30-58"""
    count: int = 0
    f: int = 0
    a: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    b: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    def resize(self, count: int, f: int) -> None:
        self.count, self.f = count, f
        self.a = np.zeros(count * f * f, np.float32)
        self.b = np.zeros(count * f, np.float32)

    def a_at(self, k: int) -> np.ndarray:
        return self.a[k * self.f * self.f:(k + 1) * self.f * self.f]

    def b_at(self, k: int) -> np.ndarray:
        return self.b[k * self.f:(k + 1) * self.f]


@dataclass
class SolverConfig:
    """solver.hpp:61-69. `bin` and `threads` are accepted and never change the result."""
    f: int = 8
    lambda_: float = 0.05
    bin: int = 16
    batch_rows: int = 4096
    accumulate_double: bool = True
    threads: int = 0
    seed: int = 42

    def _c(self) -> N.SolverConfigT:
        return N.SolverConfigT(self.f, self.lambda_, self.bin, self.batch_rows,
                               1 if self.accumulate_double else 0, self.threads, self.seed)


class BreakdownPolicy(enum.IntEnum):
    """solver.hpp:72"""
    fail = 0
    zero_row = 1


def triplets(rows, cols, values) -> np.ndarray:
    t = np.zeros(len(values), TRIPLET_DTYPE)
    t["row"], t["col"], t["value"] = rows, cols, values
    return t


# ---------------------------------------------------------------- factor init
def mix_seed(seed: int, salt: int) -> int:
    """common.hpp:70-75"""
    return int(LIB.alsk_mix_seed(seed & (2**64 - 1), salt & (2**64 - 1)))


def random_factor(rows: int, f: int, seed: int) -> FactorMatrix:
    """factor.hpp:49-54 (bit-exact mt19937_64 stream)."""
    out = np.empty(rows * f, np.float32)
    LIB.alsk_random_factor(rows, f, seed & (2**64 - 1), _p(out))
    return FactorMatrix(rows, f, out)


# ---------------------------------------------------------------- sparse plumbing
def csr_to_csc(a: CsrMatrix) -> CscMatrix:
    """sparse.hpp:185-207 (device stable transpose)."""
    c = a._c()
    col_ptr = np.empty(a.cols + 1, np.int64)
    row_idx = np.empty(a.nnz(), np.int32)
    vals = np.empty(a.nnz(), np.float32)
    _check(LIB.alsk_csr_to_csc(C.byref(c), _p(col_ptr), _p(row_idx), _p(vals)))
    return CscMatrix(a.rows, a.cols, col_ptr, row_idx, vals)


def csc_to_csr(a: CscMatrix) -> CsrMatrix:
    """sparse.hpp:209-231"""
    row_ptr = np.empty(a.rows + 1, np.int64)
    col_idx = np.empty(a.nnz(), np.int32)
    vals = np.empty(a.nnz(), np.float32)
    cp = np.ascontiguousarray(a.col_ptr, np.int64)
    ri = np.ascontiguousarray(a.row_idx, np.int32)
    va = np.ascontiguousarray(a.values, np.float32)
    _check(LIB.alsk_csc_to_csr(a.rows, a.cols, a.nnz(), _p(cp), _p(ri), _p(va),
                               _p(row_ptr), _p(col_idx), _p(vals)))
    return CsrMatrix(a.rows, a.cols, 0, row_ptr, col_idx, vals)


def transpose_of(a: CscMatrix) -> CsrMatrix:
    """sparse.hpp:235-243 — role swap (the reference copies; we share the arrays)."""
    return CsrMatrix(a.cols, a.rows, 0, a.col_ptr, a.row_idx, a.values)


def csr_from_triplets(m: int, n: int, t: np.ndarray) -> CsrMatrix:
    """sparse.hpp:132-170 (device sort + duplicate/range checks)."""
    t = np.ascontiguousarray(t, TRIPLET_DTYPE)
    row_ptr = np.empty(max(m, 0) + 1, np.int64)
    col_idx = np.empty(t.size, np.int32)
    vals = np.empty(t.size, np.float32)
    _check(LIB.alsk_csr_from_triplets(m, n, _p(t), t.size, _p(row_ptr), _p(col_idx), _p(vals)))
    return CsrMatrix(m, n, 0, row_ptr, col_idx, vals)


def csr_to_triplets(a: CsrMatrix) -> np.ndarray:
    """sparse.hpp:173-181 (host enumeration)."""
    rows = np.repeat(np.arange(a.rows, dtype=np.int64), np.diff(a.row_ptr))
    return triplets(rows, a.col_idx.astype(np.int64), a.values)


@dataclass
class GridPartition:
    """sparse.hpp:71-84 — block (i, j) at blocks[j*p + i]."""
    p: int = 1
    q: int = 1
    rows: int = 0
    cols: int = 0
    row_cuts: np.ndarray = field(default_factory=lambda: np.zeros(2, np.int64))
    col_cuts: np.ndarray = field(default_factory=lambda: np.zeros(2, np.int64))
    blocks: list = field(default_factory=list)

    def block(self, i: int, j: int) -> CsrMatrix:
        return self.blocks[j * self.p + i]


def grid_partition(r: CsrMatrix, p: int, q: int) -> GridPartition:
    """sparse.hpp:250-314 (device indexing, bit-exact)."""
    c = r._c()
    rc = np.empty(q + 1, np.int64)
    cc = np.empty(p + 1, np.int64)
    bn = np.empty(p * q, np.int64)
    _check(LIB.alsk_grid_partition_counts(C.byref(c), p, q, _p(rc), _p(cc), _p(bn)))
    blocks, rp, ci, vv = [], [], [], []
    for j in range(q):
        lr = int(rc[j + 1] - rc[j])
        for i in range(p):
            b = CsrMatrix(lr, r.cols, int(cc[i]), np.empty(lr + 1, np.int64),
                          np.empty(int(bn[j * p + i]), np.int32), np.empty(int(bn[j * p + i]), np.float32))
            blocks.append(b)
            rp.append(_p(b.row_ptr))
            ci.append(_p(b.col_idx))
            vv.append(_p(b.values))
    n = p * q
    arr = lambda xs: (C.c_void_p * n)(*xs)  # noqa: E731
    _check(LIB.alsk_grid_partition_fill(C.byref(c), p, q, arr(rp), arr(ci), arr(vv)))
    return GridPartition(p, q, r.rows, r.cols, rc, cc, blocks)


# ---------------------------------------------------------------- solver (solver.hpp)
def get_hermitian_mo_into(r: CsrMatrix, theta: FactorMatrix, cfg: SolverConfig,
                          row_begin: int, row_end: int, out: HermitianBatch) -> None:
    """solver.hpp:292-304"""
    c = r._c()
    count = max(row_end - row_begin, 0)
    out.resize(count, theta.f)
    _check(LIB.alsk_get_hermitian_mo_into(C.byref(c), _p(theta.entries), theta.rows, theta.f,
                                          C.byref(cfg._c()), row_begin, row_end, _p(out.a), _p(out.b)))


def get_hermitian_mo(r: CsrMatrix, theta: FactorMatrix, cfg: SolverConfig) -> HermitianBatch:
    """solver.hpp:309-314"""
    out = HermitianBatch()
    get_hermitian_mo_into(r, theta, cfg, 0, r.rows, out)
    return out


def get_hermitian_base(r: CsrMatrix, theta: FactorMatrix, lam: float,
                       accumulate_double: bool = True) -> HermitianBatch:
    """solver.hpp:277-287"""
    out = HermitianBatch()
    out.resize(r.rows, theta.f)
    c = r._c()
    _check(LIB.alsk_get_hermitian_base(C.byref(c), _p(theta.entries), theta.rows, theta.f, lam,
                                       1 if accumulate_double else 0, _p(out.a), _p(out.b)))
    return out


def local_hermitian(block: CsrMatrix, theta_part: FactorMatrix, cfg: SolverConfig) -> HermitianBatch:
    """parallel.hpp:412-421"""
    out = HermitianBatch()
    out.resize(block.rows, theta_part.f)
    c = block._c()
    _check(LIB.alsk_local_hermitian(C.byref(c), _p(theta_part.entries), theta_part.rows,
                                    theta_part.f, C.byref(cfg._c()), _p(out.a), _p(out.b)))
    return out


def batch_solve(batch: HermitianBatch, policy: BreakdownPolicy = BreakdownPolicy.fail,
                threads: int = 1) -> FactorMatrix:
    """solver.hpp:320-325 (reference-order double Cholesky on the device)."""
    x = FactorMatrix(batch.count, batch.f)
    a = np.ascontiguousarray(batch.a, np.float32)
    b = np.ascontiguousarray(batch.b, np.float32)
    _check(LIB.alsk_batch_solve(_p(a), _p(b), batch.count, batch.f, int(policy), _p(x.entries)))
    return x


def update_x(r: CsrMatrix, theta: FactorMatrix, cfg: SolverConfig) -> FactorMatrix:
    """solver.hpp:330-345"""
    x = FactorMatrix(r.rows, theta.f)
    c = r._c()
    _check(LIB.alsk_update_x(C.byref(c), _p(theta.entries), theta.rows, theta.f, C.byref(cfg._c()),
                             _p(x.entries)))
    return x


def update_theta(r_csc: CscMatrix, x: FactorMatrix, cfg: SolverConfig) -> FactorMatrix:
    """solver.hpp:349-352 — CSC consumed in place as the CSR of R^T (no copy)."""
    theta = FactorMatrix(r_csc.cols, x.f)
    cp = np.ascontiguousarray(r_csc.col_ptr, np.int64)
    ri = np.ascontiguousarray(r_csc.row_idx, np.int32)
    va = np.ascontiguousarray(r_csc.values, np.float32)
    _check(LIB.alsk_update_theta(r_csc.rows, r_csc.cols, r_csc.nnz(), _p(cp), _p(ri), _p(va),
                                 _p(x.entries), x.rows, x.f, C.byref(cfg._c()), _p(theta.entries)))
    return theta


def loss(r: CsrMatrix, x: FactorMatrix, theta: FactorMatrix, lam: float) -> float:
    """solver.hpp:358-390"""
    out = C.c_double()
    c = r._c()
    _check(LIB.alsk_loss(C.byref(c), _p(x.entries), x.rows, _p(theta.entries), theta.rows,
                         theta.f, lam, C.byref(out)))
    return out.value


def rmse(test: np.ndarray, x: FactorMatrix, theta: FactorMatrix) -> float:
    """solver.hpp:393-406"""
    t = np.ascontiguousarray(test, TRIPLET_DTYPE)
    out = C.c_double()
    _check(LIB.alsk_rmse(_p(t), t.size, _p(x.entries), x.rows, _p(theta.entries), theta.rows,
                         theta.f, C.byref(out)))
    return out.value


@dataclass
class IterationMetrics:
    """solver.hpp:409-413"""
    iteration: int = 0
    train_j: float = 0.0
    test_rmse: float = float("nan")


@dataclass
class AlsResult:
    """solver.hpp:415-419"""
    x: FactorMatrix = field(default_factory=FactorMatrix)
    theta: FactorMatrix = field(default_factory=FactorMatrix)
    history: list = field(default_factory=list)


IterationCallback = Callable[[int, FactorMatrix, FactorMatrix], bool]


def als_train(r: CsrMatrix, r_csc: CscMatrix, test: np.ndarray, cfg: SolverConfig, iterations: int,
              callback: Optional[IterationCallback] = None) -> AlsResult:
    """solver.hpp:432-452. Uses a device-resident session (factors stay in HBM between the
    halves); host copies are made only for the callback and the result."""
    from .session import AlsSession  # local import: session pulls torch for device memory
    if iterations < 0:
        raise InputError("iterations must be >= 0")
    if r_csc.rows != r.rows or r_csc.cols != r.cols or r_csc.nnz() != r.nnz():
        raise InputError("csr and csc inputs describe different matrices")
    res = AlsResult(random_factor(r.rows, cfg.f, cfg.seed),
                    random_factor(r.cols, cfg.f, mix_seed(cfg.seed, 1)), [])
    if iterations == 0:
        return res
    sess = AlsSession(r, r_csc, test, cfg, x0=res.x, theta0=res.theta)
    for t in range(1, iterations + 1):
        sess.half_x()
        sess.half_theta()
        m = IterationMetrics(t, sess.loss(), sess.rmse() if test is not None and len(test) else float("nan"))
        res.history.append(m)
        if callback is not None:
            x, th = sess.factors()
            if not callback(t, x, th):
                break
    res.x, res.theta = sess.factors()
    return res


# ---------------------------------------------------------------- scale-up (parallel.hpp)
def slice_cuts(count: int, p: int) -> np.ndarray:
    """parallel.hpp:160-168"""
    base, rem = divmod(count, p)
    return np.concatenate([[0], np.cumsum([base + (1 if i < rem else 0) for i in range(p)])]).astype(np.int64)


def split_factor(whole: FactorMatrix, cuts) -> list:
    """parallel.hpp:390-406"""
    cuts = [int(c) for c in cuts]
    if len(cuts) < 2 or cuts[0] != 0 or cuts[-1] != whole.rows:
        raise InputError("factor cuts must span [0, rows]")
    return [FactorMatrix(cuts[i + 1] - cuts[i], whole.f,
                         whole.entries[cuts[i] * whole.f:cuts[i + 1] * whole.f].copy())
            for i in range(len(cuts) - 1)]


def parallel_reduce(parts: Sequence[HermitianBatch], group_of=None, two_phase: bool = False) -> list:
    """parallel.hpp:474-477 (schedule parallel.hpp:436-465), executed on the device."""
    p = len(parts)
    count, f = parts[0].count, parts[0].f
    for b in parts:
        if b.count != count or b.f != f:
            raise InputError("partial batches disagree on count or rank")
    cuts = slice_cuts(count, p)
    outs = []
    for i in range(p):
        o = HermitianBatch()
        o.resize(int(cuts[i + 1] - cuts[i]), f)
        outs.append(o)
    arr = lambda xs: (C.c_void_p * p)(*xs)  # noqa: E731
    g = None if group_of is None else np.ascontiguousarray(group_of, np.int32)
    _check(LIB.alsk_parallel_reduce(arr([_p(b.a) for b in parts]), arr([_p(b.b) for b in parts]), p, count, f,
                                    _p(g), 1 if two_phase else 0, arr([_p(o.a) for o in outs]),
                                    arr([_p(o.b) for o in outs])))
    return outs


def su_als_update_x(grid: GridPartition, theta_parts: Sequence[FactorMatrix], cfg: SolverConfig,
                    group_of=None, two_phase: bool = False) -> FactorMatrix:
    """parallel.hpp:487-583 on one device (logical workers = grid.p)."""
    if len(theta_parts) != grid.p:
        raise InputError("expected one theta partition per column block")
    f = theta_parts[0].f
    for i, part in enumerate(theta_parts):
        want = int(grid.col_cuts[i + 1] - grid.col_cuts[i])
        if part.rows != want:
            raise InputError(f"theta partition {i} has {part.rows} rows, column cut wants {want}")
        if part.f != f:
            raise InputError("theta partitions disagree on rank")
    blocks = (N.CsrT * (grid.p * grid.q))(*[b._c() for b in grid.blocks])
    x = FactorMatrix(grid.rows, f)
    rc = np.ascontiguousarray(grid.row_cuts, np.int64)
    cc = np.ascontiguousarray(grid.col_cuts, np.int64)
    th = (C.c_void_p * grid.p)(*[_p(t.entries) for t in theta_parts])
    g = None if group_of is None else np.ascontiguousarray(group_of, np.int32)
    _check(LIB.alsk_su_als_update_x(blocks, grid.p, grid.q, _p(rc), _p(cc), th, f, C.byref(cfg._c()), _p(g),
                                    1 if two_phase else 0, _p(x.entries)))
    return x


# ---------------------------------------------------------------- dataio (dataio.hpp)
@dataclass
class SplitResult:
    train: CsrMatrix
    test: np.ndarray


def split_train_test(r: CsrMatrix, holdout_fraction: float, seed: int) -> SplitResult:
    """dataio.hpp:251-290 (host, bit-exact)."""
    c = r._c()
    k = C.c_int64()
    _check(LIB.alsk_split_train_test(C.byref(c), holdout_fraction, seed & (2**64 - 1), C.byref(k),
                                     None, None, None, None))
    kk = k.value
    trp = np.empty(r.rows + 1, np.int64)
    tci = np.empty(r.nnz() - kk, np.int32)
    tv = np.empty(r.nnz() - kk, np.float32)
    test = np.zeros(kk, TRIPLET_DTYPE)
    _check(LIB.alsk_split_train_test(C.byref(c), holdout_fraction, seed & (2**64 - 1), C.byref(k),
                                     _p(trp), _p(tci), _p(tv), _p(test)))
    return SplitResult(CsrMatrix(r.rows, r.cols, 0, trp, tci, tv), test)


def synth_csr(m: int, n: int, nnz: int, seed: int, threads: int = 0) -> CsrMatrix:
    """Deterministic synthetic ratings of a named shape."""
    rp = np.empty(m + 1, np.int64)
    ci = np.empty(nnz, np.int32)
    va = np.empty(nnz, np.float32)
    _check(LIB.alsk_synth_csr(m, n, nnz, seed & (2**64 - 1), threads, _p(rp), _p(ci), _p(va)))
    return CsrMatrix(m, n, 0, rp, ci, va)


# ---------------------------------------------------------------- binary ratings cache
def cache_header(path) -> tuple:
    """(rows, cols, nnz) of a binary ratings cache, after the reference's header checks
    (dataio.hpp:133-150: magic, version, bounds, exact file size)."""
    r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
    _check(LIB.alsk_cache_header(os.fsencode(path), C.byref(r), C.byref(c), C.byref(z)))
    return r.value, c.value, z.value


def save_binary_cache(a: CsrMatrix, path) -> None:
    """dataio.hpp:116-128. col_offset is not part of the format."""
    c = a._c()
    _check(LIB.alsk_save_cache(C.byref(c), os.fsencode(path)))


def load_binary_cache(path) -> CsrMatrix:
    """dataio.hpp:133-163: bit-identical to the saved matrix; truncation, bad magic/version,
    a size mismatch or CSR invariant violations raise IoError naming the file."""
    rows, cols, nnz = cache_header(path)
    rp = np.empty(rows + 1, np.int64)
    ci = np.empty(nnz, np.int32)
    va = np.empty(nnz, np.float32)
    _check(LIB.alsk_load_cache(os.fsencode(path), rows, nnz, _p(rp), _p(ci), _p(va)))
    return CsrMatrix(rows, cols, 0, rp, ci, va)


# ---------------------------------------------------------------- persisted grids (dataio.hpp:352-540)
@dataclass
class GridMeta:
    """dataio.hpp:354-361"""
    p: int = 1
    q: int = 1
    rows: int = 0
    cols: int = 0
    row_cuts: np.ndarray = field(default_factory=lambda: np.zeros(2, np.int64))
    col_cuts: np.ndarray = field(default_factory=lambda: np.zeros(2, np.int64))


@dataclass(frozen=True)
class BlockRef:
    """dataio.hpp:364-369: column partition i, row partition j."""
    i: int = 0
    j: int = 0


def block_path(dir, i: int, j: int) -> str:
    buf = C.create_string_buffer(4096)
    _check(LIB.alsk_block_path(os.fsencode(dir), i, j, buf, len(buf)))
    return os.fsdecode(buf.value)


def persist_grid(grid: GridPartition, dir) -> None:
    """dataio.hpp:381-400: grid.meta plus one binary cache per block."""
    rc = np.ascontiguousarray(grid.row_cuts, np.int64)
    cc = np.ascontiguousarray(grid.col_cuts, np.int64)
    _check(LIB.alsk_persist_grid_meta(os.fsencode(dir), grid.p, grid.q, grid.rows, grid.cols, _p(rc), _p(cc)))
    for j in range(grid.q):
        for i in range(grid.p):
            save_binary_cache(grid.block(i, j), block_path(dir, i, j))


def load_grid_meta(dir) -> GridMeta:
    """dataio.hpp:402-419"""
    p, q = C.c_int(), C.c_int()
    rows, cols = C.c_int64(), C.c_int64()
    _check(LIB.alsk_grid_meta(os.fsencode(dir), C.byref(p), C.byref(q), C.byref(rows), C.byref(cols), None, None))
    rc = np.empty(q.value + 1, np.int64)
    cc = np.empty(p.value + 1, np.int64)
    _check(LIB.alsk_grid_meta(os.fsencode(dir), C.byref(p), C.byref(q), C.byref(rows), C.byref(cols), _p(rc), _p(cc)))
    return GridMeta(p.value, q.value, rows.value, cols.value, rc, cc)


def row_major_order(meta: GridMeta) -> list:
    """dataio.hpp:528-534: row partitions outer, column partitions inner."""
    return [BlockRef(i, j) for j in range(meta.q) for i in range(meta.p)]


# ---------------------------------------------------------------- checkpoints (dataio.hpp:546-708)
class FactorKind(enum.IntEnum):
    """dataio.hpp:548: theta outranks x at the same iteration."""
    x = 0
    theta = 1


@dataclass
class Checkpoint:
    """dataio.hpp:556-561"""
    iteration: int = 0
    which: FactorKind = FactorKind.x
    factor: FactorMatrix = field(default_factory=lambda: FactorMatrix(0, 1, np.zeros(0, np.float32)))
    digest: int = 0


def checkpoint_path(dir, iteration: int, which: FactorKind) -> str:
    buf = C.create_string_buffer(4096)
    _check(LIB.alsk_checkpoint_path(os.fsencode(dir), iteration, int(which), buf, len(buf)))
    return os.fsdecode(buf.value)


def write_checkpoint(cp: Checkpoint, dir) -> str:
    """dataio.hpp:600-624: atomic temp + rename; returns the final path."""
    e = np.ascontiguousarray(cp.factor.entries, np.float32)
    _check(LIB.alsk_checkpoint_write(os.fsencode(dir), cp.iteration, int(cp.which), cp.factor.rows, cp.factor.f,
                                     cp.digest & (2**64 - 1), _p(e)))
    return checkpoint_path(dir, cp.iteration, cp.which)


def checkpoint_header(path) -> tuple:
    it, wh, f = C.c_int(), C.c_int(), C.c_int()
    rows, dg = C.c_int64(), C.c_uint64()
    _check(LIB.alsk_checkpoint_header(os.fsencode(path), C.byref(it), C.byref(wh), C.byref(rows), C.byref(f),
                                      C.byref(dg)))
    return it.value, FactorKind(wh.value), rows.value, f.value, dg.value


def read_checkpoint(path) -> Checkpoint:
    """dataio.hpp:627-651: bit-identical to what was written."""
    it, wh, rows, f, dg = checkpoint_header(path)
    e = np.empty(rows * f, np.float32)
    _check(LIB.alsk_checkpoint_read(os.fsencode(path), e.size, _p(e)))
    return Checkpoint(it, wh, FactorMatrix(rows, f, e), dg)


def latest_checkpoint_path(dir, which: Optional[FactorKind] = None) -> Optional[str]:
    buf = C.create_string_buffer(4096)
    found = C.c_int()
    _check(LIB.alsk_checkpoint_latest(os.fsencode(dir), -1 if which is None else int(which), buf, len(buf),
                                      C.byref(found)))
    return os.fsdecode(buf.value) if found.value else None


def restore_latest(dir, expected_digest: Optional[int] = None) -> Optional[Checkpoint]:
    """dataio.hpp:659-686: newest by (iteration, which); a digest mismatch is an InputError."""
    p = latest_checkpoint_path(dir)
    if p is None:
        return None
    cp = read_checkpoint(p)
    if expected_digest is not None and cp.digest != expected_digest:
        raise InputError(f"{p}: checkpoint config digest mismatch (run has {expected_digest}, checkpoint has "
                         f"{cp.digest})")
    return cp


def restore_latest_of(dir, which: FactorKind) -> Optional[Checkpoint]:
    """dataio.hpp:689-708"""
    p = latest_checkpoint_path(dir, which)
    return None if p is None else read_checkpoint(p)


FP32_ENGINES = {"auto": 0, "ffma": 1, "tensor": 2}


def set_fp32_engine(name: str) -> None:
    """Engine behind accumulate_double=False (ALSK_PREC_FP32): "auto" (tensor cores where
    16 <= f <= 119), "ffma" (CUDA-core kernel) or "tensor"."""
    N.LIB.alsk_set_fp32_engine(FP32_ENGINES[name])


def fp32_engine() -> str:
    v = N.LIB.alsk_fp32_engine()
    return {b: a for a, b in FP32_ENGINES.items()}[v]


class use_fp32_engine:
    """Context manager: run a block with the given FP32 engine, then restore."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        self.prev = fp32_engine()
        set_fp32_engine(self.name)
        return self

    def __exit__(self, *exc):
        set_fp32_engine(self.prev)


def device_available() -> bool:
    return bool(LIB.alsk_device_available())


def kernel_launch_count() -> int:
    return int(LIB.alsk_kernel_launch_count())
