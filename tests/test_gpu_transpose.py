"""The single-pass counting-sort transpose (sparse.cu tr_*; csr_to_csc, sparse.hpp:185-207)
against a host stable sort, bit for bit, on the shapes that stress it: many chunks and tiles,
empty rows (including more row boundaries in one tile than it stages, which takes the
global-search path), duplicate columns inside a row (order of appearance must survive), a
single column holding every entry, a column-skewed matrix (one owner warp doing most of
the work), the shared-memory column-table limit and one past it (radix fallback)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def host_csc(m, n, rp, ci, vv):
    order = np.argsort(ci, kind="stable")
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(rp))
    cp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(ci, minlength=n), out=cp[1:])
    return cp, rows[order].astype(np.int32), vv[order]


def random_csr(rng, m, n, nnz, skew=None, empty_frac=0.0, dup=False):
    rows = np.sort(rng.integers(0, m, nnz))
    if empty_frac:
        keep = rng.random(m) >= empty_frac
        alive = np.flatnonzero(keep)
        rows = np.sort(alive[rng.integers(0, len(alive), nnz)])
    cols = rng.integers(0, n, nnz)
    if skew is not None:
        cols = np.where(rng.random(nnz) < skew, 0, cols)
    # sort columns within each row (CSR invariant); duplicates kept when allowed
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    if not dup:
        keep = np.ones(nnz, bool)
        keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        rows, cols = rows[keep], cols[keep]
    rp = np.zeros(m + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=m), out=rp[1:])
    vv = rng.standard_normal(len(cols)).astype(np.float32)
    return rp, cols.astype(np.int32), vv


def check(A, m, n, rp, ci, vv):
    r = A.CsrMatrix(m, n, 0, rp, ci, vv)
    c = A.csr_to_csc(r)
    cp, ri, cv = host_csc(m, n, rp, ci, vv)
    assert np.array_equal(c.col_ptr, cp)
    assert np.array_equal(c.row_idx, ri)
    assert np.array_equal(c.values.view(np.uint32), cv.view(np.uint32))


@pytest.mark.parametrize("m,n,nnz,kw", [
    (300, 17, 2000, {}),
    (200_000, 17_770, 5_000_000, {}),
    (2_000_000, 1000, 150_000, {"empty_frac": 0.995}),
    (50_000, 44 * 1024, 2_000_000, {}),
    (50_000, 44 * 1024 + 1, 2_000_000, {}),
    (400_000, 1, 400_000, {"dup": True}),
    (100_000, 5000, 3_000_000, {"skew": 0.6}),
    (20_000, 300, 600_000, {"dup": True}),
])
def test_counting_transpose_bit_exact(A, gpu, m, n, nnz, kw):
    rng = np.random.default_rng(m + n + nnz)
    rp, ci, vv = random_csr(rng, m, n, nnz, **kw)
    check(A, m, n, rp, ci, vv)


def test_transpose_round_trip_and_empty(A, gpu):
    rng = np.random.default_rng(9)
    m, n = 70_000, 3000
    rp, ci, vv = random_csr(rng, m, n, 1_500_000)
    r = A.CsrMatrix(m, n, 0, rp, ci, vv)
    back = A.csc_to_csr(A.csr_to_csc(r))
    assert np.array_equal(back.row_ptr, rp) and np.array_equal(back.col_idx, ci)
    assert np.array_equal(back.values.view(np.uint32), vv.view(np.uint32))
    e = A.csr_to_csc(A.CsrMatrix(5, 4, 0, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32)))
    assert np.array_equal(e.col_ptr, np.zeros(5, np.int64))
