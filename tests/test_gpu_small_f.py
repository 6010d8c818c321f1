"""GPU parity of the small-rank kernels (f <= 15, FFMA engine): a thread per row when rows
average under 32 ratings, a warp per row otherwise (fused_fp32.cu small_update_kernel),
against the oracle's reference-order update_x. Bars: the north-star FP32 tolerance (1e-3
normwise per half-sweep); empty rows give x = 0 (solver.hpp:215-220)."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import normwise_gap
from oracle import binding

pytestmark = pytest.mark.gpu


def ocsr(r):
    return binding.csr_struct(r.rows, r.cols, r.row_ptr, r.col_idx, r.values, r.col_offset)


def rows_with_lengths(A, lengths, n, seed):
    rng = np.random.default_rng(seed)
    ptr = np.zeros(len(lengths) + 1, np.int64)
    ptr[1:] = np.cumsum(lengths)
    cols = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) if k else np.zeros(0, np.int64)
                           for k in lengths]).astype(np.int32)
    vals = rng.uniform(1.0, 5.0, size=int(ptr[-1])).astype(np.float32)
    return A.CsrMatrix(len(lengths), n, 0, ptr, cols, vals)


@pytest.mark.parametrize("f", [1, 3, 5, 10, 12, 15])
@pytest.mark.parametrize("shape", ["short", "long"])
def test_small_f_update_x(A, orc, gpu, f, shape):
    n = 2000
    if shape == "short":  # thread per row: average < 32 ratings
        lengths = ([0, 1, 2, 3, 5, 8, 13] * 60)[:400]
    else:  # warp per row
        lengths = ([0, 31, 32, 33, 64, 100, 257, 900] * 25)[:200]
    r = rows_with_lengths(A, lengths, n, 500 + f)
    th = A.random_factor(n, f, 3 + f)
    st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
    assert st == 0
    with A.use_fp32_engine("ffma"):
        x = A.update_x(r, th, A.SolverConfig(f=f, lambda_=0.05, accumulate_double=False))
    gap = normwise_gap(x.entries, xo)
    assert gap <= 1e-3, gap
    assert gap <= 1e-5, gap  # FP32 accumulation at these lengths: far inside the bar
    xs = x.entries.reshape(len(lengths), f)
    assert not xs[np.asarray(lengths) == 0].any()


def test_small_f_breakdown_names_the_row(A, gpu):
    # rows of one rating each with a negative ridge: row 0 stays SPD (rating factor 1, lambda
    # -0.25 -> 0.75), row 1's factor is 0.25 -> 0.0625 - 0.25 < 0: "batch index 1"
    f = 1
    th = A.FactorMatrix(2, 1, np.array([1.0, 0.25], np.float32))
    r = A.CsrMatrix(3, 2, 0, np.array([0, 1, 2, 3], np.int64), np.array([0, 1, 1], np.int32),
                    np.ones(3, np.float32))
    with A.use_fp32_engine("ffma"):
        with pytest.raises(A.NumericalError, match="cholesky breakdown at batch index 1"):
            A.update_x(r, th, A.SolverConfig(f=f, lambda_=-0.25, accumulate_double=False))
