"""GPU parity of the tensor-core engine (ALSK_PREC_TF32X2, tc_update.cu) against the oracle.

The oracle (pinned to the reference in test_oracle_pinning.py) runs the reference's
default double-accumulation path; the tensor-core kernel must land within the north-star
FP32 bar (factors within 1e-3 normwise after one half-sweep). The Hermitian itself is
checked entry-wise against the double oracle. Row lengths straddle every pipeline
boundary (8-rating k-groups, 32-rating stages, the 4-stage ring), rows outnumber the
persistent CTAs so both epilogue groups and both TMEM buffers cycle, and empty rows,
grid blocks (col_offset) and Cholesky breakdowns take their reference semantics."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import normwise_gap
from oracle import binding

pytestmark = pytest.mark.gpu
FP32_TOL = 1e-3


def ocsr(r):
    return binding.csr_struct(r.rows, r.cols, r.row_ptr, r.col_idx, r.values, r.col_offset)


def rows_with_lengths(A, lengths, n, seed):
    """A CSR whose row u has exactly lengths[u] distinct sorted columns, values in [1,5]."""
    rng = np.random.default_rng(seed)
    ptr = np.zeros(len(lengths) + 1, np.int64)
    ptr[1:] = np.cumsum(lengths)
    cols = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) if k else np.zeros(0, np.int64)
                           for k in lengths]).astype(np.int32)
    vals = rng.uniform(1.0, 5.0, size=int(ptr[-1])).astype(np.float32)
    return A.CsrMatrix(len(lengths), n, 0, ptr, cols, vals)


def tc_update(A, r, th, f, lam):
    with A.use_fp32_engine("tensor"):
        return A.update_x(r, th, A.SolverConfig(f=f, lambda_=lam, accumulate_double=False))


def test_engine_switch(A, gpu):
    prev = A.fp32_engine()
    with A.use_fp32_engine("ffma"):
        assert A.fp32_engine() == "ffma"
    assert A.fp32_engine() == prev


@pytest.mark.parametrize("f", [16, 24, 32, 40, 55, 64, 80, 96, 100, 103, 119])
def test_tc_update_x_ranks(A, orc, gpu, f):
    m, n = 400, 260
    r = A.synth_csr(m, n, 16000, 900 + f)
    th = A.random_factor(n, f, 7 + f)
    st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
    assert st == 0
    x = tc_update(A, r, th, f, 0.05)
    gap = normwise_gap(x.entries, xo)
    assert gap <= FP32_TOL, gap
    # the split keeps FP32-level accuracy; far inside the bar
    assert gap <= 5e-5, gap


@pytest.mark.parametrize("f", [16, 33, 100])
def test_tc_hermitian_entrywise(A, orc, gpu, f):
    from paper_1603_03820_b200.session import PREC_TF32X2, DeviceCsr, dev_hermitian
    m, n = 90, 500
    lengths = [0, 1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 40, 63, 64, 65, 96, 97, 128, 129, 200, 333] * 3
    lengths = lengths[:m] + [37] * (m - len(lengths[:m]))
    r = rows_with_lengths(A, lengths, n, 31 + f)
    th = A.random_factor(n, f, 5)
    st, ao, bo = orc.hermitian(ocsr(r), th.entries, n, f, 0.05, 1, 0, m)
    assert st == 0
    dev = torch.device("cuda")
    R = DeviceCsr.from_host(r, dev)
    T = torch.from_numpy(th.entries).to(dev)
    a = torch.empty(m * f * f, dtype=torch.float32, device=dev)
    b = torch.empty(m * f, dtype=torch.float32, device=dev)
    dev_hermitian(R, T, n, f, 0.05, PREC_TF32X2, a, b)
    a, b = a.cpu().numpy().reshape(m, f, f), b.cpu().numpy().reshape(m, f)
    ao, bo = ao.reshape(m, f, f), bo.reshape(m, f)
    assert np.array_equal(a, np.transpose(a, (0, 2, 1))), "A must be mirrored bit-exactly"
    for u in range(m):
        sa = max(np.abs(ao[u]).max(), 1e-30)
        sb = max(np.abs(bo[u]).max(), 1e-30)
        assert np.abs(a[u] - ao[u]).max() / sa <= 1e-5, (u, lengths[u])
        assert np.abs(b[u] - bo[u]).max() / sb <= 1e-5, (u, lengths[u])


def test_tc_row_lengths_and_empty_rows(A, orc, gpu):
    f, n = 100, 3000
    lengths = ([0, 1, 7, 8, 9, 31, 32, 33, 127, 128, 129, 130, 500, 2049] * 40)
    r = rows_with_lengths(A, lengths, n, 77)
    th = A.random_factor(n, f, 9)
    st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
    x = tc_update(A, r, th, f, 0.05)
    assert normwise_gap(x.entries, xo) <= 5e-5
    xs = x.entries.reshape(len(lengths), f)
    assert not xs[np.asarray(lengths) == 0].any()


def test_tc_netflix_shape_rows(A, orc, gpu):
    """X-half and Theta-half slices of the Netflix shape at f=100, tensor-core engine."""
    f = 100
    for m, n, per in [(3000, 17770, 186), (150, 480189, 5575)]:
        r = A.synth_csr(m, n, m * per, 2024 + m)
        th = A.random_factor(n, f, 42)
        st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
        x = tc_update(A, r, th, f, 0.05)
        gap = normwise_gap(x.entries, xo)
        assert gap <= 5e-5, gap


def test_tc_grid_block_col_offset(A, orc, gpu):
    """A grid block (column-global indices, col_offset = first column of the block) against
    its factor slice: the kernel gathers rows col - col_offset (sparse.hpp:34-37)."""
    f = 48
    r = A.synth_csr(500, 400, 20000, 55)
    g = A.grid_partition(r, 2, 2)
    blk = g.block(1, 1)  # rows of slab 1, columns [col_cuts[1], 400)
    lo = int(blk.col_offset)
    th_full = A.random_factor(400, f, 8)
    th = A.FactorMatrix(400 - lo, f, th_full.entries[lo * f:].copy())
    st, xo = orc.update_x(ocsr(blk), th.entries, th.rows, f, 0.05, acc_double=1)
    assert st == 0
    x = tc_update(A, blk, th, f, 0.05)
    assert normwise_gap(x.entries, xo) <= 5e-5


def test_tc_breakdown_message(A, gpu):
    # identity factors (f=16); lambda=-0.05: row 0 (all 16 columns) has A = (1-0.8) I, SPD;
    # rows 1 and 2 (one column each) turn indefinite -> the first failing row is index 1
    f = 16
    th = np.eye(f, dtype=np.float32)
    rp = np.array([0, f, f + 1, f + 2], np.int64)
    ci = np.concatenate([np.arange(f), [1], [2]]).astype(np.int32)
    r = A.CsrMatrix(3, f, 0, rp, ci, np.ones(len(ci), np.float32))
    with A.use_fp32_engine("tensor"):
        with pytest.raises(A.NumericalError, match="cholesky breakdown at batch index 1"):
            A.update_x(r, A.FactorMatrix(f, f, th.ravel()), A.SolverConfig(f=f, lambda_=-0.05, accumulate_double=False))


def test_tc_engines_agree_on_many_rows(A, orc, gpu):
    """More rows than 2 x 148 persistent CTAs: both engines within the bar of the oracle."""
    f = 64
    r = A.synth_csr(5000, 900, 5000 * 60, 4242)
    th = A.random_factor(900, f, 3)
    st, xo = orc.update_x(ocsr(r), th.entries, 900, f, 0.05, acc_double=1)
    for eng in ("ffma", "tensor"):
        with A.use_fp32_engine(eng):
            x = A.update_x(r, th, A.SolverConfig(f=f, lambda_=0.05, accumulate_double=False))
        assert normwise_gap(x.entries, xo) <= 1e-4, eng


def test_tc_long_rows_segmented_accumulation(A, orc, gpu):
    """Hugewiki-like item degrees (~78K ratings per item, the Theta-half at 3.1e9 ratings over
    39,781 items): rows of 20K-80K ratings span many 512-rating TMEM segments, each drained
    with round-to-nearest adds, so the tensor core's truncating FP32 accumulation cannot
    build up a bias. The factors must stay at FP32-level agreement with the FP64 oracle."""
    f = 100
    lengths = [20000, 40001, 78123, 511, 512, 513]
    n = 200000
    r = rows_with_lengths(A, lengths, n, 2026)
    th = A.random_factor(n, f, 11)
    st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
    assert st == 0
    x = tc_update(A, r, th, f, 0.05)
    gap = normwise_gap(x.entries, xo)
    assert gap <= 5e-5, gap


@pytest.mark.parametrize("f", [16, 37, 100])
def test_tc_partial_hermitian_f32_layout(A, orc, gpu, f):
    """alsk_dev_partial_hermitian_f32 writes the panel-blocked packed rows of kernels.cuh
    (checked entry-wise against the double oracle through the test's own packer), and
    alsk_dev_solve_packed_f32 solves them within the FP32 bar."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_distributed import unpack_panel_blocked
    from paper_1603_03820_b200.distributed import cuda_partial_hermitian_f32, cuda_solve_packed_f32, packed_stride
    from paper_1603_03820_b200.session import DeviceCsr
    m, n = 70, 800
    lengths = [0, 1, 7, 8, 9, 33, 200, 600] * 8 + [5] * 6
    r = rows_with_lengths(A, lengths, n, 99 + f)
    th = A.random_factor(n, f, 17)
    st, ao, bo = orc.hermitian(ocsr(r), th.entries, n, f, 0.05, 1, 0, m)
    assert st == 0
    dev = torch.device("cuda")
    R = DeviceCsr.from_host(r, dev)
    T = torch.from_numpy(th.entries).to(dev)
    from paper_1603_03820_b200 import _native as N
    per = packed_stride(f)
    assert N.LIB.alsk_packed_stride(f) == per
    pk = torch.empty(m * per, dtype=torch.float32, device=dev)
    cuda_partial_hermitian_f32(R, T, n, f, 0.05, 0, m, pk)
    rows = pk.cpu().numpy().reshape(m, per)
    ao, bo = ao.reshape(m, f, f), bo.reshape(m, f)
    for u in range(m):
        a, b = unpack_panel_blocked(rows[u], f)
        sa = max(np.abs(ao[u]).max(), 1e-30)
        assert np.abs(a - ao[u]).max() / sa <= 1e-5, u
        assert np.abs(b - bo[u]).max() / max(np.abs(bo[u]).max(), 1e-30) <= 1e-5, u
    x = torch.empty(m * f, dtype=torch.float32, device=dev)
    cuda_solve_packed_f32(pk, m, f, x)
    st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
    assert normwise_gap(x.cpu().numpy(), xo) <= 5e-5
    assert not x.cpu().numpy().reshape(m, f)[[u for u in range(m) if lengths[u] == 0]].any()


def test_tc_partial_hermitian_f32_grid_block(A, orc, gpu):
    """FP32 partials of a grid block (column-global indices, col_offset = its first column):
    lambda uses the block's own n_u (parallel.hpp:412-421), so the partials of a row's blocks
    add up to the whole row's A_u + lambda n_u I."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_distributed import unpack_panel_blocked
    from paper_1603_03820_b200.distributed import cuda_partial_hermitian_f32, packed_stride
    from paper_1603_03820_b200.session import DeviceCsr
    f, m, n = 24, 300, 500
    r = A.synth_csr(m, n, 12000, 314)
    th_full = A.random_factor(n, f, 2)
    g = A.grid_partition(r, 2, 1)  # two column slabs, all rows (block (i, 0) at blocks[i])
    dev = torch.device("cuda")
    per = packed_stride(f)
    total = np.zeros((m, per), np.float32)
    for i in range(2):
        blk = g.block(i, 0)
        lo, hi = int(g.col_cuts[i]), int(g.col_cuts[i + 1])
        assert int(blk.col_offset) == lo
        T = torch.from_numpy(th_full.entries[lo * f:hi * f].copy()).to(dev)
        pk = torch.empty(m * per, dtype=torch.float32, device=dev)
        cuda_partial_hermitian_f32(DeviceCsr.from_host(blk, dev), T, hi - lo, f, 0.05, 0, m, pk)
        total += pk.cpu().numpy().reshape(m, per)
    st, ao, bo = orc.hermitian(ocsr(r), th_full.entries, n, f, 0.05, 1, 0, m)
    ao, bo = ao.reshape(m, f, f), bo.reshape(m, f)
    for u in range(0, m, 7):
        a, b = unpack_panel_blocked(total[u], f)
        assert np.abs(a - ao[u]).max() <= 1e-5 * max(np.abs(ao[u]).max(), 1e-30), u
        assert np.abs(b - bo[u]).max() <= 1e-5 * max(np.abs(bo[u]).max(), 1e-30), u


@pytest.mark.parametrize("batch_rows", [4096, 2])
def test_tc_error_order_matches_reference(A, ref, gpu, batch_rows):
    """A bad column and a Cholesky breakdown in one update_x on host buffers: the reference
    assembles a whole batch (column check, solver.hpp:120-123) before solving it
    (solver.hpp:230-235), so whichever batch comes first decides the error; the sync-free
    host path resolves its deferred checks in that order. Row 1 breaks down (one rating,
    lambda < 0), row 2 holds column 25 outside the block's partition [4, 20)."""
    f = 16
    th = np.eye(f, dtype=np.float32)
    rp = np.array([0, f, f + 1, f + 3, 2 * f + 3], np.int64)
    ci = np.concatenate([np.arange(4, 20), [5], [6, 25], np.arange(4, 20)]).astype(np.int32)
    vals = np.ones(len(ci), np.float32)
    r = A.CsrMatrix(4, 30, 4, rp, ci, vals)
    cfg = A.SolverConfig(f=f, lambda_=-0.05, accumulate_double=False, batch_rows=batch_rows)
    st, _ = ref.update_x(binding.csr_struct(4, 30, rp, ci, vals, 4), th.ravel(), f, f, -0.05, acc_double=0,
                         batch_rows=batch_rows)
    assert st != 0
    msg = ref.last_error()
    with A.use_fp32_engine("tensor"):
        with pytest.raises(A.Error) as e:
            A.update_x(r, A.FactorMatrix(f, f, th.ravel()), cfg)
    if batch_rows == 4096:
        assert "column 25 outside partition [4, 20)" in msg and isinstance(e.value, A.InputError)
        assert str(e.value) == msg
    else:
        assert "cholesky breakdown at batch index 1" in msg and isinstance(e.value, A.NumericalError)
        assert str(e.value).startswith("cholesky breakdown at batch index 1")


@pytest.mark.parametrize("f", [16, 100])
def test_tc_update_x_factor_without_rows(A, orc, gpu, f):
    """A matrix of zero columns (every row empty) with a 0-row factor: the TMA row map then
    points at a zeroed dummy row and every row solves to zero, as in the reference."""
    m = 300
    r = A.CsrMatrix(m, 0, 0, np.zeros(m + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    th = A.random_factor(0, f, 3)
    x = tc_update(A, r, th, f, 0.05)
    assert x.entries.size == m * f
    assert not np.any(x.entries)


def test_tc_update_x_partial_groups(A, orc, gpu):
    """Row lengths 1..40: every remainder of the 4-row TMA gather groups and of the 8-rating
    k-groups (padding rows gathered past the map arrive as zeros)."""
    f, n = 100, 300
    lengths = [1 + (u % 40) for u in range(600)]
    r = rows_with_lengths(A, lengths, n, 11)
    th = A.random_factor(n, f, 12)
    st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
    assert st == 0
    x = tc_update(A, r, th, f, 0.05)
    assert normwise_gap(x.entries, xo) <= FP32_TOL
