"""GPU parity: every CUDA entry point, called through the C ABI (Python mirror of the
reference API), against the oracle (pinned to the reference in test_oracle_pinning.py)
and the reference's golden vectors / KATs.

Bars (north star): bit-exact for CSR/CSC/grid/partition indexing and for the
reference-order FP64 path; FP32 path factors within 1e-3 normwise after one half-sweep;
train/test RMSE within 1e-4 absolute after 10 iterations."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from helpers import csr, instance, max_rel_gap, normwise_gap, rel_gap
from oracle import binding

pytestmark = pytest.mark.gpu

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "golden.npz")
CASES = ["h6", "h4", "h13", "h32"]
FP32_TOL = 1e-3  # north star: factors within 1e-3 (normwise, test_util.hpp:123-132) per half-sweep


def gold(A, name):
    seed, m, n, nnz, f = (int(v) for v in GOLD[f"{name}_meta"])
    lam = float(GOLD[f"{name}_lam"][0])
    r = A.CsrMatrix(m, n, 0, GOLD[f"{name}_row_ptr"].copy(), GOLD[f"{name}_col_idx"].copy(),
                    GOLD[f"{name}_values"].copy())
    th = A.FactorMatrix(n, f, GOLD[f"{name}_theta"].copy())
    return seed, m, n, nnz, f, lam, r, th


def rand_csr(A, orc, seed, m, n, nnz, f):
    (rp, ci, vv), th = instance(orc, seed, m, n, nnz, f)
    return A.CsrMatrix(m, n, 0, rp, ci, vv), A.FactorMatrix(n, f, th)


def ocsr(r):
    return binding.csr_struct(r.rows, r.cols, r.row_ptr, r.col_idx, r.values, r.col_offset)


# ------------------------------------------------------------------ Hermitian ------
@pytest.mark.parametrize("name", CASES)
def test_hermitian_fp64_bit_exact_vs_golden(A, gpu, name):
    seed, m, n, nnz, f, lam, r, th = gold(A, name)
    for acc in (True, False):
        h = A.get_hermitian_mo(r, th, A.SolverConfig(f=f, lambda_=lam, accumulate_double=acc))
        if acc:
            assert np.array_equal(h.a, GOLD[f"{name}_A1"]) and np.array_equal(h.b, GOLD[f"{name}_B1"])
        else:  # float accumulation: reference is contraction-sensitive -> tolerance
            assert max_rel_gap(h.a, GOLD[f"{name}_A0"]) < 1e-5
            assert max_rel_gap(h.b, GOLD[f"{name}_B0"]) < 1e-5
        a = h.a.reshape(m, f, f)
        assert np.array_equal(a, a.transpose(0, 2, 1)), "mirror symmetry must be bit-exact"


def test_hermitian_kats(A, gpu):
    # test_solver.cpp:59-71
    r = A.CsrMatrix(1, 1, 0, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([2.0], np.float32))
    th = A.FactorMatrix(1, 1, np.array([3.0], np.float32))
    base = A.get_hermitian_base(r, th, 0.1)
    assert base.a[0] == np.float32(9.1) and base.b[0] == np.float32(6.0)
    # test_solver.cpp:42-57 empty row
    t = A.triplets([0, 2], [0, 1], [1.0, 2.0])
    r = A.csr_from_triplets(3, 2, t)
    th = A.random_factor(2, 4, 5)
    for h in (A.get_hermitian_base(r, th, 0.7), A.get_hermitian_mo(r, th, A.SolverConfig(lambda_=0.7))):
        assert not h.a_at(1).any() and not h.b_at(1).any()


def test_hermitian_discontiguous_gather_row(A, orc, gpu):
    # test_solver.cpp:109-120: one row, 200 ratings over 17,770 columns
    r, th = rand_csr(A, orc, 104, 1, 17770, 200, 4)
    th = A.random_factor(17770, 4, 105)
    h = A.get_hermitian_mo(r, th, A.SolverConfig(lambda_=0.05))
    st, Ao, Bo = orc.hermitian(ocsr(r), th.entries, 17770, 4, 0.05, 1, 0, 1)
    assert np.array_equal(h.a, Ao) and np.array_equal(h.b, Bo)


@pytest.mark.parametrize("f", [1, 7, 10, 31, 64, 100, 127, 150])
def test_hermitian_row_range_and_ranks(A, orc, gpu, f):
    r, th = rand_csr(A, orc, 300 + f, 50, 90, 1200, f)
    out = A.HermitianBatch()
    A.get_hermitian_mo_into(r, th, A.SolverConfig(lambda_=0.05), 7, 41, out)
    st, Ao, Bo = orc.hermitian(ocsr(r), th.entries, 90, f, 0.05, 1, 7, 41)
    assert np.array_equal(out.a, Ao) and np.array_equal(out.b, Bo)


def test_hermitian_errors(A, orc, gpu):
    r, th = rand_csr(A, orc, 108, 5, 4, 8, 3)
    with pytest.raises(A.InputError, match="do not match matrix columns"):
        A.get_hermitian_mo(r, A.random_factor(7, 3, 1), A.SolverConfig())
    with pytest.raises(A.InputError, match="outside matrix"):
        A.get_hermitian_mo_into(r, th, A.SolverConfig(), 2, 9, A.HermitianBatch())
    blk = A.CsrMatrix(1, 10, 4, np.array([0, 2], np.int64), np.array([4, 9], np.int32), np.ones(2, np.float32))
    with pytest.raises(A.InputError, match=r"column 9 outside partition \[4, 7\)"):
        A.local_hermitian(blk, A.random_factor(3, 2, 1), A.SolverConfig())


# ------------------------------------------------------------------ batch solve ----
@pytest.mark.parametrize("name", CASES)
def test_batch_solve_bit_exact(A, orc, gpu, name):
    seed, m, n, nnz, f, lam, r, th = gold(A, name)
    h = A.HermitianBatch(m, f, GOLD[f"{name}_A1"].copy(), GOLD[f"{name}_B1"].copy())
    x = A.batch_solve(h)
    st, xo = orc.batch_solve(h.a, h.b, m, f)
    assert st == 0 and np.array_equal(x.entries, xo)


def test_batch_solve_kats(A, gpu):
    h = A.HermitianBatch()
    h.resize(1, 4)
    for i in range(4):
        h.a_at(0)[i * 4 + i] = 1.0
        h.b_at(0)[i] = i + 1
    assert np.array_equal(A.batch_solve(h).entries, [1, 2, 3, 4])
    h.resize(1, 3)
    assert not A.batch_solve(h).entries.any()
    # test_solver.cpp:205-227
    h.resize(2, 2)
    h.a_at(0)[0], h.a_at(0)[3], h.b_at(0)[0], h.b_at(0)[1] = 2, 2, 4, 2
    h.a_at(1)[0], h.a_at(1)[3], h.b_at(1)[0] = 1, -1, 1
    with pytest.raises(A.NumericalError, match="batch index 1"):
        A.batch_solve(h)
    x = A.batch_solve(h, A.BreakdownPolicy.zero_row)
    assert x.row(0)[0] == np.float32(2.0) and x.row(0)[1] == np.float32(1.0) and not x.row(1).any()


def test_batch_solve_random_spd_residual(A, gpu):
    rng = np.random.default_rng(109)
    for f in (6, 50, 100):
        msrc = rng.random((f, f)) - 0.5
        a = (msrc.T @ msrc + np.eye(f)).astype(np.float32)
        b = (2 * rng.random(f) - 1).astype(np.float32)
        h = A.HermitianBatch(1, f, a.ravel().copy(), b.copy())
        x = A.batch_solve(h).entries.astype(np.float64)
        res = np.abs(a.astype(np.float64) @ x - b).max() / np.abs(b).max()
        assert res < 1e-5


# ------------------------------------------------------------------ update_x -------
@pytest.mark.parametrize("name", CASES)
def test_update_x_fp64_bit_exact_vs_golden(A, gpu, name):
    seed, m, n, nnz, f, lam, r, th = gold(A, name)
    x = A.update_x(r, th, A.SolverConfig(f=f, lambda_=lam, accumulate_double=True))
    assert np.array_equal(x.entries, GOLD[f"{name}_X1"])
    x32 = A.update_x(r, th, A.SolverConfig(f=f, lambda_=lam, accumulate_double=False))
    assert normwise_gap(x32.entries, GOLD[f"{name}_X1"]) <= FP32_TOL


@pytest.mark.parametrize("f", [1, 2, 8, 10, 15, 16, 31, 55, 64, 100, 103, 127, 128, 150])
def test_update_x_ranks_fp64_exact_and_fp32(A, orc, gpu, f):
    m, n = 120, 70
    r, th = rand_csr(A, orc, 500 + f, m, n, 2500, f)
    st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
    assert st == 0
    x = A.update_x(r, th, A.SolverConfig(f=f, lambda_=0.05, accumulate_double=True, batch_rows=33))
    assert np.array_equal(x.entries, xo)
    x32 = A.update_x(r, th, A.SolverConfig(f=f, lambda_=0.05, accumulate_double=False))
    assert normwise_gap(x32.entries, xo) <= FP32_TOL


def test_update_x_netflix_shape_rows(A, orc, gpu):
    """A 3,000-row slice of the Netflix X-half (n=17,770 items, ~186 ratings/row, f=100)
    and a 150-item slice of the Theta-half (~5,575 ratings/item)."""
    f = 100
    for m, n, per in [(3000, 17770, 186), (150, 480189, 5575)]:
        r = A.synth_csr(m, n, m * per, 2024 + m)
        th = A.random_factor(n, f, 42)
        st, xo = orc.update_x(ocsr(r), th.entries, n, f, 0.05, acc_double=1)
        x = A.update_x(r, th, A.SolverConfig(f=f, lambda_=0.05, accumulate_double=True))
        assert np.array_equal(x.entries, xo)
        x32 = A.update_x(r, th, A.SolverConfig(f=f, lambda_=0.05, accumulate_double=False))
        gap = normwise_gap(x32.entries, xo)
        assert gap <= FP32_TOL, gap


def test_update_x_edges(A, orc, gpu):
    # empty rows, a fully empty matrix, zero factors (A == 0 -> x == 0), lambda == 0 rank-1
    r = A.CsrMatrix(4, 3, 0, np.array([0, 0, 2, 2, 3], np.int64), np.array([0, 2, 1], np.int32),
                    np.array([1.0, 2.0, 3.0], np.float32))
    th = A.random_factor(3, 5, 3)
    for acc in (True, False):
        x = A.update_x(r, th, A.SolverConfig(lambda_=0.1, accumulate_double=acc))
        assert not x.row(0).any() and not x.row(2).any()
        z = A.update_x(r, A.FactorMatrix(3, 5), A.SolverConfig(lambda_=0.0, accumulate_double=acc))
        assert not z.entries.any()
    empty = A.CsrMatrix(0, 3, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    assert A.update_x(empty, th, A.SolverConfig()).entries.size == 0
    # test_solver.cpp:229-252 rank-1 recovery with lambda=0
    rng = np.random.default_rng(110)
    m, n = 6, 5
    theta = (0.5 + rng.random(n)).astype(np.float32)
    xs = (0.5 + rng.random(m)).astype(np.float32)
    rows, cols = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    vals = (xs[:, None].astype(np.float64) * theta[None, :]).astype(np.float32)
    r = A.csr_from_triplets(m, n, A.triplets(rows.ravel(), cols.ravel(), vals.ravel()))
    for acc in (True, False):
        got = A.update_x(r, A.FactorMatrix(n, 1, theta), A.SolverConfig(lambda_=0.0, accumulate_double=acc))
        assert max(rel_gap(a, b) for a, b in zip(got.entries, xs)) < 1e-5


def test_update_x_breakdown_message(A, gpu):
    # lambda < 0: row 0 (both unit factors) stays SPD, rows 1 and 2 turn indefinite
    r = A.CsrMatrix(3, 2, 0, np.array([0, 2, 3, 4], np.int64), np.array([0, 1, 1, 0], np.int32),
                    np.ones(4, np.float32))
    th = A.FactorMatrix(2, 2, np.array([1.0, 0.0, 0.0, 1.0], np.float32))
    for acc in (True, False):
        with pytest.raises(A.NumericalError, match="cholesky breakdown at batch index 1"):
            A.update_x(r, th, A.SolverConfig(lambda_=-0.25, accumulate_double=acc, batch_rows=4096))
        with pytest.raises(A.NumericalError, match="cholesky breakdown at batch index 0"):
            A.update_x(r, th, A.SolverConfig(lambda_=-0.25, accumulate_double=acc, batch_rows=1))


def test_update_theta_is_update_x_of_transpose(A, orc, gpu):
    r, _ = rand_csr(A, orc, 114, 30, 20, 180, 4)
    csc = A.csr_to_csc(r)
    x = A.random_factor(30, 4, 115)
    for acc in (True, False):
        cfg = A.SolverConfig(lambda_=0.1, accumulate_double=acc)
        a = A.update_theta(csc, x, cfg)
        b = A.update_x(A.transpose_of(csc), x, cfg)
        assert np.array_equal(a.entries, b.entries) and a.rows == 20


def test_update_x_batch_rows_invariance(A, orc, gpu):
    r, th = rand_csr(A, orc, 113, 40, 30, 250, 5)
    for acc in (True, False):
        a = A.update_x(r, th, A.SolverConfig(lambda_=0.05, batch_rows=1, accumulate_double=acc))
        b = A.update_x(r, th, A.SolverConfig(lambda_=0.05, batch_rows=40, accumulate_double=acc))
        assert np.array_equal(a.entries, b.entries)


# ------------------------------------------------------------------ evaluation -----
@pytest.mark.parametrize("name", CASES)
def test_loss_rmse_vs_golden(A, orc, gpu, name):
    seed, m, n, nnz, f, lam, r, th = gold(A, name)
    x0 = A.FactorMatrix(m, f, GOLD[f"{name}_x0"].copy())
    assert rel_gap(A.loss(r, x0, th, lam), float(GOLD[f"{name}_loss"][0])) < 1e-12
    t = orc.random_triplets(seed, m, n, nnz)[: max(1, nnz // 3)].copy()
    assert rel_gap(A.rmse(t, x0, th), float(GOLD[f"{name}_rmse"][0])) < 1e-12


def test_eval_kats_and_errors(A, gpu):
    r = A.csr_from_triplets(1, 1, A.triplets([0], [0], [1.0]))
    assert A.loss(r, A.FactorMatrix(1, 3), A.FactorMatrix(1, 3), 7.5) == 1.0
    x = A.FactorMatrix(1, 1, np.array([2.0], np.float32))
    t = A.FactorMatrix(1, 1, np.array([1.5], np.float32))
    assert A.rmse(A.triplets([0], [0], [3.0]), x, t) == 0.0
    one = A.FactorMatrix(1, 1, np.array([1.0], np.float32))
    assert A.rmse(A.triplets([0], [0], [3.0]), one, one) == 2.0
    with pytest.raises(A.InputError, match="empty test set"):
        A.rmse(A.triplets([], [], []), one, one)
    with pytest.raises(A.InputError, match=r"test pair \(0, 3\) outside factor shapes"):
        A.rmse(A.triplets([0], [3], [1.0]), one, one)
    with pytest.raises(A.InputError, match="x rows do not match"):
        A.loss(r, A.FactorMatrix(2, 1), one, 0.1)


# ------------------------------------------------------------------ sparse ---------
@pytest.mark.parametrize("name", CASES)
def test_transposes_bit_exact(A, gpu, name):
    seed, m, n, nnz, f, lam, r, th = gold(A, name)
    c = A.csr_to_csc(r)
    assert np.array_equal(c.col_ptr, GOLD[f"{name}_col_ptr"])
    assert np.array_equal(c.row_idx, GOLD[f"{name}_row_idx"])
    assert np.array_equal(c.values, GOLD[f"{name}_cvalues"])
    back = A.csc_to_csr(c)
    assert np.array_equal(back.row_ptr, r.row_ptr) and np.array_equal(back.col_idx, r.col_idx)
    assert np.array_equal(back.values, r.values)


def test_transpose_large_bit_exact(A, orc, gpu):
    r = A.synth_csr(20000, 3000, 2_000_000, 9)
    c = A.csr_to_csc(r)
    st, cp, ri, vv = orc.csr_to_csc(ocsr(r))
    assert np.array_equal(c.col_ptr, cp) and np.array_equal(c.row_idx, ri) and np.array_equal(c.values, vv)
    back = A.csc_to_csr(c)
    assert np.array_equal(back.col_idx, r.col_idx) and np.array_equal(back.values, r.values)


def test_csr_from_triplets(A, orc, gpu):
    t = orc.random_triplets(7, 12, 9, 40)
    a = A.csr_from_triplets(12, 9, t)
    st, rp, ci, vv = orc.csr_from_triplets(12, 9, t)
    assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci) and np.array_equal(a.values, vv)
    b = A.csr_from_triplets(12, 9, np.random.default_rng(3).permutation(t))
    assert np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.values, b.values)
    big = orc.random_triplets(8, 3000, 2000, 200000)
    a = A.csr_from_triplets(3000, 2000, big)
    st, rp, ci, vv = orc.csr_from_triplets(3000, 2000, big)
    assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci) and np.array_equal(a.values, vv)
    with pytest.raises(A.InputError, match=r"\(1, 2\)"):
        A.csr_from_triplets(3, 3, A.triplets([0, 1, 1], [1, 2, 2], [1, 2, 3]))
    for bad in ([0, 2], [-1, 0], [2, 0]):
        with pytest.raises(A.InputError, match="outside 2x2"):
            A.csr_from_triplets(2, 2, A.triplets([bad[0]], [bad[1]], [1.0]))
    assert A.csr_from_triplets(2, 2, A.triplets([], [], [])).row_ptr.tolist() == [0, 0, 0]


@pytest.mark.parametrize("name", CASES)
def test_grid_partition_bit_exact(A, gpu, name):
    seed, m, n, nnz, f, lam, r, th = gold(A, name)
    g = A.grid_partition(r, 2, 3)
    assert np.array_equal(g.row_cuts, GOLD[f"{name}_grid_row_cuts"])
    assert np.array_equal(g.col_cuts, GOLD[f"{name}_grid_col_cuts"])
    for b, blk in enumerate(g.blocks):
        assert np.array_equal(blk.row_ptr, GOLD[f"{name}_grid{b}_row_ptr"])
        assert np.array_equal(blk.col_idx, GOLD[f"{name}_grid{b}_col_idx"])
        assert np.array_equal(blk.values, GOLD[f"{name}_grid{b}_values"])


def test_grid_partition_kats(A, gpu):
    # test_sparse.cpp:161-171: identity 4x4, p=q=2 -> nnz 2/2/0/0... col_offset 2, global col idx
    r = A.csr_from_triplets(4, 4, A.triplets(range(4), range(4), [1, 2, 3, 4]))
    g = A.grid_partition(r, 2, 2)
    assert [b.nnz() for b in g.blocks] == [2, 0, 0, 2]
    assert g.block(1, 1).col_offset == 2 and g.block(1, 1).col_idx.tolist() == [2, 3]
    g1 = A.grid_partition(r, 1, 1)
    assert np.array_equal(g1.blocks[0].col_idx, r.col_idx)
    with pytest.raises(A.InputError, match="q=5 outside"):
        A.grid_partition(r, 1, 5)


# ------------------------------------------------------------------ scale-up -------
def test_parallel_reduce_bit_exact(A, orc, ref, gpu):
    rng = np.random.default_rng(5)
    p, count, f = 4, 11, 3
    parts = [A.HermitianBatch(count, f, rng.standard_normal(count * f * f).astype(np.float32),
                              rng.standard_normal(count * f).astype(np.float32)) for _ in range(p)]
    for two_phase, groups in [(False, None), (True, [0, 0, 1, 1]), (True, [0, 1, 0, 1])]:
        outs = A.parallel_reduce(parts, groups, two_phase)
        st, oa, ob = ref.parallel_reduce([b.a for b in parts], [b.b for b in parts], count, f, groups, two_phase)
        assert st == 0
        for o, a, b in zip(outs, oa, ob):
            assert np.array_equal(o.a, a) and np.array_equal(o.b, b)


def test_local_hermitians_sum_to_whole(A, orc, gpu):
    # test_parallel.cpp:126-158 / acceptance_02
    r, th = rand_csr(A, orc, 127, 30, 40, 300, 4)
    g = A.grid_partition(r, 3, 1)
    parts = A.split_factor(th, g.col_cuts)
    cfg = A.SolverConfig(lambda_=0.05)
    whole = A.get_hermitian_mo(r, th, cfg)
    acc = sum(A.local_hermitian(g.block(i, 0), parts[i], cfg).a.astype(np.float64) for i in range(3))
    assert max_rel_gap(acc, whole.a) < 1e-6


def test_su_als_update_x(A, orc, ref, gpu):
    r, th = rand_csr(A, orc, 133, 60, 48, 900, 6)
    for p, q, two in [(1, 1, 0), (2, 2, 0), (4, 3, 1)]:
        g = A.grid_partition(r, p, q)
        parts = A.split_factor(th, g.col_cuts)
        groups = [0 if i < p // 2 else 1 for i in range(p)] if two else None
        x = A.su_als_update_x(g, parts, A.SolverConfig(lambda_=0.05), groups, bool(two))
        st, xr = ref.su_als_update_x(ocsr(r), th.entries, 48, 6, p, q, 0.05, 1, two)
        assert st == 0 and np.array_equal(x.entries, xr)
        xs = A.update_x(r, th, A.SolverConfig(lambda_=0.05))
        assert normwise_gap(x.entries, xs.entries) < 1e-6


# ------------------------------------------------------------------ end to end -----
def test_als_train_ml1m_shape_rmse_parity(A, orc, gpu):
    """MovieLens-1M shape (6,040 x 3,706, 1,000,209 ratings), f=10, lambda=0.05, 10 iterations:
    the FP64 path reproduces the oracle bit for bit; the FP32 path lands within 1e-4 RMSE."""
    m, n, nnz, f, lam, iters = 6040, 3706, 1000209, 10, 0.05, 10
    R = A.synth_csr(m, n, nnz, A.mix_seed(42, 100))
    sp = A.split_train_test(R, 0.1, A.mix_seed(42, 2))
    train, test = sp.train, sp.test
    csc = A.csr_to_csc(train)
    rt = A.transpose_of(csc)
    # oracle loop (driver.hpp:255-262 order)
    x = orc.random_factor(m, f, 42)
    th = orc.random_factor(n, f, orc.mix_seed(42, 1))
    otrain, ort = ocsr(train), ocsr(rt)
    for _ in range(iters):
        st, x = orc.update_x(otrain, th, n, f, lam, acc_double=1)
        st, th = orc.update_x(ort, x, m, f, lam, acc_double=1)
    st, o_rmse = orc.rmse(test, x, m, th, n, f)
    train_t = A.csr_to_triplets(train)
    st, o_train = orc.rmse(train_t, x, m, th, n, f)
    for acc in (True, False):
        res = A.als_train(train, csc, test, A.SolverConfig(f=f, lambda_=lam, accumulate_double=acc), iters)
        rm = res.history[-1].test_rmse
        tr = A.rmse(train_t, res.x, res.theta)
        if acc:
            assert np.array_equal(res.x.entries, x) and np.array_equal(res.theta.entries, th)
        assert abs(rm - o_rmse) <= 1e-4, (acc, rm, o_rmse)
        assert abs(tr - o_train) <= 1e-4, (acc, tr, o_train)
        js = [h.train_j for h in res.history]
        assert all(b <= a * (1 + 1e-6) for a, b in zip(js, js[1:]))


# ------------------------------------------------------------------ multi-GPU paths, 1 device
def test_distributed_paths_single_device(A, orc, gpu):
    """The C++ multi-GPU session (alsk_mp) at world size 1 on the full device CSRs: the
    MODEL iteration equals update_x/update_theta bit for bit (FP64 exact); the HYBRID session's
    data-parallel Theta half (double partials -> round once -> reference-order solve) is
    bit-identical too, and its FP32 variant (tensor-core panel-blocked partials + TMEM
    Cholesky) lands within the FP32 bar."""
    import torch
    from paper_1603_03820_b200.distributed import HYBRID, MODEL, MultiGpuALS
    from paper_1603_03820_b200.session import DeviceCsr, PREC_FP32, PREC_FP64_EXACT
    r, th = rand_csr(A, orc, 777, 300, 120, 6000, 16)
    dev = torch.device("cuda")
    R = DeviceCsr.from_host(r, dev)
    RT = R.transpose()
    cfg = A.SolverConfig(f=16, lambda_=0.05)
    x1 = A.update_x(r, th, cfg)
    t1 = A.update_theta(A.csr_to_csc(r), x1, cfg)
    t0 = torch.from_numpy(th.entries).to(dev)
    for mode in (MODEL, HYBRID):
        als = MultiGpuALS(None, mode, 300, 120, 16, 0.05, PREC_FP64_EXACT, R, RT, None, t0)
        als.step()
        X, T = als.factors_host()
        als.close()
        assert np.array_equal(X, x1.entries) and np.array_equal(T, t1.entries), mode
    als = MultiGpuALS(None, HYBRID, 300, 120, 16, 0.05, PREC_FP32, R, RT, None, t0)
    als.step()
    X, T = als.factors_host()
    als.close()
    gap = max(normwise_gap(X, x1.entries), normwise_gap(T, t1.entries))
    assert gap <= FP32_TOL and gap <= 5e-5, gap
