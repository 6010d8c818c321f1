"""The batched FP32 SPD solve of panel-blocked packed rows (csrc/warp_solve.cu: one system per
warp, mma.sync Schur updates; replaces batch_solve_into, solver.hpp:204-262, at FP32
tolerance), through alsk_dev_solve_packed_f32 for every block count NB = ceil(f/8) and both
paddings (f % 8 == 0: the augmented row starts a group of its own), checked against a float64
solve; zero systems give x = 0 (solver.hpp:215-220), a non-positive pivot raises the
reference's NumericalError naming the first failing system (solver.hpp:230-235), also when
the diagonal is zero but the matrix is not."""
import numpy as np
import pytest
import torch

from helpers import normwise_gap

pytestmark = pytest.mark.gpu


def pack_panel_blocked(a, b):
    """kernels.cuh pb_block layout: per 8-column block k, rows 8k..f of 8 floats (row f = b)."""
    f = a.shape[0]
    nb = (f + 7) // 8
    out = []
    for k in range(nb):
        blk = np.zeros((f + 1 - 8 * k, 8), np.float32)
        for i in range(8 * k, f + 1):
            for j in range(8 * k, min(8 * k + 8, f)):
                if i < f and j <= i:
                    blk[i - 8 * k, j - 8 * k] = a[i, j]
                elif i == f:
                    blk[i - 8 * k, j - 8 * k] = b[j]
        out.append(blk.ravel())
    return np.concatenate(out)


def spd(rng, f, cond_scale=1.0):
    g = rng.standard_normal((f, f + 8)).astype(np.float64)
    a = g @ g.T / (f + 8) + 0.05 * cond_scale * np.eye(f)
    return a.astype(np.float32)


def solve(count, f, packed):
    from paper_1603_03820_b200.distributed import cuda_solve_packed_f32
    dev = torch.device("cuda")
    pk = torch.from_numpy(packed).to(dev)
    x = torch.empty(count * f, dtype=torch.float32, device=dev)
    cuda_solve_packed_f32(pk, count, f, x)
    return x.cpu().numpy().reshape(count, f)


@pytest.mark.parametrize("f", [16, 17, 23, 24, 25, 31, 32, 33, 40, 63, 64, 65, 96, 99, 100, 101, 104, 111, 112,
                               113, 119, 120, 121, 127, 128])
def test_warp_solve_matches_float64(A, gpu, f):
    from paper_1603_03820_b200.distributed import packed_stride
    rng = np.random.default_rng(1000 + f)
    count = 157  # not a multiple of the warps per CTA; several systems per warp on some SMs
    rows, xs = [], []
    for _ in range(count):
        a = spd(rng, f)
        b = rng.standard_normal(f).astype(np.float32)
        rows.append(pack_panel_blocked(a, b))
        xs.append(np.linalg.solve(a.astype(np.float64), b.astype(np.float64)))
    pk = np.concatenate(rows)
    assert pk.size == count * packed_stride(f)
    x = solve(count, f, pk)
    assert normwise_gap(x, np.array(xs)) <= 1e-4


def test_warp_solve_many_systems_and_zero_rows(A, gpu):
    """More systems than the grid's warps (persistent loop + next-system prefetch); all-zero
    systems (no ratings) give x = 0 without an error."""
    rng = np.random.default_rng(7)
    f, count = 100, 148 * 10 * 3 + 11
    base = [(spd(rng, f), rng.standard_normal(f).astype(np.float32)) for _ in range(16)]
    rows, xs = [], []
    for i in range(count):
        if i % 97 == 5:
            rows.append(pack_panel_blocked(np.zeros((f, f), np.float32), np.zeros(f, np.float32)))
            xs.append(np.zeros(f))
            continue
        a, b = base[i % 16]
        rows.append(pack_panel_blocked(a, b))
        xs.append(np.linalg.solve(a.astype(np.float64), b.astype(np.float64)))
    x = solve(count, f, np.concatenate(rows))
    assert normwise_gap(x, np.array(xs)) <= 1e-4
    assert not x[[i for i in range(count) if i % 97 == 5]].any()


@pytest.mark.parametrize("f,bad_col", [(24, 0), (100, 57), (104, 103)])
def test_warp_solve_breakdown_names_the_first_system(A, gpu, f, bad_col):
    rng = np.random.default_rng(f)
    good = spd(rng, f)
    b = rng.standard_normal(f).astype(np.float32)
    bad = good.copy()
    bad[bad_col, bad_col] = -1.0  # indefinite at (or before) column bad_col
    rows = [pack_panel_blocked(good, b), pack_panel_blocked(good, b), pack_panel_blocked(bad, b),
            pack_panel_blocked(bad, b), pack_panel_blocked(good, b)]
    with pytest.raises(A.NumericalError, match=rf"cholesky breakdown at batch index 2 \(pivot .* at column {bad_col}\)"):
        solve(len(rows), f, np.concatenate(rows))


def test_warp_solve_zero_diagonal_is_a_breakdown_not_a_zero_system(A, gpu):
    """Only an all-zero A is the empty-row case; a zero diagonal with nonzero off-diagonal
    entries is a non-positive pivot at column 0."""
    f = 32
    a = np.zeros((f, f), np.float32)
    a[5, 3] = a[3, 5] = 1.0
    rows = [pack_panel_blocked(np.zeros((f, f), np.float32), np.ones(f, np.float32)), pack_panel_blocked(a, np.ones(f, np.float32))]
    with pytest.raises(A.NumericalError, match=r"cholesky breakdown at batch index 1 \(pivot .* at column 0\)"):
        solve(2, f, np.concatenate(rows))
