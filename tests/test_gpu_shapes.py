"""Parity at the other named shapes (BASELINE.json configs), on one GPU:

* YahooMusic shape (1,000,990 x 624,961, 252.8M ratings, lambda = 1.4): the FP32 half-sweeps
  against the oracle (our restatement, pinned to the reference) on row samples of both
  halves — users, and items of R^T — computed from the full-size factor; and the full-size
  half-sweeps against the reference-order FP64 mode (normwise 1e-3, test_util.hpp:123-132).
* More than 2^31 nonzeros (int64 row_ptr, sparse.hpp:42): a 2.3e9-rating matrix at f = 16.
  The transpose round trip's row pointers and the FP32 X half are checked against the FP64
  mode at full size, and the rows whose ratings sit beyond offset 2^31 against the oracle.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from helpers import normwise_gap  # noqa: E402

pytestmark = pytest.mark.gpu


def _sample_rows(d, rows):
    """Host CSR of the given rows of a device CSR (local row pointers)."""
    rp = d.row_ptr.cpu().numpy()
    parts_c, parts_v, ptr = [], [], [0]
    for u in rows:
        k0, k1 = int(rp[u]), int(rp[u + 1])
        parts_c.append(d.col_idx[k0:k1].cpu().numpy())
        parts_v.append(d.values[k0:k1].cpu().numpy())
        ptr.append(ptr[-1] + (k1 - k0))
    ci = np.concatenate(parts_c) if parts_c else np.zeros(0, np.int32)
    vv = np.concatenate(parts_v) if parts_v else np.zeros(0, np.float32)
    return np.asarray(ptr, np.int64), ci.astype(np.int32), vv.astype(np.float32)


def _oracle_rows(orc, rows_csr, cols, theta, f, lam):
    from oracle import binding
    rp, ci, vv = rows_csr
    st, x = orc.update_x(binding.csr_struct(len(rp) - 1, cols, rp, ci, vv), theta, cols, f, lam, acc_double=1)
    assert st == 0, orc.last_error()
    return x.reshape(-1, f)


@pytest.mark.timeout(1500)
def test_yahoo_shape_parity(A, orc, gpu):
    import bench
    from paper_1603_03820_b200 import datagen as G
    from paper_1603_03820_b200.session import PREC_FP32, PREC_FP64_EXACT, dev_update
    m, n, nnz, f, lam = bench.CONFIGS["yahoo"]
    assert lam == 1.4
    dev = torch.device("cuda", 0)
    mask = G.holdout_mask(nnz, 0.1, G.split_seed())
    rd = G.build_rank_data("yahoo", 0, 1, dev, mask)
    T0 = torch.from_numpy(A.random_factor(n, f, A.mix_seed(42, 1)).entries).to(dev)
    x32 = torch.empty(m * f, dtype=torch.float32, device=dev)
    x64 = torch.empty_like(x32)
    dev_update(rd.x, T0, n, f, lam, PREC_FP32, x32)
    dev_update(rd.x, T0, n, f, lam, PREC_FP64_EXACT, x64)
    t32 = torch.empty(n * f, dtype=torch.float32, device=dev)
    t64 = torch.empty_like(t32)
    dev_update(rd.t, x32, m, f, lam, PREC_FP32, t32)
    dev_update(rd.t, x32, m, f, lam, PREC_FP64_EXACT, t64)
    gx = normwise_gap(x32.cpu().numpy(), x64.cpu().numpy())
    gt = normwise_gap(t32.cpu().numpy(), t64.cpu().numpy())
    assert gx <= 1e-3 and gt <= 1e-3, (gx, gt)
    # row samples of both halves against the oracle (double accumulation, reference order)
    rng = np.random.default_rng(14)
    users = np.sort(rng.choice(m, 400, replace=False))
    items = np.sort(rng.choice(n, 60, replace=False))
    theta = T0.cpu().numpy()
    xo = _oracle_rows(orc, _sample_rows(rd.x, users), n, theta, f, lam)
    X32 = x32.cpu().numpy().reshape(m, f)
    assert normwise_gap(X32[users], xo) <= 1e-3
    assert np.array_equal(x64.cpu().numpy().reshape(m, f)[users], xo)  # FP64 mode: bit-exact
    to = _oracle_rows(orc, _sample_rows(rd.t, items), m, x32.cpu().numpy(), f, lam)
    assert normwise_gap(t32.cpu().numpy().reshape(n, f)[items], to) <= 1e-3
    assert np.array_equal(t64.cpu().numpy().reshape(n, f)[items], to)


@pytest.mark.timeout(1500)
def test_more_than_2_31_nonzeros(A, orc, gpu):
    """int64 offsets end to end: 2.3e9 ratings (m = 30M, n = 40,000), f = 16."""
    from paper_1603_03820_b200 import datagen as G
    from paper_1603_03820_b200.session import PREC_FP32, PREC_FP64_EXACT, dev_update
    m, n, nnz, f, lam = 30_000_000, 40_000, 2_300_000_000, 16, 0.05
    dev = torch.device("cuda", 0)
    parts = [G.dev_synth_rows(m, n, nnz, 987654321, u0, u1, dev) for u0, u1 in G._chunks(m, nnz, 0, m, 1 << 28)]
    R = G.concat_rows(parts, n, dev)
    del parts
    assert R.nnz == nnz and int(R.row_ptr[-1]) == nnz > 2**31
    RT = R.transpose()
    assert int(RT.row_ptr[-1]) == nnz
    back = RT.transpose()
    assert torch.equal(back.row_ptr, R.row_ptr)
    assert torch.equal(back.col_idx[-1000000:], R.col_idx[-1000000:])
    del back, RT
    T0 = torch.from_numpy(A.random_factor(n, f, 7).entries).to(dev)
    x32 = torch.empty(m * f, dtype=torch.float32, device=dev)
    x64 = torch.empty_like(x32)
    dev_update(R, T0, n, f, lam, PREC_FP32, x32)
    dev_update(R, T0, n, f, lam, PREC_FP64_EXACT, x64)
    g = normwise_gap(x32.cpu().numpy(), x64.cpu().numpy())
    assert g <= 1e-3, g
    # the last rows: their ratings live past offset 2^31
    rp = R.row_ptr.cpu().numpy()
    users = np.arange(m - 300, m)
    assert rp[users[0]] > 2**31
    xo = _oracle_rows(orc, _sample_rows(R, users), n, T0.cpu().numpy(), f, lam)
    assert np.array_equal(x64.cpu().numpy().reshape(m, f)[users], xo)
    assert normwise_gap(x32.cpu().numpy().reshape(m, f)[users], xo) <= 1e-3
