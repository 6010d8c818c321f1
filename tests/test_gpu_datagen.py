"""The per-rank workload builder (paper_1603_03820_b200/datagen.py) against the host path:
device generator == host generator (alsk_synth_csr) bit for bit; the broadcast holdout mask
applied per row chunk == split_train_test on the whole matrix (dataio.hpp:251-290, itself
pinned to oracle/_ref in test_split.py); every rank's slices (model-parallel item slices of
R^T, hybrid user slabs) == the corresponding rows of the single-process matrices."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

pytestmark = pytest.mark.gpu


def _host(cfg_shape, seed):
    from paper_1603_03820_b200 import alskit as A
    m, n, nnz, f, lam = cfg_shape
    R = A.synth_csr(m, n, nnz, seed)
    sp = A.split_train_test(R, 0.1, A.mix_seed(42, 2))
    return R, sp.train, sp.test


def _np(t):
    return t.cpu().numpy()


def _csr_np(d):
    return _np(d.row_ptr[: d.rows + 1]), _np(d.col_idx[: d.nnz]), _np(d.values[: d.nnz])


@pytest.mark.parametrize("shape", [(500, 300, 20000, 8, 0.05), (97, 1000, 51234, 16, 0.05), (64, 40, 64 * 40, 4, 0.1)])
def test_device_generator_matches_host(shape):
    import torch
    from paper_1603_03820_b200 import alskit as A
    from paper_1603_03820_b200 import datagen as G
    m, n, nnz, f, lam = shape
    R = A.synth_csr(m, n, nnz, 1234)
    dev = torch.device("cuda", 0)
    for rb, re in [(0, m), (0, 1), (m // 3, m // 2 + 1), (m - 1, m), (5, 5)]:
        d = G.dev_synth_rows(m, n, nnz, 1234, rb, re, dev)
        rp, ci, vv = _csr_np(d)
        k0, k1 = int(R.row_ptr[rb]), int(R.row_ptr[re])
        assert np.array_equal(rp, R.row_ptr[rb:re + 1] - k0)
        assert np.array_equal(ci, R.col_idx[k0:k1])
        assert np.array_equal(vv.view(np.uint32), R.values[k0:k1].view(np.uint32))


@pytest.mark.parametrize("world,mode", [(1, "model"), (3, "model"), (3, "hybrid"), (2, "hybrid")])
def test_rank_data_matches_single_process(world, mode):
    import torch
    from paper_1603_03820_b200 import alskit as A
    from paper_1603_03820_b200 import datagen as G
    shape = (700, 90, 700 * 30, 8, 0.05)
    seed = G.data_seed("ml1m")
    R, train, test = _host(shape, seed)
    csc = A.csr_to_csc(train)
    m, n, nnz = shape[:3]
    mask = G.holdout_mask(nnz, 0.1, G.split_seed())
    dev = torch.device("cuda", 0)
    seen_test = []
    for rank in range(world):
        rd = G.build_rank_data("ml1m", rank, world, dev, mask, mode=mode, chunk_nnz=4000, shape=shape)
        rb, re = rd.xs
        cb, ce = rd.ts
        rp, ci, vv = _csr_np(rd.x)
        k0, k1 = int(train.row_ptr[rb]), int(train.row_ptr[re])
        assert np.array_equal(rp, train.row_ptr[rb:re + 1] - k0)
        assert np.array_equal(ci, train.col_idx[k0:k1])
        assert np.array_equal(vv, train.values[k0:k1])
        trp, tci, tvv = _csr_np(rd.t)
        if mode == "model":
            c0, c1 = int(csc.col_ptr[cb]), int(csc.col_ptr[ce])
            assert rd.t.rows == ce - cb and rd.t.cols == m
            assert np.array_equal(trp, csc.col_ptr[cb:ce + 1] - c0)
            assert np.array_equal(tci, csc.row_idx[c0:c1])
            assert np.array_equal(tvv, csc.values[c0:c1])
        else:
            sub = A.CsrMatrix(re - rb, n, 0, train.row_ptr[rb:re + 1] - k0, train.col_idx[k0:k1], train.values[k0:k1])
            sc = A.csr_to_csc(sub)
            assert rd.t.rows == n and rd.t.cols == re - rb
            assert np.array_equal(trp, sc.col_ptr) and np.array_equal(tci, sc.row_idx)
            assert np.array_equal(tvv, sc.values)
        seen_test.append(_np(rd.test).view(A.TRIPLET_DTYPE).reshape(-1))
    allt = np.concatenate(seen_test)
    assert np.array_equal(allt["row"], test["row"]) and np.array_equal(allt["col"], test["col"])
    assert np.array_equal(allt["value"], test["value"])


def test_netflix_shape_device_data_bit_identical():
    """The bench's workload: device generation + mask split + transpose at the full Netflix
    shape equals the host generator + host split + transpose."""
    import torch
    from paper_1603_03820_b200 import alskit as A
    from paper_1603_03820_b200 import datagen as G
    shape = G.CONFIGS["netflix"]
    R, train, test = _host(shape, G.data_seed("netflix"))
    mask = G.holdout_mask(shape[2], 0.1, G.split_seed())
    rd = G.build_rank_data("netflix", 0, 1, torch.device("cuda", 0), mask)
    rp, ci, vv = _csr_np(rd.x)
    assert np.array_equal(rp, train.row_ptr) and np.array_equal(ci, train.col_idx)
    assert np.array_equal(vv, train.values)
    t = _np(rd.test).view(A.TRIPLET_DTYPE).reshape(-1)
    assert np.array_equal(t["row"], test["row"]) and np.array_equal(t["value"], test["value"])
