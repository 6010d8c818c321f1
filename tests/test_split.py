"""split_train_test on the device (dataio.hpp:251-290): the held-out
positions come from the reference's Fisher-Yates on the host, the CSR compaction runs in
HBM. Bar: bit-identical train CSR and test triplets to the host split (itself pinned to the
reference in test_abi.py / test_oracle_pinning.py) and, where oracle/_ref is built, to the
reference directly; the reference's edge cases (test_dataio.cpp:148-170)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle import binding


def test_fraction_outside_unit_interval_is_an_input_error(A):
    from paper_1603_03820_b200 import _native as N
    r = A.synth_csr(20, 6, 10, 1)
    c = r._c()
    k = C.c_int64()
    for frac in (0.0, 1.0, -0.3):
        st = N.LIB.alsk_dev_split_train_test(C.byref(c), frac, 1, C.byref(k), None, None, None, None, None)
        assert st == 1
        assert N.LIB.alsk_last_error().decode() == "holdout fraction must lie strictly between 0 and 1"
        with pytest.raises(A.InputError, match="^holdout fraction must lie strictly between 0 and 1$"):
            A.split_train_test(r, frac, 1)  # the host split reports the same text
    assert N.LIB.alsk_dev_split_train_test(C.byref(c), 0.25, 1, C.byref(k), None, None, None, None, None) == 0
    assert k.value == 2  # floor(10 * 0.25)


def _dev_split(A, r, frac, seed):
    import torch
    from paper_1603_03820_b200.session import DeviceCsr
    d = DeviceCsr.from_host(r, torch.device("cuda"))
    tr, te = d.split_train_test(frac, seed)
    torch.cuda.synchronize()
    test = np.frombuffer(te.cpu().numpy().tobytes(), dtype=A.TRIPLET_DTYPE)
    return tr, test


def _same(A, tr, test, sp):
    assert np.array_equal(tr.row_ptr.cpu().numpy(), sp.train.row_ptr)
    assert np.array_equal(tr.col_idx.cpu().numpy(), sp.train.col_idx)
    assert tr.values.cpu().numpy().tobytes() == sp.train.values.tobytes()
    assert len(test) == len(sp.test)
    for fld in ("row", "col", "value"):
        assert test[fld].tobytes() == np.ascontiguousarray(sp.test)[fld].tobytes(), fld


@pytest.mark.gpu
@pytest.mark.parametrize("shape,frac,seed", [((22, 30, 300), 0.2, 99), ((500, 80, 9000), 0.1, 7),
                                             ((3000, 2000, 200_000), 0.35, 12345), ((21, 6, 10), 0.01, 7),
                                             ((40, 4000, 40_000), 0.5, 3)])
def test_device_split_matches_the_host_split(A, gpu, shape, frac, seed):
    r = A.synth_csr(*shape, seed)
    tr, test = _dev_split(A, r, frac, seed)
    _same(A, tr, test, A.split_train_test(r, frac, seed))


@pytest.mark.gpu
def test_device_split_matches_the_reference(A, gpu, ref):
    r = A.synth_csr(300, 50, 4000, 5)
    tr, test = _dev_split(A, r, 0.1, A.mix_seed(42, 2))
    st, (trp, tci, tv, rtest) = binding.Oracle.split_train_test(ref,
        binding.csr_struct(r.rows, r.cols, r.row_ptr, r.col_idx, r.values), 0.1, A.mix_seed(42, 2))
    assert st == 0
    assert np.array_equal(tr.row_ptr.cpu().numpy(), trp) and np.array_equal(tr.col_idx.cpu().numpy(), tci)
    assert tr.values.cpu().numpy().tobytes() == tv.tobytes()
    assert test.tobytes() == np.ascontiguousarray(rtest).tobytes()


@pytest.mark.gpu
def test_device_split_full_size(A, gpu):
    """Netflix shape, the bench's split (driver.hpp:113 seed): identical to the host split;
    train and test partition the input exactly."""
    import bench
    m, n, nnz, _, _ = bench.CONFIGS["netflix"]
    r = A.synth_csr(m, n, nnz, A.mix_seed(42, 100 + bench.SHAPE_ID["netflix"]))
    tr, test = _dev_split(A, r, 0.1, A.mix_seed(42, 2))
    sp = A.split_train_test(r, 0.1, A.mix_seed(42, 2))
    _same(A, tr, test, sp)
    assert tr.nnz + len(test) == r.nnz() and len(test) == int(np.floor(0.1 * r.nnz()))
