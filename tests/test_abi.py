"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every symbol the
header declares, fails loudly without a device, and its host-side helpers (factor init,
seed mixing, holdout split) are bit-exact with the oracle."""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from helpers import csr, instance

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "alskit_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(alsk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(A):
    import ctypes
    lib = ctypes.CDLL(str(A.N.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"declared in include/alskit_cuda.h but not exported: {missing}"
    assert len(declared_symbols()) >= 30


def test_no_cpu_fallback(A):
    if A.device_available():
        pytest.skip("device present")
    r = A.CsrMatrix(1, 1, 0, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([2.0], np.float32))
    th = A.FactorMatrix(1, 1, np.array([3.0], np.float32))
    with pytest.raises(A.DeviceError, match="no CUDA device"):
        A.update_x(r, th, A.SolverConfig(f=1))


def test_host_helpers_bit_exact(A, orc):
    for rows, f, seed in [(7, 5, 9001), (100, 3, 42), (1, 100, A.mix_seed(42, 1))]:
        assert np.array_equal(A.random_factor(rows, f, seed).entries, orc.random_factor(rows, f, seed))
    for s, t in [(42, 1), (42, 2), (0, 0), (2**63, 7)]:
        assert A.mix_seed(s, t) == orc.mix_seed(s, t)
    (rp, ci, vv), _ = instance(orc, 77, 60, 50, 700, 2)
    r = A.CsrMatrix(60, 50, 0, rp, ci, vv)
    sp = A.split_train_test(r, 0.1, A.mix_seed(42, 2))
    st, (trp, tci, tv, test) = orc.split_train_test(csr(60, 50, (rp, ci, vv)), 0.1, orc.mix_seed(42, 2))
    assert np.array_equal(sp.train.row_ptr, trp) and np.array_equal(sp.train.col_idx, tci)
    assert np.array_equal(sp.train.values, tv) and np.array_equal(sp.test.view(np.uint8), test.view(np.uint8))


def test_synthetic_generator_shape_and_determinism(A):
    a = A.synth_csr(1000, 300, 20000, 7, threads=4)
    b = A.synth_csr(1000, 300, 20000, 7, threads=3)
    assert a.row_ptr[-1] == 20000 and np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.values, b.values)
    d = np.diff(a.row_ptr)
    assert d.min() >= 19 and d.max() <= 21
    for u in range(0, 1000, 97):
        seg = a.col_idx[a.row_ptr[u]:a.row_ptr[u + 1]]
        assert np.all(np.diff(seg) > 0) and seg.min() >= 0 and seg.max() < 300


def test_packed_stride_matches_the_python_layout():
    """alsk_packed_stride (C ABI, no device needed) and distributed.packed_stride agree: for
    f <= 15 the compact [lower(A) | b] row of the register kernels, otherwise the panel-blocked
    packed row of kernels.cuh, one 8-float row segment per (block, row)."""
    from paper_1603_03820_b200 import _native as N
    from paper_1603_03820_b200.distributed import packed_stride
    for f in range(1, 131):
        nb = (f + 7) // 8
        want = f * (f + 1) // 2 + f if f <= 15 else sum(8 * (f + 1 - 8 * b) for b in range(nb))
        assert N.LIB.alsk_packed_stride(f) == packed_stride(f) == want
