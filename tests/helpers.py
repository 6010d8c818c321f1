"""Test helpers: reference-test instances rebuilt seed for seed, and the reference's
comparison metrics (tests/test_util.hpp:109-132)."""
from __future__ import annotations

import numpy as np

from oracle import binding


def rel_gap(a: float, b: float) -> float:
    scale = max(abs(a), abs(b), 1e-30)
    return abs(a - b) / scale


def max_rel_gap(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-30)
    return float((np.abs(a - b) / scale).max(initial=0.0))


def normwise_gap(a, b) -> float:
    """max|a-b| / max|b| (test_util.hpp:123-132)"""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max(initial=0.0) / max(np.abs(b).max(initial=0.0), 1e-30))


def instance(orc, seed, m, n, nnz, f):
    """random_instance (test_solver.cpp:29-36): CSR of random_triplets + random_factor(n, f, seed+1)."""
    t = orc.random_triplets(seed, m, n, nnz)
    st, rp, ci, vv = orc.csr_from_triplets(m, n, t)
    assert st == 0
    theta = orc.random_factor(n, f, seed + 1)
    return (rp, ci, vv), theta


def csr(m, n, arrs, col_offset=0):
    rp, ci, vv = arrs
    return binding.csr_struct(m, n, rp, ci, vv, col_offset)


def synth_split(cfg: str):
    """The bench's input on the host: the shared synthetic generator's matrix for a named
    shape (bench.CONFIGS) and the reference driver's split (driver.hpp:113)."""
    import bench
    from paper_1603_03820_b200 import alskit as A
    m, n, nnz, f, lam = bench.CONFIGS[cfg]
    R = A.synth_csr(m, n, nnz, bench.data_seed(cfg))
    sp = A.split_train_test(R, 0.1, A.mix_seed(42, 2))
    return sp.train, sp.test
