"""Host side of the per-rank workload builder (no device needed): the holdout bitmask is the
reference split's held-out set (dataio.hpp:251-290), the generator's row offsets, and the mask
popcount used to size each chunk's test triplets."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def test_holdout_mask_is_the_reference_split():
    from oracle import binding
    from paper_1603_03820_b200 import alskit as A
    from paper_1603_03820_b200 import datagen as G
    m, n, nnz = 300, 200, 9000
    R = A.synth_csr(m, n, nnz, 77)
    seed = A.mix_seed(42, 2)
    mask = G.holdout_mask(nnz, 0.1, seed)
    held = np.unpackbits(mask.view(np.uint8), bitorder="little")[:nnz].astype(bool)
    ref = binding.reference()
    if ref is not None:
        st, (trp, tci, tvv, test) = ref.split_train_test(binding.csr_struct(m, n, R.row_ptr, R.col_idx, R.values),
                                                          0.1, seed)
        assert st == 0
    else:
        sp = A.split_train_test(R, 0.1, seed)
        trp, tci, tvv = sp.train.row_ptr, sp.train.col_idx, sp.train.values
    assert held.sum() == int(0.1 * nnz)
    assert np.array_equal(R.col_idx[~held], tci) and np.array_equal(R.values[~held], tvv)
    rows = np.repeat(np.arange(m), np.diff(R.row_ptr))
    kept_per_row = np.bincount(rows[~held], minlength=m)
    assert np.array_equal(np.concatenate([[0], np.cumsum(kept_per_row)]), trp)
    for b0, b1 in [(0, nnz), (3, 77), (32, 64), (100, 100), (8999, 9000)]:
        assert int(G.LIB.alsk_mask_count(mask.ctypes.data, b0, b1)) == int(held[b0:b1].sum())


def test_row_offsets():
    from paper_1603_03820_b200 import alskit as A
    from paper_1603_03820_b200 import datagen as G
    R = A.synth_csr(97, 1000, 51234, 5)
    assert all(G.row_start(97, 51234, u) == R.row_ptr[u] for u in range(98))
    m, nnz = G.CONFIGS["sparkals"][0], G.CONFIGS["sparkals"][2]
    assert G.row_start(m, nnz, m) == nnz and G.row_start(m, nnz, m // 2) == nnz * (m // 2) // m
