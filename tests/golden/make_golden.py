"""Generate tests/golden/golden.npz from the UNMODIFIED reference (oracle/_ref, compiled
from /root/reference by oracle/Makefile). Run here (the reference is not on the GPU box):

    python tests/golden/make_golden.py

Every array stored is a reference output on a seeded input that the tests can rebuild
(random_triplets / random_factor are restated bit-exactly in the oracle and pinned below).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import binding  # noqa: E402


def main() -> None:
    ref = binding.reference()
    orc = binding.oracle()
    assert ref is not None, "build oracle/_ref first (make -C oracle)"
    out = {}

    def inst(seed, m, n, nnz, f):
        t = orc.random_triplets(seed, m, n, nnz)
        st, rp, ci, vv = ref.csr_from_triplets(m, n, t)
        assert st == 0
        return t, (rp, ci, vv), ref.random_factor(n, f, seed + 1)

    # hermitian + solve + update_x, double and float accumulation
    for name, (seed, m, n, nnz, f, lam) in {
        "h6": (103, 20, 30, 200, 6, 0.05),
        "h4": (111, 50, 40, 300, 4, 0.1),
        "h13": (131, 40, 60, 500, 13, 1.4),
        "h32": (132, 30, 80, 700, 32, 0.05),
    }.items():
        t, (rp, ci, vv), th = inst(seed, m, n, nnz, f)
        c = binding.csr_struct(m, n, rp, ci, vv)
        out[f"{name}_meta"] = np.array([seed, m, n, nnz, f], np.int64)
        out[f"{name}_lam"] = np.array([lam])
        out[f"{name}_row_ptr"], out[f"{name}_col_idx"], out[f"{name}_values"] = rp, ci, vv
        out[f"{name}_theta"] = th
        for acc in (1, 0):
            st, A, B = ref.hermitian_mo(c, th, n, f, lam, acc, 0, m)
            assert st == 0
            out[f"{name}_A{acc}"], out[f"{name}_B{acc}"] = A, B
            st, X = ref.update_x(c, th, n, f, lam, acc_double=acc)
            assert st == 0, ref.last_error()
            out[f"{name}_X{acc}"] = X
        st, cp, ri, cv = ref.csr_to_csc(c)
        out[f"{name}_col_ptr"], out[f"{name}_row_idx"], out[f"{name}_cvalues"] = cp, ri, cv
        x0 = ref.random_factor(m, f, seed + 2)
        st, L = ref.loss(c, x0, m, th, n, f, lam)
        out[f"{name}_x0"], out[f"{name}_loss"] = x0, np.array([L])
        st, R = ref.rmse(t[: max(1, nnz // 3)].copy(), x0, m, th, n, f)
        out[f"{name}_rmse"] = np.array([R])
        st, g = ref.grid_partition(c, 2, 3)
        rc, cc, blocks = g
        out[f"{name}_grid_row_cuts"], out[f"{name}_grid_col_cuts"] = rc, cc
        for b, (brp, bci, bv) in enumerate(blocks):
            out[f"{name}_grid{b}_row_ptr"], out[f"{name}_grid{b}_col_idx"], out[f"{name}_grid{b}_values"] = brp, bci, bv
        st, sp = ref.split_train_test(c, 0.1, ref.mix_seed(42, 2))
        out[f"{name}_split_row_ptr"], out[f"{name}_split_col_idx"], out[f"{name}_split_values"], test = sp
        out[f"{name}_split_test"] = test.view(np.uint8)
    # seed/init KATs
    out["mix_seed_42_1"] = np.array([ref.mix_seed(42, 1)], np.uint64)
    out["mix_seed_42_2"] = np.array([ref.mix_seed(42, 2)], np.uint64)
    out["random_factor_7x5_9001"] = ref.random_factor(7, 5, 9001)
    path = Path(__file__).resolve().parent / "golden.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
