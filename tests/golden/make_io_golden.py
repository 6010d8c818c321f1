"""Generate the IO golden files from the reference itself (oracle/_ref, the unmodified
reference compiled by __graft_entry__.build()): a binary ratings cache and an X checkpoint
written by the reference's save_binary_cache / write_checkpoint (dataio.hpp:116-128,
600-624), plus the arrays they hold (io_golden.npz). tests/test_io_golden.py loads them
through the repo's loaders, so the formats stay pinned where oracle/_ref is not built.
usage: python tests/golden/make_io_golden.py"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle import binding  # noqa: E402


def main():
    ref = binding.reference()
    if ref is None:
        raise SystemExit("oracle/_ref is not built (run __graft_entry__.build() here first)")
    rng = np.random.default_rng(20261017)
    m, n = 9, 13
    rows = [np.sort(rng.choice(n, size=int(rng.integers(0, 6)), replace=False)) for _ in range(m)]
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate(rows).astype(np.int32)
    vals = rng.uniform(0.5, 5.0, size=ci.size).astype(np.float32)
    st = ref.save_cache(binding.csr_struct(m, n, rp, ci, vals), str(HERE / "ref_ratings.cache"))
    assert st == 0, ref.last_error()
    f = 5
    fac = rng.standard_normal(m * f).astype(np.float32)
    tmp = HERE / "_ckpt"
    st = ref.write_checkpoint(str(tmp), 7, 0, m, f, 0x0123456789ABCDEF, fac)
    assert st == 0, ref.last_error()
    (tmp / "ckpt_000007_x.bin").replace(HERE / "ref_ckpt_000007_x.bin")
    tmp.rmdir()
    np.savez(HERE / "io_golden.npz", rows=m, cols=n, row_ptr=rp, col_idx=ci, values=vals, f=f, factor=fac,
             iteration=7, digest=np.uint64(0x0123456789ABCDEF))
    print("wrote", HERE / "ref_ratings.cache", HERE / "ref_ckpt_000007_x.bin", HERE / "io_golden.npz")


if __name__ == "__main__":
    main()
