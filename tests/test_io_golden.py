"""IO formats pinned to files the reference itself wrote (tests/golden/make_io_golden.py:
oracle/_ref's save_binary_cache and write_checkpoint, dataio.hpp:116-128 and 600-624).
Runs without oracle/_ref: the repo's loaders must read the reference's bytes exactly, and
its writers must reproduce them byte for byte."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

G = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def gold():
    return np.load(G / "io_golden.npz")


def test_reference_cache_loads_bit_exactly(A, gold):
    a = A.load_binary_cache(G / "ref_ratings.cache")
    assert (a.rows, a.cols) == (int(gold["rows"]), int(gold["cols"]))
    assert np.array_equal(a.row_ptr, gold["row_ptr"]) and np.array_equal(a.col_idx, gold["col_idx"])
    assert a.values.tobytes() == gold["values"].tobytes()


def test_cache_writer_reproduces_the_reference_bytes(A, gold, tmp_path):
    a = A.CsrMatrix(int(gold["rows"]), int(gold["cols"]), 0, gold["row_ptr"], gold["col_idx"], gold["values"])
    A.save_binary_cache(a, tmp_path / "mine.cache")
    assert (tmp_path / "mine.cache").read_bytes() == (G / "ref_ratings.cache").read_bytes()


def test_reference_checkpoint_reads_and_rewrites(A, gold, tmp_path):
    cp = A.read_checkpoint(G / "ref_ckpt_000007_x.bin")
    assert (cp.iteration, cp.which, cp.digest) == (int(gold["iteration"]), A.FactorKind.x, int(gold["digest"]))
    assert (cp.factor.rows, cp.factor.f) == (int(gold["rows"]), int(gold["f"]))
    assert cp.factor.entries.tobytes() == gold["factor"].tobytes()
    p = A.write_checkpoint(cp, tmp_path)
    assert Path(p).read_bytes() == (G / "ref_ckpt_000007_x.bin").read_bytes()
