"""Persisted grids and the out-of-core block stream (dataio.hpp:352-540):

* persist_grid writes grid.meta in the reference's text format plus one binary cache per
  block; load_grid_meta reads it back; corrupt metadata is an IoError;
* (gpu) the device block stream yields every block in plan order, bit-identical to
  grid_partition's (col_offset restored from grid.meta), with the reference's error texts
  ("block (i, j): ..."), and an out-of-core X half over the streamed grid matches the
  in-core tensor-core half-sweep within the FP32 bar.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import normwise_gap


def _grid(A, tmp_path, p=3, q=2, m=400, n=250, nnz=9000, seed=21):
    r = A.synth_csr(m, n, nnz, seed)
    g = A.grid_partition(r, p, q)
    d = tmp_path / "grid"
    A.persist_grid(g, d)
    return r, g, d


@pytest.mark.gpu  # grid_partition runs on the device
def test_persist_and_load_grid_meta(A, gpu, tmp_path):
    r, g, d = _grid(A, tmp_path)
    text = (d / "grid.meta").read_text()
    lines = text.splitlines()
    assert lines[0] == "alskit-grid 1"
    assert lines[1] == f"{g.p} {g.q} {g.rows} {g.cols}"
    assert lines[2] == " ".join(str(int(c)) for c in g.row_cuts)
    assert lines[3] == " ".join(str(int(c)) for c in g.col_cuts)
    meta = A.load_grid_meta(d)
    assert (meta.p, meta.q, meta.rows, meta.cols) == (g.p, g.q, g.rows, g.cols)
    assert np.array_equal(meta.row_cuts, g.row_cuts) and np.array_equal(meta.col_cuts, g.col_cuts)
    for j in range(g.q):
        for i in range(g.p):
            b = A.load_binary_cache(A.block_path(d, i, j))
            want = g.block(i, j)
            assert np.array_equal(b.row_ptr, want.row_ptr) and np.array_equal(b.col_idx, want.col_idx)
            assert b.values.tobytes() == want.values.tobytes()
    assert [(b.i, b.j) for b in A.row_major_order(meta)] == [(i, j) for j in range(2) for i in range(3)]


def test_corrupt_grid_meta(A, tmp_path):
    d = tmp_path / "grid"
    A.persist_grid(A.GridPartition(1, 1, 0, 0, np.zeros(2, np.int64), np.zeros(2, np.int64),
                                   [A.CsrMatrix(0, 0)]), d)
    assert A.load_grid_meta(d).p == 1
    (d / "grid.meta").write_text("alskit-grid 2\n1 1 3 3\n0 3\n0 3\n")
    with pytest.raises(A.IoError, match="grid.meta: corrupt grid metadata"):
        A.load_grid_meta(d)
    (d / "grid.meta").write_text("alskit-grid 1\n2 2 3 3\n0 3\n")
    with pytest.raises(A.IoError, match="corrupt grid metadata"):
        A.load_grid_meta(d)
    with pytest.raises(A.IoError, match="cannot open"):
        A.load_grid_meta(tmp_path / "nothing")


@pytest.mark.gpu
@pytest.mark.parametrize("order", ["row_major", "custom"])
def test_stream_yields_the_grid_blocks(A, gpu, tmp_path, order):
    from paper_1603_03820_b200.session import DeviceBlockStream
    r, g, d = _grid(A, tmp_path)
    meta = A.load_grid_meta(d)
    plan = A.row_major_order(meta) if order == "row_major" else \
        [A.BlockRef(2, 1), A.BlockRef(0, 0), A.BlockRef(2, 1), A.BlockRef(1, 0)]
    seen = []
    with DeviceBlockStream(d, plan) as bs:
        for ref, blk in bs:
            seen.append(ref)
            h = blk.to_host()
            want = g.block(ref.i, ref.j)
            assert (h.rows, h.cols, h.col_offset) == (want.rows, want.cols, want.col_offset)
            assert np.array_equal(h.row_ptr, want.row_ptr) and np.array_equal(h.col_idx, want.col_idx)
            assert h.values.tobytes() == want.values.tobytes()
    assert seen == plan


@pytest.mark.gpu
def test_stream_errors_name_the_block(A, gpu, tmp_path):
    from paper_1603_03820_b200.session import DeviceBlockStream
    _, g, d = _grid(A, tmp_path)
    meta = A.load_grid_meta(d)
    # an out-of-range block surfaces at the next() that would return it, after the blocks
    # planned before it (BlockStream::next, dataio.hpp:498-506)
    got = []
    with pytest.raises(A.InputError, match=r"block \(3, 0\) lies outside the 3x2 grid"):
        with DeviceBlockStream(d, [A.BlockRef(0, 0), A.BlockRef(3, 0)]) as bs:
            for ref, _ in bs:
                got.append(ref)
    assert got == [A.BlockRef(0, 0)]
    missing = A.block_path(d, 1, 1)
    import os
    os.remove(missing)
    got = []
    with pytest.raises(A.IoError) as e:
        with DeviceBlockStream(d, A.row_major_order(meta)) as bs:
            for ref, _ in bs:
                got.append(ref)
    assert str(e.value) == f"block (1, 1): cannot open {missing}"
    assert got == [A.BlockRef(0, 0), A.BlockRef(1, 0), A.BlockRef(2, 0), A.BlockRef(0, 1)]
    A.save_binary_cache(A.CsrMatrix(7, g.cols, 0, np.zeros(8, np.int64)), missing)  # wrong shape for (1, 1)
    with pytest.raises(A.IoError, match=r"block \(1, 1\): shape does not match the grid metadata"):
        with DeviceBlockStream(d, [A.BlockRef(1, 1)]) as bs:
            list(bs)


@pytest.mark.gpu
@pytest.mark.parametrize("p,q", [(1, 1), (3, 2), (4, 5)])
def test_out_of_core_x_half_matches_in_core(A, gpu, tmp_path, p, q):
    import torch
    from paper_1603_03820_b200.session import PREC_FP32, DeviceCsr, dev_update, out_of_core_update_x
    f, lam = 32, 0.05
    r, g, d = _grid(A, tmp_path, p, q, m=3000, n=1200, nnz=120_000, seed=5)
    dev = torch.device("cuda")
    T = torch.from_numpy(A.random_factor(r.cols, f, 9).entries).to(dev)
    x_ooc = torch.zeros(r.rows * f, dtype=torch.float32, device=dev)
    out_of_core_update_x(d, T, f, lam, x_ooc)
    with A.use_fp32_engine("tensor"):
        x_in = torch.zeros_like(x_ooc)
        dev_update(DeviceCsr.from_host(r, dev), T, r.cols, f, lam, PREC_FP32, x_in)
    gap = normwise_gap(x_ooc.cpu().numpy(), x_in.cpu().numpy())
    assert gap <= 1e-3, gap
    assert gap <= 1e-4, gap


def _ocsr(r):
    from oracle import binding
    return binding.csr_struct(r.rows, r.cols, r.row_ptr, r.col_idx, r.values, r.col_offset)


@pytest.mark.gpu
@pytest.mark.parametrize("p,q", [(1, 1), (2, 2), (3, 2), (4, 3)])
def test_out_of_core_fp64_matches_reference_su_als(A, ref, gpu, tmp_path, p, q):
    """FP64-exact out-of-core half-sweeps -- X over the persisted grid of R, Theta over the
    persisted grid of R^T with that X -- are bit-identical to the reference's own
    su_als_update_x (parallel.hpp:487-583) on the same p x q grids."""
    import torch
    from paper_1603_03820_b200.session import PREC_FP64_EXACT, out_of_core_update_x
    f, lam, m, n = 6, 0.05, 150, 70
    r = A.synth_csr(m, n, 2600, 17)
    th = A.random_factor(n, f, 3)
    dev = torch.device("cuda")
    A.persist_grid(A.grid_partition(r, p, q), tmp_path / "gx")
    x = torch.zeros(m * f, dtype=torch.float32, device=dev)
    out_of_core_update_x(tmp_path / "gx", torch.from_numpy(th.entries).to(dev), f, lam, x, PREC_FP64_EXACT)
    st, xr = ref.su_als_update_x(_ocsr(r), th.entries, n, f, p, q, lam, 1, 0)
    assert st == 0 and np.array_equal(x.cpu().numpy(), xr)
    rt = A.transpose_of(A.csr_to_csc(r))
    A.persist_grid(A.grid_partition(rt, p, q), tmp_path / "gt")
    t = torch.zeros(n * f, dtype=torch.float32, device=dev)
    out_of_core_update_x(tmp_path / "gt", x, f, lam, t, PREC_FP64_EXACT)
    st, tr = ref.su_als_update_x(_ocsr(rt), xr, m, f, p, q, lam, 1, 0)
    assert st == 0 and np.array_equal(t.cpu().numpy(), tr)


@pytest.mark.gpu
@pytest.mark.parametrize("f", [10, 24, 100, 130])
def test_out_of_core_fp32_within_bar_of_fp64(A, gpu, tmp_path, f):
    """The FP32 out-of-core path (tensor-core packed partials for 16 <= f <= 119, float
    partials through the reduce otherwise) stays within the FP32 bar of the FP64-exact one."""
    import torch
    from paper_1603_03820_b200.session import PREC_FP32, PREC_FP64_EXACT, out_of_core_update_x
    r, g, d = _grid(A, tmp_path, 3, 2, m=900, n=400, nnz=40_000, seed=8)
    dev = torch.device("cuda")
    T = torch.from_numpy(A.random_factor(r.cols, f, 9).entries).to(dev)
    x32 = torch.zeros(r.rows * f, dtype=torch.float32, device=dev)
    x64 = torch.zeros_like(x32)
    out_of_core_update_x(d, T, f, 0.05, x32, PREC_FP32)
    out_of_core_update_x(d, T, f, 0.05, x64, PREC_FP64_EXACT)
    assert normwise_gap(x32.cpu().numpy(), x64.cpu().numpy()) <= 1e-4


@pytest.mark.gpu
def test_out_of_core_errors(A, gpu, tmp_path):
    """Factor rows must match the grid's columns; a block column outside its slab raises the
    reference's message (solver.hpp:120-123) naming the column."""
    import torch
    from paper_1603_03820_b200.session import PREC_FP32, out_of_core_update_x
    r, g, d = _grid(A, tmp_path, 2, 1, m=40, n=30, nnz=300, seed=2)
    f = 24
    dev = torch.device("cuda")
    x = torch.zeros(r.rows * f, dtype=torch.float32, device=dev)
    with pytest.raises(A.InputError, match="factor rows 29 do not match matrix columns 30"):
        out_of_core_update_x(d, torch.zeros(29 * f, device=dev), f, 0.05, x, PREC_FP32)
    # block (0, 0) holds the columns [0, cut); move one of its entries into slab 1
    cut = int(g.col_cuts[1])
    b00 = A.load_binary_cache(A.block_path(d, 0, 0))
    ci = b00.col_idx.copy()
    u = int(np.argmax(np.diff(b00.row_ptr) > 0))  # a row with entries: its last one moves past the cut
    ci[int(b00.row_ptr[u + 1]) - 1] = cut + 1
    A.save_binary_cache(A.CsrMatrix(b00.rows, b00.cols, 0, b00.row_ptr, ci, b00.values), A.block_path(d, 0, 0))
    with pytest.raises(A.InputError, match=rf"column {cut + 1} outside partition \[0, {cut}\)"):
        out_of_core_update_x(d, torch.zeros(30 * f, device=dev), f, 0.05, x, PREC_FP32)
