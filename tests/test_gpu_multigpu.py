"""The C++ multi-GPU session (alsk_mp_*, csrc/multigpu.cu) and its communicators, on one GPU.

* world 1 (no communicator): the MODEL session's iteration is the single-GPU update_x /
  update_theta — bit-identical to the host API in FP32 (same kernels, batching-independent
  rows) and to the oracle in FP64-exact mode; the HYBRID session's data-parallel Theta half
  (partials -> solve) is within the FP32 bar of the oracle for f = 10 (register partials) and
  f = 16 / 100 (tensor-core partials), and bit-identical to update_x in FP64 mode.
* world 2 on one GPU: two processes drive their own rank's session on the same device with
  the collectives over a host transport (alsk_comm_init_custom + gloo; NCCL refuses two
  ranks on one device). MODEL is bit-identical to world 1; HYBRID matches within 1e-6 (FP64:
  double reassociation, the reference's SU bound test_parallel.cpp:329-338) / the FP32 bar.
* NCCL: libalskit_cuda loads it, and a one-rank NCCL communicator runs its collectives.
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import normwise_gap

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

pytestmark = pytest.mark.gpu


def _problem(m, n, nnz, f, seed=5):
    from oracle import binding
    orc = binding.oracle()
    t = orc.random_triplets(seed, m, n, nnz)
    st, rp, ci, vv = orc.csr_from_triplets(m, n, t)
    assert st == 0
    th = orc.random_factor(n, f, orc.mix_seed(42, 1))
    return orc, (rp, ci, vv), th


def _slices(rp, ci, vv, m, n, rank, world):
    """This rank's MODEL slices: CSR rows [xb, xe) and R^T rows [tb, te) (host arrays)."""
    from oracle import binding
    orc = binding.oracle()
    cx, ct = -(-m // world), -(-n // world)
    xb, xe = min(m, rank * cx), min(m, (rank + 1) * cx)
    tb, te = min(n, rank * ct), min(n, (rank + 1) * ct)
    st, cp, ri, cv = orc.csr_to_csc(binding.csr_struct(m, n, rp, ci, vv))
    x = (rp[xb:xe + 1] - rp[xb], ci[rp[xb]:rp[xe]], vv[rp[xb]:rp[xe]])
    t = (cp[tb:te + 1] - cp[tb], ri[cp[tb]:cp[te]], cv[cp[tb]:cp[te]])
    return (xb, xe, x), (tb, te, t)


def _hybrid_t(rp, ci, vv, m, n, xb, xe):
    """Every item's ratings from users [xb, xe), user ids local to the slab."""
    rows = np.repeat(np.arange(m), np.diff(rp))
    keep = (rows >= xb) & (rows < xe)
    order = np.lexsort((rows[keep], ci[keep]))
    items, users, vals = ci[keep][order], rows[keep][order] - xb, vv[keep][order]
    tp = np.zeros(n + 1, np.int64)
    np.add.at(tp, items + 1, 1)
    return np.cumsum(tp), users.astype(np.int32), vals.astype(np.float32)


def _run(m, n, f, lam, prec, mode, rank, world, arrs, th, comm, iters=2):
    import torch
    from paper_1603_03820_b200.distributed import HYBRID, MultiGpuALS
    from paper_1603_03820_b200.session import DeviceCsr
    dev = torch.device("cuda", 0)
    rp, ci, vv = arrs
    (xb, xe, x), (tb, te, t) = _slices(rp, ci, vv, m, n, rank, world)
    X = DeviceCsr(xe - xb, n, *x, dev)
    if mode == HYBRID:
        T = DeviceCsr(n, xe - xb, *_hybrid_t(rp, ci, vv, m, n, xb, xe), dev)
    else:
        T = DeviceCsr(te - tb, m, *t, dev)
    als = MultiGpuALS(comm, mode, m, n, f, lam, prec, X, T, None, torch.from_numpy(th).to(dev))
    for _ in range(iters):
        als.step()
    Xh, Th = als.factors_host()
    als.close()
    return Xh, Th


def _oracle_iters(orc, m, n, f, lam, arrs, th, iters=2, acc_double=1):
    from oracle import binding
    rp, ci, vv = arrs
    st, cp, ri, cv = orc.csr_to_csc(binding.csr_struct(m, n, rp, ci, vv))
    R, RT = binding.csr_struct(m, n, rp, ci, vv), binding.csr_struct(n, m, cp, ri, cv)
    x, t = None, th
    for _ in range(iters):
        st, x = orc.update_x(R, t, n, f, lam, acc_double=acc_double)
        st, t = orc.update_x(RT, x, m, f, lam, acc_double=acc_double)
    return x, t


@pytest.mark.parametrize("f", [10, 16, 100])
def test_mp_model_world1_matches_single_gpu(A, gpu, f):
    from paper_1603_03820_b200.distributed import MODEL
    from paper_1603_03820_b200.session import PREC_FP32, PREC_FP64_EXACT
    m, n, lam = 301, 127, 0.05
    orc, arrs, th = _problem(m, n, 7000, f)
    # FP32: the host API's update_x / update_theta run the same kernels
    X, T = _run(m, n, f, lam, PREC_FP32, MODEL, 0, 1, arrs, th, None, iters=1)
    r = A.CsrMatrix(m, n, 0, *arrs)
    cfg = A.SolverConfig(f=f, lambda_=lam, accumulate_double=False)
    x1 = A.update_x(r, A.FactorMatrix(n, f, th), cfg)
    t1 = A.update_theta(A.csr_to_csc(r), x1, cfg)
    assert np.array_equal(X, x1.entries) and np.array_equal(T, t1.entries)
    # FP64 exact: bit-identical to the oracle
    X, T = _run(m, n, f, lam, PREC_FP64_EXACT, MODEL, 0, 1, arrs, th, None, iters=2)
    xo, to = _oracle_iters(orc, m, n, f, lam, arrs, th, iters=2)
    assert np.array_equal(X, xo) and np.array_equal(T, to)


@pytest.mark.parametrize("f", [10, 16, 100])
def test_mp_hybrid_world1(A, gpu, f):
    """The data-parallel Theta half at one rank: packed partials (register kernel for f <= 15,
    tensor cores otherwise) -> solve, against the oracle's iteration."""
    from paper_1603_03820_b200.distributed import HYBRID
    from paper_1603_03820_b200.session import PREC_FP32, PREC_FP64_EXACT
    m, n, lam = 400, 90, 0.05
    orc, arrs, th = _problem(m, n, 9000, f, seed=11)
    xo, to = _oracle_iters(orc, m, n, f, lam, arrs, th, iters=2)
    X, T = _run(m, n, f, lam, PREC_FP32, HYBRID, 0, 1, arrs, th, None, iters=2)
    assert normwise_gap(X, xo) <= 1e-4 and normwise_gap(T, to) <= 1e-4, (normwise_gap(X, xo), normwise_gap(T, to))
    X, T = _run(m, n, f, lam, PREC_FP64_EXACT, HYBRID, 0, 1, arrs, th, None, iters=2)
    assert np.array_equal(X, xo) and np.array_equal(T, to)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, cases):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1603_03820_b200.distributed import HostTransportComm
        comm = HostTransportComm.from_process_group(0)
        out = []
        for (m, n, nnz, f, lam, prec, mode) in cases:
            orc, arrs, th = _problem(m, n, nnz, f, seed=17)
            X, T = _run(m, n, f, lam, prec, mode, rank, world, arrs, th, comm, iters=2)
            out.append((X, T))
        q.put((rank, out))
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_mp_world2_on_one_gpu_host_transport(A, gpu):
    import torch.multiprocessing as mp
    from paper_1603_03820_b200.distributed import HYBRID, MODEL
    from paper_1603_03820_b200.session import PREC_FP32, PREC_FP64_EXACT
    cases = [(333, 121, 8000, 16, 0.05, PREC_FP32, MODEL), (333, 121, 8000, 100, 0.05, PREC_FP32, MODEL),
             (333, 121, 8000, 10, 0.05, PREC_FP32, MODEL), (333, 121, 8000, 16, 0.05, PREC_FP64_EXACT, MODEL),
             (500, 97, 9000, 10, 0.05, PREC_FP32, HYBRID), (500, 97, 9000, 32, 0.05, PREC_FP32, HYBRID),
             (500, 97, 9000, 12, 0.05, PREC_FP64_EXACT, HYBRID)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, cases)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (m, n, nnz, f, lam, prec, mode) in enumerate(cases):
        X1, T1 = _run(m, n, f, lam, prec, mode, 0, 1, *_problem(m, n, nnz, f, seed=17)[1:], None, iters=2)
        if mode == MODEL:
            for r in (0, 1):
                X2, T2 = res[r][i]
                assert np.array_equal(X2, X1) and np.array_equal(T2, T1), f"case {i} rank {r}"
        else:
            # X slabs of both ranks stacked == the one-rank X; Theta replicated
            Xs = np.concatenate([res[0][i][0][: (-(-m // 2)) * f], res[1][i][0][: (m - (-(-m // 2))) * f]])
            tol = 1e-6 if prec == PREC_FP64_EXACT else 5e-5
            for r in (0, 1):
                assert normwise_gap(res[r][i][1], T1) <= tol, (i, r, normwise_gap(res[r][i][1], T1))
            assert normwise_gap(Xs, X1) <= tol, (i, normwise_gap(Xs, X1))


def test_nccl_loads_and_one_rank_communicator_runs(A, gpu):
    import ctypes as C
    import torch
    from paper_1603_03820_b200 import _native as N
    assert N.LIB.alsk_comm_available() == 1, "libalskit_cuda could not load NCCL"
    assert N.LIB.alsk_nccl_version() >= 22000
    uid = (C.c_uint8 * 128)()
    assert N.LIB.alsk_comm_unique_id(uid) == 0
    h = C.c_void_p()
    assert N.LIB.alsk_comm_init_rank(uid, 1, 0, 0, C.byref(h)) == 0, N.LIB.alsk_last_error()
    buf = torch.arange(12, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert N.LIB.alsk_comm_allgather(h, buf.data_ptr(), 12, 0, s) == 0
    out = torch.empty(12, dtype=torch.float32, device="cuda")
    assert N.LIB.alsk_comm_reduce_scatter(h, buf.data_ptr(), out.data_ptr(), 12, 0, s) == 0
    assert N.LIB.alsk_comm_wait(h, s, 30.0) == 0
    assert torch.equal(out, buf)
    N.LIB.alsk_comm_destroy(h)
