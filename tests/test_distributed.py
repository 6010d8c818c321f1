"""Multi-GPU host logic on CPU: world_size-2 gloo runs of the partitioning model
(tests/mp_model.py, the Python restatement of libalskit_cuda's alsk_mp slicing and
collectives) with the compute steps replaced by CPU stand-ins (the oracle for update_x, numpy for the packed
partial Hermitians). Checks the partitioning, padding, all-gather and reduce-scatter
plumbing: model-parallel halves are bit-identical to one process; the data-parallel
Theta-half matches the single-process update within 1e-6 normwise (double reassociation,
the reference's own SU bound, test_parallel.cpp:329-338)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class HostCsr:
    def __init__(self, rows, cols, rp, ci, vv):
        self.rows, self.cols, self.rp, self.ci, self.vv = rows, cols, rp, ci, vv


def _problem():
    from oracle import binding
    orc = binding.oracle()
    m, n, f, lam = 37, 23, 5, 0.05
    t = orc.random_triplets(2718, m, n, 400)
    st, rp, ci, vv = orc.csr_from_triplets(m, n, t)
    st, cp, ri, cv = orc.csr_to_csc(binding.csr_struct(m, n, rp, ci, vv))
    x0 = orc.random_factor(m, f, 42)
    t0 = orc.random_factor(n, f, orc.mix_seed(42, 1))
    return orc, m, n, f, lam, HostCsr(m, n, rp, ci, vv), HostCsr(n, m, cp, ri, cv), x0, t0


def _cpu_compute():
    from oracle import binding
    from mp_model import Compute
    orc = binding.oracle()

    def update_rows(R, theta, theta_rows, f, lam, precision, rb, re, out):
        rp = (R.rp[rb:re + 1] - R.rp[rb]).copy()
        k0, k1 = int(R.rp[rb]), int(R.rp[re])
        sub = binding.csr_struct(re - rb, R.cols, rp, R.ci[k0:k1].copy(), R.vv[k0:k1].copy())
        st, x = orc.update_x(sub, theta.numpy()[: theta_rows * f].copy(), theta_rows, f, lam, acc_double=1)
        assert st == 0, orc.last_error()
        out[: (re - rb) * f].copy_(torch.from_numpy(x))

    def partial_hermitian(R, theta, theta_rows, f, lam, rb, re, out):
        X = theta.numpy()[: theta_rows * f].reshape(theta_rows, f).astype(np.float64)
        per = f * (f + 1) // 2 + f
        il = np.tril_indices(f)
        for v in range(rb, re):
            k0, k1 = int(R.rp[v]), int(R.rp[v + 1])
            xs = X[R.ci[k0:k1]]
            a = xs.T @ xs + lam * (k1 - k0) * np.eye(f)
            b = xs.T @ R.vv[k0:k1].astype(np.float64)
            o = out[(v - rb) * per:(v - rb + 1) * per].numpy()
            packed = np.empty(per)
            packed[: f * (f + 1) // 2] = a[il[0], il[1]]  # row-major lower: (i, j<=i)
            packed[f * (f + 1) // 2:] = b
            o[:] = packed

    def solve_packed(packed, count, f, out):
        per = f * (f + 1) // 2 + f
        p = packed.numpy()[: count * per].reshape(count, per)
        il = np.tril_indices(f)
        A = np.zeros((count, f, f), np.float32)
        A[:, il[0], il[1]] = p[:, : f * (f + 1) // 2].astype(np.float32)
        A[:, il[1], il[0]] = p[:, : f * (f + 1) // 2].astype(np.float32)
        B = p[:, f * (f + 1) // 2:].astype(np.float32)
        st, x = orc.batch_solve(np.ascontiguousarray(A.reshape(-1)), np.ascontiguousarray(B.reshape(-1)), count, f)
        assert st == 0
        out[: count * f].copy_(torch.from_numpy(x))

    def partial_hermitian_f32(R, theta, theta_rows, f, lam, rb, re, out):
        from paper_1603_03820_b200.distributed import packed_stride
        X = theta.numpy()[: theta_rows * f].reshape(theta_rows, f).astype(np.float64)
        per = packed_stride(f)
        for v in range(rb, re):
            k0, k1 = int(R.rp[v]), int(R.rp[v + 1])
            xs = X[R.ci[k0:k1]]
            a = xs.T @ xs + lam * (k1 - k0) * np.eye(f)
            b = xs.T @ R.vv[k0:k1].astype(np.float64)
            out[(v - rb) * per:(v - rb + 1) * per] = torch.from_numpy(pack_row(a, b, f))

    def solve_packed_f32(packed, count, f, out):
        from paper_1603_03820_b200.distributed import packed_stride
        per = packed_stride(f)
        p = packed.numpy()[: count * per].reshape(count, per)
        A = np.zeros((count, f, f), np.float32)
        B = np.zeros((count, f), np.float32)
        for v in range(count):
            A[v], B[v] = unpack_row(p[v], f)
        st, x = orc.batch_solve(np.ascontiguousarray(A.reshape(-1)), np.ascontiguousarray(B.reshape(-1)), count, f)
        assert st == 0
        out[: count * f].copy_(torch.from_numpy(x))

    return Compute(update_rows, partial_hermitian, solve_packed, partial_hermitian_f32, solve_packed_f32)


def pack_row(a, b, f):
    """The FP32 packed partial row (distributed.packed_stride): compact [lower(A) | b] for
    f <= 15, panel-blocked otherwise."""
    if f <= 15:
        il = np.tril_indices(f)
        return np.concatenate([a[il[0], il[1]], b]).astype(np.float32)
    return pack_panel_blocked(a, b, f)


def unpack_row(row, f):
    if f <= 15:
        na = f * (f + 1) // 2
        il = np.tril_indices(f)
        a = np.zeros((f, f), np.float32)
        a[il[0], il[1]] = row[:na]
        a[il[1], il[0]] = row[:na]
        return a, np.asarray(row[na:na + f], np.float32)
    return unpack_panel_blocked(row, f)


def pack_panel_blocked(a, b, f):
    """The panel-blocked packed row of kernels.cuh: for each 8-column block k, rows 8k..f of
    8 floats (A lower, then b as row f; zeros above the diagonal and at columns >= f)."""
    from paper_1603_03820_b200.distributed import packed_stride
    out = np.zeros(packed_stride(f), np.float32)
    off = 0
    for k in range((f + 7) // 8):
        for i in range(8 * k, f + 1):
            for j in range(8 * k, 8 * k + 8):
                if i < f and j <= i:
                    out[off + 8 * (i - 8 * k) + (j - 8 * k)] = a[i, j]
                elif i == f and j < f:
                    out[off + 8 * (i - 8 * k) + (j - 8 * k)] = b[j]
        off += 8 * (f + 1 - 8 * k)
    return out


def unpack_panel_blocked(row, f):
    a = np.zeros((f, f), np.float32)
    b = np.zeros(f, np.float32)
    off = 0
    for k in range((f + 7) // 8):
        for i in range(8 * k, f + 1):
            for j in range(8 * k, min(8 * k + 8, f)):
                v = row[off + 8 * (i - 8 * k) + (j - 8 * k)]
                if i < f and j <= i:
                    a[i, j] = a[j, i] = v
                elif i == f:
                    b[j] = v
        off += 8 * (f + 1 - 8 * k)
    return a, b


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from mp_model import DataParallelThetaHalf, ModelParallelALS
        from paper_1603_03820_b200.distributed import even_slices
        orc, m, n, f, lam, R, RT, x0, t0 = _problem()
        comp = _cpu_compute()
        mp_als = ModelParallelALS(R, RT, m, n, f, lam, 0, torch.from_numpy(x0), torch.from_numpy(t0), compute=comp)
        for _ in range(2):
            mp_als.step()
        X, T = mp_als.factors()
        # data-parallel Theta half from the model-parallel X: rank r keeps users of its X slab
        cx, xs = even_slices(m, world)
        ub, ue = xs[rank]
        rows, cols = np.repeat(np.arange(m), np.diff(R.rp)), R.ci
        keep = (rows >= ub) & (rows < ue)
        order = np.lexsort((rows[keep], cols[keep]))
        items, users, vals = cols[keep][order], rows[keep][order], R.vv[keep][order]
        rp = np.zeros(n + 1, np.int64)
        np.add.at(rp, items + 1, 1)
        rp = np.cumsum(rp)
        RTl = HostCsr(n, m, rp, users.astype(np.int32), vals.astype(np.float32))
        dp = DataParallelThetaHalf(RTl, m, n, f, lam, compute=comp)
        ct, _ = even_slices(n, world)
        T_dp = torch.zeros(ct * world * f)
        dp.half_theta(X.clone(), T_dp)
        dp32 = DataParallelThetaHalf(RTl, m, n, f, lam, compute=comp, fp32=True)
        T_dp32 = torch.zeros(ct * world * f)
        dp32.half_theta(X.clone(), T_dp32)
        if rank == 0:
            q.put((X.numpy().copy(), T.numpy().copy(), T_dp[: n * f].numpy().copy(), T_dp32[: n * f].numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_model_and_data_parallel_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    X, T, T_dp, T_dp32 = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process oracle run of the same two iterations (driver.hpp:255-262)
    from oracle import binding
    orc, m, n, f, lam, R, RT, x0, t0 = _problem()
    cR = binding.csr_struct(m, n, R.rp, R.ci, R.vv)
    cRT = binding.csr_struct(n, m, RT.rp, RT.ci, RT.vv)
    x, th = x0, t0
    for _ in range(2):
        st, x = orc.update_x(cR, th, n, f, lam)
        st, th = orc.update_x(cRT, x, m, f, lam)
    assert np.array_equal(X, x) and np.array_equal(T, th), "model-parallel must be bit-identical to 1 process"
    st, th_single = orc.update_x(cRT, X, m, f, lam)
    gap = np.abs(T_dp - th_single).max() / np.abs(th_single).max()
    assert gap <= 1e-6, gap
    # FP32 panel-blocked partials, FP32 reduce-scatter: within the FP32 bar
    gap32 = np.linalg.norm(T_dp32 - th_single) / np.linalg.norm(th_single)
    assert gap32 <= 1e-5, gap32


def test_panel_blocked_pack_round_trip():
    from paper_1603_03820_b200.distributed import packed_stride
    rng = np.random.default_rng(3)
    for f in (1, 5, 8, 9, 15, 16, 17, 100):
        m = rng.standard_normal((f, f))
        a = (m @ m.T).astype(np.float32)
        b = rng.standard_normal(f).astype(np.float32)
        row = pack_row(a, b, f)
        assert row.size == packed_stride(f)
        a2, b2 = unpack_row(row, f)
        il = np.tril_indices(f)
        assert np.array_equal(a2[il], a[il]) and np.array_equal(b2, b)


def test_even_slices_and_slice_cuts():
    from paper_1603_03820_b200.distributed import even_slices, slice_cuts
    chunk, sl = even_slices(10, 4)
    assert chunk == 3 and sl == [(0, 3), (3, 6), (6, 9), (9, 10)]
    assert even_slices(2, 4)[1] == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert slice_cuts(5, 4) == [0, 2, 3, 4, 5]
