"""Probe (not a test): where the host-buffer iteration (alsk_update_x + alsk_update_theta on
pinned host buffers, bench.py's e2e leg) spends its time at the Netflix shape: wall time of
each call, the same halves device-resident (alsk_dev_update_*), and the raw pinned H2D / D2H
rates of the bytes each call moves. usage: python scripts/probes/e2e_breakdown.py [reps=5]"""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_03820_b200 import _native as N  # noqa: E402
from paper_1603_03820_b200 import alskit as A  # noqa: E402
from paper_1603_03820_b200 import datagen as G  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
m, n, nnz, f, lam = bench.CONFIGS["netflix"]
dev = torch.device("cuda", 0)
mask = G.holdout_mask(nnz, 0.1, G.split_seed())
rd = G.build_rank_data("netflix", 0, 1, dev, mask)
x, t = rd.x, rd.t
pin = lambda a: a.cpu().pin_memory()  # noqa: E731
rp, ci, vv = pin(x.row_ptr[: x.rows + 1]), pin(x.col_idx[: x.nnz]), pin(x.values[: x.nnz])
cp, ri, cv = pin(t.row_ptr[: t.rows + 1]), pin(t.col_idx[: t.nnz]), pin(t.values[: t.nnz])
theta_h = pin(torch.from_numpy(A.random_factor(n, f, A.mix_seed(42, 1)).entries))
X = torch.zeros(m * f, dtype=torch.float32).pin_memory()
T = theta_h.clone().pin_memory()
csr = N.CsrT(m, n, 0, x.nnz, rp.data_ptr(), ci.data_ptr(), vv.data_ptr())
cfg = N.SolverConfigT(f, lam, 16, 4096, 0, 0, 42)


def wall(fn):
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts[1:]))


ux = wall(lambda: A._check(N.LIB.alsk_update_x(C.byref(csr), T.data_ptr(), n, f, C.byref(cfg), X.data_ptr())))
ut = wall(lambda: A._check(N.LIB.alsk_update_theta(m, n, x.nnz, cp.data_ptr(), ri.data_ptr(), cv.data_ptr(),
                                                   X.data_ptr(), m, f, C.byref(cfg), T.data_ptr())))
# raw copies of the same bytes
dx = [torch.empty_like(a, device=dev) for a in (rp, ci, vv)]
dt = [torch.empty_like(a, device=dev) for a in (cp, ri, cv)]
dX = torch.empty(m * f, dtype=torch.float32, device=dev)


def h2d(srcs, dsts):
    for s_, d_ in zip(srcs, dsts):
        d_.copy_(s_, non_blocking=True)


bx = sum(a.nbytes for a in (rp, ci, vv)) + theta_h.nbytes
bt = sum(a.nbytes for a in (cp, ri, cv)) + X.nbytes
cx = wall(lambda: h2d([rp, ci, vv], dx))
ct = wall(lambda: h2d([cp, ri, cv, X], dt + [dX]))
d2h = wall(lambda: X.copy_(dX, non_blocking=True))
print(f"alsk_update_x {ux:.1f} ms | alsk_update_theta {ut:.1f} ms | sum {ux + ut:.1f} ms")
print(f"H2D X-half inputs {bx / 1e9:.3f} GB in {cx:.1f} ms ({bx / cx / 1e6:.1f} GB/s); "
      f"Theta-half inputs {bt / 1e9:.3f} GB in {ct:.1f} ms ({bt / ct / 1e6:.1f} GB/s); D2H X {X.nbytes / d2h / 1e6:.1f} GB/s")

# device-resident X half (alsk_dev_update, default scratch), alone, in 9 ranges, and with a
# concurrent pinned H2D stream of the same bytes
from paper_1603_03820_b200.session import PREC_FP32, dev_update  # noqa: E402

Td = theta_h.to(dev)
Xd = torch.empty(m * f, dtype=torch.float32, device=dev)
cuts = [0] + [int(np.searchsorted(rp.numpy(), c * x.nnz)) for c in (1 / 64, 1 / 16, 3 / 16, 6 / 16, 9 / 16, 12 / 16,
                                                                      15 / 16, 63 / 64)] + [m]
one = wall(lambda: dev_update(x, Td, n, f, lam, PREC_FP32, Xd))
ranged = wall(lambda: [dev_update(x, Td, n, f, lam, PREC_FP32, Xd[a * f:], a, b) for a, b in zip(cuts[:-1], cuts[1:])])
cs = torch.cuda.Stream()


def with_copy():
    with torch.cuda.stream(cs):
        h2d([rp, ci, vv], dx)
    dev_update(x, Td, n, f, lam, PREC_FP32, Xd)


both = wall(with_copy)
print(f"device X half: one call {one:.1f} ms | 9 ranges {ranged:.1f} ms | one call + concurrent H2D {both:.1f} ms")


def ranged_with_copy():
    with torch.cuda.stream(cs):
        for _ in range(3):
            h2d([rp, ci, vv], dx)
    for a, b in zip(cuts[:-1], cuts[1:]):
        dev_update(x, Td, n, f, lam, PREC_FP32, Xd[a * f:], a, b)


def ev_time(fn):
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(e1)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[1:]))


def ranged_with_copy_ev(e1):
    with torch.cuda.stream(cs):
        for _ in range(3):
            h2d([rp, ci, vv], dx)
    for a, b in zip(cuts[:-1], cuts[1:]):
        dev_update(x, Td, n, f, lam, PREC_FP32, Xd[a * f:], a, b)
    e1.record()


def ranged_ev(e1):
    for a, b in zip(cuts[:-1], cuts[1:]):
        dev_update(x, Td, n, f, lam, PREC_FP32, Xd[a * f:], a, b)
    e1.record()


print(f"device X half in 9 ranges, compute stream only: alone {ev_time(ranged_ev):.1f} ms, "
      f"with 3 concurrent H2D passes {ev_time(ranged_with_copy_ev):.1f} ms")
