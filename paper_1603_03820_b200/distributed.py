"""Multi-GPU ALS on one box: one process per GPU, torch.distributed (NCCL over NVLink /
NVSwitch) for the exchanges, libalskit_cuda for every half-sweep.

Two splits, both from the paper (§4 "SU-ALS"; reference parallel.hpp:487-583):

* ModelParallelALS — rows of X (then of Theta) are cut into P equal slices (one per rank,
  padded to ceil(rows/P) so NCCL's equal-count all-gather applies); the other factor is
  replicated. Each rank solves its slice, then an in-place all-gather refreshes the whole
  factor on every rank. Per row the arithmetic is the single-GPU kernel's, so results are
  bit-identical to one GPU for any P.

* DataParallelThetaHalf — rank i owns a slab of users (X rows) and their ratings, viewed
  item-major; the Theta-half forms per-item partial Hermitians over the local users only
  (lambda * n_v^local on the diagonal, parallel.hpp:408-411), a reduce-scatter in double
  sums them so rank i receives item slice i (the reference's one-phase reduce_batches,
  parallel.hpp:206-280), the slice is rounded to float once and solved, and an all-gather
  refreshes Theta. X never moves in this half.

The compute steps are injectable so the host-side partitioning and collectives can be
tested on CPU with the gloo backend (tests/test_distributed.py); the defaults are the CUDA
entry points and there is no CPU fallback in the product path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import _native as N


def even_slices(rows: int, world: int) -> tuple[int, list[tuple[int, int]]]:
    """Equal-count (padded) slices: chunk = ceil(rows/world); rank r owns [r*chunk, min(rows, (r+1)*chunk))."""
    chunk = -(-rows // world) if rows else 0
    return chunk, [(min(rows, r * chunk), min(rows, (r + 1) * chunk)) for r in range(world)]


def slice_cuts(count: int, p: int) -> list[int]:
    """parallel.hpp:160-168 — first count % p slices take one extra entry."""
    base, rem = divmod(count, p)
    cuts = [0]
    for i in range(p):
        cuts.append(cuts[-1] + base + (1 if i < rem else 0))
    return cuts


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else 0


def _check(st: int) -> None:
    if st != 0:
        from .alskit import _ERR, Error
        raise _ERR.get(st, Error)(N.LIB.alsk_last_error().decode(errors="replace"))


# ---------------------------------------------------------------- default (CUDA) compute
def cuda_update_rows(R, theta: torch.Tensor, theta_rows: int, f: int, lam: float, precision: int,
                     row_begin: int, row_end: int, out: torch.Tensor) -> None:
    """update_x of rows [row_begin,row_end) of the device CSR `R` into `out` (rows-local)."""
    _check(N.LIB.alsk_dev_update(C.byref(R.c), theta.data_ptr(), theta_rows, f, lam, precision, 4096,
                                 row_begin, row_end, out.data_ptr(), _stream()))


def cuda_partial_hermitian(R, theta: torch.Tensor, theta_rows: int, f: int, lam: float, row_begin: int,
                           row_end: int, out: torch.Tensor) -> None:
    """Packed-lower double partial Hermitians (+ B) of rows [row_begin,row_end)."""
    _check(N.LIB.alsk_dev_partial_hermitian(C.byref(R.c), theta.data_ptr(), theta_rows, f, lam, row_begin,
                                            row_end, out.data_ptr(), _stream()))


def cuda_solve_packed(packed: torch.Tensor, count: int, f: int, out: torch.Tensor) -> None:
    _check(N.LIB.alsk_dev_solve_packed(packed.data_ptr(), count, f, out.data_ptr(), _stream()))


def packed_stride(f: int) -> int:
    """Floats per panel-blocked packed row (kernels.cuh pb_block): for each 8-column block b,
    rows 8b..f of 8 floats."""
    nb = (f + 7) // 8
    return 8 * (nb * (f + 1) - 4 * nb * (nb - 1))


def cuda_partial_hermitian_f32(R, theta: torch.Tensor, theta_rows: int, f: int, lam: float, row_begin: int,
                               row_end: int, out: torch.Tensor) -> None:
    """Panel-blocked FP32 partial Hermitians (+ B) of rows [row_begin,row_end), tensor cores."""
    _check(N.LIB.alsk_dev_partial_hermitian_f32(C.byref(R.c), theta.data_ptr(), theta_rows, f, lam, row_begin,
                                                row_end, out.data_ptr(), _stream()))


def cuda_solve_packed_f32(packed: torch.Tensor, count: int, f: int, out: torch.Tensor) -> None:
    _check(N.LIB.alsk_dev_solve_packed_f32(packed.data_ptr(), count, f, out.data_ptr(), _stream()))


@dataclass
class Compute:
    update_rows: Callable = cuda_update_rows
    partial_hermitian: Callable = cuda_partial_hermitian
    solve_packed: Callable = cuda_solve_packed
    partial_hermitian_f32: Callable = cuda_partial_hermitian_f32
    solve_packed_f32: Callable = cuda_solve_packed_f32


def _all_gather_inplace(buf: torch.Tensor, chunk_elems: int, rank: int, world: int, group=None) -> None:
    """Every rank contributes buf[rank*chunk:(rank+1)*chunk]; afterwards buf is complete."""
    if world == 1:
        return
    mine = buf[rank * chunk_elems:(rank + 1) * chunk_elems]
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, mine, group=group)  # in place over NVLink
    else:
        parts = list(buf.view(world, chunk_elems).unbind(0))
        dist.all_gather(parts, mine.clone(), group=group)


class ModelParallelALS:
    """Row-partitioned ALS: X rows, then Theta rows, split over the ranks; factors
    refreshed by all-gather after every half."""

    def __init__(self, R, RT, m: int, n: int, f: int, lam: float, precision: int, x0: torch.Tensor,
                 theta0: torch.Tensor, group=None, compute: Optional[Compute] = None):
        self.R, self.RT, self.m, self.n, self.f, self.lam, self.precision = R, RT, m, n, f, lam, precision
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.compute = compute or Compute()
        self.cx, self.xs = even_slices(m, self.world)
        self.ct, self.ts = even_slices(n, self.world)
        dev = x0.device
        self.X = torch.zeros(self.cx * self.world * f, dtype=torch.float32, device=dev)
        self.T = torch.zeros(self.ct * self.world * f, dtype=torch.float32, device=dev)
        self.X[: m * f].copy_(x0.reshape(-1))
        self.T[: n * f].copy_(theta0.reshape(-1))

    def half_x(self) -> None:
        rb, re = self.xs[self.rank]
        if re > rb:
            self.compute.update_rows(self.R, self.T, self.n, self.f, self.lam, self.precision, rb, re,
                                     self.X[rb * self.f:])
        _all_gather_inplace(self.X, self.cx * self.f, self.rank, self.world, self.group)

    def half_theta(self) -> None:
        rb, re = self.ts[self.rank]
        if re > rb:
            self.compute.update_rows(self.RT, self.X, self.m, self.f, self.lam, self.precision, rb, re,
                                     self.T[rb * self.f:])
        _all_gather_inplace(self.T, self.ct * self.f, self.rank, self.world, self.group)

    def step(self) -> None:
        self.half_x()
        self.half_theta()

    def factors(self) -> tuple[torch.Tensor, torch.Tensor]:
        return self.X[: self.m * self.f], self.T[: self.n * self.f]


class DataParallelThetaHalf:
    """Theta-half with a data-parallel split over users: per-item partial Hermitians from
    the local user slab, reduce-scatter (slice i -> rank i), solve, all-gather.

    `RT_local` is the CSR of (R restricted to this rank's users)^T, i.e. items x all users
    with only local users' ratings; theta rows are solved for all n items.

    fp32=False (default): packed-lower double partials, double reduce-scatter, one rounding
    to f32 and the reference-order solve (parallel.hpp:487-583). fp32=True: panel-blocked
    FP32 partials from the tensor cores, FP32 reduce-scatter and the batched TMEM Cholesky
    (the north star's FP32 tolerance; half the bytes on NVLink)."""

    def __init__(self, RT_local, m: int, n: int, f: int, lam: float, group=None, compute: Optional[Compute] = None,
                 fp32: bool = False):
        self.RT, self.m, self.n, self.f, self.lam = RT_local, m, n, f, lam
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.compute = compute or Compute()
        self.fp32 = fp32
        self.per = packed_stride(f) if fp32 else f * (f + 1) // 2 + f
        self.ct, self.ts = even_slices(n, self.world)

    def half_theta(self, X: torch.Tensor, T_out: torch.Tensor) -> None:
        dev = X.device
        dt = torch.float32 if self.fp32 else torch.float64
        partial = torch.zeros(self.ct * self.world * self.per, dtype=dt, device=dev)
        if self.n:
            herm = self.compute.partial_hermitian_f32 if self.fp32 else self.compute.partial_hermitian
            herm(self.RT, X, self.m, self.f, self.lam, 0, self.n, partial)
        mine = torch.empty(self.ct * self.per, dtype=dt, device=dev)
        if self.world > 1:
            if dist.get_backend(self.group) == "nccl":
                dist.reduce_scatter_tensor(mine, partial, op=dist.ReduceOp.SUM, group=self.group)
            else:
                ins = list(partial.view(self.world, -1).unbind(0))
                dist.reduce_scatter(mine, ins, op=dist.ReduceOp.SUM, group=self.group)
        else:
            mine.copy_(partial)
        rb, re = self.ts[self.rank]
        if re > rb:
            solve = self.compute.solve_packed_f32 if self.fp32 else self.compute.solve_packed
            solve(mine, re - rb, self.f, T_out[rb * self.f:])
        _all_gather_inplace(T_out, self.ct * self.f, self.rank, self.world, self.group)
