"""CPU model of the multi-GPU partitioning (TEST INFRASTRUCTURE ONLY).

The product's multi-GPU path is C++ inside libalskit_cuda.so (alsk_mp_*, csrc/multigpu.cu)
over NCCL. This module restates its slicing and collectives in Python with injectable
compute so the partitioning logic can be checked on CPU with the gloo backend at world
size > 1 (tests/test_distributed.py) against the oracle:

* ModelParallelALS — rows of X (then of Theta) cut into P equal (padded) slices, solved per
  rank, refreshed by an in-place all-gather (bit-identical to one process for any P);
* DataParallelThetaHalf — per-item partial Hermitians over a rank's user slab
  (lambda n_v^local, parallel.hpp:408-411), reduce-scatter (parallel.hpp:206-280), solve of
  the rank's item slice, all-gather of Theta.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist

from paper_1603_03820_b200.distributed import even_slices, packed_stride


@dataclass
class Compute:
    update_rows: Callable
    partial_hermitian: Callable
    solve_packed: Callable
    partial_hermitian_f32: Callable
    solve_packed_f32: Callable


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
        self.compute = compute
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
        self.compute = compute
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
