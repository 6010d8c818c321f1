"""Multi-GPU ALS on one box: a thin Python caller of libalskit_cuda's C++ multi-GPU session
(alsk_mp_*, csrc/multigpu.cu) and its NCCL communicators.

One process per GPU. torch.distributed is plumbing only: the rendezvous that ships NCCL's
128-byte unique id to every rank, barriers and the max-over-ranks of a timing. Every
half-sweep and every collective (ncclAllGather / ncclReduceScatter over NVLink/NVSwitch) is
issued by the C++ session on the caller's CUDA stream; there is no torch op and no CPU
fallback on the data path.

Two splits, both from the paper (§4 "SU-ALS"; reference parallel.hpp:487-583):
* MODEL (Netflix / YahooMusic / Hugewiki): X rows, then Theta rows, in P equal (padded)
  slices, the other factor replicated; an in-place all-gather after every half. Per row the
  arithmetic is the one-GPU kernel's, so results are bit-identical for any P.
* HYBRID (SparkALS): model-parallel X half with X kept in per-rank slabs; data-parallel
  Theta half — per-item partial Hermitians over the local users (lambda n_v^local,
  parallel.hpp:408-411) summed by reduce-scatter, the rank's item slice solved, Theta
  all-gathered.

The CPU restatement of this partitioning used by the gloo tests is tests/mp_model.py.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N

MODEL = 0
HYBRID = 1


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


def packed_stride(f: int) -> int:
    """Floats per packed FP32 partial row: f <= 15 the compact [lower(A) row-major | b]
    (f(f+1)/2 + f); otherwise the panel-blocked row of kernels.cuh pb_block (for each 8-column
    block b, rows 8b..f of 8 floats)."""
    if f <= 15:
        return f * (f + 1) // 2 + f
    nb = (f + 7) // 8
    return 8 * (nb * (f + 1) - 4 * nb * (nb - 1))


def cuda_partial_hermitian_f32(R, theta: torch.Tensor, theta_rows: int, f: int, lam: float, row_begin: int,
                               row_end: int, out: torch.Tensor) -> None:
    """Packed FP32 partial Hermitians (+ B) of rows [row_begin,row_end) (layout: packed_stride)."""
    _check(N.LIB.alsk_dev_partial_hermitian_f32(C.byref(R.c), theta.data_ptr(), theta_rows, f, lam, row_begin,
                                                row_end, out.data_ptr(), _stream()))


def cuda_solve_packed_f32(packed: torch.Tensor, count: int, f: int, out: torch.Tensor) -> None:
    _check(N.LIB.alsk_dev_solve_packed_f32(packed.data_ptr(), count, f, out.data_ptr(), _stream()))


# ---------------------------------------------------------------- communicators
class NativeComm:
    """An NCCL communicator inside libalskit_cuda (alsk_comm_init_rank). Rank 0 draws the
    unique id; torch.distributed (any backend) ships it to the other ranks."""

    def __init__(self, handle: int, rank: int, world: int, keep=None):
        self.handle, self.rank, self.world = handle, rank, world
        self._keep = keep  # transport callbacks of a custom communicator

    @classmethod
    def from_process_group(cls, device_index: int, group=None) -> "NativeComm":
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if N.LIB.alsk_comm_available() != 1:
            raise RuntimeError("NCCL could not be loaded by libalskit_cuda (alsk_comm_available() == 0)")
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _check(N.LIB.alsk_comm_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        _check(N.LIB.alsk_comm_init_rank(uid, world, rank, device_index, C.byref(h)))
        return cls(h.value, rank, world)

    def close(self) -> None:
        if self.handle:
            N.LIB.alsk_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostTransportComm(NativeComm):
    """A communicator whose collectives run over torch.distributed on host copies
    (alsk_comm_init_custom). TEST TRANSPORT: it lets several ranks' C++ sessions share one
    GPU (NCCL refuses two ranks on one device) so the multi-rank session logic is exercised
    where only one GPU exists. NCCL (NativeComm) is the product path."""

    @classmethod
    def from_process_group(cls, device_index: int = 0, group=None) -> "HostTransportComm":
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        dtypes = {0: (np.float32, 4), 1: (np.float64, 8)}

        def host(ptr, count, dtype, stream):
            npd, size = dtypes[dtype]
            buf = np.empty(count, npd)
            _check(N.LIB.alsk_dev_to_host(buf.ctypes.data, ptr, count * size, stream))
            return torch.from_numpy(buf)

        def device(ptr, t: torch.Tensor, stream):
            a = np.ascontiguousarray(t.numpy())
            _check(N.LIB.alsk_host_to_dev(ptr, a.ctypes.data, a.nbytes, stream))

        def allgather(user, buf, chunk, dtype, stream):
            try:
                whole = host(buf, chunk * world, dtype, stream)
                mine = whole[rank * chunk:(rank + 1) * chunk].clone()
                parts = [torch.empty(chunk, dtype=mine.dtype) for _ in range(world)]
                dist.all_gather(parts, mine, group=group)
                device(buf, torch.cat(parts), stream)
                return 0
            except Exception:  # noqa: BLE001 — reported to the C side as a transport failure
                return 1

        def reduce_scatter(user, src, dst, chunk, dtype, stream):
            try:
                whole = host(src, chunk * world, dtype, stream)
                dist.all_reduce(whole, op=dist.ReduceOp.SUM, group=group)
                device(dst, whole[rank * chunk:(rank + 1) * chunk].contiguous(), stream)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        ag = N.ALLGATHER_FN(allgather)
        rs = N.REDUCE_SCATTER_FN(reduce_scatter)
        ops = N.CommOpsT(ag, rs, None)
        h = C.c_void_p()
        _check(N.LIB.alsk_comm_init_custom(world, rank, C.byref(ops), C.byref(h)))
        return cls(h.value, rank, world, keep=(ag, rs, ops))


# ---------------------------------------------------------------- the session
class MultiGpuALS:
    """One rank's share of a multi-GPU ALS run (alsk_mp_*). comm=None is the single-GPU run.

    x_local: the train ratings of this rank's user slice [xb, xe) as a local CSR (global item
    ids). t_local: MODEL — the rank's item slice [tb, te) of R^T (global user ids); HYBRID —
    every item's ratings from the rank's users (n rows, user ids local to the slab).
    x0 / theta0: device tensors with all m*f / n*f initial entries (or None for zeros)."""

    def __init__(self, comm: Optional[NativeComm], mode: int, m: int, n: int, f: int, lam: float, precision: int,
                 x_local, t_local, x0: Optional[torch.Tensor], theta0: Optional[torch.Tensor],
                 workspace: Optional[int] = None):
        self.comm, self.mode, self.m, self.n, self.f, self.lam = comm, mode, m, n, f, lam
        self.x_local, self.t_local = x_local, t_local  # keep the device CSRs alive
        h = C.c_void_p()
        _check(N.LIB.alsk_mp_create(comm.handle if comm else None, mode, m, n, f, lam, precision,
                                    C.byref(x_local.c), C.byref(t_local.c),
                                    x0.data_ptr() if x0 is not None else None,
                                    theta0.data_ptr() if theta0 is not None else None, workspace, _stream(),
                                    C.byref(h)))
        self.handle = h.value
        xb, xe, tb, te = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        N.LIB.alsk_mp_slices(self.handle, C.byref(xb), C.byref(xe), C.byref(tb), C.byref(te))
        self.xs, self.ts = (xb.value, xe.value), (tb.value, te.value)

    def half_x(self) -> None:
        _check(N.LIB.alsk_mp_half_x(self.handle, _stream()))

    def half_theta(self) -> None:
        _check(N.LIB.alsk_mp_half_theta(self.handle, _stream()))

    def step(self) -> None:
        self.half_x()
        self.half_theta()

    def check(self) -> None:
        """Synchronise (polling NCCL errors) and raise a recorded Cholesky breakdown."""
        _check(N.LIB.alsk_mp_check(self.handle, _stream()))

    def pointers(self) -> tuple[int, int, int]:
        """(X device pointer, global row of X's first row, Theta device pointer)."""
        x, xb, t = C.c_void_p(), C.c_int64(), C.c_void_p()
        _check(N.LIB.alsk_mp_factors(self.handle, C.byref(x), C.byref(xb), C.byref(t)))
        return x.value, xb.value, t.value

    def factors_host(self) -> tuple[np.ndarray, np.ndarray]:
        """Copies of X (MODEL: all m rows; HYBRID: this rank's slab) and Theta (n rows)."""
        self.check()
        x, xb, t = self.pointers()
        rows = self.m if self.mode == MODEL else self.xs[1] - self.xs[0]
        X = np.empty(rows * self.f, np.float32)
        T = np.empty(self.n * self.f, np.float32)
        _check(N.LIB.alsk_dev_to_host(X.ctypes.data, x, X.nbytes, _stream()))
        _check(N.LIB.alsk_dev_to_host(T.ctypes.data, t, T.nbytes, _stream()))
        return X, T

    def collective_stats(self) -> tuple[int, int]:
        b, c = C.c_int64(), C.c_int64()
        N.LIB.alsk_mp_collective_stats(self.handle, C.byref(b), C.byref(c))
        return b.value, c.value

    def close(self) -> None:
        if self.handle:
            N.LIB.alsk_mp_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
