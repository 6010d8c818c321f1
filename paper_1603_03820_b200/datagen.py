"""Per-rank synthetic workloads built in HBM (bench and multi-GPU setup; not the hot path).

The generator is row-seeded: row u's degree, columns and values depend only
on (seed, u), so every rank generates exactly the rows it needs on its own GPU
(alsk_dev_synth_rows, bit-identical to the host generator alsk_synth_csr). The reference
driver's holdout split (split_train_test(R, 0.1, mix_seed(42, 2)), driver.hpp:113,
dataio.hpp:251-290) is a sequential Fisher-Yates over all positions; it runs once on one
host (alsk_holdout_mask, 4-byte positions below 2^32 entries) and travels as a bitmask of
nnz/8 bytes, which each rank applies to its rows in HBM (alsk_dev_split_mask).

Per rank r of P (model-parallel):
  x : the train ratings of its user slice [rb, re) as a local CSR (rows re-rb, global item ids)
  t : the Theta-half matrix
        mode "model":  its item slice [cb, ce) of R^T as a local CSR (rows ce-cb, global user
                       ids): every row chunk of R is generated, split, filtered to the slice's
                       columns and finally transposed (stable, so users stay ascending);
        mode "hybrid": the transpose of its own user slab (all items, local user ids) for the
                       data-parallel Theta half (partial Hermitians + reduce-scatter).
  test: the held-out triplets of its users (global ids), row-major like the reference.
Slices are equal-count (ceil(rows/P)) so the NCCL collectives move equal chunks.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .alskit import TRIPLET_DTYPE, _check, mix_seed
from .session import DeviceCsr

LIB = N.LIB

# name: (m, n, nnz_total, f, lambda); lambdas from PAPER.md Table 4 / BASELINE.json
CONFIGS = {
    "ml1m": (6040, 3706, 1000209, 10, 0.05),
    "netflix": (480189, 17770, 99_000_000, 100, 0.05),
    "yahoo": (1000990, 624961, 252_800_000, 100, 1.4),
    "hugewiki": (50082604, 39781, 3_100_000_000, 100, 0.05),
    "sparkals": (660_000_000, 2_400_000, 3_500_000_000, 10, 0.05),
}
SHAPE_ID = {"ml1m": 0, "netflix": 1, "yahoo": 2, "hugewiki": 3, "sparkals": 4}
RUN_SEED = 42  # SolverConfig default seed (solver.hpp:68)


def data_seed(cfg: str) -> int:
    return mix_seed(RUN_SEED, 100 + SHAPE_ID[cfg])


def split_seed() -> int:
    return mix_seed(RUN_SEED, 2)


def even_slices(rows: int, world: int):
    chunk = -(-rows // world) if rows else 0
    return chunk, [(min(rows, r * chunk), min(rows, (r + 1) * chunk)) for r in range(world)]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def row_start(m: int, nnz: int, u: int) -> int:
    return int(LIB.alsk_synth_row_start(m, nnz, u))


def holdout_mask(nnz: int, holdout: float, seed: int) -> np.ndarray:
    """Bitmask (uint32 words) of split_train_test's held-out positions."""
    k = C.c_int64()
    mask = np.zeros(max(1, (nnz + 31) // 32), np.uint32)
    _check(LIB.alsk_holdout_mask(nnz, holdout, seed & (2**64 - 1), mask.ctypes.data, C.byref(k)))
    return mask


def dev_synth_rows(m: int, n: int, nnz: int, seed: int, rb: int, re: int, device) -> DeviceCsr:
    """Rows [rb, re) of the synthetic matrix as a local device CSR (row_ptr from 0)."""
    k0, k1 = row_start(m, nnz, rb), row_start(m, nnz, re)
    rp = torch.empty(re - rb + 1, dtype=torch.int64, device=device)
    ci = torch.empty(max(1, k1 - k0), dtype=torch.int32, device=device)
    va = torch.empty(max(1, k1 - k0), dtype=torch.float32, device=device)
    _check(LIB.alsk_dev_synth_rows(m, n, nnz, seed & (2**64 - 1), rb, re, rp.data_ptr(), ci.data_ptr(),
                                   va.data_ptr(), _stream()))
    return DeviceCsr(re - rb, n, rp, ci[: k1 - k0], va[: k1 - k0], device)


def dev_split_mask(r: DeviceCsr, dmask: torch.Tensor, bit_offset: int, row_base: int, held: int):
    """Train CSR (local rows) and held-out triplets (global rows) of a row chunk."""
    dev = r.values.device
    rp = torch.empty(r.rows + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(1, r.nnz), dtype=torch.int32, device=dev)
    va = torch.empty(max(1, r.nnz), dtype=torch.float32, device=dev)
    te = torch.empty((max(1, held), TRIPLET_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    kept = C.c_int64()
    _check(LIB.alsk_dev_split_mask(C.byref(r.c), dmask.data_ptr(), bit_offset, row_base, rp.data_ptr(),
                                   ci.data_ptr(), va.data_ptr(), te.data_ptr(), C.byref(kept), _stream()))
    keep = kept.value
    assert keep + held == r.nnz, (keep, held, r.nnz)
    return DeviceCsr(r.rows, r.cols, rp, ci[:keep], va[:keep], dev), te[:held]


def dev_filter_columns(r: DeviceCsr, lo: int, hi: int) -> DeviceCsr:
    dev = r.values.device
    rp = torch.empty(r.rows + 1, dtype=torch.int64, device=dev)
    tot = C.c_int64()
    _check(LIB.alsk_dev_filter_columns(C.byref(r.c), lo, hi, rp.data_ptr(), None, None, C.byref(tot), _stream()))
    ci = torch.empty(max(1, tot.value), dtype=torch.int32, device=dev)
    va = torch.empty(max(1, tot.value), dtype=torch.float32, device=dev)
    _check(LIB.alsk_dev_filter_columns(C.byref(r.c), lo, hi, rp.data_ptr(), ci.data_ptr(), va.data_ptr(),
                                       C.byref(tot), _stream()))
    return DeviceCsr(r.rows, hi - lo, rp, ci[: tot.value], va[: tot.value], dev)


def concat_rows(parts: list, cols: int, device) -> DeviceCsr:
    """Stack local CSRs of consecutive row chunks into one CSR."""
    if len(parts) == 1:
        return parts[0]
    rows = sum(p.rows for p in parts)
    nnz = sum(p.nnz for p in parts)
    rp = torch.empty(rows + 1, dtype=torch.int64, device=device)
    ci = torch.empty(max(1, nnz), dtype=torch.int32, device=device)
    va = torch.empty(max(1, nnz), dtype=torch.float32, device=device)
    r0 = k0 = 0
    for p in parts:
        rp[r0:r0 + p.rows + 1] = p.row_ptr[: p.rows + 1] + k0
        ci[k0:k0 + p.nnz] = p.col_idx[: p.nnz]
        va[k0:k0 + p.nnz] = p.values[: p.nnz]
        r0 += p.rows
        k0 += p.nnz
    return DeviceCsr(rows, cols, rp, ci[:nnz], va[:nnz], device)


def _chunks(m: int, nnz: int, rb: int, re: int, chunk_nnz: int):
    """Row ranges of [rb, re) holding about chunk_nnz ratings each."""
    per_row = max(1, nnz // max(1, m))
    step = max(1, chunk_nnz // per_row)
    u = rb
    while u < re:
        yield u, min(re, u + step)
        u += step


@dataclass
class RankData:
    cfg: str
    m: int
    n: int
    f: int
    lam: float
    rank: int
    world: int
    mode: str
    xs: tuple  # (rb, re) user slice
    ts: tuple  # (cb, ce) item slice
    x: DeviceCsr  # train rows of the user slice (local rows)
    t: DeviceCsr  # Theta-half matrix (see module doc)
    test: torch.Tensor  # held-out triplets of the user slice (uint8 rows of TRIPLET_DTYPE)
    nnz_total: int
    nnz_train_local: int


def build_rank_data(cfg: str, rank: int, world: int, device, mask: np.ndarray, mode: str = "model",
                    chunk_nnz: int = 1 << 28, shape: Optional[tuple] = None) -> RankData:
    """This rank's share of the workload, built in HBM from the row-seeded generator and the
    broadcast holdout mask (see the module doc)."""
    m, n, nnz, f, lam = shape if shape is not None else CONFIGS[cfg]
    seed = data_seed(cfg)
    _, xs = even_slices(m, world)
    _, ts = even_slices(n, world)
    rb, re = xs[rank]
    cb, ce = ts[rank]
    dmask = torch.from_numpy(mask).to(device)

    def rows_split(u0, u1):
        raw = dev_synth_rows(m, n, nnz, seed, u0, u1, device)
        k0, k1 = row_start(m, nnz, u0), row_start(m, nnz, u1)
        held = int(LIB.alsk_mask_count(mask.ctypes.data, k0, k1))
        tr, te = dev_split_mask(raw, dmask, k0, u0, held)
        del raw
        return tr, te

    xparts, tests = [], []
    for u0, u1 in _chunks(m, nnz, rb, re, chunk_nnz):
        tr, te = rows_split(u0, u1)
        xparts.append(tr)
        tests.append(te)
    x = concat_rows(xparts, n, device) if xparts else DeviceCsr(0, n, torch.zeros(1, dtype=torch.int64, device=device),
                                                                torch.zeros(0, dtype=torch.int32, device=device),
                                                                torch.zeros(0, dtype=torch.float32, device=device),
                                                                device)
    del xparts
    test = torch.cat(tests) if len(tests) > 1 else (tests[0] if tests else
                                                     torch.zeros((0, TRIPLET_DTYPE.itemsize), dtype=torch.uint8,
                                                                 device=device))
    if mode == "hybrid" or world == 1:
        t = x.transpose()  # items x local users (all of them at world 1)
    elif mode == "model":
        parts = []
        for u0, u1 in _chunks(m, nnz, 0, m, chunk_nnz):
            tr, _ = rows_split(u0, u1)
            parts.append(dev_filter_columns(tr, cb, ce))
            del tr
        sub = concat_rows(parts, ce - cb, device)
        del parts
        t = sub.transpose()  # (ce-cb) x m, user ids global
        del sub
    else:
        raise ValueError(f"unknown mode {mode!r}")
    return RankData(cfg, m, n, f, lam, rank, world, mode, (rb, re), (cb, ce), x, t, test, nnz, x.nnz)
