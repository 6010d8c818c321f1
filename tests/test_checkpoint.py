"""Factor checkpoints (dataio.hpp:546-786, driver.hpp:183-262), after
the reference's checkpoint and resume tests (test_dataio.cpp, test_driver.cpp:280-317):

* write -> read is bit-exact; files are byte-identical to the reference writer's and each
  side reads the other's;
* names, atomic rename (no .tmp left behind), newest-wins ordering with theta outranking x,
  restore_latest_of, the digest-mismatch InputError;
* every IoError text matches oracle/_ref's;
* (gpu) the device writer snapshots HBM factors in the background, by value, and a run
  interrupted after X@t or Theta@t resumes to bit-identical factors.
"""
from __future__ import annotations

import struct

import numpy as np
import pytest


def factor(A, rows, f, seed):
    return A.random_factor(rows, f, seed)


def test_write_read_round_trip(A, tmp_path):
    fm = factor(A, 37, 7, 3)
    p = A.write_checkpoint(A.Checkpoint(5, A.FactorKind.theta, fm, 0xDEADBEEFCAFEF00D), tmp_path / "ck")
    assert p.endswith("ckpt_000005_theta.bin")
    assert sorted(x.name for x in (tmp_path / "ck").iterdir()) == ["ckpt_000005_theta.bin"]  # no .tmp left
    cp = A.read_checkpoint(p)
    assert (cp.iteration, cp.which, cp.digest) == (5, A.FactorKind.theta, 0xDEADBEEFCAFEF00D)
    assert (cp.factor.rows, cp.factor.f) == (37, 7)
    assert cp.factor.entries.tobytes() == fm.entries.tobytes()
    assert (tmp_path / "ck" / "ckpt_000005_theta.bin").stat().st_size == 56 + 37 * 7 * 4


def test_files_match_the_reference_writer(A, ref, tmp_path):
    fm = factor(A, 50, 9, 8)
    mine = A.write_checkpoint(A.Checkpoint(12, A.FactorKind.x, fm, 77), tmp_path / "mine")
    assert ref.write_checkpoint(str(tmp_path / "ref"), 12, 0, 50, 9, 77, fm.entries) == 0
    theirs = tmp_path / "ref" / "ckpt_000012_x.bin"
    assert open(mine, "rb").read() == theirs.read_bytes()
    cp = A.read_checkpoint(theirs)
    assert cp.factor.entries.tobytes() == fm.entries.tobytes() and cp.digest == 77
    st, it, wh, rows, f, dg, e = ref.read_checkpoint(mine, 50 * 9)
    assert (st, it, wh, rows, f, dg) == (0, 12, 0, 50, 9, 77)
    assert e.tobytes() == fm.entries.tobytes()


def _populate(A, d, entries):
    fm = factor(A, 4, 2, 1)
    for it, wh in entries:
        A.write_checkpoint(A.Checkpoint(it, wh, fm, 5), d)
    (d / "ckpt_99_junk.bin").write_bytes(b"x")  # not a checkpoint name: ignored
    (d / "notes.txt").write_bytes(b"x")
    (d / "ckpt_000100_x.bin.tmp").write_bytes(b"x")


def test_newest_wins_theta_outranks_x(A, ref, tmp_path):
    X, T = A.FactorKind.x, A.FactorKind.theta
    assert A.restore_latest(tmp_path / "missing") is None
    _populate(A, tmp_path, [(1, X), (1, T), (2, X), (10, X)])
    cp = A.restore_latest(tmp_path)
    assert (cp.iteration, cp.which) == (10, X)
    assert ref.restore_latest(str(tmp_path)) == (0, (10, 0))
    A.write_checkpoint(A.Checkpoint(10, T, factor(A, 4, 2, 1), 5), tmp_path)
    cp = A.restore_latest(tmp_path)
    assert (cp.iteration, cp.which) == (10, T)
    assert ref.restore_latest(str(tmp_path)) == (0, (10, 1))
    assert A.restore_latest_of(tmp_path, X).iteration == 10
    with pytest.raises(A.InputError, match="checkpoint config digest mismatch"):
        A.restore_latest(tmp_path, expected_digest=6)


def _corrupt(A, tmp_path):
    fm = factor(A, 3, 2, 1)
    good = A.write_checkpoint(A.Checkpoint(1, A.FactorKind.x, fm, 9), tmp_path / "g")
    raw = bytearray(open(good, "rb").read())
    out = []

    def put(name, data):
        p = tmp_path / f"{name}.bin"
        p.write_bytes(bytes(data))
        out.append((name, p))

    put("truncated", raw[:-3])
    put("junk", b"definitely not a checkpoint, but long enough to read a header from")
    put("short", raw[:30])
    bad = bytearray(raw); bad[8:16] = struct.pack("<Q", 3); put("version", bad)
    bad = bytearray(raw); bad[24:32] = struct.pack("<Q", 2); put("kind", bad)
    bad = bytearray(raw); bad[40:48] = struct.pack("<Q", 1 << 21); put("header", bad)
    put("trailing", raw + b"\0")
    return out


EXPECTED = {
    "truncated": "checkpoint size does not match its header",
    "junk": "not a checkpoint (bad magic)",
    "short": "truncated while reading which",
    "version": "unsupported checkpoint version",
    "kind": "corrupt checkpoint (bad factor kind)",
    "header": "corrupt checkpoint header",
    "trailing": "checkpoint size does not match its header",
}


def test_errors_match_the_reference(A, ref, tmp_path):
    for name, p in _corrupt(A, tmp_path):
        with pytest.raises(A.IoError) as e:
            A.read_checkpoint(p)
        assert str(e.value) == f"{p}: {EXPECTED[name]}", name
        st, *_ = ref.read_checkpoint(str(p), 64)
        assert st == 4 and ref.last_error() == str(e.value), name
    with pytest.raises(A.IoError, match="cannot open /nonexistent/ck.bin"):
        A.read_checkpoint("/nonexistent/ck.bin")
    blocker = tmp_path / "file"
    blocker.write_bytes(b"")
    with pytest.raises(A.IoError, match="cannot create directory"):
        A.write_checkpoint(A.Checkpoint(1, A.FactorKind.x, factor(A, 2, 2, 1), 0), blocker / "sub")


# ---------------------------------------------------------------- device writer and resume
def _session(A, seed=3, fp64=True):
    from paper_1603_03820_b200.session import AlsSession
    r = A.synth_csr(700, 300, 9000, seed)
    cfg = A.SolverConfig(f=24, lambda_=0.05, accumulate_double=fp64)
    x0 = A.random_factor(r.rows, cfg.f, 42)
    t0 = A.random_factor(r.cols, cfg.f, A.mix_seed(42, 1))
    return r, cfg, lambda: AlsSession(r, None, None, cfg, x0, t0)


def test_host_writer_needs_no_device(A, tmp_path):
    """The C-ABI writer's host submit runs without a GPU, like the reference's pure-host
    CheckpointWriter (dataio.hpp:717-786): files identical to write_checkpoint's, errors
    sticky."""
    import ctypes as C
    from paper_1603_03820_b200 import _native as N
    fm = factor(A, 33, 5, 4)
    h = C.c_void_p()
    A._check(N.LIB.alsk_ckpt_writer_create(str(tmp_path / "w").encode(), C.byref(h)))
    try:
        for it, wh in ((1, 0), (1, 1), (2, 0)):
            A._check(N.LIB.alsk_ckpt_writer_submit_host(h, it, wh, 33, 5, 9, fm.entries.ctypes.data))
        A._check(N.LIB.alsk_ckpt_writer_flush(h))
    finally:
        N.LIB.alsk_ckpt_writer_destroy(h)
    want = A.write_checkpoint(A.Checkpoint(2, A.FactorKind.x, fm, 9), tmp_path / "direct")
    assert (tmp_path / "w" / "ckpt_000002_x.bin").read_bytes() == open(want, "rb").read()
    assert sorted(x.name for x in (tmp_path / "w").iterdir()) == [
        "ckpt_000001_theta.bin", "ckpt_000001_x.bin", "ckpt_000002_x.bin"]
    blocker = tmp_path / "file"
    blocker.write_bytes(b"")
    A._check(N.LIB.alsk_ckpt_writer_create(str(blocker / "sub").encode(), C.byref(h)))
    try:
        A._check(N.LIB.alsk_ckpt_writer_submit_host(h, 1, 0, 33, 5, 9, fm.entries.ctypes.data))
        for _ in range(2):
            with pytest.raises(A.IoError, match="cannot create directory"):
                A._check(N.LIB.alsk_ckpt_writer_flush(h))
    finally:
        N.LIB.alsk_ckpt_writer_destroy(h)


@pytest.mark.gpu
def test_device_writer_snapshots_by_value(A, gpu, tmp_path):
    import torch
    from paper_1603_03820_b200.session import DeviceCheckpointWriter
    f, rows = 16, 100_000
    t = torch.arange(rows * f, dtype=torch.float32, device="cuda")
    with DeviceCheckpointWriter(tmp_path) as w:
        w.submit(1, A.FactorKind.x, t, rows, f, 11)
        t.mul_(-1.0)  # overwrite at once: the snapshot must hold the old values
        w.submit(1, A.FactorKind.theta, t, rows, f, 11)
        w.flush()
    a = A.read_checkpoint(tmp_path / "ckpt_000001_x.bin")
    b = A.read_checkpoint(tmp_path / "ckpt_000001_theta.bin")
    want = np.arange(rows * f, dtype=np.float32)
    assert a.factor.entries.tobytes() == want.tobytes()
    assert b.factor.entries.tobytes() == (-want).tobytes()


@pytest.mark.gpu
def test_device_writer_errors_are_sticky(A, gpu, tmp_path):
    import torch
    from paper_1603_03820_b200.session import DeviceCheckpointWriter
    blocker = tmp_path / "file"
    blocker.write_bytes(b"")
    t = torch.zeros(8, device="cuda")
    with DeviceCheckpointWriter(blocker / "sub") as w:
        w.submit(1, A.FactorKind.x, t, 4, 2, 0)
        with pytest.raises(A.IoError, match="cannot create directory"):
            w.flush()
        with pytest.raises(A.IoError, match="cannot create directory"):
            w.submit(2, A.FactorKind.x, t, 4, 2, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32_tensor"])
@pytest.mark.parametrize("stop_after", ["x", "theta"])
def test_resume_is_bit_exact(A, gpu, tmp_path, stop_after, precision):
    """test_driver.cpp:280-317: a run interrupted and resumed ends with the same factors as
    an uninterrupted one. Interrupted after Theta@2, or after X@3 (the dangling X case:
    Theta@3 is recomputed first). Both precisions: the tensor-core path is deterministic
    too (no atomics in the Hermitian or the solve)."""
    from paper_1603_03820_b200.session import train_resumable
    r, cfg, make = _session(A, fp64=precision == "fp64")
    full = make()
    start, rows = train_resumable(full, 5, tmp_path / "full", digest=99)
    assert start == 1 and [m.iteration for m in rows] == [1, 2, 3, 4, 5]
    X_full, T_full = full.factors()

    d = tmp_path / "cut"
    part = make()
    train_resumable(part, 2, d, digest=99)
    if stop_after == "x":  # X@3 written, Theta@3 not
        part.half_x()
        A.write_checkpoint(A.Checkpoint(3, A.FactorKind.x, part.factors()[0], 99), d)
    resumed = make()
    start, rows = train_resumable(resumed, 5, d, digest=99)
    assert start == (3 if stop_after == "x" else 3)
    assert [m.iteration for m in rows] == [3, 4, 5]
    X, T = resumed.factors()
    assert X.entries.tobytes() == X_full.entries.tobytes()
    assert T.entries.tobytes() == T_full.entries.tobytes()
    for t in range(1, 6):
        a = A.read_checkpoint(d / f"ckpt_{t:06d}_theta.bin")
        b = A.read_checkpoint(tmp_path / "full" / f"ckpt_{t:06d}_theta.bin")
        assert a.factor.entries.tobytes() == b.factor.entries.tobytes(), t
    with pytest.raises(A.InputError, match="digest mismatch"):
        train_resumable(make(), 6, d, digest=100)
