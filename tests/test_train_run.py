"""The C++ train_run (include/alskit/driver.hpp) against the
reference's own train_run (driver.hpp:107-268, compiled into oracle/_ref) on the same binary
cache, seed and config:

* FP64 mode (accumulate_double, the reference default): final factors bit-identical,
  every checkpoint file byte-identical, the metrics CSV identical in layout and iteration
  rows, train_J / test_RMSE equal to 1e-12 (device eval sums in a fixed two-level order,
  the reference serially);
* kill and resume: a run stopped after iteration 2 and resumed reaches the uninterrupted
  run's factors bit for bit, appending to the metrics file;
* a dangling X (x@t without theta@t) is finished first, as in the reference;
* resuming from checkpoints the reference wrote continues the reference's run exactly;
* FP32 mode: within the north-star bars of the reference run."""
from __future__ import annotations

import ctypes as C
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from helpers import normwise_gap

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "tests" / "cpp" / "train_run_cli"
M, N, NNZ, F, LAM, SEED = 700, 260, 30000, 12, 0.05, 42

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cache(ref, tmp_path_factory):
    if not EXE.exists():
        from paper_1603_03820_b200 import build as B
        B.build_cpp_tests()
    p = tmp_path_factory.mktemp("cache") / "r.cache"
    assert ref.bench_write_cache(M, N, NNZ, 2024, p) == 0
    return p


def ours(cache, out, iters, acc=1, ckpt="-", metrics="-", resume=0, stop=-1, plan=None):
    cmd = [str(EXE), str(cache), str(F), repr(LAM), str(iters), str(SEED), str(acc), str(ckpt), str(metrics),
           str(resume), str(out)] + ([str(stop)] if stop > 0 or plan else [])
    if plan:  # (capacity, force_p, force_q)
        cmd += [str(v) for v in plan]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    x = np.fromfile(f"{out}_x.f32", np.float32)
    t = np.fromfile(f"{out}_theta.f32", np.float32)
    start = int(res.stdout.split("start=")[1].split()[0])
    return x, t, start


def theirs(ref, cache, iters, acc=1, ckpt=None, metrics=None, resume=0, stop=-1):
    x = np.zeros(M * F, np.float32)
    t = np.zeros(N * F, np.float32)
    start, dg = C.c_int(), C.c_uint64()
    st = ref.call("train_run", str(cache).encode(), F, C.c_double(LAM), iters, C.c_uint64(SEED), acc,
                  str(ckpt).encode() if ckpt else None, str(metrics).encode() if metrics else None, resume, stop,
                  x.ctypes.data_as(C.c_void_p), t.ctypes.data_as(C.c_void_p), C.byref(start), C.byref(dg))
    assert st == 0, ref.last_error()
    return x, t, start.value


def _csv(p):
    lines = Path(p).read_text().splitlines()
    return lines[0], [l for l in lines[1:] if l.startswith("#")], [l.split(",") for l in lines[1:] if not l.startswith("#")]


def test_train_run_fp64_matches_reference(ref, cache, tmp_path):
    a, b = tmp_path / "ours", tmp_path / "ref"
    xo, to, so = ours(cache, tmp_path / "o", 4, ckpt=a, metrics=tmp_path / "o.csv")
    xr, tr, sr = theirs(ref, cache, 4, ckpt=b, metrics=tmp_path / "r.csv")
    assert so == sr == 1
    assert np.array_equal(xo, xr) and np.array_equal(to, tr)
    names = sorted(p.name for p in a.iterdir())
    assert names == sorted(p.name for p in b.iterdir()) and len(names) == 8
    for nm in names:
        assert (a / nm).read_bytes() == (b / nm).read_bytes(), nm
    ho, co, ro = _csv(tmp_path / "o.csv")
    hr, cr, rr = _csv(tmp_path / "r.csv")
    assert ho == hr == "iteration,wall_seconds,train_J,test_RMSE" and co == cr
    assert [r[0] for r in ro] == [r[0] for r in rr] == ["1", "2", "3", "4"]
    for x, y in zip(ro, rr):
        for k in (2, 3):
            assert abs(float(x[k]) - float(y[k])) <= 1e-12 * abs(float(y[k])), (x, y)


def test_train_run_kill_resume_and_dangling_x(ref, cache, tmp_path):
    xr, tr, _ = theirs(ref, cache, 4)
    d = tmp_path / "ck"
    ours(cache, tmp_path / "a", 4, ckpt=d, metrics=tmp_path / "m.csv", stop=2)  # killed after iteration 2
    x2, t2, start = ours(cache, tmp_path / "b", 4, ckpt=d, metrics=tmp_path / "m.csv", resume=1)
    assert start == 3 and np.array_equal(x2, xr) and np.array_equal(t2, tr)
    _, _, rows = _csv(tmp_path / "m.csv")
    assert [r[0] for r in rows] == ["1", "2", "3", "4"]
    # dangling X: drop theta@4, resume: theta@4 is recomputed from x@4
    (d / "ckpt_000004_theta.bin").unlink()
    x3, t3, start = ours(cache, tmp_path / "c", 4, ckpt=d, resume=1)
    assert start == 4 and np.array_equal(x3, xr) and np.array_equal(t3, tr)


def test_train_run_resumes_reference_checkpoints(ref, cache, tmp_path):
    d = tmp_path / "ck"
    theirs(ref, cache, 4, ckpt=d, stop=2)  # the reference wrote iterations 1-2
    xr, tr, _ = theirs(ref, cache, 4)
    x, t, start = ours(cache, tmp_path / "o", 4, ckpt=d, resume=1)
    assert start == 3 and np.array_equal(x, xr) and np.array_equal(t, tr)


def test_train_run_fp32_within_bars(ref, cache, tmp_path):
    xr, tr, _ = theirs(ref, cache, 4)
    x, t, _ = ours(cache, tmp_path / "o", 4, acc=0)
    assert normwise_gap(x, xr) <= 1e-3 and normwise_gap(t, tr) <= 1e-3


@pytest.mark.parametrize("plan", [(60000, 0, 0), (0, 2, 3)])
def test_train_run_split_sides_match_reference(ref, cache, tmp_path, plan):
    """The planner fields (config.hpp:54-60): a capacity that makes plan_partition split the
    rows (q = 4 for X, 2 for Theta here) or a forced 2 x 3 grid. Our train_run persists each
    split side's grid and runs its half-sweeps out of core (alsk_ooc_update, blocks streamed
    into HBM); the reference's train_run runs su_als_update_x on the same grids in memory.
    FP64: factors bit-identical, the metrics CSV equal."""
    x, t, _ = ours(cache, tmp_path / "o", 3, metrics=tmp_path / "o.csv", plan=plan)
    xr = np.zeros(M * F, np.float32)
    tr = np.zeros(N * F, np.float32)
    st = ref.call("train_run_plan", str(cache).encode(), F, C.c_double(LAM), 3, C.c_uint64(SEED), 1,
                  str(tmp_path / "r.csv").encode(), C.c_int64(plan[0]), plan[1], plan[2],
                  xr.ctypes.data_as(C.c_void_p), tr.ctypes.data_as(C.c_void_p))
    assert st == 0, ref.last_error()
    assert np.array_equal(x, xr) and np.array_equal(t, tr)
    _, _, ro = _csv(tmp_path / "o.csv")
    _, _, rr = _csv(tmp_path / "r.csv")
    assert [r[0] for r in ro] == [r[0] for r in rr] == ["1", "2", "3"]
    for a, b in zip(ro, rr):
        for k in (2, 3):
            assert abs(float(a[k]) - float(b[k])) <= 1e-12 * abs(float(b[k])), (a, b)
    # and the split really happened (the CLI reports the X side's grid)
    res = subprocess.run([str(EXE), str(cache), str(F), repr(LAM), "1", str(SEED), "1", "-", "-", "0",
                          str(tmp_path / "p"), "-1", *map(str, plan)], capture_output=True, text=True, timeout=300)
    pq = res.stdout.split("p=")[1].split()
    assert (int(pq[0]), int(pq[1].split("=")[1])) == ((2, 3) if plan[1] else (1, 4)), res.stdout


def test_train_run_split_fp32_within_bars(ref, cache, tmp_path):
    """FP32 with split sides (tensor-core partials out of core) stays within the FP32 bar of the
    reference's FP64 train_run on the same grids."""
    x, t, _ = ours(cache, tmp_path / "o", 3, acc=0, plan=(0, 2, 3))
    xr = np.zeros(M * F, np.float32)
    tr = np.zeros(N * F, np.float32)
    st = ref.call("train_run_plan", str(cache).encode(), F, C.c_double(LAM), 3, C.c_uint64(SEED), 1, None,
                  C.c_int64(0), 2, 3, xr.ctypes.data_as(C.c_void_p), tr.ctypes.data_as(C.c_void_p))
    assert st == 0, ref.last_error()
    assert normwise_gap(x, xr) <= 1e-3 and normwise_gap(t, tr) <= 1e-3
