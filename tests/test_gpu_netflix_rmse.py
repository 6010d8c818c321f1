"""Netflix-shape RMSE parity with the reference itself (north star: "train and test RMSE
within 1e-4 absolute after 10 iterations"). The fixtures tests/golden/netflix_ref_10iter.csv
(train_run's metrics CSV, driver.hpp:207-246) and netflix_ref_10iter.json (final train and
test RMSE of the reference's factors) were written by the UNMODIFIED reference's train_run
(oracle/_ref, accumulate_double, 10 iterations on the box's host cores) on the same binary
cache, by scripts/netflix_rmse_parity.py; here our C++ train_run (include/alskit/driver.hpp)
runs the FP32 tensor-core mode on that cache, rebuilt with our own writer from the shared
generator (byte-identical to the reference's save_binary_cache: tests/test_io_golden.py)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"
EXE = ROOT / "tests" / "cpp" / "train_run_cli"


def _csv(p):
    lines = Path(p).read_text().splitlines()
    return lines[0], [[float(v) for v in l.split(",")] for l in lines[1:] if not l.startswith("#")]


def test_netflix_shape_10_iterations_match_the_reference(A, gpu, tmp_path):
    import bench
    if not EXE.exists():
        from paper_1603_03820_b200 import build as B
        B.build_cpp_tests()
    m, n, nnz, f, lam = bench.CONFIGS["netflix"]
    seed = bench.RUN_SEED
    ref = json.loads((GOLD / "netflix_ref_10iter.json").read_text())
    assert ref["shape"] == {"m": m, "n": n, "nnz": nnz, "f": f, "lambda": lam, "seed": seed, "iterations": 10}
    cache = tmp_path / "netflix.cache"
    A.save_binary_cache(A.synth_csr(m, n, nnz, bench.data_seed("netflix")), cache)
    res = subprocess.run([str(EXE), str(cache), str(f), repr(lam), "10", str(seed), "0", "-", str(tmp_path / "o.csv"),
                          "0", str(tmp_path / "o")], capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout + res.stderr
    head, ours = _csv(tmp_path / "o.csv")
    head_r, theirs = _csv(GOLD / "netflix_ref_10iter.csv")
    assert head == head_r == "iteration,wall_seconds,train_J,test_RMSE"
    assert [r[0] for r in ours] == [r[0] for r in theirs] == list(range(1, 11))
    for a, b in zip(ours, theirs):
        assert abs(a[3] - b[3]) <= 1e-4, (a, b)            # test RMSE, absolute
        assert abs(a[2] - b[2]) <= 1e-4 * abs(b[2]), (a, b)  # train objective J, relative
    # final train / test RMSE of our factors on the reference's split of the cache
    x = A.FactorMatrix(m, f, np.fromfile(tmp_path / "o_x.f32", np.float32))
    t = A.FactorMatrix(n, f, np.fromfile(tmp_path / "o_theta.f32", np.float32))
    sp = A.split_train_test(A.load_binary_cache(cache), 0.1, A.mix_seed(seed, 2))
    train = A.rmse(A.csr_to_triplets(sp.train), x, t)
    test = A.rmse(sp.test, x, t)
    assert abs(train - ref["train_rmse_final"]["ref"]) <= 1e-4
    assert abs(test - ref["test_rmse_final"]["ref"]) <= 1e-4
