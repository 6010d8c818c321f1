"""Netflix-shape RMSE parity against the reference itself (BASELINE north star: "train and
test RMSE within 1e-4 absolute after 10 iterations"), run on the GPU box:

* one binary cache written by the reference's save_binary_cache from the shared synthetic
  generator (bench.py's netflix shape and seed);
* the reference's own train_run (oracle/_ref, driver.hpp:107-268, accumulate_double = its
  default, all host threads) for 10 iterations with its metrics CSV;
* our C++ train_run (include/alskit/driver.hpp via tests/cpp/train_run_cli) on the same
  cache in the FP32 tensor-core mode and in the FP64-exact mode;
* per-iteration train J and test RMSE from both CSVs, the final factors compared (FP64 mode:
  bit for bit; FP32: normwise), and the final train RMSE of both factor pairs (the
  reference's split of the cache, evaluated by the same kernel).

Writes <out>/netflix_rmse_parity.json and copies the reference CSV to
tests/golden/netflix_ref_10iter.csv (the fixture tests/test_gpu_netflix_rmse.py checks).
usage: python scripts/netflix_rmse_parity.py [out_dir=gpurun_out] [iterations=10]"""
import ctypes as C
import json
import shutil
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import binding  # noqa: E402

out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
out.mkdir(parents=True, exist_ok=True)
scratch = Path("/tmp") / "netflix_rmse_parity"  # factor dumps (hundreds of MB) stay off gpurun_out
scratch.mkdir(parents=True, exist_ok=True)
m, n, nnz, f, lam = bench.CONFIGS["netflix"]
seed = bench.RUN_SEED
exe = ROOT / "tests" / "cpp" / "train_run_cli"
ref = binding.reference()
assert ref is not None, "oracle/_ref not built"

cache = Path("/tmp") / f"netflix_{bench.data_seed('netflix'):016x}.cache"
if not cache.exists():
    tmp = cache.with_suffix(".tmp")
    assert ref.bench_write_cache(m, n, nnz, bench.data_seed("netflix"), tmp) == 0, ref.last_error()
    tmp.replace(cache)


def ours(acc: int):
    pre = scratch / f"ours{acc}"
    t = time.perf_counter()
    res = subprocess.run([str(exe), str(cache), str(f), repr(lam), str(iters), str(seed), str(acc), "-",
                          str(out / f"ours{acc}.csv"), "0", str(pre)], capture_output=True, text=True, timeout=3600)
    assert res.returncode == 0, res.stdout + res.stderr
    return (np.fromfile(f"{pre}_x.f32", np.float32), np.fromfile(f"{pre}_theta.f32", np.float32),
            time.perf_counter() - t)


def theirs():
    x = np.zeros(m * f, np.float32)
    t = np.zeros(n * f, np.float32)
    start, dg = C.c_int(), C.c_uint64()
    t0 = time.perf_counter()
    st = ref.call("train_run", str(cache).encode(), f, C.c_double(lam), iters, C.c_uint64(seed), 1, None,
                  str(out / "ref.csv").encode(), 0, -1, x.ctypes.data_as(C.c_void_p), t.ctypes.data_as(C.c_void_p),
                  C.byref(start), C.byref(dg))
    assert st == 0, ref.last_error()
    return x, t, time.perf_counter() - t0


def csv_rows(p):
    lines = Path(p).read_text().splitlines()
    return [[float(v) for v in l.split(",")] for l in lines[1:] if not l.startswith("#")]


x32, t32, s32 = ours(0)
x64, t64, s64 = ours(1)
xr, tr, sr = theirs()

# final train RMSE of each factor pair on the reference's own split of the cache
from paper_1603_03820_b200 import alskit as A  # noqa: E402

r = A.load_binary_cache(cache)
sp = A.split_train_test(r, 0.1, A.mix_seed(seed, 2))
train_trip = A.csr_to_triplets(sp.train)


def rm(trip, x, t):
    return A.rmse(trip, A.FactorMatrix(rows=m, f=f, entries=x), A.FactorMatrix(rows=n, f=f, entries=t))


ro, r64, rr = csv_rows(out / "ours0.csv"), csv_rows(out / "ours1.csv"), csv_rows(out / "ref.csv")
res = {
    "shape": {"m": m, "n": n, "nnz": nnz, "f": f, "lambda": lam, "seed": seed, "iterations": iters},
    "seconds": {"ours_fp32_run": s32, "ours_fp64_run": s64, "reference_run": sr},
    "per_iteration": [{"iteration": int(a[0]), "ref_train_J": c[2], "ref_test_RMSE": c[3], "fp32_train_J": a[2],
                       "fp32_test_RMSE": a[3], "fp64_train_J": b[2], "fp64_test_RMSE": b[3]}
                      for a, b, c in zip(ro, r64, rr)],
    "max_abs_test_rmse_gap_fp32": max(abs(a[3] - c[3]) for a, c in zip(ro, rr)),
    "max_rel_train_J_gap_fp32": max(abs(a[2] - c[2]) / abs(c[2]) for a, c in zip(ro, rr)),
    "fp64_factors_bit_identical": bool(np.array_equal(x64, xr) and np.array_equal(t64, tr)),
    "fp64_csv_identical": (out / "ours1.csv").read_text().splitlines()[1:] == (out / "ref.csv").read_text().splitlines()[1:],
    "fp32_factor_normwise_gap": {"x": float(np.linalg.norm(x32 - xr) / np.linalg.norm(xr)),
                                 "theta": float(np.linalg.norm(t32 - tr) / np.linalg.norm(tr))},
    "train_rmse_final": {"ref": rm(train_trip, xr, tr), "fp32": rm(train_trip, x32, t32),
                         "fp64": rm(train_trip, x64, t64)},
    "test_rmse_final": {"ref": rm(sp.test, xr, tr), "fp32": rm(sp.test, x32, t32), "fp64": rm(sp.test, x64, t64)},
}
res["train_rmse_gap_fp32"] = abs(res["train_rmse_final"]["fp32"] - res["train_rmse_final"]["ref"])
res["test_rmse_gap_fp32"] = abs(res["test_rmse_final"]["fp32"] - res["test_rmse_final"]["ref"])
(out / "netflix_rmse_parity.json").write_text(json.dumps(res, indent=1))
shutil.copy(out / "ref.csv", out / "netflix_ref_10iter.csv")
print(json.dumps({k: res[k] for k in ("max_abs_test_rmse_gap_fp32", "max_rel_train_J_gap_fp32",
                                      "fp64_factors_bit_identical", "train_rmse_gap_fp32", "test_rmse_gap_fp32",
                                      "seconds")}))
