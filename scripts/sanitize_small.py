"""Small shapes through every kernel family, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): tensor-core half-sweep (tc_update + tc_solve, long and short rows,
f = 16 / 37 / 100), FFMA and small-f engines, FP64-exact path, data-parallel partials,
transposes (counting and radix), device split, loss / RMSE.
usage: compute-sanitizer --tool <tool> python scripts/sanitize_small.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_03820_b200 import alskit as A  # noqa: E402
from paper_1603_03820_b200.distributed import HYBRID, MODEL, MultiGpuALS  # noqa: E402
from paper_1603_03820_b200.session import DeviceCsr, PREC_FP32, PREC_FP64_EXACT  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
for (m, n, nnz, f) in [(300, 120, 9000, 100), (200, 700, 30000, 37), (150, 90, 3000, 16), (400, 300, 5000, 10)]:
    R = A.synth_csr(m, n, nnz, int(rng.integers(1 << 30)))
    th = A.random_factor(n, f, 7)
    for acc in (False, True):
        cfg = A.SolverConfig(f=f, lambda_=0.05, accumulate_double=acc)
        x = A.update_x(R, th, cfg)
        t = A.update_theta(A.csr_to_csc(R), x, cfg)
        A.loss(R, x, t, 0.05)
    d = DeviceCsr.from_host(R, dev)
    dt = d.transpose()
    for mode in (MODEL, HYBRID):
        for prec in (PREC_FP32, PREC_FP64_EXACT):
            als = MultiGpuALS(None, mode, m, n, f, 0.05, prec, d, dt, None, torch.from_numpy(th.entries).to(dev))
            als.step()
            als.check()
            als.close()
    tr, te = d.split_train_test(0.1, 99)
torch.cuda.synchronize()
print("sanitize workload done")
