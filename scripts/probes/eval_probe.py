"""Bring-up probe: device loss (J) and RMSE at the Netflix shape (solver.hpp:358-406).
usage: python scripts/probes/eval_probe.py"""
import sys
import time
sys.path.insert(0, '.')
import torch
import bench
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import AlsSession

train, test = bench.make_data("netflix")
cfg = A.SolverConfig(f=100, lambda_=0.05, accumulate_double=False)
sess = AlsSession(train, None, test, cfg, A.random_factor(train.rows, 100, 42),
                  A.random_factor(train.cols, 100, A.mix_seed(42, 1)))
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); J = sess.loss(); tl = time.perf_counter() - t
    t = time.perf_counter(); e = sess.rmse(); tr = time.perf_counter() - t
print(f"loss {tl * 1e3:.2f} ms (J={J!r}), rmse {tr * 1e3:.2f} ms (rmse={e!r})", flush=True)
