"""Bring-up probe: cost of per-half checkpoints on the device session at the Netflix shape
(train_resumable with the device writer) against the same iterations without snapshots.
usage: python scripts/probes/ckpt_probe.py [iterations]"""
import sys
import tempfile
import time
sys.path.insert(0, '.')
import torch
import bench
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import AlsSession, train_resumable

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
train, test = bench.make_data("netflix")
cfg = A.SolverConfig(f=100, lambda_=0.05, accumulate_double=False)
x0 = A.random_factor(train.rows, 100, 42)
t0 = A.random_factor(train.cols, 100, A.mix_seed(42, 1))
sess = AlsSession(train, None, test, cfg, x0, t0)
sess.half_x(); sess.half_theta(); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(iters):
    sess.half_x(); sess.half_theta(); sess.loss(); sess.rmse()
torch.cuda.synchronize()
plain = (time.perf_counter() - t) / iters
with tempfile.TemporaryDirectory() as d:
    sess2 = AlsSession(train, None, test, cfg, x0, t0)
    t = time.perf_counter()
    train_resumable(sess2, iters, d, digest=1, resume=False)
    torch.cuda.synchronize()
    ck = (time.perf_counter() - t) / iters
print(f"per iteration (with loss+rmse): {plain * 1e3:.1f} ms plain, {ck * 1e3:.1f} ms with X and Theta "
      f"checkpoints ({(train.rows + train.cols) * 400 / 1e6:.0f} MB per iteration)", flush=True)
