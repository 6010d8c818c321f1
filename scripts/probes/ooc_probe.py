"""Bring-up probe: out-of-core X half over a persisted Netflix-shape grid (block stream into
HBM + FP32 partial Hermitians + batched Cholesky) vs the in-core tensor-core half-sweep.
usage: python scripts/probes/ooc_probe.py [p q ...]"""
import sys
import tempfile
import time
from pathlib import Path
sys.path.insert(0, '.')
import torch
import bench
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import PREC_FP32, DeviceCsr, dev_update, out_of_core_update_x

grids = [int(a) for a in sys.argv[1:]] or [1, 4, 2, 4, 4, 8]
m, n, nnz, _, _ = bench.CONFIGS["netflix"]
train = A.split_train_test(A.synth_csr(m, n, nnz, bench.data_seed("netflix")), 0.1, A.mix_seed(42, 2)).train
f, lam = 100, 0.05
dev = torch.device("cuda")
T = torch.from_numpy(A.random_factor(train.cols, f, 9).entries).to(dev)
R = DeviceCsr.from_host(train, dev)
x_in = torch.zeros(train.rows * f, dtype=torch.float32, device=dev)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    dev_update(R, T, train.cols, f, lam, PREC_FP32, x_in)
    torch.cuda.synchronize(); ti = time.perf_counter() - t
print(f"in-core X half {ti * 1e3:.1f} ms", flush=True)
for p, q in zip(grids[::2], grids[1::2]):
    with tempfile.TemporaryDirectory() as tmp:
        g = A.grid_partition(train, p, q)
        A.persist_grid(g, Path(tmp) / "g")
        x = torch.zeros_like(x_in)
        for _ in range(2):
            torch.cuda.synchronize(); t = time.perf_counter()
            out_of_core_update_x(Path(tmp) / "g", T, f, lam, x)
            torch.cuda.synchronize(); to = time.perf_counter() - t
        gap = float((x - x_in).abs().max() / x_in.abs().max())
        print(f"out-of-core {p}x{q}: {to * 1e3:.1f} ms (gap {gap:.2e})", flush=True)
