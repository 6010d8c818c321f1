"""Bring-up probe: device half-sweep time for small ranks (the FFMA engine, f < 16) on a
SparkALS-like sparse shape (many short rows): rows x cols with ~5 ratings per row.
usage: python scripts/probes/small_f_probe.py [rows] [cols] [per_row] [f ...]"""
import sys
import time
sys.path.insert(0, '.')
import torch
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import DeviceCsr, dev_update

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
per = int(sys.argv[3]) if len(sys.argv) > 3 else 5
fs = [int(a) for a in sys.argv[4:]] or [10]
R = A.synth_csr(rows, cols, rows * per, 11)
dev = torch.device('cuda')
Rd = DeviceCsr.from_host(R, dev)
RT = Rd.transpose()
nnz = rows * per
for f in fs:
    T = torch.from_numpy(A.random_factor(cols, f, 5).entries).to(dev)
    X = torch.from_numpy(A.random_factor(rows, f, 6).entries).to(dev)
    for it in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        dev_update(Rd, T, cols, f, 0.05, 1, X)
        torch.cuda.synchronize()
        tx = time.perf_counter() - t
        t = time.perf_counter()
        dev_update(RT, X, rows, f, 0.05, 1, T)
        torch.cuda.synchronize()
        tt = time.perf_counter() - t
    gb = nnz * (8 + 4 * f) / 1e9
    print(f"f={f}: X-half {tx * 1e3:.2f} ms ({gb / tx:.0f} GB/s gathered), Theta-half {tt * 1e3:.2f} ms "
          f"({gb / tt:.0f} GB/s)", flush=True)
