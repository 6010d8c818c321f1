"""Bring-up probe: device half-sweep time (tensor-core engine) across factor ranks on a
Netflix-like X-half slice (200K users x 17,770 items, ~186 ratings per user).
usage: python scripts/probes/f_sweep.py [f ...]"""
import sys
import time
sys.path.insert(0, '.')
import torch
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import DeviceCsr, dev_update

fs = [int(a) for a in sys.argv[1:]] or [16, 32, 64, 96, 100, 112, 119]
m, n = 200_000, 17770
R = A.synth_csr(m, n, m * 186, 77)
dev = torch.device('cuda')
Rd = DeviceCsr.from_host(R, dev)
for f in fs:
    T = torch.from_numpy(A.random_factor(n, f, 5).entries).to(dev)
    X = torch.empty(m * f, dtype=torch.float32, device=dev)
    for it in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        dev_update(Rd, T, n, f, 0.05, 2, X)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"f={f:4d}: {dt * 1e3:7.2f} ms  ({dt * 1e9 / (m * 186):.2f} ns/rating)", flush=True)
