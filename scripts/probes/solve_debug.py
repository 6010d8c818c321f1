"""Bring-up probe: the TMEM Cholesky solve on a few tiny systems, with a watchdog."""
import sys, os, time
sys.path.insert(0, '.')
import numpy as np
from paper_1603_03820_b200 import alskit as A
f = int(sys.argv[1]) if len(sys.argv) > 1 else 16
m = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = 40
r = A.synth_csr(m, n, m * 10, 5)
th = A.random_factor(n, f, 7)
t0 = time.time()
with A.use_fp32_engine("tensor"):
    x = A.update_x(r, th, A.SolverConfig(f=f, lambda_=0.05, accumulate_double=False))
print("tensor done", time.time() - t0, flush=True)
x64 = A.update_x(r, th, A.SolverConfig(f=f, lambda_=0.05, accumulate_double=True))
print("gap", np.abs(x.entries - x64.entries).max() / np.abs(x64.entries).max())
