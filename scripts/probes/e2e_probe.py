"""Bring-up probe: host-buffer API (alsk_update_x) timing per engine at Netflix shape."""
import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_1603_03820_b200 import _native as N, alskit as A
train, test = bench.make_data('netflix')
m, n, f, lam = 480189, 17770, 100, 0.05
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
rp, ci, vv = pin(train.row_ptr), pin(train.col_idx), pin(train.values)
T = pin(A.random_factor(n, f, A.mix_seed(42, 1)).entries)
X = pin(A.random_factor(m, f, 42).entries)
nz = int(train.row_ptr[-1])
csr = N.CsrT(m, n, 0, nz, rp.data_ptr(), ci.data_ptr(), vv.data_ptr())
cfg = N.SolverConfigT(f, lam, 16, 4096, 0, 0, 42)
for eng in ("tensor", "ffma", "tensor"):
    A.set_fp32_engine(eng)
    for it in range(3):
        t = time.perf_counter()
        A._check(N.LIB.alsk_update_x(C.byref(csr), T.data_ptr(), n, f, C.byref(cfg), X.data_ptr()))
        print(eng, it, f"{(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
