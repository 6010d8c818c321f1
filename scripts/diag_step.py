"""Per-half timing of the device path at Netflix shape: CUDA events around alsk_dev_update
and the library's kernel-only events. usage: diag_step.py [precision=1] [iters=4]"""
import ctypes as C, sys, time
sys.path.insert(0, '.')
import torch
import bench
from paper_1603_03820_b200 import _native as N, alskit as A
from paper_1603_03820_b200.session import DeviceCsr, dev_update
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
train, test = bench.make_data('netflix')
dev = torch.device('cuda')
R = DeviceCsr.from_host(train, dev); RT = R.transpose()
m, n, f = 480189, 17770, 100
X = torch.from_numpy(A.random_factor(m, f, 42).entries).to(dev)
T = torch.from_numpy(A.random_factor(n, f, A.mix_seed(42, 1)).entries).to(dev)
for it in range(iters):
    for name, Rd, th, tr, out in (('x', R, T, n, X), ('t', RT, X, m, T)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        N.LIB.alsk_profile_begin()
        h0 = time.perf_counter(); e0.record()
        dev_update(Rd, th, tr, f, 0.05, prec, out)
        e1.record(); torch.cuda.synchronize(); h1 = time.perf_counter()
        kms, kl = C.c_double(), C.c_uint64(); N.LIB.alsk_profile_end(C.byref(kms), C.byref(kl))
        print(f"prec{prec} it{it} {name}: events {e0.elapsed_time(e1):7.2f} ms  host {1e3*(h1-h0):7.2f} ms  kernel {kms.value:7.2f} ms")
