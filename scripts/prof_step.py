"""One Netflix-shape ALS iteration (X-half then Theta-half) through alsk_dev_update with the
chosen precision, for ncu captures: python scripts/prof_step.py [precision] [iters]."""
import sys
sys.path.insert(0, '.')
import torch
import bench
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import DeviceCsr, dev_update
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
train, test = bench.make_data('netflix')
dev = torch.device('cuda')
R = DeviceCsr.from_host(train, dev); RT = R.transpose()
m, n, f = 480189, 17770, 100
X = torch.from_numpy(A.random_factor(m, f, 42).entries).to(dev)
T = torch.from_numpy(A.random_factor(n, f, A.mix_seed(42, 1)).entries).to(dev)
for it in range(iters):
    dev_update(R, T, n, f, 0.05, prec, X)
    dev_update(RT, X, m, f, 0.05, prec, T)
torch.cuda.synchronize()
print("done")
