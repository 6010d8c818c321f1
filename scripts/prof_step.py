"""The benched iteration for ncu captures: bench.py's single-GPU path (the C++ session
alsk_mp with its own packed-row workspace, the same data builder), without bench.py's
extra legs. usage: python scripts/prof_step.py [config=netflix] [iters=1] [precision=fp32]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_03820_b200 import alskit as A  # noqa: E402
from paper_1603_03820_b200 import datagen as G  # noqa: E402
from paper_1603_03820_b200.distributed import MODEL, MultiGpuALS  # noqa: E402
from paper_1603_03820_b200.session import PREC_FP32, PREC_FP64_EXACT  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "netflix"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prec = PREC_FP64_EXACT if (len(sys.argv) > 3 and sys.argv[3] == "fp64") else PREC_FP32
m, n, nnz, f, lam = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
mask = G.holdout_mask(nnz, 0.1, G.split_seed())
rd = G.build_rank_data(cfg, 0, 1, dev, mask)
theta0 = torch.from_numpy(A.random_factor(n, f, A.mix_seed(42, 1)).entries).to(dev)
als = MultiGpuALS(None, MODEL, m, n, f, lam, prec, rd.x, rd.t, None, theta0)
for _ in range(iters):
    als.step()
als.check()
torch.cuda.synchronize()
print("done")
