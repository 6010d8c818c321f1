"""Probe (not a test): time the batched FP32 solve alone on packed rows of the Netflix-shape
X half (the first ROWS users), CUDA events on the launching stream; prints ms scaled to the
whole X half. usage: python scripts/probes/solve_bench.py [rows=200000] [reps=5] [f=100]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_03820_b200 import alskit as A  # noqa: E402
from paper_1603_03820_b200 import datagen as G  # noqa: E402
from paper_1603_03820_b200.distributed import cuda_partial_hermitian_f32, cuda_solve_packed_f32, packed_stride  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
m, n, nnz, f, lam = bench.CONFIGS["netflix"]
if len(sys.argv) > 3:
    f = int(sys.argv[3])
dev = torch.device("cuda", 0)
mask = G.holdout_mask(nnz, 0.1, G.split_seed())
rd = G.build_rank_data("netflix", 0, 1, dev, mask)
theta = torch.from_numpy(A.random_factor(n, f, A.mix_seed(42, 1)).entries).to(dev)
pk = torch.empty(rows * packed_stride(f), dtype=torch.float32, device=dev)
x = torch.empty(rows * f, dtype=torch.float32, device=dev)
cuda_partial_hermitian_f32(rd.x, theta, n, f, lam, 0, rows, pk)
torch.cuda.synchronize()
ts = []
for _ in range(reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cuda_solve_packed_f32(pk, rows, f, x)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = sorted(ts[1:])
med = ts[len(ts) // 2]
print(f"solve f={f} rows={rows}: {med:.3f} ms median ({ts[0]:.3f} min) -> {med * m / rows:.2f} ms per X half "
      f"({rows * packed_stride(f) * 4 / med / 1e6:.0f} GB/s of packed rows); x checksum {float(x.double().sum()):.6e}")
