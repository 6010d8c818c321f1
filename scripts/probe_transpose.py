"""Device CSR -> CSC timing at a named shape (bench.CONFIGS train matrix, built in HBM):
CUDA events around alsk_dev_csr_to_csc, best of N after a warm-up, and the algorithmic
HBM bytes (col_idx read twice + values read once + row_idx/values written + pointers).
usage: python scripts/probe_transpose.py [config=netflix] [reps=5]
(ALSK_TRANSPOSE_RADIX=1 selects the two-pass radix path for comparison)"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_03820_b200 import _native as N  # noqa: E402
from paper_1603_03820_b200 import datagen as G  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "netflix"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
m, n, nnz, f, lam = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
mask = G.holdout_mask(nnz, 0.1, G.split_seed())
x = G.build_rank_data(cfg, 0, 1, dev, mask).x if cfg in ("ml1m", "netflix", "yahoo") else None
if x is None:  # big shapes: the train rows only (no transpose inside build_rank_data)
    x = G.concat_rows([G.dev_split_mask(G.dev_synth_rows(m, n, nnz, G.data_seed(cfg), u0, u1, dev),
                                        torch.from_numpy(mask).to(dev), G.row_start(m, nnz, u0), u0,
                                        int(N.LIB.alsk_mask_count(mask.ctypes.data, G.row_start(m, nnz, u0),
                                                                  G.row_start(m, nnz, u1))))[0]
                       for u0, u1 in G._chunks(m, nnz, 0, m, 1 << 28)], n, dev)
cp = torch.empty(n + 1, dtype=torch.int64, device=dev)
ri = torch.empty(x.nnz, dtype=torch.int32, device=dev)
cv = torch.empty(x.nnz, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
times = []
for i in range(reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    st = N.LIB.alsk_dev_csr_to_csc(C.byref(x.c), cp.data_ptr(), ri.data_ptr(), cv.data_ptr(), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    assert st == 0, N.LIB.alsk_last_error()
    if i:
        times.append(e0.elapsed_time(e1))
algo = x.nnz * 16 + 8 * (m + n + 2)  # read col+value, write row+value (the counting pass re-read is overhead)
best = min(times)
print(json.dumps({"config": cfg, "path": "radix" if os.environ.get("ALSK_TRANSPOSE_RADIX") else "counting",
                  "nnz": x.nnz, "ms_best": best, "ms_all": times, "algorithmic_bytes": algo,
                  "gbs": algo / (best * 1e-3) / 1e9}))
