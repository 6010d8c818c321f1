"""Bring-up probe: split_train_test at the Netflix shape, host (alsk_split_train_test) vs
device compaction (alsk_dev_split_train_test, host Fisher-Yates + HBM scatter), and the
binary cache -> HBM loader against the host loader + upload.
usage: python scripts/probes/split_probe.py"""
import sys
import tempfile
import time
from pathlib import Path
sys.path.insert(0, '.')
import torch
import bench
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import DeviceCsr

m, n, nnz, _, _ = bench.CONFIGS["netflix"]
r = A.synth_csr(m, n, nnz, A.mix_seed(42, 100 + bench.SHAPE_ID["netflix"]))
dev = torch.device("cuda")
d = DeviceCsr.from_host(r, dev)
seed = A.mix_seed(42, 2)
for it in range(2):
    t = time.perf_counter(); A.split_train_test(r, 0.1, seed); th = time.perf_counter() - t
    torch.cuda.synchronize(); t = time.perf_counter(); d.split_train_test(0.1, seed); torch.cuda.synchronize()
    td = time.perf_counter() - t
    print(f"split: host {th:.3f} s, device {td:.3f} s", flush=True)
with tempfile.TemporaryDirectory() as tmp:
    p = Path(tmp) / "r.cache"
    t = time.perf_counter(); A.save_binary_cache(r, p); ts = time.perf_counter() - t
    for it in range(2):
        t = time.perf_counter(); h = A.load_binary_cache(p); DeviceCsr.from_host(h, dev); torch.cuda.synchronize()
        th = time.perf_counter() - t
        t = time.perf_counter(); DeviceCsr.from_cache(p, dev); torch.cuda.synchronize(); td = time.perf_counter() - t
        gb = p.stat().st_size / 1e9
        print(f"cache ({gb:.2f} GB, save {ts:.2f} s): host load+upload {th:.3f} s, streamed to HBM {td:.3f} s "
              f"({gb / td:.1f} GB/s)", flush=True)
