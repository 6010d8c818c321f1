"""Bring-up probe: the block stream alone (no compute) over persisted Netflix-shape grids,
to split the out-of-core X half's time into loading and compute.
usage: python scripts/probes/stream_probe.py [p q ...]"""
import sys
import tempfile
import time
from pathlib import Path
sys.path.insert(0, '.')
import torch
import bench
from paper_1603_03820_b200 import alskit as A
from paper_1603_03820_b200.session import DeviceBlockStream

grids = [int(a) for a in sys.argv[1:]] or [1, 4, 4, 8, 8, 16]
train, _ = bench.make_data("netflix")
for p, q in zip(grids[::2], grids[1::2]):
    with tempfile.TemporaryDirectory() as tmp:
        d = Path(tmp) / "g"
        A.persist_grid(A.grid_partition(train, p, q), d)
        order = A.row_major_order(A.load_grid_meta(d))
        for _ in range(2):
            torch.cuda.synchronize(); t = time.perf_counter()
            with DeviceBlockStream(d, order) as bs:
                n = sum(1 for _ in bs)
            torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(f"stream only {p}x{q}: {dt * 1e3:.1f} ms for {n} blocks ({dt / n * 1e3:.2f} ms per block)", flush=True)
