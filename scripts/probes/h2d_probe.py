"""Bring-up probe: pinned host<->device copy bandwidth on this box (what bounds the serial
part of the host-buffer API: the gathered factor must be resident before a half-sweep)."""
import time
import torch

for mb in (64, 256, 1024):
    n = mb << 18  # floats
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device='cuda')
    for direction in ("h2d", "d2h"):
        for _ in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            if direction == "h2d":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
        print(f"{direction} {mb:5d} MB: {dt * 1e3:7.2f} ms  {mb / 1024 / dt:6.1f} GB/s", flush=True)
