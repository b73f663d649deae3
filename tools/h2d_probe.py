"""Pinned host->device copy throughput on this box: one stream vs two streams
(both copy engines), for the e2e wire size (19.7 MB).  Debug aid."""
import time

import torch

n = 19_656_196
x = torch.empty(n, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = (n + streams - 1) // streams
    t = time.perf_counter()
    for _ in range(30):
        for k, st in enumerate(ss):
            with torch.cuda.stream(st):
                y[k * chunk:(k + 1) * chunk].copy_(x[k * chunk:(k + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 30
    print(f"H2D {n / 1e6:.1f} MB over {streams} stream(s): {dt * 1e3:.3f} ms  {n / dt / 1e9:.1f} GB/s")
