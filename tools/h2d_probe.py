"""Pinned host<->device copy throughput on this box: H2D alone (1 / 2 / 4
streams), D2H alone, and both directions at once (the e2e wire sizes:
19.7 MB in, 3.3 MB out).  Debug aid."""
import time

import torch

n, m = 19_656_196, 3_300_008
x = torch.empty(n, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
xo = torch.empty(m, dtype=torch.uint8).pin_memory()
yo = torch.empty(m, dtype=torch.uint8, device="cuda")
for _ in range(3):
    y.copy_(x, non_blocking=True)
    xo.copy_(yo, non_blocking=True)
torch.cuda.synchronize()


def timed(fn, reps=30):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
        torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = (n + streams - 1) // streams

    def h2d():
        for k, st in enumerate(ss):
            with torch.cuda.stream(st):
                y[k * chunk:(k + 1) * chunk].copy_(x[k * chunk:(k + 1) * chunk], non_blocking=True)

    dt = timed(h2d)
    print(f"H2D {n / 1e6:.1f} MB over {streams} stream(s): {dt * 1e3:.3f} ms  {n / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def d2h():
    with torch.cuda.stream(s2):
        xo.copy_(yo, non_blocking=True)


dt = timed(d2h)
print(f"D2H {m / 1e6:.1f} MB: {dt * 1e3:.3f} ms  {m / dt / 1e9:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        y.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(6):  # ~20 MB out while 19.7 MB go in
            xo.copy_(yo, non_blocking=True)


dt = timed(both)
print(f"H2D {n / 1e6:.1f} MB || D2H {6 * m / 1e6:.1f} MB: {dt * 1e3:.3f} ms")
e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
f1, f2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
with torch.cuda.stream(s1):
    e1.record()
    y.copy_(x, non_blocking=True)
    e2.record()
with torch.cuda.stream(s2):
    f1.record()
    for _ in range(6):
        xo.copy_(yo, non_blocking=True)
    f2.record()
torch.cuda.synchronize()
print(f"  concurrent: H2D {e1.elapsed_time(e2):.3f} ms ({n / e1.elapsed_time(e2) / 1e6:.1f} GB/s), "
      f"D2H {f1.elapsed_time(f2):.3f} ms ({6 * m / f1.elapsed_time(f2) / 1e6:.1f} GB/s)")
