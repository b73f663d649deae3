"""Per-call timing of the e2e host pass (bench's C2 trace) + raw PCIe copy rates."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06374_b200.detect_pass import DetectorPass  # noqa: E402

dev = torch.device("cuda", 0)
for nbytes in (19_656_196, 31_405_288):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    print(f"H2D {nbytes/1e6:.1f} MB: {dt*1e3:.3f} ms = {nbytes/dt/1e9:.1f} GB/s")
    t0 = time.perf_counter()
    for _ in range(20):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    print(f"D2H {nbytes/1e6:.1f} MB: {dt*1e3:.3f} ms = {nbytes/dt/1e9:.1f} GB/s")

tr = bench.build_trace(0, bench.N_ITER, use_oracle=False)
p = DetectorPass(tr, dev)
p.run()
torch.cuda.synchronize()


class A:
    warmup = 1
    steps = 1


ts = []
for k in range(12):
    r = bench.run_e2e(tr, p, A, dev)
    ts.append(r["step_s"] * 1e3)
print("per-call ms (each run_e2e call = 1 warmup + 1 timed):", [round(x, 3) for x in ts])
os.environ["RH_NO_GRAPH"] = "1"
r = bench.run_e2e(tr, p, A, dev)
print("no-graph call ms", round(r["step_s"] * 1e3, 3))
from paper_2605_06374_b200 import _lib  # noqa: E402
print("graph in use:", "see RH_NO_GRAPH comparison above")
