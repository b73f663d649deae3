"""Time the detect kernel on SURVEY trace R at its full 10^5 iterations (a 10^4
sample tiled 10x in HBM, as bench.py's trace_R line), for A/B builds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06374_b200.detect_pass import DetectorPass, synthesize_measurements  # noqa: E402
from paper_2605_06374_b200.scenarios import c2_trace  # noqa: E402

tr = c2_trace(10_000, seed=0, tp=8, dp=32, pp=16, layers=80, M=512)
synthesize_measurements(tr, seed=0)
tr = bench.tile_trace(tr, 10)
p = DetectorPass(tr)
for _ in range(2):
    p.detect(prepare_screen=False)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(7):
    ev[0].record()
    p.detect(prepare_screen=False)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ts.sort()
nb = bench.algorithmic_bytes(tr)
print(f"trace R 10^5: detect median {ts[3]:.3f} ms min {ts[0]:.3f} ms -> {nb / (ts[3] * 1e-3) / 1e9:.0f} GB/s "
      f"({nb / (ts[3] * 1e-3) / 1e9 / 6536.7:.3f} of HBM)")
