"""Time the detect kernel on a SURVEY trace-R-shape sample (C5 shape), for A/B."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_06374_b200.detect_pass import DetectorPass, synthesize_measurements  # noqa: E402
from paper_2605_06374_b200.scenarios import c2_trace  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
tr = c2_trace(n, seed=0, tp=8, dp=32, pp=16, layers=80, M=512)
synthesize_measurements(tr, seed=0)
p = DetectorPass(tr)
for _ in range(3):
    p.detect(prepare_screen=False)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(10):
    ev[0].record()
    p.detect(prepare_screen=False)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ts.sort()
nbytes = sum(tr.nbytes_per_iter().values()) * n
print(f"trace R sample n={n}: detect median {ts[5]*1e3:.1f} us min {ts[0]*1e3:.1f} us "
      f"-> {nbytes / (ts[5] * 1e-3) / 1e9:.0f} GB/s")
