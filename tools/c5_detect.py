"""One C5-shape detect pass (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_06374_b200.detect_pass import DetectorPass, synthesize_measurements  # noqa: E402
from paper_2605_06374_b200.scenarios import c2_trace  # noqa: E402

tr = c2_trace(int(sys.argv[1]) if len(sys.argv) > 1 else 2000, seed=0, tp=8, dp=32, pp=16,
              layers=80, M=512)
synthesize_measurements(tr, seed=0)
p = DetectorPass(tr)
for _ in range(2):
    p.detect(prepare_screen=False)
torch.cuda.synchronize()
