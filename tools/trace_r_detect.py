"""One detect launch on SURVEY trace R (10^5 iterations, a 10^4 sample tiled
10x; for ncu: the second launch is the measured one)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06374_b200.detect_pass import DetectorPass, synthesize_measurements  # noqa: E402
from paper_2605_06374_b200.scenarios import c2_trace  # noqa: E402

sample = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
tr = c2_trace(sample, seed=0, tp=8, dp=32, pp=16, layers=80, M=512)
synthesize_measurements(tr, seed=0)
tr = bench.tile_trace(tr, reps)
p = DetectorPass(tr)
for _ in range(2):
    p.detect(prepare_screen=False)
torch.cuda.synchronize()
print("bytes", bench.algorithmic_bytes(tr), "iterations", tr.n_iter)
