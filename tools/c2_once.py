"""Run the bench's C2 Detector pass a few times (an ncu target; debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06374_b200.detect_pass import DetectorPass  # noqa: E402

dev = torch.device("cuda", 0)
tr = bench.build_trace(0, bench.N_ITER, use_oracle=False)
p = DetectorPass(tr, dev)
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    fl.fill_(k & 255)
    p.run()
torch.cuda.synchronize()
print("ok", int(p.results()["status"].sum()))
