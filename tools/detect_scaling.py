"""Detect-kernel time vs trace length on the C2 shape (wave / fixed-cost study).  Debug aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06374_b200.detect_pass import DetectorPass  # noqa: E402

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
for n_iter in [int(x) for x in (sys.argv[1:] or ["1480", "2960", "5920", "10000", "11840", "23680"])]:
    tr = bench.build_trace(0, n_iter, use_oracle=False)
    p = DetectorPass(tr, dev)
    for _ in range(3):
        fl.fill_(1)
        p.run()
    torch.cuda.synchronize()
    n = 100
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n)]
    for k in range(n):
        fl.fill_(k & 255)
        ev[k][0].record(st)
        p.detect()
        ev[k][1].record(st)
        p.screen()
        ev[k][2].record(st)
    torch.cuda.synchronize()
    d = sum(e[0].elapsed_time(e[1]) for e in ev) / n * 1e3
    s = sum(e[1].elapsed_time(e[2]) for e in ev) / n * 1e3
    print(f"n_iter {n_iter:6d}  CTAs {(n_iter + 7) // 8:5d}  detect {d:7.2f} us  screen {s:7.2f} us"
          f"  per-iter detect {d / n_iter * 1e3:6.2f} ns", flush=True)
