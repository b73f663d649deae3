"""Detector pass throughput at other BASELINE shapes (C1, C5 / SURVEY §8d trace R)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_06374_b200.detect_pass import DetectorPass, synthesize_measurements  # noqa: E402
from paper_2605_06374_b200.scenarios import c2_trace  # noqa: E402

shapes = {
    "C1": dict(tp=4, dp=4, pp=2, layers=32, M=16),
    "C2": dict(tp=4, dp=16, pp=4, layers=40, M=128),
    "C5": dict(tp=8, dp=32, pp=16, layers=80, M=512),
}
n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
for name, kw in shapes.items():
    t0 = time.perf_counter()
    tr = c2_trace(n_iter, seed=0, **kw)
    synthesize_measurements(tr, seed=0)
    build_s = time.perf_counter() - t0
    p = DetectorPass(tr)
    for _ in range(3):
        p.run()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    reps = 20
    det = scr = 0.0
    for _ in range(reps):
        e[0].record(); p.detect(); e[1].record(); p.screen(); e[2].record()
        torch.cuda.synchronize()
        det += e[0].elapsed_time(e[1]); scr += e[1].elapsed_time(e[2])
    det /= reps; scr /= reps
    nbytes = sum(tr.nbytes_per_iter().values()) * tr.n_iter
    dev = kw["tp"] * kw["dp"] * kw["pp"]
    print(f"{name}: {n_iter} it x {dev} dev, trace {nbytes/1e6:.1f} MB, detect {det*1e3:.1f} us "
          f"({nbytes/det/1e6:.0f} GB/s), screen {scr*1e3:.1f} us, "
          f"{n_iter*dev/((det+scr)*1e-3):.3e} samples/s (build {build_s:.1f}s)")
