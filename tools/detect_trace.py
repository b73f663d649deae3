"""Phase timeline of pass_small_kernel on the bench's C2 trace (debug aid).

Needs the traced build: tools/ab_build.sh dtrace -DRH_DETECT_TRACE.  Prints,
for CTAs of the first and of later waves, the median duration of each phase
(warp 0's globaltimer): setup loads, TMA wait + sum l^2, base costs, walk,
block barrier, epilogue.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("RESIHP_B200_LIB", os.path.join(ROOT, "tools", "ab", "lib_dtrace.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06374_b200 import _lib  # noqa: E402
from paper_2605_06374_b200.detect_pass import DetectorPass  # noqa: E402

n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else bench.N_ITER
dev = torch.device("cuda", 0)
tr = bench.build_trace(0, n_iter, use_oracle=False)
p = DetectorPass(tr, dev)
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
for _ in range(3):
    fl.fill_(1)
    p.run()
fl.fill_(2)
p.detect()
torch.cuda.synchronize()
buf = (C.c_ulonglong * (4096 * 8))()
_lib.load_library().rh_debug_detect_trace(buf)
n_blk = min(4096, (n_iter + 3) // 4)  # 64-thread CTAs of 4 iterations (dp 16)
t = np.array(buf[:], np.int64).reshape(4096, 8)[:n_blk]
t0 = t[:, 0].min()
start = t[:, 0] - t0
end = t[:, 6] - t0
print(f"CTAs {n_blk}  kernel span {end.max() / 1e3:.2f} us  (first start -> last end)")
names = ["setup", "tma-wait", "sumsq", "base", "walk", "epilogue"]  # (mark 5: after the TMA wait)
first = start < 1000  # started within 1 us of the first CTA
for label, sel in (("wave 1", first), ("later", ~first)):
    if not sel.any():
        continue
    tt = t[sel][:, [0, 1, 5, 2, 3, 4, 6]]
    d = np.diff(tt, axis=1) / 1e3
    med = np.median(d, axis=0)
    print(f"{label:7s} n={sel.sum():5d} start med {np.median(start[sel]) / 1e3:6.2f} us  life med "
          f"{np.median((end - start)[sel]) / 1e3:6.2f} us  " +
          "  ".join(f"{n} {m:5.2f}" for n, m in zip(names, med)))
sm = t[:, 7]
print("CTAs per SM (max):", np.bincount(sm[first].astype(int)).max() if first.any() else 0)
