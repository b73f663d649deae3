"""Phase timeline of pass_wide_kernel on a trace-R sample (debug aid).

Needs the traced build: tools/ab_build.sh wtrace -DRH_WIDE_TRACE (run with
RESIHP_B200_LIB pointing at it).  Prints, for the first wave of CTAs and for
later ones, the median duration of each phase (thread 0's globaltimer).
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_06374_b200 import _lib  # noqa: E402
from paper_2605_06374_b200.detect_pass import DetectorPass, synthesize_measurements  # noqa: E402
from paper_2605_06374_b200.scenarios import c2_trace  # noqa: E402

tr = c2_trace(10_000, seed=0, tp=8, dp=32, pp=16, layers=80, M=512)
synthesize_measurements(tr, seed=0)
p = DetectorPass(tr)
for _ in range(3):
    p.detect(prepare_screen=False)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (4096 * 8))()
_lib.load_library().rh_debug_wide_trace(buf)
t = np.array(buf[:], np.int64).reshape(4096, 8)
t = t - t[:, 0].min()
names = ["setup issue", "TMA wait", "sum l^2", "checks", "walk", "epilogue", "barrier + stores"]
t = t[:, [0, 1, 2, 7, 3, 4, 5, 6]]
order = np.argsort(t[:, 0])
wave = 148 * 8
print(f"CTAs 4096 of 5000, span of these {t[:, 7].max() / 1e3:.1f} us")
for label, sel in (("first wave", order[:wave]), ("later", order[wave:])):
    d = np.diff(t[sel, :8], axis=1) / 1e3
    life = (t[sel, 7] - t[sel, 0]) / 1e3
    print(f"{label:10s} lifetime median {np.median(life):6.1f} us | " +
          " | ".join(f"{n} {np.median(d[:, k]):5.1f}" for k, n in enumerate(names)))
