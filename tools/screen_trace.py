"""Per-round timeline of the cooperative screen kernel on the bench's C2 trace.

Builds a traced copy of the library (-DRH_SCREEN_TRACE) into tools/_trace/ and
prints, per Jacobi round: block 0's compute time, its barrier wait, the slowest
block's compute time, and the number of changed decisions.  Debug aid only.
"""
import ctypes as C
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
out = ROOT / "tools" / "_trace" / "libresihp_trace.so"
if not out.exists() or "--rebuild" in sys.argv:
    import __graft_entry__ as g

    out.parent.mkdir(exist_ok=True)
    srcs = sorted((ROOT / "paper_2605_06374_b200" / "csrc").glob("*.cu"))
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", *g.NVCC_FLAGS, "-DRH_SCREEN_TRACE",
                           "-shared", *map(str, srcs), "-o", str(out)])
    if "--build-only" in sys.argv:
        sys.exit(0)
os.environ["RESIHP_B200_LIB"] = str(out)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06374_b200 import _lib  # noqa: E402
from paper_2605_06374_b200.detect_pass import DetectorPass  # noqa: E402

dev = torch.device("cuda", 0)
shape = next((a for a in sys.argv[1:] if a in ("C1", "C5")), None)
if shape:  # another BASELINE shape (tools/detect_shapes.py's parameters), 4000 iterations
    from paper_2605_06374_b200.detect_pass import synthesize_measurements
    from paper_2605_06374_b200.scenarios import c2_trace

    kw = {"C1": dict(tp=4, dp=4, pp=2, layers=32, M=16),
          "C5": dict(tp=8, dp=32, pp=16, layers=80, M=512)}[shape]
    tr = c2_trace(4000, seed=0, **kw)
    synthesize_measurements(tr, seed=0)
else:
    tr = bench.build_trace(0, bench.N_ITER, use_oracle=False)
p = DetectorPass(tr, dev)
fn = _lib.load_library().rh_debug_screen_trace
t = (C.c_ulonglong * 96)()
slow = (C.c_ulonglong * 32)()
chg = (C.c_uint * 32)()
for rep in range(3):
    p.detect()
    p.screen()
    torch.cuda.synchronize()
fn(t, slow, chg)
tt = np.array(t[:], np.int64).reshape(32, 3)
for r in range(32):
    if tt[r, 0] == 0:
        break
    print(f"round {r}: block0 compute {(tt[r,1]-tt[r,0])/1e3:6.2f} us  barrier "
          f"{(tt[r,2]-tt[r,1])/1e3:6.2f} us  slowest block {slow[r]/1e3:6.2f} us  "
          f"changes {chg[r]}")
