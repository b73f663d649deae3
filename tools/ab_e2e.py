"""A/B of the e2e host pass (bench.run_e2e, C2) across library builds.  Debug aid."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, torch
sys.path.insert(0, %r)
import bench
from paper_2605_06374_b200.detect_pass import DetectorPass
dev = torch.device('cuda', 0)
tr = bench.build_trace(0, bench.N_ITER, use_oracle=False)
p = DetectorPass(tr, dev); p.run(); torch.cuda.synchronize()
class A: warmup = 5; steps = 60
r = bench.run_e2e(tr, p, A, dev)
print('%%.1f us per call' %% (r['step_s'] * 1e6))
""" % ROOT
for rep in range(3):
    for lib in sys.argv[1:]:
        env = dict(os.environ, RESIHP_B200_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print(rep, os.path.basename(lib), (out.stdout.strip().splitlines() or [out.stderr[-300:]])[-1], flush=True)
