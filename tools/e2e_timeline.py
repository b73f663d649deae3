"""Device timeline of one e2e host pass (C2): RH_HOST_TRACE milestones
(copy / detect / read-back per chunk, screen) relative to the call's first
event, from the replayed CUDA graph (RH_NO_GRAPH=1: direct enqueue).  Debug aid."""
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
class A: warmup = 3; steps = 3
r = bench.run_e2e(tr, p, A, dev)
print('%%.1f us per call (with trace events)' %% (r['step_s'] * 1e6))
""" % ROOT
env = dict(os.environ, RH_HOST_TRACE="1")
out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
lines = [l for l in out.stderr.splitlines() if l.startswith("rh_host_trace")]
last = max((k for k, l in enumerate(lines) if " call " in l), default=None)
print("\n".join(lines[last:] if last is not None else out.stderr.splitlines()[-20:]))
print(out.stdout.strip())
print("\n".join(l for l in out.stderr.splitlines()[-8:] if not l.startswith("rh_host_trace")))
