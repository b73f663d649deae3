"""A/B timing of the C2 device-resident Detector pass across library builds.

usage: python tools/ab_detect.py lib_a.so lib_b.so ...   (each timed in its own
process via RESIHP_B200_LIB; bench.py's protocol: L2 flush, event-timed detect
and screen, 200 steps, repeated 3 times interleaved).  Debug aid only.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json, torch
sys.path.insert(0, %r)
import bench
from paper_2605_06374_b200.detect_pass import DetectorPass
dev = torch.device('cuda', 0)
tr = bench.build_trace(0, bench.N_ITER, use_oracle=False)
p = DetectorPass(tr, dev)
st = torch.cuda.current_stream(dev)
fl = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
for _ in range(5):
    fl.fill_(1); p.run()
torch.cuda.synchronize()
n = 200
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n)]
import os
noflush = bool(os.environ.get("AB_NOFLUSH"))
for k in range(n):
    if not noflush:
        fl.fill_(k & 255)
    ev[k][0].record(st); p.detect(); ev[k][1].record(st); p.screen(); ev[k][2].record(st)
torch.cuda.synchronize()
d = sorted(e[0].elapsed_time(e[1]) for e in ev)
s = sorted(e[1].elapsed_time(e[2]) for e in ev)
r = p.results()
print(json.dumps({"det_us": 1e3 * sum(d) / n, "det_med": 1e3 * d[n // 2], "scr_us": 1e3 * sum(s) / n,
                  "scr_med": 1e3 * s[n // 2], "alarm": int(r["status"].sum())}))
""" % ROOT

for rep in range(3):
    for lib in sys.argv[1:]:
        env = dict(os.environ, RESIHP_B200_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
        print(rep, os.path.basename(lib), line, flush=True)
