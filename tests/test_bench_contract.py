"""bench.py's reference arm is the reference algorithm on the host cores and
nothing else: its process must never map the product library (the driver
voids the comparison otherwise).  CPU only."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

PROBE = r"""
import runpy, sys
sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3']
runpy.run_path('bench.py', run_name='__main__')
maps = open('/proc/self/maps').read()
print('MAPS', 'libresihp_b200' in maps, 'liboracle' in maps)
"""


def test_reference_arm_never_loads_the_product_library():
    out = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = out.stdout.strip().splitlines()
    rec = json.loads(next(l for l in lines if l.startswith("{")))
    assert rec["impl"] == "reference" and rec["value"] > 0
    assert rec["cpu_baseline"]["kind"] in ("port", "reference")
    assert lines[-1] == "MAPS False True", lines[-1]
