"""Run the reference's own unit tests against the drop-in.

The test modules in this directory are the reference's tests, copied
unmodified from /root/reference/pkg/tests (provenance and sha256 in
README.md) -- /root/reference does not exist on the GPU box.  This conftest
makes `import resilsim.<module>` resolve to this repository's drop-in
package (paper_2605_06374_b200.<module>), so every `from resilsim.pipeline
import simulate_iteration` in them exercises the B200 implementation.  It is
collected only by tests/test_gpu_reference_suite.py (a GPU test), never by
the main suite (tests/conftest.py ignores this directory).
"""

import importlib
import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

_MODULES = ("cluster", "comm", "workload", "pipeline", "detector", "scheduler", "policies")

pkg = importlib.import_module("paper_2605_06374_b200")
shim = types.ModuleType("resilsim")
shim.__path__ = []  # a package, so `import resilsim.x` consults sys.modules
shim.__dict__.update({k: v for k, v in vars(pkg).items() if not k.startswith("__")})
sys.modules["resilsim"] = shim
for name in _MODULES:
    mod = importlib.import_module(f"paper_2605_06374_b200.{name}")
    sys.modules[f"resilsim.{name}"] = mod
    setattr(shim, name, mod)
