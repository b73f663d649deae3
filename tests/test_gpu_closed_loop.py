"""the batched closed loop (closed_loop.run_batch) -- all
scenarios in lockstep, one predictor launch per iteration for all of them --
reproduces the reference's run_scenario rows bit for bit: observed and
predicted iteration times, alarms (candidate / benign / escalate /
confirmed / unconfirmed / adapt), charged wall time, plans and aborts, on
acceptance criterion 4's fail-slow scenarios plus fail-stop, slow-link and
multi-failure scenarios (tests/golden/closed_loop.json)."""

import numpy as np
import pytest

from tests.golden_io import load

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.float64(x).view(np.uint64)


def test_batched_closed_loop_matches_run_scenario(cuda_device):
    from paper_2605_06374_b200.closed_loop import run_batch

    cases = load("closed_loop")["cases"]
    got = run_batch([c["mapping"] for c in cases])
    for c, g in zip(cases, got):
        seed = c["mapping"]["seed"]
        assert g["aborted_at"] == c["aborted_at"], seed
        assert [list(p) for p in g["plans"]] == c["plans"], seed
        assert len(g["rows"]) == len(c["rows"]), seed
        for a, b in zip(g["rows"], c["rows"]):
            assert a["iteration"] == b["iteration"]
            assert a["alarms"] == b["alarms"], (seed, a["iteration"], a["alarms"], b["alarms"])
            assert _bits(a["observed_s"]) == _bits(b["observed_s"]), (seed, a["iteration"])
            assert _bits(a["predicted_s"]) == _bits(b["predicted_s"]), (seed, a["iteration"])
            assert _bits(a["wall_s"]) == _bits(b["wall_s"]), (seed, a["iteration"])
            assert a["active_devices"] == b["active_devices"]
            assert a["migrations"] == b["migrations"]
