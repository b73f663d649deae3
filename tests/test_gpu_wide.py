"""GPU parity of the long-pipeline Detector kernels (5 <= P <= 16): the
thread-per-replica pass_wide_kernel and the lane-per-stage pass_kernel it
replaced (still the path for D > 64 or P outside the wide instantiations),
bit-exact against the oracle, including SURVEY §8(d)'s roofline trace R shape
(TP8 x DP32 x PP16, 80 layers, 512 micro-batches) with its fault phases."""

import numpy as np
import pytest

from tests.helpers import random_trace, with_measurements

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _check_detect(tr, oracle, keep_stage_cost=True):
    from paper_2605_06374_b200.detect_pass import DetectorPass

    p = DetectorPass(tr, keep_stage_cost=keep_stage_cost)
    p.detect()
    r = p.results()
    oms, ost, osc, ofl, osv = oracle.detect(tr)
    np.testing.assert_array_equal(r["status"], ost)
    np.testing.assert_array_equal(_bits(r["makespan"]), _bits(oms))
    if keep_stage_cost:
        np.testing.assert_array_equal(_bits(r["stage_cost"]), _bits(osc))
    np.testing.assert_array_equal(r["stage_flag"], ofl)
    np.testing.assert_array_equal(r["severity"].view(np.uint32), osv.view(np.uint32))
    return p, ost


@pytest.mark.parametrize("seed", range(24))
def test_wide_kernel_matches_oracle(seed, oracle, cuda_device):
    """P in {8, 16}: 1..64 replicas (partial warps, one replica per CTA),
    micro-batch counts below, at and above P (level-table, steady walks),
    slow / stopped stages (division, warp-mixed unit and non-unit), hops and
    all-reduce, both schedules."""
    rng = np.random.default_rng(3000 + seed)
    pp = [8, 16][seed % 2]
    dp = int(rng.choice([1, 2, 5, 16, 31, 32, 33, 64]))
    per = int(rng.choice([max(1, pp - 3), pp - 1, pp, pp + 1, 2 * pp + 3]))
    tr = with_measurements(
        random_trace(3100 + seed, n_iter=int(rng.integers(30, 120)), pp=pp, dp=dp,
                     M=per * dp + int(rng.integers(0, dp)), stop=seed % 7 == 3,
                     unit=seed % 5 == 0, schedule=["1f1b", "zbh"][(seed // 2) % 2]),
        oracle, noise=0.02, seed=seed)
    _check_detect(tr, oracle)


@pytest.mark.parametrize("schedule", ["1f1b", "zbh"])
@pytest.mark.parametrize("pp", [8, 16])
def test_wide_steady_boundaries_and_capacity(pp, schedule, oracle, cuda_device):
    from paper_2605_06374_b200.detect_pass import DetectorPass

    for m in sorted({1, pp - 1, pp, pp + 1, 2 * pp, 37}):
        dp = 3
        tr = with_measurements(random_trace(5200 + 10 * pp + m, n_iter=10, pp=pp, dp=dp,
                                            M=m * dp, schedule=schedule, n_seg=1),
                               oracle, noise=0.02, seed=m)
        p, _ = _check_detect(tr, oracle)
        for cap in (1, pp // 2, pp, pp + 2):
            ms, st, _ = p.pipeline("actual", capacity=cap)
            oms2, ost2, _ = oracle.pipeline(tr, view="actual", capacity=cap)
            np.testing.assert_array_equal(st.cpu().numpy(), ost2)
            np.testing.assert_array_equal(_bits(ms.cpu().numpy()), _bits(oms2))


@pytest.mark.parametrize("kernel", ["wide", "lane"])
def test_trace_r_shape_matches_oracle(kernel, oracle, cuda_device, monkeypatch):
    """SURVEY §8(d)'s roofline trace R shape -- 4096 GPUs, TP8 x DP32 x PP16,
    80 layers, 512 micro-batches, the C2 fault phases (fail-slow, link,
    fail-stop subgroup, proportional re-split) -- detect + screen vs the
    oracle, on the wide kernel (the bench path) and on the lane kernel
    (forced: D * next_pow2(P) = 512 lanes -> its 1024-thread instantiation)."""
    from paper_2605_06374_b200.detect_pass import DetectorPass
    from paper_2605_06374_b200.scenarios import c2_trace

    if kernel == "lane":
        monkeypatch.setenv("RH_FORCE_LANE_KERNEL", "1")
    else:
        monkeypatch.delenv("RH_FORCE_LANE_KERNEL", raising=False)
    tr = c2_trace(400, seed=0, tp=8, dp=32, pp=16, layers=80, M=512)
    ms, st, sc = oracle.pipeline(tr, view="actual")
    tr.attach_measurements(sc, ms, seed=0)
    p, ost = _check_detect(tr, oracle)
    p.screen()
    r = p.results()
    ooc, oln = oracle.screen(tr.observed, ost, reset=tr.reset)
    np.testing.assert_array_equal(r["outcome"], ooc)
    assert r["series_len"] == oln


def test_lane_kernel_1024_thread_instantiation(oracle, cuda_device):
    """The widest shapes: 64 replicas of a 16-stage pipeline on the wide kernel
    (one iteration per CTA), and a stage count without a wide instantiation
    (P = 9, pw = 16) on the lane kernel at 64 x 16 = 1024 lanes per iteration,
    its 1024-thread instantiation, both schedules."""
    tr = with_measurements(random_trace(6100, n_iter=40, pp=16, dp=64, M=64 * 17,
                                        schedule="1f1b"), oracle, noise=0.02, seed=2)
    _check_detect(tr, oracle)
    for k, sched in enumerate(["1f1b", "zbh"]):
        tr = with_measurements(random_trace(6101 + k, n_iter=30, pp=9, dp=64, M=64 * 10,
                                            schedule=sched), oracle, noise=0.02, seed=3)
        _check_detect(tr, oracle)


@pytest.mark.parametrize("pp", [8, 12, 16])
def test_wide_outputs_at_unaligned_addresses(pp, oracle, cuda_device):
    """The wide kernel stores a replica's contiguous outputs as vectors (4 flags
    per u32, float4 severities, double2 costs) only when the caller's pointers
    are aligned for them; outputs at odd offsets take the scalar stores and
    must be identical."""
    import torch

    from paper_2605_06374_b200.detect_pass import DetectorPass

    tr = with_measurements(random_trace(6100 + pp, n_iter=40, pp=pp, dp=7, M=7 * pp + 3),
                           oracle, noise=0.02, seed=pp)
    p = DetectorPass(tr, keep_stage_cost=True)
    n, G = tr.n_iter, tr.cfg.dp * tr.cfg.pp
    dev = p.stage_flag.device
    flag_buf = torch.zeros(n * G + 16, dtype=torch.uint8, device=dev)
    sev_buf = torch.zeros(n * G + 8, dtype=torch.float32, device=dev)
    cost_buf = torch.zeros(n * G + 4, dtype=torch.float64, device=dev)
    p.stage_flag, p.severity, p.stage_cost = flag_buf[1:1 + n * G], sev_buf[1:1 + n * G], \
        cost_buf[1:1 + n * G]
    p.detect()
    r = p.results()
    oms, ost, osc, ofl, osv = oracle.detect(tr)
    np.testing.assert_array_equal(r["status"], ost)
    np.testing.assert_array_equal(_bits(r["stage_cost"]), _bits(osc))
    np.testing.assert_array_equal(r["stage_flag"], ofl)
    np.testing.assert_array_equal(r["severity"].view(np.uint32), osv.view(np.uint32))
    assert int(flag_buf[0]) == 0 and int(flag_buf[1 + n * G]) == 0  # nothing outside
