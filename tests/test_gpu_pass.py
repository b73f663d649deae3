"""GPU parity: the fused predictor / Detector pass vs the CPU oracle.

Bit-exact comparisons (fp64 bit patterns, flags, status bits) on seeded
random traces covering 1F1B and ZBH, 1..6 stages, 1..4 replicas, uneven and
empty micro-batch ownership, slow and subgroup stages, hop and all-reduce
weights, stopped stages and the activation-capacity check.
"""

import numpy as np
import pytest

from tests.helpers import random_trace, with_measurements

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("seed", range(40))
def test_pipeline_matches_oracle(seed, oracle, cuda_device):
    from paper_2605_06374_b200.detect_pass import DetectorPass

    tr = random_trace(seed, stop=(seed % 7 == 3))
    p = DetectorPass(tr)
    for view in ("known", "actual"):
        ms, st, sc = p.pipeline(view)
        oms, ost, osc = oracle.pipeline(tr, view=view)
        np.testing.assert_array_equal(st.cpu().numpy(), ost)
        np.testing.assert_array_equal(_bits(ms.cpu().numpy()), _bits(oms))
        np.testing.assert_array_equal(_bits(sc.cpu().numpy()), _bits(osc))


@pytest.mark.parametrize("seed", range(12))
def test_pipeline_capacity_matches_oracle(seed, oracle, cuda_device):
    from paper_2605_06374_b200.detect_pass import DetectorPass

    tr = random_trace(100 + seed, pp=int(2 + seed % 5))
    p = DetectorPass(tr)
    for cap in (1, 2, 3, tr.cfg.pp + 2):
        ms, st, _ = p.pipeline("actual", capacity=cap)
        oms, ost, _ = oracle.pipeline(tr, view="actual", capacity=cap)
        np.testing.assert_array_equal(st.cpu().numpy(), ost)
        np.testing.assert_array_equal(_bits(ms.cpu().numpy()), _bits(oms))


@pytest.mark.parametrize("seed", range(24))
def test_detect_matches_oracle(seed, oracle, cuda_device):
    from paper_2605_06374_b200.detect_pass import DetectorPass

    tr = with_measurements(random_trace(200 + seed, n_iter=24), oracle, noise=0.02, seed=seed)
    p = DetectorPass(tr, keep_stage_cost=True)
    p.detect()
    r = p.results()
    oms, ost, osc, ofl, osv = oracle.detect(tr)
    np.testing.assert_array_equal(r["status"], ost)
    np.testing.assert_array_equal(_bits(r["makespan"]), _bits(oms))
    np.testing.assert_array_equal(_bits(r["stage_cost"]), _bits(osc))
    np.testing.assert_array_equal(r["stage_flag"], ofl)
    np.testing.assert_array_equal(r["severity"].view(np.uint32), osv.view(np.uint32))


@pytest.mark.parametrize("seed", range(40))
def test_screen_matches_oracle(seed, oracle, cuda_device):
    """rh_screen (Jacobi fixpoint) == the sequential state machine: windows
    1..64 (above 32 the lane-0 path), with and without resets, long pop runs
    (multi-chunk backward scans) and quantised series (ties in the sorts)."""
    from paper_2605_06374_b200.detector import _screen

    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000)) if seed % 4 else int(rng.integers(3000, 40000))
    base = 10.0 + rng.standard_normal(n) * rng.choice([0.05, 0.5, 2.0])
    if seed % 5 == 0:
        base = np.round(base, 1)
    spikes = rng.random(n) < rng.choice([0.02, 0.1, 0.3, 0.6])
    obs = np.where(spikes, base * rng.uniform(1.1, 3.0, n), base)
    st = np.zeros(n, np.uint8)
    st |= (rng.random(n) < rng.choice([0.05, 0.3])).astype(np.uint8)  # escalate
    st |= ((rng.random(n) < 0.2).astype(np.uint8) << 1)  # stage flag
    reset = None if seed % 3 == 0 else (rng.random(n) < 0.003).astype(np.uint8)
    w = int(rng.choice([1, 2, 3, 5, 20, 21, 32, 33, 64]))
    fe = bool(rng.integers(0, 2))
    L0 = int(rng.choice([0, 2, w, 50]))
    hist = list(10.0 + rng.standard_normal(min(L0, w)))
    oc, ln = _screen(L0, hist, obs, st, w, 3.0, fe, reset=reset)
    ooc, oln = oracle.screen(obs, st, window=w, kappa=3.0, filter_enabled=fe, series_len=L0,
                             hist=hist, reset=reset)
    np.testing.assert_array_equal(oc, ooc)
    assert ln == oln


@pytest.mark.parametrize("seed", range(3))
def test_detector_pass_host_chunked(seed, oracle, cuda_device):
    """rh_detector_pass_host (host buffers, chunked H2D/compute overlap) == oracle."""
    import ctypes as C

    from paper_2605_06374_b200 import _lib
    from paper_2605_06374_b200.tables import pipe_shape
    from paper_2605_06374_b200.workload import cost_model_c
    from tests.oracle_bind import HostSegments

    tr = with_measurements(random_trace(300 + seed, n_iter=3000 + 517 * seed, n_seg=3,
                                        pp=int(2 + seed * 3)), oracle, noise=0.02, seed=seed)
    tr.reset[::700] = 1
    segs = HostSegments(tr.known)
    n, G = tr.n_iter, tr.cfg.dp * tr.cfg.pp
    keep = [np.ascontiguousarray(a) for a in (tr.seg, tr.mb_off, tr.doc_len,
                                               tr.device_time.astype(np.float32), tr.observed,
                                               tr.reset)]
    seg, off, doc, dt, obs, rst = keep
    ms, st = np.zeros(n), np.zeros(n, np.uint8)
    fl, sv = np.zeros(n * G, np.uint8), np.zeros(n * G, np.float32)
    oc, ln = np.zeros(n, np.uint8), C.c_int64()
    trc = _lib.Trace(n, seg.ctypes.data, off.ctypes.data, doc.ctypes.data, dt.ctypes.data,
                     obs.ctypes.data)
    out = _lib.PassOut(ms.ctypes.data, st.ctypes.data, None, fl.ctypes.data, sv.ctypes.data)
    shape = pipe_shape(tr.cfg, tr.M, tr.N, has_allreduce=tr.has_allreduce, max_mb=segs.max_mb)
    sp = _lib.ScreenParams(20, 1, 3.0)
    lib = _lib.load_library()
    _lib.check(lib.rh_detector_pass_host(_lib.context(), C.byref(shape),
                                         C.byref(cost_model_c(tr.model)), C.byref(segs.c),
                                         C.byref(trc), 1.25, C.byref(sp), 0, None,
                                         rst.ctypes.data, C.byref(out), oc.ctypes.data,
                                         C.byref(ln), None), "rh_detector_pass_host")
    oms, ost, _, ofl, osv = oracle.detect(tr)
    ooc, oln = oracle.screen(tr.observed, ost, reset=tr.reset)
    np.testing.assert_array_equal(st, ost)
    np.testing.assert_array_equal(_bits(ms), _bits(oms))
    np.testing.assert_array_equal(fl, ofl.reshape(-1))
    np.testing.assert_array_equal(sv.view(np.uint32), osv.reshape(-1).view(np.uint32))
    np.testing.assert_array_equal(oc, ooc)
    assert ln.value == oln


@pytest.mark.parametrize("seed", range(3))
def test_screen_prepare_protocol(seed, oracle, cuda_device):
    """rh_screen_prepare on a side stream + rh_screen == the oracle; a prepare
    with different arguments is ignored (rh_screen recomputes); repeated
    prepare/screen pairs do not race on the shared results."""
    import torch

    from paper_2605_06374_b200 import _lib

    rng = np.random.default_rng(100 + seed)
    n = 5000 + 1000 * seed
    obs_h = 10.0 + rng.standard_normal(n) * 0.5
    obs_h = np.where(rng.random(n) < 0.1, obs_h * 2.0, obs_h)
    st_h = ((rng.random(n) < 0.3) | ((rng.random(n) < 0.2) << 1)).astype(np.uint8)
    rst_h = (rng.random(n) < 0.002).astype(np.uint8)
    dev = torch.device("cuda", 0)
    obs = torch.from_numpy(obs_h).to(dev)
    st = torch.from_numpy(st_h).to(dev)
    rst = torch.from_numpy(rst_h).to(dev)
    hist = torch.zeros(1, dtype=torch.float64, device=dev)
    lib, ctx = _lib.load_library(), _lib.context(0)
    side = torch.cuda.Stream(dev)
    main = torch.cuda.current_stream(dev)

    def run(w_prep, w_screen):
        oc = torch.empty(n, dtype=torch.uint8, device=dev)
        ln = torch.zeros(1, dtype=torch.int64, device=dev)
        ev = torch.cuda.Event()
        ev.record(main)
        side.wait_event(ev)
        _lib.check(lib.rh_screen_prepare(ctx, _lib.C.byref(_lib.ScreenParams(w_prep, 1, 3.0)), 0,
                                         hist.data_ptr(), n, obs.data_ptr(), rst.data_ptr(),
                                         _lib.stream_handle(side)), "prepare")
        _lib.check(lib.rh_screen(ctx, _lib.C.byref(_lib.ScreenParams(w_screen, 1, 3.0)), 0,
                                 hist.data_ptr(), n, obs.data_ptr(), st.data_ptr(),
                                 rst.data_ptr(), oc.data_ptr(), ln.data_ptr(),
                                 _lib.stream_handle(main)), "screen")
        return oc, ln

    for w_prep, w_screen in [(20, 20), (20, 20), (7, 20), (20, 5), (20, 20)]:
        outs = [run(w_prep, w_screen) for _ in range(3)]
        torch.cuda.synchronize()
        ooc, oln = oracle.screen(obs_h, st_h, window=w_screen, reset=rst_h)
        for oc, ln in outs:
            np.testing.assert_array_equal(oc.cpu().numpy(), ooc)
            assert int(ln.item()) == oln


@pytest.mark.parametrize("seed", range(3))
def test_detector_pass_host_packed(seed, oracle, cuda_device):
    """rh_detector_pass_host_packed (uint16 docs, uint8 counts, device-side CSR
    rebuild per chunk) == oracle, including chunk boundaries and empty
    micro-batches."""
    import ctypes as C

    from paper_2605_06374_b200 import _lib
    from paper_2605_06374_b200.tables import pipe_shape
    from paper_2605_06374_b200.workload import cost_model_c
    from tests.oracle_bind import HostSegments

    tr = with_measurements(random_trace(400 + seed, n_iter=2600 + 911 * seed, n_seg=3,
                                        pp=int(2 + seed * 2)), oracle, noise=0.02, seed=seed)
    tr.reset[::500] = 1
    pk = tr.packed()
    segs = HostSegments(tr.known)
    n, G = tr.n_iter, tr.cfg.dp * tr.cfg.pp
    keep = [np.ascontiguousarray(a) for a in (tr.seg, tr.device_time.astype(np.float32),
                                               tr.observed, tr.reset)]
    seg, dt, obs, rst = keep
    ms, st = np.zeros(n), np.zeros(n, np.uint8)
    fl, sv = np.zeros(n * G, np.uint8), np.zeros(n * G, np.float32)
    oc, ln = np.zeros(n, np.uint8), C.c_int64()
    trc = _lib.TracePacked(n, seg.ctypes.data, pk["iter_doc"].ctypes.data,
                           pk["mb_docs"].ctypes.data, pk["doc_len"].ctypes.data,
                           dt.ctypes.data, obs.ctypes.data)
    out = _lib.PassOut(ms.ctypes.data, st.ctypes.data, None, fl.ctypes.data, sv.ctypes.data)
    shape = pipe_shape(tr.cfg, tr.M, tr.N, has_allreduce=tr.has_allreduce, max_mb=segs.max_mb)
    sp = _lib.ScreenParams(20, 1, 3.0)
    lib = _lib.load_library()
    _lib.check(lib.rh_detector_pass_host_packed(
        _lib.context(), C.byref(shape), C.byref(cost_model_c(tr.model)), C.byref(segs.c),
        C.byref(trc), 1.25, C.byref(sp), 0, None, rst.ctypes.data, C.byref(out),
        oc.ctypes.data, C.byref(ln), None), "rh_detector_pass_host_packed")
    oms, ost, _, ofl, osv = oracle.detect(tr)
    ooc, oln = oracle.screen(tr.observed, ost, reset=tr.reset)
    np.testing.assert_array_equal(st, ost)
    np.testing.assert_array_equal(_bits(ms), _bits(oms))
    np.testing.assert_array_equal(fl, ofl.reshape(-1))
    np.testing.assert_array_equal(sv.view(np.uint32), osv.reshape(-1).view(np.uint32))
    np.testing.assert_array_equal(oc, ooc)
    assert ln.value == oln


def test_detector_pass_host_graph_replay(oracle, cuda_device):
    """Repeated host passes on the same buffers run direct, then capture a CUDA
    graph, then replay it: each call must see the CURRENT buffer contents."""
    import ctypes as C

    from paper_2605_06374_b200 import _lib
    from paper_2605_06374_b200.tables import pipe_shape
    from paper_2605_06374_b200.workload import cost_model_c
    from tests.oracle_bind import HostSegments

    tr = with_measurements(random_trace(777, n_iter=4100, n_seg=2, pp=3), oracle, noise=0.02,
                           seed=7)
    tr.reset[::900] = 1
    pk = tr.packed()
    segs = HostSegments(tr.known)
    n, G = tr.n_iter, tr.cfg.dp * tr.cfg.pp
    seg = np.ascontiguousarray(tr.seg)
    dt = np.ascontiguousarray(tr.device_time.astype(np.float32))
    obs = np.ascontiguousarray(tr.observed.copy())
    rst = np.ascontiguousarray(tr.reset)
    ms, st = np.zeros(n), np.zeros(n, np.uint8)
    fl, sv = np.zeros(n * G, np.uint8), np.zeros(n * G, np.float32)
    oc, ln = np.zeros(n, np.uint8), C.c_int64()
    trc = _lib.TracePacked(n, seg.ctypes.data, pk["iter_doc"].ctypes.data,
                           pk["mb_docs"].ctypes.data, pk["doc_len"].ctypes.data,
                           dt.ctypes.data, obs.ctypes.data)
    out = _lib.PassOut(ms.ctypes.data, st.ctypes.data, None, fl.ctypes.data, sv.ctypes.data)
    shape = pipe_shape(tr.cfg, tr.M, tr.N, has_allreduce=tr.has_allreduce, max_mb=segs.max_mb)
    sp = _lib.ScreenParams(20, 1, 3.0)
    lib, ctx = _lib.load_library(), _lib.context()
    model = cost_model_c(tr.model)
    base_obs, base_dt = obs.copy(), dt.copy()
    rng = np.random.default_rng(5)
    for call in range(4):
        # new measurements in place (same pointers): 1.0x, then perturbed
        scale = 1.0 if call == 0 else float(rng.uniform(0.8, 1.6))
        obs[:] = base_obs * scale
        dt[:] = base_dt * np.float32(scale)
        _lib.check(lib.rh_detector_pass_host_packed(
            ctx, C.byref(shape), C.byref(model), C.byref(segs.c), C.byref(trc), 1.25,
            C.byref(sp), 0, None, rst.ctypes.data, C.byref(out), oc.ctypes.data, C.byref(ln),
            None), "rh_detector_pass_host_packed")
        tr.observed, tr.device_time = obs.copy(), dt.copy().reshape(tr.device_time.shape)
        oms, ost, _, ofl, osv = oracle.detect(tr)
        ooc, oln = oracle.screen(obs, ost, reset=rst)
        np.testing.assert_array_equal(st, ost)
        np.testing.assert_array_equal(_bits(ms), _bits(oms))
        np.testing.assert_array_equal(fl, ofl.reshape(-1))
        np.testing.assert_array_equal(sv.view(np.uint32), osv.reshape(-1).view(np.uint32))
        np.testing.assert_array_equal(oc, ooc)
        assert ln.value == oln


def test_host_pass_graph_survives_workspace_growth(oracle, cuda_device):
    """replay the captured host pass after OTHER calls on the
    same context grew the shared scratch (a longer screen on the same stream,
    a large general DAG): the graph must not replay into retired buffers --
    the pass is re-captured and still equals the oracle."""
    import ctypes as C

    import torch

    from paper_2605_06374_b200 import _lib
    from paper_2605_06374_b200.detector import _screen
    from paper_2605_06374_b200.tables import pipe_shape
    from paper_2605_06374_b200.workload import cost_model_c
    from tests.oracle_bind import HostSegments

    tr = with_measurements(random_trace(4242, n_iter=3000, n_seg=2, pp=3), oracle, noise=0.02,
                           seed=3)
    tr.reset[::700] = 1
    pk = tr.packed()
    segs = HostSegments(tr.known)
    n, G = tr.n_iter, tr.cfg.dp * tr.cfg.pp
    seg = np.ascontiguousarray(tr.seg)
    dt = np.ascontiguousarray(tr.device_time.astype(np.float32))
    obs = np.ascontiguousarray(tr.observed)
    rst = np.ascontiguousarray(tr.reset)
    ms, st = np.zeros(n), np.zeros(n, np.uint8)
    fl, sv = np.zeros(n * G, np.uint8), np.zeros(n * G, np.float32)
    oc, ln = np.zeros(n, np.uint8), C.c_int64()
    trc = _lib.TracePacked(n, seg.ctypes.data, pk["iter_doc"].ctypes.data,
                           pk["mb_docs"].ctypes.data, pk["doc_len"].ctypes.data,
                           dt.ctypes.data, obs.ctypes.data)
    out = _lib.PassOut(ms.ctypes.data, st.ctypes.data, None, fl.ctypes.data, sv.ctypes.data)
    shape = pipe_shape(tr.cfg, tr.M, tr.N, has_allreduce=tr.has_allreduce, max_mb=segs.max_mb)
    sp = _lib.ScreenParams(20, 1, 3.0)
    lib, ctx = _lib.load_library(), _lib.context()
    model = cost_model_c(tr.model)
    oms, ost, _, ofl, osv = oracle.detect(tr)
    ooc, oln = oracle.screen(obs, ost, reset=rst)

    def host_pass():
        ms[:] = 0
        oc[:] = 0
        _lib.check(lib.rh_detector_pass_host_packed(
            ctx, C.byref(shape), C.byref(model), C.byref(segs.c), C.byref(trc), 1.25,
            C.byref(sp), 0, None, rst.ctypes.data, C.byref(out), oc.ctypes.data, C.byref(ln),
            None), "rh_detector_pass_host_packed")
        np.testing.assert_array_equal(st, ost)
        np.testing.assert_array_equal(_bits(ms), _bits(oms))
        np.testing.assert_array_equal(oc, ooc)
        assert ln.value == oln

    rng = np.random.default_rng(9)
    for grow in range(3):
        host_pass()
        host_pass()  # captured here (or replayed)
        # grow the legacy stream's screen scratch: a much longer series
        m = 60_000 * (grow + 2)
        big = 10.0 + rng.standard_normal(m)
        bst = np.zeros(m, np.uint8)
        with torch.cuda.stream(torch.cuda.default_stream()):
            oc_big, _ = _screen(0, [], big, bst, 20, 3.0, True, reset=None)
        ooc_big, _ = oracle.screen(big, bst)
        np.testing.assert_array_equal(oc_big, ooc_big)
        torch.cuda.synchronize()
        host_pass()  # must not replay into the retired buffers
    torch.cuda.synchronize()


def test_two_streams_concurrent_screens(oracle, cuda_device):
    """Per-stream scratch: rh_screen enqueued on two streams of one context
    back to back (no synchronisation between the calls, so the kernels may
    overlap) equals the oracle on both."""
    import ctypes as C

    import torch

    from paper_2605_06374_b200 import _lib

    lib, ctx = _lib.load_library(), _lib.context()
    rng = np.random.default_rng(11)
    dev = torch.device("cuda", torch.cuda.current_device())
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    params = _lib.ScreenParams(20, 1, 3.0)
    cases = []
    for k in range(2):
        n = 50_000 + 7_777 * k
        base = 10.0 + rng.standard_normal(n) * 0.5
        obs = np.where(rng.random(n) < 0.1, base * 2.0, base)
        stt = (rng.random(n) < 0.2).astype(np.uint8)
        cases.append(dict(obs=obs, st=stt, t_obs=torch.as_tensor(obs).to(dev),
                          t_st=torch.as_tensor(stt).to(dev), hist=torch.zeros(1, dtype=torch.float64, device=dev),
                          out=torch.empty(n, dtype=torch.uint8, device=dev),
                          ln=torch.empty(1, dtype=torch.int64, device=dev)))
    torch.cuda.synchronize()
    for rep in range(3):
        for c, s in zip(cases, streams):
            _lib.check(lib.rh_screen(ctx, C.byref(params), 0, c["hist"].data_ptr(), len(c["obs"]),
                                     c["t_obs"].data_ptr(), c["t_st"].data_ptr(), None,
                                     c["out"].data_ptr(), c["ln"].data_ptr(), s.cuda_stream),
                       "rh_screen")
        torch.cuda.synchronize()
        for c in cases:
            ooc, oln = oracle.screen(c["obs"], c["st"])
            np.testing.assert_array_equal(c["out"].cpu().numpy(), ooc)
            assert int(c["ln"].item()) == oln


def test_division_selftest(cuda_device):
    """The hot path's hoisted-reciprocal division equals __ddiv_rn bit for bit
    (2^28 seeded pairs over divisor regimes, on the device)."""
    import ctypes as C

    from paper_2605_06374_b200 import _lib

    bad = C.c_int64(-1)
    _lib.check(_lib.load_library().rh_selftest_division(_lib.context(), 1 << 28, 12345,
                                                        C.byref(bad)), "rh_selftest_division")
    assert bad.value == 0


@pytest.mark.parametrize("n_iter", [800, 2500])
def test_c2_scenario_matches_oracle(n_iter, oracle, cuda_device):
    """The headline configuration itself (bench.py's C2 trace: 256 GPUs,
    TP4 x DP16 x PP4, 128 micro-batches, fail-stop / fail-slow / link phases,
    resets) through DetectorPass -- detect + screen -- vs the oracle."""
    from paper_2605_06374_b200.detect_pass import DetectorPass
    from paper_2605_06374_b200.scenarios import c2_trace

    tr = c2_trace(n_iter, seed=3)
    ms, st, sc = oracle.pipeline(tr, view="actual")
    tr.attach_measurements(sc, ms, seed=3)
    p = DetectorPass(tr, keep_stage_cost=True)
    p.run()
    r = p.results()
    oms, ost, osc, ofl, osv = oracle.detect(tr)
    np.testing.assert_array_equal(r["status"], ost)
    np.testing.assert_array_equal(_bits(r["makespan"]), _bits(oms))
    np.testing.assert_array_equal(_bits(r["stage_cost"]), _bits(osc))
    np.testing.assert_array_equal(r["stage_flag"], ofl)
    np.testing.assert_array_equal(r["severity"].view(np.uint32), osv.view(np.uint32))
    ooc, oln = oracle.screen(tr.observed, ost, reset=tr.reset)
    np.testing.assert_array_equal(r["outcome"], ooc)
    assert r["series_len"] == oln


@pytest.mark.parametrize("seed", range(16))
def test_wide_replica_shapes_match_oracle(seed, oracle, cuda_device):
    """Shapes the small random traces do not reach: 8..128 replicas, up to 384
    micro-batches (micro-batch counts past the unrolled walks' 12), long
    documents (the unstaged-document fallback), slow stages (division)."""
    from paper_2605_06374_b200.detect_pass import DetectorPass

    rng = np.random.default_rng(500 + seed)
    dp = int(rng.choice([8, 16, 32, 64, 128]))
    pp = int(rng.integers(1, 5))
    M = int(rng.integers(dp, 3 * dp + 1)) if seed % 3 else int(rng.integers(dp, 384 + 1))
    mean = 4.0 if seed % 4 == 0 else 7.0  # short documents: many per micro-batch
    tr = with_measurements(random_trace(700 + seed, n_iter=int(rng.integers(40, 200)), dp=dp,
                                        pp=pp, M=M, mean=mean, sigma=1.0), oracle, noise=0.02,
                           seed=seed)
    p = DetectorPass(tr, keep_stage_cost=True)
    p.detect()
    r = p.results()
    oms, ost, osc, ofl, osv = oracle.detect(tr)
    np.testing.assert_array_equal(r["status"], ost)
    np.testing.assert_array_equal(_bits(r["makespan"]), _bits(oms))
    np.testing.assert_array_equal(_bits(r["stage_cost"]), _bits(osc))
    np.testing.assert_array_equal(r["stage_flag"], ofl)
    np.testing.assert_array_equal(r["severity"].view(np.uint32), osv.view(np.uint32))


@pytest.mark.parametrize("seed", range(8))
def test_extreme_cost_model_matches_oracle(seed, oracle, cuda_device):
    """Base costs far outside the hoisted-reciprocal range (tiny and huge cost
    models): the walks fall back to correctly rounded division, bit-exact."""
    from paper_2605_06374_b200.detect_pass import DetectorPass
    from paper_2605_06374_b200.workload import CostModel

    tr = random_trace(900 + seed, n_iter=20, pp=[2, 4, 6, 12][seed % 4])
    alpha, beta = ((1e-300, 1e-310), (1e270, 1e262))[seed % 2]
    tr.model = CostModel(alpha=alpha, beta=beta, chunk_ratios=tr.model.chunk_ratios)
    p = DetectorPass(tr)
    for view in ("known", "actual"):
        ms, st, sc = p.pipeline(view)
        oms, ost, osc = oracle.pipeline(tr, view=view)
        np.testing.assert_array_equal(st.cpu().numpy(), ost)
        np.testing.assert_array_equal(_bits(ms.cpu().numpy()), _bits(oms))
        np.testing.assert_array_equal(_bits(sc.cpu().numpy()), _bits(osc))


@pytest.mark.parametrize("schedule", ["1f1b", "zbh"])
@pytest.mark.parametrize("pp", [1, 2, 3, 4])
def test_steady_walk_boundaries_match_oracle(pp, schedule, oracle, cuda_device):
    """Replicas at and around the steady-state walk's boundary (m = P-1, P, P+1,
    2P, and long runs), 1F1B and ZBH: warm-up, steady loop, cool-down and the ZBH
    W tail reproduce the level-ordered walk bit for bit, with stage-cost sums and
    capacity checks."""
    from paper_2605_06374_b200.detect_pass import DetectorPass

    for m in sorted({max(1, pp - 1), pp, pp + 1, 2 * pp, 13, 37}):
        dp = 4
        tr = with_measurements(random_trace(1200 + 10 * pp + m, n_iter=12, pp=pp, dp=dp,
                                            M=m * dp, schedule=schedule, n_seg=1),
                               oracle, noise=0.02, seed=m)
        p = DetectorPass(tr, keep_stage_cost=True)
        p.detect()
        r = p.results()
        oms, ost, osc, ofl, osv = oracle.detect(tr)
        np.testing.assert_array_equal(r["status"], ost)
        np.testing.assert_array_equal(_bits(r["makespan"]), _bits(oms))
        np.testing.assert_array_equal(_bits(r["stage_cost"]), _bits(osc))
        np.testing.assert_array_equal(r["stage_flag"], ofl)
        for cap in (1, pp, pp + 2):
            ms, st, _ = p.pipeline("actual", capacity=cap)
            oms2, ost2, _ = oracle.pipeline(tr, view="actual", capacity=cap)
            np.testing.assert_array_equal(st.cpu().numpy(), ost2)
            np.testing.assert_array_equal(_bits(ms.cpu().numpy()), _bits(oms2))


@pytest.mark.parametrize("dp", [3, 16, 48, 64])
def test_cta_width_variants_match_oracle(dp, oracle, cuda_device, monkeypatch):
    """The thread-per-replica kernel runs 64-thread CTAs for dp <= 64 and
    128-thread CTAs otherwise (`RH_SMALL_WIDE=1` forces 128). Both widths must
    give the oracle's bits: dp = 48 leaves a 64-wide CTA partly empty (one
    iteration of 48 replicas), dp = 3 packs 21 iterations per CTA."""
    from paper_2605_06374_b200.detect_pass import DetectorPass

    tr = with_measurements(random_trace(900 + dp, n_iter=150, dp=dp, pp=4, schedule="1f1b",
                                        M=2 * dp + 1), oracle, noise=0.02, seed=dp)
    oms, ost, osc, ofl, osv = oracle.detect(tr)
    for wide in (False, True):
        if wide:
            monkeypatch.setenv("RH_SMALL_WIDE", "1")
        else:
            monkeypatch.delenv("RH_SMALL_WIDE", raising=False)
        p = DetectorPass(tr, keep_stage_cost=True)
        p.detect()
        r = p.results()
        np.testing.assert_array_equal(r["status"], ost)
        np.testing.assert_array_equal(_bits(r["makespan"]), _bits(oms))
        np.testing.assert_array_equal(_bits(r["stage_cost"]), _bits(osc))
        np.testing.assert_array_equal(r["stage_flag"], ofl)
        np.testing.assert_array_equal(r["severity"].view(np.uint32), osv.view(np.uint32))
