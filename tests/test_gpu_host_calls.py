"""GPU parity of the per-call host entry points (rh_*_host: one staged copy
in, one copy out) against the CPU oracle, plus their argument checks."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2605_06374_b200 import _lib

    return _lib, _lib.load_library(), _lib.context()


def test_quad_load_host_matches_oracle(oracle, cuda_device):
    L, lib, ctx = _lib()
    rng = np.random.default_rng(1)
    for n_mb in (1, 7, 300):
        counts = rng.integers(0, 6, n_mb)
        off = np.zeros(n_mb + 1, np.int32)
        np.cumsum(counts, out=off[1:])
        docs = rng.integers(1, 40000, max(1, int(off[-1]))).astype(np.int32)
        out = np.zeros(n_mb, np.int64)
        assert lib.rh_quad_load_host(ctx, n_mb, off.ctypes.data, docs.ctypes.data,
                                     out.ctypes.data) == 0
        want = [oracle.quad_load(docs[off[j]:off[j + 1]]) for j in range(n_mb)]
        assert out.tolist() == want


def test_chunk_time_host_matches_oracle(oracle, cuda_device):
    from paper_2605_06374_b200.workload import CostModel, cost_model_c

    L, lib, ctx = _lib()
    rng = np.random.default_rng(2)
    n = 500
    m = cost_model_c(CostModel(2e-6, 5e-10, {"F": 1.0, "B": 2.0, "W": 1.5}))
    quad = rng.integers(0, 2**34, n).astype(np.int64)
    budget = rng.integers(1, 70000, n).astype(np.int32)
    kind = rng.integers(0, 4, n).astype(np.uint8)
    layers = rng.integers(1, 40, n).astype(np.int32)
    speed = rng.uniform(-0.2, 1.0, n)
    speed[::7] = 1.0
    t = np.zeros(n)
    bad = np.zeros(n, np.uint8)
    assert lib.rh_chunk_time_host(ctx, C.byref(m), n, quad.ctypes.data, budget.ctypes.data,
                                  kind.ctypes.data, layers.ctypes.data, speed.ctypes.data,
                                  t.ctypes.data, bad.ctypes.data) == 0
    for i in range(n):
        if speed[i] <= 0:
            assert bad[i] == 1 and t[i] == 0.0
        else:
            want = oracle.chunk_time(m, int(kind[i]), int(quad[i]), int(budget[i]),
                                     int(layers[i]), float(speed[i]))
            assert bad[i] == 0 and t[i].tobytes() == np.float64(want).tobytes(), i


def test_validate_host_rule(cuda_device):
    L, lib, ctx = _lib()
    rng = np.random.default_rng(3)
    n = 1000
    meas = rng.uniform(-0.1, 3.0, n)
    exp = rng.uniform(-0.1, 2.0, n)
    flag = np.zeros(n, np.uint8)
    sev = np.zeros(n)
    assert lib.rh_validate_host(ctx, n, meas.ctypes.data, exp.ctypes.data, 1.25,
                                flag.ctypes.data, sev.ctypes.data) == 0
    want = (exp > 0) & (meas > 0) & (meas > 1.25 * exp)
    assert np.array_equal(flag.astype(bool), want)
    np.testing.assert_array_equal(sev[want], exp[want] / meas[want])
    assert (sev[~want] == 0).all()


@pytest.mark.parametrize("seed", range(6))
def test_screen_host_matches_oracle(seed, oracle, cuda_device):
    L, lib, ctx = _lib()
    rng = np.random.default_rng(10 + seed)
    n = int(rng.integers(50, 3000))
    obs = 1.0 + 0.01 * rng.standard_normal(n)
    obs[rng.random(n) < 0.05] *= 1.6
    st = (rng.random(n) < 0.3).astype(np.uint8) * L.RH_IT_ESCALATE
    st |= (rng.random(n) < 0.1).astype(np.uint8) * L.RH_IT_STAGE_FLAG
    reset = (rng.random(n) < 0.01).astype(np.uint8)
    series_len = int(rng.integers(0, 40))
    hist = 1.0 + 0.01 * rng.standard_normal(max(1, min(series_len, 20)))
    params = L.ScreenParams(20, seed % 2, 3.0)
    oc = np.zeros(n, np.uint8)
    ln = np.zeros(1, np.int64)
    assert lib.rh_screen_host(ctx, C.byref(params), series_len, hist.ctypes.data, n,
                              obs.ctypes.data, st.ctypes.data, reset.ctypes.data, oc.ctypes.data,
                              ln.ctypes.data) == 0
    woc, wln = oracle.screen(obs, st, 20, 3.0, bool(seed % 2), series_len=series_len,
                             hist=hist[:min(series_len, 20)], reset=reset)
    assert np.array_equal(oc, woc) and int(ln[0]) == wln


def test_host_calls_reject_bad_arguments(cuda_device):
    L, lib, ctx = _lib()
    x = np.zeros(4)
    assert lib.rh_quad_load_host(ctx, 3, None, None, None) == L.RH_E_INVALID
    assert lib.rh_validate_host(ctx, 4, None, None, 1.25, None, None) == L.RH_E_INVALID
    assert lib.rh_chunk_time_host(ctx, None, 4, x.ctypes.data, None, None, None, None, None,
                                  None) == L.RH_E_INVALID
    params = L.ScreenParams(20, 1, 3.0)
    # a non-empty series without its history
    assert lib.rh_screen_host(ctx, C.byref(params), 5, None, 4, x.ctypes.data, None, None, None,
                              None) == L.RH_E_INVALID


@pytest.mark.parametrize("seed", range(4))
def test_observe_host_sequence_matches_oracle_screen(seed, oracle, cuda_device):
    """rh_observe_host called once per observation (the drop-in's
    DetectorState.observe) equals the oracle's batch screen of the whole
    sequence, with the validation flags folded into each status."""
    L, lib, ctx = _lib()
    rng = np.random.default_rng(40 + seed)
    n, w, fe = 400, 20, seed % 2
    obs = 1.0 + 0.01 * rng.standard_normal(n)
    obs[rng.random(n) < 0.06] *= 1.5
    esc = rng.random(n) < 0.3
    params = L.ScreenParams(w, fe, 3.0)
    series = []
    st_all = np.zeros(n, np.uint8)
    oc_all = np.zeros(n, np.uint8)
    for i in range(n):
        ns, nl = 6, 2
        meas = rng.uniform(0.5, 1.6, ns)
        exp = np.ones(ns)
        lr = rng.uniform(0.8, 1.3, nl)
        do_val = bool(esc[i] or not fe)
        sf, ss = np.zeros(ns, np.uint8), np.zeros(ns)
        lf, ls = np.zeros(nl, np.uint8), np.zeros(nl)
        h = min(len(series), w)
        hist = np.asarray(series[len(series) - h:] if h else [0.0], np.float64)
        oc, ln = np.zeros(1, np.uint8), np.zeros(1, np.int64)
        assert lib.rh_observe_host(ctx, C.byref(params), len(series), hist.ctypes.data,
                                   float(obs[i]), int(esc[i]), int(do_val), ns, meas.ctypes.data,
                                   exp.ctypes.data, nl, lr.ctypes.data, 1.25, sf.ctypes.data,
                                   ss.ctypes.data, lf.ctypes.data, ls.ctypes.data, oc.ctypes.data,
                                   ln.ctypes.data) == 0
        st = L.RH_IT_ESCALATE if esc[i] else 0
        if do_val:
            want_sf = (meas > 1.25 * exp)
            assert np.array_equal(sf.astype(bool), want_sf)
            assert np.array_equal(lf.astype(bool), lr > 1.25)
            if want_sf.any():
                st |= L.RH_IT_STAGE_FLAG
            if (lr > 1.25).any():
                st |= L.RH_IT_LINK_FLAG
        st_all[i], oc_all[i] = st, oc[0]
        series.append(float(obs[i]))
        if oc[0] & L.RH_SC_POPPED:
            series.pop()
        assert int(ln[0]) == len(series)
    woc, wln = oracle.screen(obs, st_all, w, 3.0, bool(fe))
    assert np.array_equal(oc_all, woc) and wln == len(series)
