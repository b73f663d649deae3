"""Pin the CPU oracle (and the host-side table builders) to the reference.

Every fixture under tests/golden was produced by running the reference
implementation itself (tests/golden/make_golden.py).  These tests need no
GPU: the oracle is plain C, the tables are host Python, and the native FFD
packer is a host function of the CUDA library.
"""

import numpy as np
import pytest

from paper_2605_06374_b200 import _lib
from paper_2605_06374_b200.cluster import dp_counts_or_even
from paper_2605_06374_b200.pipeline import _busy_idle
from paper_2605_06374_b200.tables import segment_for_view, used_link_ratios
from paper_2605_06374_b200.trace import DetectorTrace, pack_ffd
from paper_2605_06374_b200.workload import CostModel, KIND_CODE, cost_model_c
from tests.golden_io import (bits, cfg_of, comm_of, keyed, load, mbs_of, model_of, state_of)


def test_quad_load_golden(oracle):
    for docs, q in load("workload")["quad_load"]:
        assert oracle.quad_load(docs) == q


def test_chunk_time_golden(oracle):
    for docs, budget, m, kind, layers, speed, t in load("workload")["chunk_time"]:
        mc = cost_model_c(model_of(m))
        got = oracle.chunk_time(mc, KIND_CODE[kind], oracle.quad_load(docs), budget, layers, speed)
        assert bits(got) == bits(t), (docs, kind, layers, speed)


def test_oracle_ffd_pack_golden(oracle):
    """The oracle's literal FFD (bench.py's reference arm packs with it) equals
    the reference's pack_sequences on every golden packing."""
    for docs, budget, bins in load("workload")["pack"]:
        off, flat = oracle.pack_sequences(np.asarray(docs, np.int32), budget)
        got = [list(map(int, flat[off[i]:off[i + 1]])) for i in range(len(off) - 1)]
        assert got == bins
    with pytest.raises(ValueError):
        oracle.pack_sequences(np.array([5000]), 4096)


def test_native_ffd_pack_golden():
    for docs, budget, bins in load("workload")["pack"]:
        off, flat = pack_ffd(np.asarray(docs, np.int32), budget)
        got = [flat[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)]
        assert got == bins


def test_native_ffd_bulk_runs_match_oracle(oracle):
    """The native FFD places runs of equal lengths in bulk (one tree descent per
    bin a run touches); the packing must equal the oracle's literal first-fit
    scan -- many duplicates, tiny and large budgets, truncation to max_bins --
    and the fused quad loads (rh_pack_sequences_quad) must equal sum l^2."""
    from paper_2605_06374_b200.replan_scenarios import pack_workload

    rng = np.random.default_rng(5)
    for t in range(120):
        n = int(rng.integers(1, 2500))
        budget = int(rng.integers(4, 6000))
        if t % 3 == 0:  # heavy duplication
            docs = rng.integers(1, min(budget, 9) + 1, n)
        else:
            docs = np.minimum(budget, np.maximum(1, rng.lognormal(np.log(budget / 4), 0.8, n)))
        docs = np.rint(docs).astype(np.int32)
        off, flat = pack_ffd(docs, budget)
        o2, f2 = oracle.pack_sequences(docs, budget)
        assert np.array_equal(off, o2) and np.array_equal(flat, f2), t
        nb = len(off) - 1
        m = max(1, nb // 2)
        poff, packed, quad = pack_workload(docs, budget, m)
        q = [int((flat[off[b]:off[b + 1]].astype(np.int64) ** 2).sum()) for b in range(m)]
        assert quad.tolist() == q and np.array_equal(poff, off[:m + 1]), t


def test_native_ffd_rejects_bad_lengths():
    with pytest.raises(ValueError):
        pack_ffd(np.array([5000]), 4096)
    with pytest.raises(ValueError):
        pack_ffd(np.array([0]), 4096)


def _trace_for_case(case):
    """Two-iteration trace (actual view, healthy view) of one simulate case."""
    state, cfg = state_of(case["state"]), cfg_of(case["cfg"])
    mbs, model, comm = mbs_of(case["mbs"]), model_of(case["model"]), comm_of(case["comm"])
    M, N = len(mbs), mbs[0].token_budget
    counts = dp_counts_or_even(M, cfg.dp, case["dp_counts"])
    a = segment_for_view(state, cfg, M, N, comm=comm, dp_counts=counts)
    h = segment_for_view(state, cfg, M, N, comm=comm, dp_counts=counts, healthy=True,
                         clean_links=True)
    from paper_2605_06374_b200.workload import csr_of

    off, docs = csr_of(mbs)
    tr = DetectorTrace(cfg=cfg, model=model, M=M, N=N, has_allreduce=comm is not None,
                       seg=np.array([0, 1], np.int32),
                       mb_off=np.concatenate([off, off[1:] + off[-1]]).astype(np.int32),
                       doc_len=np.concatenate([docs, docs]).astype(np.int32),
                       known=[a, h], actual=[a, h], reset=np.zeros(2, np.uint8))
    return tr, state, cfg, counts


def test_simulate_iteration_golden(oracle):
    n_ok = n_err = 0
    for case in load("pipeline")["simulate"]:
        tr, state, cfg, counts = _trace_for_case(case)
        ms, st, sc = oracle.pipeline(tr, capacity=case["capacity"])
        if "error" in case:
            n_err += 1
            if "completeness" in case["error"]:
                assert st[0] & _lib.RH_IT_STOPPED
            else:
                assert "capacity" in case["error"]
                assert st[0] & _lib.RH_IT_CAPACITY
            continue
        n_ok += 1
        res = case["result"]
        assert st[0] == 0
        assert bits(ms[0]) == bits(res["observed"])
        assert bits(ms[1]) == bits(res["predicted"])
        P = cfg.pp
        exp = keyed(res["stage_cost"])
        exp_ref = keyed(res["stage_cost_reference"])
        assert set(exp) == {(d, s) for d in range(cfg.dp) if counts[d] for s in range(P)}
        for (d, s), v in exp.items():
            assert bits(sc[0, d * P + s]) == bits(v)
            assert bits(sc[1, d * P + s]) == bits(exp_ref[(d, s)])
        busy, idle = _busy_idle(state, exp, res["observed"])
        assert [[k, v] for k, v in busy.items()] == res["busy"]
        assert [[k, v] for k, v in idle.items()] == res["idle"]
        assert keyed(res["link_ratio"]) == (used_link_ratios(state, cfg)
                                            if case["comm"] is not None else {})
    assert n_ok > 60 and n_err > 5


def test_critical_path_golden(oracle):
    for g in load("pipeline")["dags"]:
        e = np.asarray(g["edges"], dtype=np.float64).reshape(-1, 3)
        starts, ms, cyc = oracle.critical_path(g["cost"], e[:, 0].astype(np.int32),
                                               e[:, 1].astype(np.int32), e[:, 2])
        assert not cyc
        assert bits(ms) == bits(g["makespan"])
        np.testing.assert_array_equal(bits(starts), bits(g["starts"]))


def test_unit_1f1b_makespan_is_six(oracle):
    """test_pipeline.py:138-149: 2 stages x 2 micro-batches of unit chunks -> 6.0."""
    g = load("pipeline")["dags"][-1]
    assert g["makespan"] == 6.0


def test_change_point_golden(oracle):
    for series, w, kappa, idx in load("detector_units")["change_point"]:
        assert oracle.change_point(series, w, kappa) == (idx is not None)


def test_validate_golden(oracle):
    import ctypes as C

    for stages, links, confirmed, deg_s, deg_l in load("detector_units")["validate"]:
        stages = sorted(stages, key=lambda r: (r[0], r[1]))
        m = np.array([r[2] for r in stages] or [0.0])
        e = np.array([r[3] for r in stages] or [0.0])
        f = np.zeros(len(m), np.uint8)
        s = np.zeros(len(m))
        oracle.lib.orc_validate(len(stages), m.ctypes.data, e.ctypes.data, 1.25, f.ctypes.data,
                                s.ctypes.data)
        got = {(r[0], r[1]): s[i] for i, r in enumerate(stages) if f[i]}
        assert {k: bits(v) for k, v in got.items()} == {k: bits(v) for k, v in keyed(deg_s).items()}
        lr = np.array([r[2] for r in links] or [0.0])
        lf = np.zeros(len(lr), np.uint8)
        ls = np.zeros(len(lr))
        oracle.lib.orc_validate(len(links), lr.ctypes.data, None, 1.25, lf.ctypes.data,
                                ls.ctypes.data)
        gl = {(r[0], r[1]): ls[i] for i, r in enumerate(links) if lf[i]}
        assert gl == keyed(deg_l)
        assert confirmed == bool(got or gl)


def detector_trace_of(fx):
    """A DetectorTrace of a reference closed-loop detector run (one segment
    per iteration: the known view can change after each confirmation)."""
    from paper_2605_06374_b200.tables import Segment

    cfg, model = cfg_of(fx["cfg"]), model_of(fx["model"])
    its = fx["iterations"]
    n, D, P, T = len(its), cfg.dp, cfg.pp, cfg.tp
    M = len(its[0]["mbs"])
    known, offs, docs = [], [0], []
    dt = np.zeros((n, D, P, T), np.float32)
    for i, it in enumerate(its):
        state = state_of(it["known"])
        seg = segment_for_view(state, cfg, M, 4096, comm=__import__(
            "paper_2605_06374_b200.comm", fromlist=["CommSpec"]).CommSpec())
        seg.link_ratio = np.array([r[2] for r in it["link_ratio"]], np.float64)
        known.append(seg)
        for mb in it["mbs"]:
            docs.extend(mb)
            offs.append(len(docs))
        for d, s, v in it["noisy"]:
            dt[i, d, s, 0] = np.float32(v)
            dt[i, d, s, 1:] = np.float32(v) * np.float32(0.95)
    reset = np.zeros(n, np.uint8)
    for i, it in enumerate(its[:-1]):
        if it["reset_after"]:
            reset[i + 1] = 1
    tr = DetectorTrace(cfg=cfg, model=model, M=M, N=4096, has_allreduce=D > 1,
                       seg=np.arange(n, dtype=np.int32), mb_off=np.asarray(offs, np.int32),
                       doc_len=np.asarray(docs, np.int32), known=known, actual=known,
                       reset=reset, device_time=dt,
                       observed=np.array([it["observed"] for it in its]))
    return tr


def outcome_alarms(oc: int, degraded) -> list[str]:
    """The reference's alarm list for one outcome code (detector.py:217-271)."""
    out = []
    if oc & _lib.RH_SC_CANDIDATE:
        out.append("candidate")
    if oc & _lib.RH_SC_FILTERED and not oc & _lib.RH_SC_ESCALATED:
        if oc & _lib.RH_SC_POPPED:
            out.append("benign")
        return out
    if not oc & _lib.RH_SC_ESCALATED:
        return out
    out.append("escalate")
    if oc & _lib.RH_SC_CONFIRMED:
        targets = [f"d{d}s{s}" for d, s in sorted(degraded)]
        out.append("confirmed:" + "+".join(targets))
    else:
        out.append("unconfirmed")
    return out


@pytest.mark.parametrize("k", range(6))
def test_detector_trace_golden(oracle, k):
    fx = load("detector_traces")["traces"][k]
    tr = detector_trace_of(fx)
    ms, st, sc, fl, sv = oracle.detect(tr)
    its = fx["iterations"]
    P = tr.cfg.pp
    for i, it in enumerate(its):
        assert bits(ms[i]) == bits(it["predicted"])
        for d, s, v in it["expected"]:
            assert bits(sc[i, d * P + s]) == bits(v)
        if it["degraded"] is not None:
            got = {(g // P, g % P): float(sv[i, g]) for g in np.nonzero(fl[i])[0]}
            exp = keyed(it["degraded"])
            assert set(got) == set(exp)
            for key, v in exp.items():
                assert np.float32(v) == np.float32(got[key])
    oc, ln = oracle.screen(tr.observed, st, window=fx["window"], kappa=fx["kappa"],
                           filter_enabled=fx["filter_enabled"], reset=tr.reset)
    for i, it in enumerate(its):
        degraded = keyed(it["degraded"]) if it["degraded"] else {}
        links = [key for key in () ]
        alarms = outcome_alarms(int(oc[i]), degraded)
        # link targets are appended after stage targets by the reference
        if alarms and alarms[-1].startswith("confirmed:") and it["alarms"][-1] != alarms[-1]:
            assert it["alarms"][-1].startswith(alarms[-1])
            alarms[-1] = it["alarms"][-1]
        assert alarms == it["alarms"], (i, oc[i], it["alarms"])
    # final series length (reset after a confirmation happens outside observe)
    assert (0 if its[-1]["reset_after"] else ln) == its[-1]["series_len"]


def test_packed_trace_roundtrip():
    """DetectorTrace.packed(): the wire form decodes back to the int32 CSR."""
    from tests.helpers import random_trace

    for seed in range(4):
        tr = random_trace(900 + seed, n_iter=57)
        pk = tr.packed()
        n, M = tr.n_iter, tr.M
        assert pk["iter_doc"].dtype == np.int32 and pk["iter_doc"].shape == (n + 1,)
        assert pk["mb_docs"].dtype == np.uint8 and pk["mb_docs"].shape == (n * M,)
        assert pk["doc_len"].dtype == np.uint16
        off = np.concatenate([[0], np.cumsum(pk["mb_docs"].astype(np.int64))])
        np.testing.assert_array_equal(off, tr.mb_off)
        np.testing.assert_array_equal(pk["iter_doc"], tr.mb_off[::M])
        np.testing.assert_array_equal(pk["doc_len"].astype(np.int32), tr.doc_len)
    tr.doc_len[0] = 70000
    with pytest.raises(ValueError):
        tr.packed()
