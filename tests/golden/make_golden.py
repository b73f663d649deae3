"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (needs /root/reference, which does not
exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package (resilsim, from
/root/reference/pkg/src), evaluates it on seeded inputs and writes JSON
fixtures next to this script.  Floats are stored with repr() (exact
round-trip).  The fixtures are committed; tests read only the fixtures.
"""

from __future__ import annotations

import json
import os
import random
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("RESIHP_REFERENCE", "/root/reference/pkg/src"))
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF))
sys.path.insert(1, str(Path(__file__).resolve().parents[2]))  # this repo (oracle decode)

import resilsim  # noqa: E402
from resilsim import cluster as rc  # noqa: E402
from resilsim import detector as rd  # noqa: E402
from resilsim import pipeline as rp  # noqa: E402
from resilsim import policies as rpol  # noqa: E402
from resilsim import scheduler as rs  # noqa: E402
from resilsim import workload as rw  # noqa: E402
from resilsim.comm import CommSpec  # noqa: E402

OUT = Path(__file__).resolve().parent


def dump(name, obj):
    path = OUT / f"{name}.json"
    path.write_text(json.dumps(obj, separators=(",", ":")) + "\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


# ----------------------------------------------------------------- helpers
def state_to_json(state):
    return {
        "devices": [[d.id, d.node_id, d.speed, d.status] for d in state.devices],
        "devices_per_node": state.devices_per_node,
        "tp_groups": [[k[0], k[1], list(v)] for k, v in state.tp_groups.items()],
        "intra_bw": state.intra_bw,
        "inter_bw": state.inter_bw,
        "link_factors": [[k[0], k[1], v] for k, v in state.link_factors.items()],
    }


def cfg_to_json(cfg):
    return {"tp": cfg.tp, "dp": cfg.dp, "pp": cfg.pp, "schedule": cfg.schedule,
            "layer_partition": list(cfg.layer_partition)}


def model_to_json(m):
    return {"alpha": m.alpha, "beta": m.beta, "chunk_ratios": dict(m.chunk_ratios)}


def mbs_to_json(mbs):
    return [[mb.id, list(mb.doc_lengths), mb.token_budget] for mb in mbs]


def keyed(d):
    return [[k[0], k[1], v] for k, v in d.items()]


def random_scenario(rng: random.Random, *, allow_fail_stop=False):
    tp = rng.choice([1, 2, 4])
    dp = rng.choice([1, 2, 3, 4])
    pp = rng.choice([1, 2, 3, 4, 6])
    schedule = rng.choice(["1f1b", "zbh"])
    layers = [rng.randint(1, 5) for _ in range(pp)]
    cfg = rc.ParallelismConfig(tp=tp, dp=dp, pp=pp, schedule=schedule, layer_partition=layers)
    n_dev = tp * dp * pp
    dpn = 8
    nodes = max(1, -(-n_dev // dpn))
    state = rc.build_cluster(nodes, dpn, cfg, rng.choice([300e9, 300.0 * 2**30]),
                             rng.choice([25e9, 25.0 * 2**30]))
    events = []
    for _ in range(rng.randint(0, 3)):
        events.append(rc.FailureEvent(kind="fail_slow_compute", start=0.0,
                                      device=rng.randrange(n_dev),
                                      severity=rng.choice([0.5, 0.3, 0.75, 0.62])))
    if nodes > 1 and rng.random() < 0.4:
        a, b = rng.sample(range(nodes), 2)
        events.append(rc.FailureEvent(kind="fail_slow_comm", start=0.0, link=(a, b),
                                      severity=rng.choice([0.5, 0.4])))
    if allow_fail_stop and rng.random() < 0.3:
        events.append(rc.FailureEvent(kind="fail_stop", start=0.0, device=rng.randrange(n_dev)))
    if events:
        state = rc.apply_failures(state, events, 0.0)
    budget = rng.choice([1024, 2048, 4096])
    M = dp * rng.randint(1, 5)
    docs = [max(1, min(budget, int(rng.lognormvariate(6.8, 0.9)))) for _ in range(M * 6)]
    mbs = rw.pack_sequences(docs, budget)[:M]
    model = rw.CostModel(alpha=rng.uniform(1e-6, 4e-6), beta=rng.uniform(1e-10, 9e-10),
                         chunk_ratios={"F": 1.0, "B": rng.choice([1.0, 0.5]),
                                       "W": rng.choice([1.0, 0.75])})
    comm = CommSpec(p2p_optimized=rng.random() < 0.7) if rng.random() < 0.7 else None
    return state, cfg, mbs, model, comm


# ----------------------------------------------------------------- workload
def gen_workload():
    rng = random.Random(1)
    quad = [[[4096], 16777216], [[1024] * 4, 4194304], [[3000, 1000], 10000000]]
    for _ in range(200):
        docs = [rng.randint(1, 32768) for _ in range(rng.randint(1, 12))]
        quad.append([docs, rw.quad_load(rc.MicroBatch(0, tuple(docs), sum(docs)))])
    chunk = []
    for _ in range(400):
        docs = [rng.randint(1, 8192) for _ in range(rng.randint(1, 8))]
        budget = sum(docs) + rng.choice([0, 0, rng.randint(1, 4096)])
        if budget > sum(docs):
            docs.append(budget - sum(docs))
        mb = rc.MicroBatch(0, tuple(docs), budget)
        m = rw.CostModel(alpha=rng.choice([0.0, rng.uniform(1e-7, 5e-6)]),
                         beta=rng.uniform(1e-13, 1e-9),
                         chunk_ratios={"F": rng.choice([1.0, 0.7]), "B": rng.choice([1.0, 1.3]),
                                       "W": rng.choice([1.0, 0.4])})
        kind = rng.choice(["F", "B", "W", "BW"])
        layers = rng.randint(0, 12)
        speed = rng.choice([1.0, 0.5, 0.25, rng.uniform(0.05, 1.0)])
        chunk.append([docs, budget, model_to_json(m), kind, layers, speed,
                      rw.predict_chunk_time(mb, kind, m, layers, speed)])
    pack = []
    for _ in range(120):
        budget = rng.choice([512, 1024, 4096, 8192])
        docs = [rng.randint(1, budget) for _ in range(rng.randint(0, 60))]
        pack.append([docs, budget, [list(mb.doc_lengths) for mb in rw.pack_sequences(docs, budget)]])
    pack.append([[3000, 2000, 1000], 4096, [[3000, 1000, 96], [2000, 2096]]])
    dump("workload", {"quad_load": quad, "chunk_time": chunk, "pack": pack})


# ----------------------------------------------------------------- pipeline
def gen_pipeline():
    rng = random.Random(2)
    cases = []
    while len(cases) < 160:
        state, cfg, mbs, model, comm = random_scenario(rng, allow_fail_stop=True)
        counts = None
        if rng.random() < 0.4 and cfg.dp > 1:
            cuts = sorted(rng.randint(0, len(mbs)) for _ in range(cfg.dp - 1))
            counts = [b - a for a, b in zip([0] + cuts, cuts + [len(mbs)])]
        plan = rs.AdaptationPlan(dp_assignment=counts) if counts else None
        capacity = rng.choice([None, None, cfg.pp + 2, 2, 1])
        case = {"state": state_to_json(state), "cfg": cfg_to_json(cfg), "mbs": mbs_to_json(mbs),
                "model": model_to_json(model),
                "comm": None if comm is None else [comm.hidden_bytes_per_token, comm.layer_bytes,
                                                   comm.p2p_optimized],
                "dp_counts": counts, "capacity": capacity}
        try:
            rec = rp.simulate_iteration(state, cfg, mbs, model, plan, comm=comm,
                                        capacity=capacity)
            case["result"] = {
                "observed": rec.observed_time, "predicted": rec.predicted_healthy_time,
                "stage_cost": keyed(rec.stage_cost),
                "stage_cost_reference": keyed(rec.stage_cost_reference),
                "busy": [[k, v] for k, v in rec.per_device_busy.items()],
                "idle": [[k, v] for k, v in rec.per_device_idle.items()],
                "link_ratio": keyed(rec.link_ratio),
            }
        except rp.SimulationError as exc:
            case["error"] = str(exc)
        cases.append(case)
    # critical_path on the reference's DAGs, including migrated plans whose
    # stage orders come from plan_migration (general DAGs)
    dags = []
    while len(dags) < 60:
        state, cfg, mbs, model, comm = random_scenario(rng)
        speeds = rp._stage_speed_maps(state, cfg)[0]
        executors, orders = {}, None
        if cfg.dp > 1 and rng.random() < 0.6:
            res = rs.plan_migration(cfg, mbs, model, speeds, delta=rng.choice([0, 1]),
                                    capacity=cfg.pp + 2)
            executors = {(m.mb, m.stage): m.executor for m in res.migrations}
            orders = res.stage_orders if res.migrations else None
        dag = rp.build_dag(cfg, mbs, model, speeds, rng.choice([0.0, 1e-3]),
                           executors=executors, stage_orders=orders,
                           allreduce_seconds=rng.choice([None, 0.01]))
        starts, ms = rp.critical_path(dag)
        dags.append({"cost": [v.cost for v in dag.vertices],
                     "kind": [v.kind for v in dag.vertices],
                     "edges": [[e.src, e.dst, e.weight] for e in dag.edges],
                     "starts": starts, "makespan": ms, "migrated": bool(executors)})
    # unit-cost KATs from the reference tests (test_pipeline.py:125-149)
    unit = rw.CostModel(alpha=1.0, beta=0.0, chunk_ratios={"F": 1.0, "B": 0.5, "W": 0.5})
    ub = [rc.MicroBatch(i, (1,), 1) for i in range(2)]
    d = rp.build_dag(rc.ParallelismConfig(1, 1, 2, layer_partition=[1, 1]), ub, unit, 1.0)
    s, m = rp.critical_path(d)
    dags.append({"cost": [v.cost for v in d.vertices], "kind": [v.kind for v in d.vertices],
                 "edges": [[e.src, e.dst, e.weight] for e in d.edges], "starts": s,
                 "makespan": m, "migrated": False})
    dump("pipeline", {"simulate": cases, "dags": dags})


# ----------------------------------------------------------------- detector
def gen_detector():
    rng = random.Random(3)
    cp = []
    for _ in range(300):
        w = rng.choice([3, 5, 20])
        n = rng.randint(w - 1, w + 5)
        scale = rng.choice([0.0, 0.01, 0.3])
        series = [10.0 + rng.choice([0.0, scale * rng.gauss(0, 1)]) for _ in range(n)]
        if rng.random() < 0.5:
            series.append(10.0 * rng.choice([1.05, 1.3, 2.0]))
        cp.append([series, w, 3.0, rd.detect_change_point(series, w, 3.0)])
    val = []
    for _ in range(200):
        st = {}
        for d in range(rng.randint(1, 3)):
            for s in range(rng.randint(1, 3)):
                e = rng.choice([0.0, rng.uniform(0.1, 1.0)])
                st[(d, s)] = (e * rng.choice([1.0, 1.2, 1.25, 1.3, 2.0, 0.0]), e)
        lr = {(a, a + 1): rng.choice([1.0, 1.25, 1.26, 2.5]) for a in range(rng.randint(0, 2))}
        r = rd.validate(st, lr, threshold=1.25)
        val.append([[[k[0], k[1], v[0], v[1]] for k, v in st.items()],
                    [[k[0], k[1], v] for k, v in lr.items()], r.confirmed,
                    keyed(r.degraded_stages), keyed(r.degraded_links)])
    dump("detector_units", {"change_point": cp, "validate": val})

    # closed-loop detector traces: the reference's own observe() on records
    # from the reference simulator, noisy stage costs rounded to float32 so a
    # float32 device trace reproduces them exactly
    traces = []
    for seed in range(6):
        traces.append(detector_trace(seed))
    dump("detector_traces", {"traces": traces})


def detector_trace(seed: int):
    rng = np.random.default_rng([seed, 7])
    tp, dp, pp = [(4, 2, 2), (2, 4, 2), (4, 2, 4), (2, 2, 3), (1, 4, 2), (4, 4, 2)][seed]
    schedule = "zbh" if seed % 3 == 2 else "1f1b"
    cfg = rc.ParallelismConfig(tp=tp, dp=dp, pp=pp, schedule=schedule,
                               layer_partition=[4] * pp)
    nodes = max(1, -(-tp * dp * pp // 8))
    state0 = rc.build_cluster(nodes, 8, cfg, 300.0 * 2**30, 25.0 * 2**30)
    model = rw.CostModel(alpha=2e-6, beta=5e-10)
    comm = CommSpec()
    n_iter = 90
    slow_dev = int(rng.integers(tp * dp * pp))
    events = [rc.FailureEvent(kind="fail_slow_compute", start=0.0, device=slow_dev,
                              severity=float(rng.choice([0.4, 0.5, 0.6])))]
    if nodes > 1:
        events.append(rc.FailureEvent(kind="fail_slow_comm", start=0.0, link=(0, 1),
                                      severity=0.5))
    onset = [40, 70]
    det = rd.DetectorState(window=int(rng.choice([10, 20])), filter_enabled=seed % 4 != 3)
    known_speeds: dict[int, float] = {}
    known_links: dict = {}
    docs = np.random.default_rng([seed, 0])
    M = dp * 4
    iters = []
    for k in range(n_iter):
        act = [e for i, e in enumerate(events) if k >= onset[min(i, 1)]]
        state = rc.apply_failures(state0, act, 0.0) if act else state0.copy()
        lengths = [int(max(1, min(4096, round(docs.lognormal(7.2, 0.8))))) for _ in range(M * 4)]
        mbs = rw.pack_sequences(lengths, 4096)[:M]
        rec = rp.simulate_iteration(state, cfg, mbs, model, comm=comm)
        known = state.copy()
        for dev in known.devices:
            if dev.status != rc.FAIL_STOP:
                dev.speed = min(1.0, known_speeds.get(dev.id, 1.0))
        known.link_factors = dict(known_links)
        ref = rp.simulate_iteration(known, cfg, mbs, model, comm=comm)
        noisy = {key: float(np.float32(v * (1.0 + 0.01 * float(rng.standard_normal()))))
                 for key, v in sorted(rec.stage_cost.items())}
        import dataclasses

        rec2 = dataclasses.replace(rec, stage_cost=noisy)
        out = det.observe(rec2, ref.observed_time, reference_stage_cost=ref.stage_cost)
        reset = False
        if out.validation is not None and out.validation.confirmed:
            for key in sorted(out.validation.degraded_stages):
                for dev_id in state.tp_groups.get(key, ()):
                    known_speeds[dev_id] = state.devices[dev_id].speed
            for link in out.validation.degraded_links:
                known_links[link] = state.link_factors.get(link, 1.0)
            det.reset_series()
            reset = True
        iters.append({
            "mbs": [list(mb.doc_lengths) for mb in mbs],
            "known": state_to_json(known),
            "observed": rec.observed_time,
            "noisy": keyed(noisy),
            "link_ratio": keyed(rec.link_ratio),
            "predicted": ref.observed_time,
            "expected": keyed(ref.stage_cost),
            "alarms": out.alarms,
            "verdict": out.verdict,
            "confirmed": None if out.validation is None else out.validation.confirmed,
            "degraded": None if out.validation is None else keyed(out.validation.degraded_stages),
            "reset_after": reset,
            "series_len": len(det.series),
        })
    return {"cfg": cfg_to_json(cfg), "model": model_to_json(model), "window": det.window,
            "kappa": det.kappa, "filter_enabled": det.filter_enabled, "iterations": iters,
            "stats": vars(det.stats)}


# ----------------------------------------------------------------- scheduler
def gen_scheduler():
    rng = random.Random(4)
    degrees = []
    for _ in range(100):
        g = rng.randint(1, 12)
        f = rng.randint(0, g)
        k = rng.choice([1, 2, 4])
        degrees.append([g, f, k, sorted(rs.candidate_tp_degrees(g, f, k))])
    subgroup = []
    for _ in range(400):
        n = rng.randint(1, 10)
        speeds = {i: rng.choice([1.0, 0.5, rng.uniform(0.01, 1.0)]) for i in range(n)}
        degs = rs.candidate_tp_degrees(n, 0, rng.choice([1, 2]))
        try:
            chosen, standby = rs.select_tp_subgroup(speeds, degs)
            subgroup.append([list(speeds.values()), sorted(degs), list(chosen), list(standby)])
        except rs.GroupUnrecoverable:
            subgroup.append([list(speeds.values()), sorted(degs), None, None])
    repart = [[[1.0, 0.5, 1.0], 12, 1, [5, 2, 5]]]
    for _ in range(400):
        P = rng.randint(1, 16)
        speeds = [rng.choice([1.0, 1.0, 0.5, rng.uniform(0.05, 1.0)]) for _ in range(P)]
        L = P * rng.randint(1, 6) + rng.randint(0, P)
        ml = rng.choice([1, 1, 2])
        try:
            repart.append([speeds, L, ml, rs.repartition_layers(speeds, L, ml)])
        except ValueError:
            repart.append([speeds, L, ml, None])
    prop = []
    for _ in range(300):
        D = rng.randint(1, 12)
        w = [rng.choice([1.0, 0.5, 0.0, rng.uniform(0.0, 1.0)]) for _ in range(D)]
        total = rng.randint(0, 200)
        try:
            prop.append([total, w, rpol.proportional_split(total, w)])
        except ValueError:
            prop.append([total, w, None])
    dump("scheduler_units", {"tp_degrees": degrees, "subgroup": subgroup,
                             "repartition": repart, "proportional": prop})


# ----------------------------------------------------------------- search
def search_cases():
    """Small re-plan problems: (name, nodes, dpn, cfg, events, M, N, comm, capacity, sched)."""
    return [
        ("slow32", 4, 8, (4, 4, 2), [("fail_slow_compute", 5, 0.5)], 16, 4096, True, 8, "1f1b"),
        ("stop32", 4, 8, (4, 4, 2), [("fail_stop", 3, None), ("fail_slow_compute", 17, 0.6)],
         16, 4096, True, 8, "1f1b"),
        ("link32", 4, 8, (2, 4, 4), [("fail_slow_comm", (1, 2), 0.4)], 16, 2048, True, 6, "zbh"),
        ("nocomm16", 2, 8, (2, 2, 4), [("fail_slow_compute", 9, 0.3)], 12, 4096, False, 0,
         "1f1b"),
    ]


def gen_search():
    """Reference evaluate_plan + reconfig_cost on candidates of the re-plan space.

    The candidate space is this repo's definition; the
    oracle decodes candidate indices (placement, partition, counts) and the
    REFERENCE scores them, which pins the oracle's and the GPU's scores."""
    from paper_2605_06374_b200 import cluster as mc
    from paper_2605_06374_b200.search import build_desc
    from tests.oracle_bind import Oracle

    oracle = Oracle()
    out = []
    for name, nodes, dpn, (T, D, P), evs, M, N, has_comm, cap, sched in search_cases():
        rng = random.Random(sum(map(ord, name)))
        L = 8 * P
        cfg_r = rc.ParallelismConfig(tp=T, dp=D, pp=P, schedule=sched, layer_partition=[8] * P)
        st_r = rc.build_cluster(nodes, dpn, cfg_r, 300.0 * 2**30, 25.0 * 2**30)
        events = []
        for kind, target, sev in evs:
            if kind == "fail_slow_comm":
                events.append(rc.FailureEvent(kind=kind, start=0.0, link=target, severity=sev))
            else:
                events.append(rc.FailureEvent(kind=kind, start=0.0, device=target, severity=sev))
        st_r = rc.apply_failures(st_r, events, 0.0)
        docs = [max(1, min(N, int(rng.lognormvariate(7.2, 0.8)))) for _ in range(M * 8)]
        mbs_r = rw.pack_sequences(docs, N)[:M]
        model_r = rw.CostModel(alpha=2e-6, beta=5e-10)
        comm_r = CommSpec() if has_comm else None
        # the same problem in this package's types for the descriptor
        st_m = mc.ClusterState(
            devices=[mc.Device(d.id, d.node_id, d.speed, d.status) for d in st_r.devices],
            devices_per_node=dpn, tp_groups=dict(st_r.tp_groups), intra_bw=st_r.intra_bw,
            inter_bw=st_r.inter_bw, link_factors=dict(st_r.link_factors))
        cfg_m = mc.ParallelismConfig(T, D, P, sched, [8] * P)
        from paper_2605_06374_b200.comm import CommSpec as MCS

        quad = [rw.quad_load(mb) for mb in mbs_r]
        inp = build_desc(st_m, cfg_m, mbs_r, model_r, MCS() if has_comm else None,
                         capacity=cap or None, quad=quad, min_utilization=0.6)
        srch = oracle.search(inp)
        best, bi = srch.best()
        picks = sorted({0, bi, srch.size - 1} | {rng.randrange(srch.size) for _ in range(90)})
        rows = []
        for idx in picks:
            c = srch.decode(idx)
            if not c.feasible:  # a move out of an empty replica / below min_layers
                rows.append([idx, None, "infeasible variant"])
                continue
            st2 = st_r.copy()
            st2.tp_groups = {(g // c.pp, g % c.pp): tuple(m) for g, m in enumerate(c.groups)}
            members = {m for g in c.groups for m in g}
            for dev in st2.devices:
                if dev.status == rc.FAIL_STOP:
                    continue
                dev.status = ((rc.FAIL_SLOW if dev.speed < 1.0 else rc.HEALTHY)
                              if dev.id in members else rc.STANDBY)
            cfg2 = rc.ParallelismConfig(tp=T, dp=c.dp, pp=c.pp, schedule=sched,
                                        layer_partition=list(c.partition))
            plan = rs.AdaptationPlan(dp_assignment=list(c.counts))
            try:
                ms = rs.evaluate_plan(plan, st2, cfg2, mbs_r, model_r, comm=comm_r,
                                      capacity=cap or None)
            except rp.SimulationError as exc:
                rows.append([idx, None, str(exc)[:40]])
                continue
            same = (c.tp == T and c.dp == D and c.pp == P and
                    all(tuple(sorted(st_r.tp_groups[(g // P, g % P)])) == tuple(m)
                        for g, m in enumerate(c.groups)))
            if same:  # the reference's own reconfig_cost
                rplan = rs.AdaptationPlan(layer_partition=list(c.partition))
                reconf = rs.reconfig_cost(rplan, st_r, cfg_r, layer_bytes=256.0 * 2**20)
            else:      # DESIGN.md §5 extension: full reshard over the worst link
                moved = (sum(max(0, a - b) for a, b in zip(c.partition, cfg_r.layer_partition))
                         if c.pp == P else 0)
                reshard = 0.0
                for _d in range(c.dp):
                    for q in range(c.pp):
                        reshard += c.partition[q] * (256.0 * 2**20)
                worst = rc.ClusterState.copy(st_r).inter_bw * min(
                    st_r.link_factors.values(), default=1.0)
                reconf = 2.0 + (moved * (256.0 * 2**20) + reshard) / worst
            rows.append([idx, ms, reconf / max(1, 25)])
        out.append({"name": name, "nodes": nodes, "dpn": dpn, "cfg": [T, D, P], "sched": sched,
                    "events": [[k, list(t) if isinstance(t, tuple) else t, s] for k, t, s in evs],
                    "mbs": [list(mb.doc_lengths) for mb in mbs_r], "N": N, "comm": has_comm,
                    "capacity": cap, "size": srch.size, "best": [best, bi], "rows": rows})
        print(name, "size", srch.size, "best", best, bi)
    dump("search", {"cases": out})


# ------------------------------------------------ benchmarked search spaces
_SB = {}  # (reference problem, oracle) of the space being scored (fork-shared)


def _ref_state_of(st_m):
    """This package's ClusterState -> the reference's (same fields)."""
    return rc.ClusterState(
        devices=[rc.Device(d.id, d.node_id, d.speed, d.status) for d in st_m.devices],
        devices_per_node=st_m.devices_per_node, tp_groups=dict(st_m.tp_groups),
        intra_bw=st_m.intra_bw, inter_bw=st_m.inter_bw, link_factors=dict(st_m.link_factors))


def _ref_score(idx):
    """The reference's evaluate_plan + reconfig_cost of candidate idx (decoded
    by the oracle: placement groups, partition, counts) -> [idx, ms, extra]."""
    st_r, cfg_r, mbs_r, model_r, comm_r, cap, srch = _SB["problem"]
    c = srch.decode(idx)
    if not c.feasible:
        return [idx, None, "infeasible variant"]
    st2 = st_r.copy()
    st2.tp_groups = {(g // c.pp, g % c.pp): tuple(m) for g, m in enumerate(c.groups)}
    members = {m for g in c.groups for m in g}
    for dev in st2.devices:
        if dev.status == rc.FAIL_STOP:
            continue
        dev.status = ((rc.FAIL_SLOW if dev.speed < 1.0 else rc.HEALTHY)
                      if dev.id in members else rc.STANDBY)
    # the config keeps the NOMINAL TP degree: a c.tp-wide group runs at
    # slowest * c.tp / nominal (effective_stage_speed, cluster.py:155-169)
    cfg2 = rc.ParallelismConfig(tp=cfg_r.tp, dp=c.dp, pp=c.pp, schedule=cfg_r.schedule,
                                layer_partition=list(c.partition))
    plan = rs.AdaptationPlan(dp_assignment=list(c.counts))
    try:
        ms = rs.evaluate_plan(plan, st2, cfg2, mbs_r, model_r, comm=comm_r, capacity=cap)
    except rp.SimulationError as exc:
        return [idx, None, str(exc)[:40]]
    T, D, P = cfg_r.tp, cfg_r.dp, cfg_r.pp
    same = (c.tp == T and c.dp == D and c.pp == P and
            all(tuple(sorted(st_r.tp_groups[(g // P, g % P)])) == tuple(m)
                for g, m in enumerate(c.groups)))
    if same:  # the reference's own reconfig_cost
        rplan = rs.AdaptationPlan(layer_partition=list(c.partition))
        reconf = rs.reconfig_cost(rplan, st_r, cfg_r, layer_bytes=256.0 * 2**20)
    else:      # DESIGN.md §5 extension: full reshard over the worst link
        moved = (sum(max(0, a - b) for a, b in zip(c.partition, cfg_r.layer_partition))
                 if c.pp == P else 0)
        reshard = 0.0
        for _d in range(c.dp):
            for q in range(c.pp):
                reshard += c.partition[q] * (256.0 * 2**20)
        worst = st_r.inter_bw * min(st_r.link_factors.values(), default=1.0)
        reconf = 2.0 + (moved * (256.0 * 2**20) + reshard) / worst
    return [idx, ms, reconf / max(1, 25)]


def gen_search_bench(per_config=1200):
    """Reference-scored candidates of the BENCHMARKED re-plan spaces (bench.py's
    C3 / C4 / C5, replan_scenarios.py): per config >= 10^3 indices -- every
    layout's first and last candidate, the oracle's full-space winner and its
    neighbourhood, stratified random picks per layout (proportional to its
    size, at least 4 each) and uniform random picks -- each scored by the
    reference's evaluate_plan + reconfig_cost on the decoded plan, in parallel
    over the host cores (one process per candidate batch)."""
    import multiprocessing as mp

    from paper_2605_06374_b200.comm import CommSpec as MCS  # noqa: F401
    from paper_2605_06374_b200.replan_scenarios import replan_problem
    from tests.oracle_bind import Oracle

    oracle = Oracle()
    out = {}
    for name in ("C3", "C4", "C5"):
        st_m, cfg_m, mbs_m, inputs = replan_problem(name)
        srch = oracle.search(inputs)
        best, bi = srch.best_memo()
        rng = random.Random(sum(map(ord, name)) * 7)
        picks = {0, srch.size - 1, bi}
        picks |= {min(srch.size - 1, max(0, bi + k)) for k in range(-24, 25)}
        d = inputs.desc
        # layouts: bases from decode of increasing indices (the oracle's order)
        lay = {}
        i = 0
        while i < srch.size:  # walk the layouts: (layout, partition, count) blocks
            c = srch.decode(i)
            lay.setdefault(len(lay), [i, i])
            # jump to the next layout: its size is nv * nu
            nv = 2 + c.pp * (c.pp - 1)
            nu = 2 + c.dp * (c.dp - 1)
            j = i - (c.partition_variant * nu + c.count_variant) + nv * nu
            lay[len(lay) - 1][1] = j - 1
            i = j
        for li, (a, b) in lay.items():
            picks |= {a, b}
            k = max(4, int(per_config * 0.6 * (b - a + 1) / srch.size))
            picks |= {rng.randint(a, b) for _ in range(k)}
        while len(picks) < per_config:
            picks.add(rng.randrange(srch.size))
        picks = sorted(picks)
        st_r = _ref_state_of(st_m)
        cfg_r = rc.ParallelismConfig(tp=cfg_m.tp, dp=cfg_m.dp, pp=cfg_m.pp, schedule=cfg_m.schedule,
                                     layer_partition=list(cfg_m.layer_partition))
        mbs_r = [rw.MicroBatch(id=mb.id, doc_lengths=tuple(mb.doc_lengths),
                               token_budget=mb.token_budget) for mb in mbs_m]
        model_r = rw.CostModel(alpha=2e-6, beta=5e-10)
        _SB["problem"] = (st_r, cfg_r, mbs_r, model_r, CommSpec(), cfg_m.pp + 2, srch)
        with mp.get_context("fork").Pool(os.cpu_count() or 1) as pool:
            rows = pool.map(_ref_score, picks, chunksize=4)
        n_ok = sum(r[1] is not None for r in rows)
        out[name] = {"size": srch.size, "devices": d.n_devices, "layouts": len(lay),
                     "oracle_best": [best, bi], "rows": rows}
        print(name, "size", srch.size, "layouts", len(lay), "scored", len(rows), "finite", n_ok,
              "best", best, bi, flush=True)
    dump("search_bench", out)


# --------------------------------------------------- batched closed loop
def closed_loop_mappings():
    """Acceptance criterion 4's fail-slow scenarios (test_acceptance.py:193-223:
    16 GPUs TP4 x DP2 x PP2, 24 micro-batches of lognormal(7.0, 0.25), one
    fail-slow of random device / severity near iteration 25, resihp, 34
    iterations; the same random.Random(99) draws), the first 16 trials, plus
    mixed scenarios: a fail-stop with heartbeats, a slow link, two staggered
    fail-slows on a wider pipeline."""
    from resilsim.harness import run_scenario, scenario_from_mapping

    def det(seed, iterations, policy, failures=()):
        return {"name": "detect", "seed": seed, "iterations": iterations, "policy": policy,
                "cluster": {"nodes": 2, "devices_per_node": 8},
                "parallelism": {"tp": 4, "dp": 2, "pp": 2, "layers": 8},
                "workload": {"token_budget": 4096, "micro_batches": 24,
                             "doc_lengths": {"kind": "lognormal", "mean": 7.0,
                                             "sigma": 0.25}},
                "failures": list(failures)}

    probe = det(0, 12, "none")
    h = run_scenario(scenario_from_mapping(probe)).summary["avg_iteration_s"]
    rng = random.Random(99)
    out = []
    for i in range(16):
        severity = rng.uniform(0.3, 0.7)
        device = rng.randrange(16)
        out.append(det(1000 + i, 34, "resihp", [{"kind": "fail_slow_compute", "device": device,
                                                 "start": h * 25.4, "severity": severity}]))
    out.append(det(3001, 30, "resihp", [{"kind": "fail_stop", "device": 6, "start": h * 9.5}]))
    out.append(det(3002, 30, "resihp", [{"kind": "fail_slow_comm", "link": [0, 1],
                                         "start": h * 12.2, "severity": 0.4}]))
    wide = det(3003, 40, "resihp", [
        {"kind": "fail_slow_compute", "device": 3, "start": h * 8.3, "severity": 0.5},
        {"kind": "fail_slow_compute", "device": 27, "start": h * 21.7, "severity": 0.6}])
    wide["cluster"] = {"nodes": 4, "devices_per_node": 8}
    wide["parallelism"] = {"tp": 4, "dp": 2, "pp": 4, "layers": 16}
    out.append(wide)
    out.append(det(3004, 20, "none", [{"kind": "fail_slow_compute", "device": 9,
                                       "start": h * 5.0, "severity": 0.5}]))
    return out


def gen_closed_loop():
    """The reference's run_scenario rows / plans / detections on the
    closed-loop scenarios (harness.py:283-475)."""
    from resilsim.harness import run_scenario, scenario_from_mapping

    cases = []
    for m in closed_loop_mappings():
        res = run_scenario(scenario_from_mapping(m))
        cases.append({"mapping": m, "rows": res.iteration_rows,
                      "plans": [[k, p.reason] for k, p in res.plans],
                      "aborted_at": res.summary["aborted_at"]})
        print(m["seed"], len(res.iteration_rows), "plans", [k for k, _ in res.plans], flush=True)
    dump("closed_loop", {"cases": cases})


# ----------------------------------------------------------------- migration
def gen_migration():
    """Reference plan_migration (scheduler.py:272-513) on random problems."""
    rng = random.Random(6)
    cases = []
    while len(cases) < 80:
        state, cfg, mbs, model, comm = random_scenario(rng, allow_fail_stop=False)
        if cfg.dp < 2:
            continue
        speeds = rp._stage_speed_maps(state, cfg)[0]
        kind = rng.random()
        if kind < 0.3:  # a dead stage to drain
            d0, s0 = rng.randrange(cfg.dp), rng.randrange(cfg.pp)
            speeds[(d0, s0)] = 0.0
        counts = None
        if rng.random() < 0.3:
            cuts = sorted(rng.randint(0, len(mbs)) for _ in range(cfg.dp - 1))
            counts = [b - a for a, b in zip([0] + cuts, cuts + [len(mbs)])]
        edge = None
        if comm is not None:
            links = rc.ClusterState.copy(state)
            from resilsim.comm import LinkModel

            edge = rp.edge_cost_fn(state, cfg, comm, LinkModel.from_cluster(state),
                                   mbs[0].token_budget)
        delta = rng.choice([0, 0, 1, 2, 10**9])
        capacity = rng.choice([cfg.pp + 2, 8, 3])
        migrate = rng.random() < 0.85
        preset = {}
        if not migrate or rng.random() < 0.2:
            for mb in mbs[: max(1, len(mbs) // 3)]:
                preset[(mb.id, rng.randrange(cfg.pp))] = rng.randrange(cfg.dp)
        case = {"cfg": cfg_to_json(cfg), "mbs": mbs_to_json(mbs), "model": model_to_json(model),
                "speeds": keyed(speeds), "counts": counts, "delta": delta, "capacity": capacity,
                "migrate": migrate, "preset": [[j, s, d] for (j, s), d in preset.items()],
                "edges": None}
        if edge is not None:
            P, D = cfg.pp, cfg.dp
            case["edges"] = {
                "next": [[[edge(s, a, s + 1, b) if s + 1 < P else 0.0 for b in range(D)]
                          for a in range(D)] for s in range(P)],
                "prev": [[[edge(s, a, s - 1, b) if s > 0 else 0.0 for b in range(D)]
                          for a in range(D)] for s in range(P)],
                "same": [[[edge(s, a, s, b) for b in range(D)] for a in range(D)]
                         for s in range(P)]}
        try:
            res = rs.plan_migration(cfg, mbs, model, speeds, dp_counts=counts, delta=delta,
                                    capacity=capacity, edge_seconds=edge,
                                    preset_executors=preset or None, migrate=migrate)
            case["result"] = {
                "migrations": [[m.mb, m.stage, m.source, m.executor] for m in res.migrations],
                "makespan": res.makespan,
                "orders": [[d, s, [[k, j] for k, j in seq]]
                           for (d, s), seq in sorted(res.stage_orders.items())]}
        except rs.StrandedWorkload as exc:
            case["error"] = str(exc)
        cases.append(case)
    dump("migration", {"cases": cases})


# ----------------------------------------------------------------- policies
def gen_policies():
    """Reference resihp_adapt (policies.py:189-352) decisions on random contexts."""
    rng = random.Random(8)
    cases = []
    while len(cases) < 40:
        tp = rng.choice([2, 4])
        dp = rng.choice([1, 2, 3])
        pp = rng.choice([2, 3, 4])
        layers = pp * rng.randint(2, 4)
        cfg = rc.ParallelismConfig(tp=tp, dp=dp, pp=pp,
                                   schedule=rng.choice(["1f1b", "zbh"]),
                                   layer_partition=[layers // pp] * pp)
        n_dev = tp * dp * pp
        nodes = max(1, -(-n_dev // 8)) + rng.choice([0, 0, 1])
        state = rc.build_cluster(nodes, 8, cfg, 300.0 * 2**30, 25.0 * 2**30)
        events, known, new_stop = [], {}, []
        for _ in range(rng.randint(1, 3)):
            dev = rng.randrange(n_dev)
            if rng.random() < 0.35:
                events.append(rc.FailureEvent(kind="fail_stop", start=0.0, device=dev))
                new_stop.append("stop")
            else:
                sev = rng.choice([0.2, 0.4, 0.5, 0.7])
                events.append(rc.FailureEvent(kind="fail_slow_compute", start=0.0, device=dev,
                                              severity=sev))
                known[dev] = sev
        state = rc.apply_failures(state, events, 0.0)
        M = dp * rng.randint(2, 6)
        docs = [max(1, min(4096, int(rng.lognormvariate(7.2, 0.8)))) for _ in range(M * 6)]
        mbs = rw.pack_sequences(docs, 4096)[:M]
        if len(mbs) < M:
            continue
        confirmed = None
        slow_keys = sorted({k for k, g in state.tp_groups.items() if any(d in known for d in g)})
        if slow_keys:
            confirmed = rd.ValidationResult(True, {k: 0.5 for k in slow_keys}, {}, 3.0)
        ctx = rpol.PlanningContext(state=state, cfg=cfg, model=rw.CostModel(2e-6, 5e-10),
                                   micro_batches=mbs, comm=CommSpec(), known_speeds=known,
                                   new_fail_stop=new_stop, confirmed=confirmed,
                                   delta=rng.choice([0, 1]), capacity=pp + 2)
        case = {"nodes": nodes, "cfg": cfg_to_json(cfg),
                "events": [[e.kind, e.device, e.severity] for e in events],
                "known": [[k, v] for k, v in known.items()], "mbs": mbs_to_json(mbs),
                "confirmed": [list(k) for k in slow_keys], "new_fail_stop": len(new_stop),
                "delta": ctx.delta, "capacity": ctx.capacity}
        try:
            plan = rpol.resihp_adapt(ctx)
            case["plan"] = {
                "tp_subgroups": [[d, s, list(m), list(sb)]
                                 for (d, s), (m, sb) in sorted(plan.tp_subgroups.items())],
                "excluded": [list(k) for k in plan.excluded_groups],
                "layer_partition": plan.layer_partition, "dp_assignment": plan.dp_assignment,
                "migrations": [[m.mb, m.stage, m.source, m.executor] for m in plan.migrations],
                "predicted": plan.predicted_makespan_s}
        except (rs.StrandedWorkload, rs.GroupUnrecoverable) as exc:
            case["error"] = type(exc).__name__
        cases.append(case)
    dump("policies", {"cases": cases})


if __name__ == "__main__":
    which = sys.argv[1:] or ["workload", "pipeline", "detector", "scheduler", "search",
                             "search_bench", "migration", "policies", "closed_loop"]
    for w in which:
        globals()[f"gen_{w}"]()
