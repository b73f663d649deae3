"""Batched closed loop across scenarios (harness.py:283-475).

S seeded scenarios advance in lockstep, one iteration at a time.  Per
iteration the host runs each scenario's control logic (failure injection,
heartbeat declarations, the document stream, ResiHP re-planning when the
Detector confirmed a fail-slow or a fail-stop was declared, the known-speed
bookkeeping) and the GPU does the predictor work of ALL scenarios at once:
the actual run and the known-view reference of every scenario -- each with
its healthy twin -- go through `simulate_iteration_batch`, one
rh_pipeline_batch launch per distinct pipeline shape instead of 2S
simulate_iteration calls.  Detection feeds back into adaptation exactly as in
run_scenario: confirmed stages update the known speeds (with the
measurement-noise draw of harness.py:446-449) and trigger resihp_adapt on the
next iteration.

Scenario mappings use the reference's schema (harness.scenario_from_mapping);
the per-iteration rows equal run_scenario's (tests/golden/closed_loop.json,
made by importing the reference).  Out of scope: output files,
the summary's idle-amplification tracker and the recycle / greyhound
baselines.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np

from .cluster import (FAIL_STOP, STANDBY, FailureEvent, ParallelismConfig, apply_failures,
                      build_cluster, validate_cluster)
from .comm import CommSpec
from .detector import DetectorState, HeartbeatConfig, HeartbeatMonitor
from .pipeline import SimulationError, simulate_iteration_batch
from .policies import PlanningContext, make_policy
from .scheduler import AdaptationPlan, StrandedWorkload, apply_plan
from .workload import CostModel, pack_sequences

GIB = float(2**30)


@dataclass
class _Spec:
    """The fields of harness.Scenario this loop reads (harness.py:66-128)."""

    name: str = "scenario"
    seed: int = 0
    iterations: int = 50
    policy: str = "resihp"
    nodes: int = 2
    devices_per_node: int = 8
    intra_bw: float = 300.0 * GIB
    inter_bw: float = 25.0 * GIB
    cfg: ParallelismConfig = None
    token_budget: int = 4096
    micro_batches: int = 8
    doc_kind: str = "lognormal"
    doc_length: int = 0
    mean_log: float = 7.0
    sigma_log: float = 0.8
    model: CostModel = None
    comm: CommSpec = None
    det: dict = field(default_factory=dict)
    sched: dict = field(default_factory=dict)
    failures: list = field(default_factory=list)

    @property
    def capacity(self) -> int:
        return self.sched["activation_capacity"] or self.cfg.pp + 2


def spec_from_mapping(data: dict) -> _Spec:
    """harness.scenario_from_mapping (harness.py:131-224), lognormal / fixed
    document lengths."""
    sc = _Spec()
    sc.name = str(data.get("name", sc.name))
    sc.seed = int(data.get("seed", 0))
    sc.iterations = int(data.get("iterations", 50))
    sc.policy = str(data.get("policy", "resihp"))
    cl = data.get("cluster", {})
    sc.nodes = int(cl.get("nodes", 2))
    sc.devices_per_node = int(cl.get("devices_per_node", 8))
    sc.intra_bw = float(cl.get("intra_bw_gbps", 300.0)) * GIB
    sc.inter_bw = float(cl.get("inter_bw_gbps", 25.0)) * GIB
    par = data.get("parallelism", {})
    tp, dp, pp = int(par.get("tp", 4)), int(par.get("dp", 2)), int(par.get("pp", 2))
    if "layer_partition" in par:
        part = [int(x) for x in par["layer_partition"]]
    else:
        layers = int(par.get("layers", 8 * pp))
        b, e = divmod(layers, pp)
        part = [b + (1 if i < e else 0) for i in range(pp)]
    sc.cfg = ParallelismConfig(tp=tp, dp=dp, pp=pp,
                               schedule=str(par.get("schedule", "1f1b")).lower(),
                               layer_partition=part)
    wl = data.get("workload", {})
    sc.token_budget = int(wl.get("token_budget", 4096))
    sc.micro_batches = int(wl.get("micro_batches", 8))
    doc = wl.get("doc_lengths", {"kind": "lognormal"})
    sc.doc_kind = str(doc.get("kind", "lognormal"))
    if sc.doc_kind == "fixed":
        sc.doc_length = int(doc.get("length", sc.token_budget))
    elif sc.doc_kind == "lognormal":
        sc.mean_log = float(doc.get("mean", 7.0))
        sc.sigma_log = float(doc.get("sigma", 0.8))
    else:
        raise NotImplementedError(f"document source {sc.doc_kind!r}")
    cm = data.get("cost_model", {})
    sc.model = CostModel(alpha=float(cm.get("alpha", 2e-6)), beta=float(cm.get("beta", 5e-10)))
    if "chunk_ratios" in cm:
        sc.model.chunk_ratios.update({k: float(v) for k, v in cm["chunk_ratios"].items()})
    co = data.get("comm", {})
    sc.comm = CommSpec(hidden_bytes_per_token=float(co.get("hidden_bytes_per_token", 8192.0)),
                       layer_bytes=float(co.get("layer_bytes_mib", 256.0)) * 2**20,
                       p2p_optimized=bool(co.get("p2p_optimized", True)))
    det = data.get("detector", {})
    sc.det = dict(heartbeat_interval_s=float(det.get("heartbeat_interval_s", 1.0)),
                  heartbeat_miss_threshold=int(det.get("heartbeat_miss_threshold", 3)),
                  window=int(det.get("window", 20)), kappa=float(det.get("kappa", 3.0)),
                  escalation_factor=float(det.get("escalation_factor", 1.25)),
                  filter_cost_s=float(det.get("filter_cost_s", 0.05)),
                  validation_cost_s=float(det.get("validation_cost_s", 3.0)),
                  measurement_noise=float(det.get("measurement_noise", 0.01)))
    sch = data.get("scheduler", {})
    sc.sched = dict(k_min=int(sch.get("k_min", 2)), delta=int(sch.get("delta", 0)),
                    min_layers=int(sch.get("min_layers", 1)),
                    activation_capacity=int(sch.get("activation_capacity", 0)),
                    group_rebuild_s=float(sch.get("group_rebuild_s", 2.0)))
    for ev in data.get("failures", []):
        sc.failures.append(FailureEvent(
            kind=str(ev["kind"]), start=float(ev["start"]),
            device=int(ev["device"]) if "device" in ev else None,
            link=tuple(int(x) for x in ev["link"]) if "link" in ev else None,
            end=float(ev["end"]) if "end" in ev else None,
            severity=float(ev["severity"]) if "severity" in ev else None))
    sc.failures.sort(key=lambda e: e.start)
    return sc


class _DocSource:
    """harness._DocSource (harness.py:235-263): the same numpy stream."""

    def __init__(self, sc: _Spec):
        self.sc = sc
        self.rng = np.random.default_rng([sc.seed, 0])

    def micro_batches(self):
        sc = self.sc
        target = sc.micro_batches * sc.token_budget
        docs, total = [], 0
        while total < target:
            if sc.doc_kind == "fixed":
                x = min(sc.doc_length or sc.token_budget, sc.token_budget)
            else:
                raw = self.rng.lognormal(sc.mean_log, sc.sigma_log)
                x = int(max(1.0, min(round(raw), sc.token_budget)))
            docs.append(x)
            total += x
        return pack_sequences(docs, sc.token_budget)[:sc.micro_batches]


def _known_view(state, known_speeds, known_links):
    """harness.known_cluster_view (harness.py:514-521)."""
    out = state.copy()
    for dev in out.devices:
        if dev.status != FAIL_STOP:
            dev.speed = min(1.0, known_speeds.get(dev.id, 1.0))
    out.link_factors = dict(known_links)
    return out


def _active_count(state) -> int:
    return sum(1 for d in state.devices if d.status not in (FAIL_STOP, STANDBY))


def _has_dead_active_stage(state) -> bool:
    return any(g and any(state.devices[d].status == FAIL_STOP for d in g)
               for g in state.tp_groups.values())


def _absolute_severity(record, key) -> float:
    ref = record.stage_cost_reference.get(key, 0.0)
    act = record.stage_cost.get(key, 0.0)
    return 1.0 if act <= 0 or ref <= 0 else ref / act


class _Run:
    """One scenario's state between iterations (the locals of run_scenario)."""

    def __init__(self, sc: _Spec):
        self.sc = sc
        self.cfg = sc.cfg.copy()
        self.state = build_cluster(sc.nodes, sc.devices_per_node, self.cfg, sc.intra_bw,
                                   sc.inter_bw)
        bad = validate_cluster(self.state, self.cfg)
        if bad:
            raise ValueError("invalid scenario: " + "; ".join(bad))
        self.policy = make_policy(sc.policy)
        d = sc.det
        self.detector = DetectorState(window=d["window"], kappa=d["kappa"],
                                      escalation_factor=d["escalation_factor"],
                                      filter_enabled=self.policy.filter_enabled,
                                      filter_cost_s=d["filter_cost_s"],
                                      validation_cost_s=d["validation_cost_s"])
        self.monitor = HeartbeatMonitor(HeartbeatConfig(
            interval_s=d["heartbeat_interval_s"], miss_threshold=d["heartbeat_miss_threshold"]))
        self.docs = _DocSource(sc)
        self.noise = np.random.default_rng([sc.seed, 1])
        self.known_speeds, self.known_links = {}, {}
        self.live = AdaptationPlan()
        self.pending_fail_stop, self.confirmed = [], None
        self.now = self.wall = 0.0
        self.rows, self.plans, self.fail_slow_log, self.fail_stop = [], [], [], []
        self.aborted_at = None
        self.done = False


def run_batch(mappings, *, iterations: int | None = None):
    """Run every scenario mapping to completion in lockstep; returns, per
    scenario, {"rows": [...], "plans": [(iteration, reason)], "fail_slow":
    [...], "fail_stop": [...], "aborted_at": k or None}."""
    runs = [_Run(spec_from_mapping(m)) for m in mappings]
    n_iter = max(r.sc.iterations for r in runs) if iterations is None else iterations
    for k in range(n_iter):
        items, owners = [], []
        pending = []
        for r in runs:
            if r.done or k >= r.sc.iterations:
                r.done = True
                continue
            sc = r.sc
            r.state = apply_failures(r.state, sc.failures, r.now)
            for dec in r.monitor.scan(r.state, r.now):
                r.pending_fail_stop.append(dec)
                r.fail_stop.append({"node": dec.node_id, "devices": list(dec.device_ids),
                                    "failed_at": dec.failed_at, "declared_at": dec.declared_at,
                                    "latency_s": dec.declared_at - dec.failed_at})
            mbs = r.docs.micro_batches()
            undeclared = [r.monitor.declare_time(dev.failed_at) for dev in r.state.devices
                          if dev.status == FAIL_STOP and dev.failed_at is not None
                          and dev.id not in r.monitor.declared]
            if undeclared and _has_dead_active_stage(r.state):
                stall = max(r.now, min(undeclared)) - r.now
                r.now += stall
                r.wall += stall
                r.rows.append({"iteration": k, "observed_s": stall, "predicted_s": 0.0,
                               "alarms": "stall:fail_stop",
                               "active_devices": _active_count(r.state), "migrations": 0,
                               "wall_s": stall})
                continue
            charges, alarms = 0.0, []
            try:
                if r.pending_fail_stop or r.confirmed is not None:
                    ctx = PlanningContext(
                        state=r.state, cfg=r.cfg, model=sc.model, micro_batches=mbs,
                        comm=sc.comm, dp_counts=r.live.dp_assignment,
                        known_speeds=r.known_speeds, live_plan=r.live,
                        new_fail_stop=list(r.pending_fail_stop), confirmed=r.confirmed,
                        k_min=sc.sched["k_min"], delta=sc.sched["delta"], capacity=sc.capacity,
                        min_layers=sc.sched["min_layers"], layer_bytes=sc.comm.layer_bytes,
                        group_rebuild_s=sc.sched["group_rebuild_s"])
                    plan = r.policy.plan(ctx)
                    if plan is not None:
                        r.state, r.cfg = apply_plan(r.state, r.cfg, plan)
                        r.live = AdaptationPlan(
                            migrations=plan.migrations,
                            dp_assignment=plan.dp_assignment or r.live.dp_assignment,
                            stage_orders=plan.stage_orders)
                        charges += plan.reconfig_cost_s
                        r.plans.append((k, plan.reason))
                        r.detector.reset_series()
                        alarms.append("adapt:" + plan.reason)
                    r.pending_fail_stop, r.confirmed = [], None
            except (StrandedWorkload, SimulationError) as exc:
                r.aborted_at = k
                r.rows.append({"iteration": k, "observed_s": 0.0, "predicted_s": 0.0,
                               "alarms": "aborted:" + type(exc).__name__,
                               "active_devices": _active_count(r.state), "migrations": 0,
                               "wall_s": 0.0})
                r.done = True
                continue
            known = _known_view(r.state, r.known_speeds, r.known_links)
            items.append((r.state, r.cfg, mbs, sc.model, r.live, sc.comm, k, sc.capacity))
            items.append((known, r.cfg, mbs, sc.model, r.live, sc.comm, k, None))
            owners.append(r)
            pending.append((charges, alarms))
        if not items:
            continue
        # ---- the GPU step: every scenario's actual + reference run at once
        results = simulate_iteration_batch(items)
        for q, r in enumerate(owners):
            sc = r.sc
            charges, alarms = pending[q]
            record, reference = results[2 * q], results[2 * q + 1]
            bad = record if isinstance(record, Exception) else (
                reference if isinstance(reference, Exception) else None)
            if bad is not None:
                if not isinstance(bad, (StrandedWorkload, SimulationError)):
                    raise bad
                r.aborted_at = k
                r.rows.append({"iteration": k, "observed_s": 0.0, "predicted_s": 0.0,
                               "alarms": "aborted:" + type(bad).__name__,
                               "active_devices": _active_count(r.state), "migrations": 0,
                               "wall_s": 0.0})
                r.done = True
                continue
            record.predicted_healthy_time = reference.observed_time
            record.alarms = alarms
            if r.policy.detector_enabled:
                sigma = sc.det["measurement_noise"]
                noisy = dataclasses.replace(record, stage_cost={
                    key: value * (1.0 + sigma * float(r.noise.standard_normal()))
                    for key, value in sorted(record.stage_cost.items())})
                outcome = r.detector.observe(noisy, reference.observed_time,
                                             reference_stage_cost=reference.stage_cost)
                charges += outcome.charged_s
                record.alarms.extend(outcome.alarms)
                if outcome.validation is not None and outcome.validation.confirmed:
                    r.confirmed = outcome.validation
                    for key in sorted(r.confirmed.degraded_stages):
                        r.fail_slow_log.append({"kind": "fail_slow", "stage": list(key),
                                                "confirmed_iteration": k,
                                                "severity_estimate":
                                                    _absolute_severity(record, key)})
                        for dev_id in r.state.tp_groups.get(key, ()):
                            true = r.state.devices[dev_id].speed
                            est = true * (1.0 + sigma * float(r.noise.standard_normal()))
                            r.known_speeds[dev_id] = float(min(1.0, max(0.01, est)))
                    for link in sorted(r.confirmed.degraded_links):
                        factor = r.state.link_factors.get(link,
                                                          r.confirmed.degraded_links[link])
                        r.known_links[link] = factor
                        r.fail_slow_log.append({"kind": "fail_slow_comm", "link": list(link),
                                                "confirmed_iteration": k,
                                                "severity_estimate": factor})
            wall_iter = record.observed_time + charges
            r.now += wall_iter
            r.wall += wall_iter
            r.rows.append({"iteration": k, "observed_s": record.observed_time,
                           "predicted_s": record.predicted_healthy_time,
                           "alarms": ";".join(record.alarms),
                           "active_devices": _active_count(r.state),
                           "migrations": record.migrations, "wall_s": wall_iter})
    return [{"rows": r.rows, "plans": r.plans, "fail_slow": r.fail_slow_log,
             "fail_stop": r.fail_stop, "aborted_at": r.aborted_at} for r in runs]
