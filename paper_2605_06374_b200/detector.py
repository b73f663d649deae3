"""Fail-slow detection (mirror of resilsim/detector.py) on the GPU.

Single-iteration calls keep the reference API (``DetectorState.observe``,
``detect_change_point``, ``filter_candidate``, ``validate``).  The batched
product entry point is ``DetectorPass`` (rh_detect_batch + rh_screen): the
predictor on the known view, the workload-aware filter, validation and the
change-point state machine for a whole trace of iterations in two launches.
Fail-stop heartbeats (detector.py:42-91) are event-time bookkeeping outside
this hot path; HeartbeatMonitor is provided for API completeness.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cluster import FAIL_STOP

BENIGN = "benign"
ESCALATE = "escalate"


@dataclass
class HeartbeatConfig:
    interval_s: float = 1.0
    miss_threshold: int = 3

    def __post_init__(self):
        if self.interval_s <= 0:
            raise ValueError("heartbeat interval must be positive")
        if self.miss_threshold < 1:
            raise ValueError("miss threshold must be >= 1")


@dataclass
class FailStopDecision:
    node_id: int
    device_ids: tuple[int, ...]
    failed_at: float
    declared_at: float


class HeartbeatMonitor:
    """detector.py:42-83: declare at the first tick >= t0 + m * interval."""

    def __init__(self, config: HeartbeatConfig | None = None):
        self.config = config or HeartbeatConfig()
        self.declared: set[int] = set()

    def declare_time(self, failed_at: float) -> float:
        c = self.config
        return math.ceil((failed_at + c.miss_threshold * c.interval_s) / c.interval_s
                         - 1e-12) * c.interval_s

    def scan(self, state, t: float) -> list[FailStopDecision]:
        per_node: dict[int, list[tuple[int, float, float]]] = {}
        for dev in state.devices:
            if dev.status != FAIL_STOP or dev.id in self.declared or dev.failed_at is None:
                continue
            at = self.declare_time(dev.failed_at)
            if at <= t:
                per_node.setdefault(dev.node_id, []).append((dev.id, dev.failed_at, at))
        out = []
        for node in sorted(per_node):
            rows = sorted(per_node[node])
            ids = tuple(r[0] for r in rows)
            self.declared.update(ids)
            out.append(FailStopDecision(node, ids, min(r[1] for r in rows),
                                        max(r[2] for r in rows)))
        return out


def heartbeat_scan(monitor: HeartbeatMonitor, state, t: float) -> set[int]:
    return {d for dec in monitor.scan(state, t) for d in dec.device_ids}


@dataclass
class ValidationResult:
    confirmed: bool
    degraded_stages: dict[tuple[int, int], float]
    degraded_links: dict[tuple[int, int], float]
    cost_s: float


@dataclass
class DetectorStats:
    candidates: int = 0
    filter_checks: int = 0
    benign_filtered: int = 0
    escalations: int = 0
    validations: int = 0
    false_alarms: int = 0
    filter_cost_s: float = 0.0
    validation_cost_s: float = 0.0


@dataclass
class DetectorOutcome:
    candidate: bool = False
    verdict: str | None = None
    validation: ValidationResult | None = None
    charged_s: float = 0.0
    alarms: list[str] = field(default_factory=list)


# ------------------------------------------------------------ GPU helpers
def _dev():
    import torch

    return torch.device("cuda", torch.cuda.current_device())


def _screen(series_len: int, hist: list[float], observed, it_status, window: int, kappa: float,
            filter_enabled: bool, reset=None):
    """rh_screen (rh_screen_host: one copy in, one copy out) -> (outcome
    uint8[n], final series length)."""
    n = len(observed)
    h = min(series_len, window)
    t_hist = np.asarray(list(hist[len(hist) - h:]) if h else [0.0], dtype=np.float64)
    t_obs = np.ascontiguousarray(observed, dtype=np.float64)
    t_st = np.ascontiguousarray(it_status, dtype=np.uint8)
    t_rst = None if reset is None else np.ascontiguousarray(reset, dtype=np.uint8)
    out = np.zeros(max(n, 1), dtype=np.uint8)
    t_len = np.zeros(1, dtype=np.int64)
    params = _lib.ScreenParams(int(window), 1 if filter_enabled else 0, float(kappa))
    lib = _lib.load_library()
    _lib.check(lib.rh_screen_host(_lib.context(), _lib.C.byref(params), int(series_len),
                                  t_hist.ctypes.data, n, t_obs.ctypes.data, t_st.ctypes.data,
                                  None if t_rst is None else t_rst.ctypes.data, out.ctypes.data,
                                  t_len.ctypes.data), "rh_screen_host")
    return out[:n], int(t_len[0])


def _validate_arrays(measured, expected, threshold):
    n = len(measured)
    if n == 0:
        return np.zeros(0, bool), np.zeros(0)
    m = np.ascontiguousarray(measured, dtype=np.float64)
    e = None if expected is None else np.ascontiguousarray(expected, dtype=np.float64)
    flag = np.empty(n, dtype=np.uint8)
    sev = np.empty(n, dtype=np.float64)
    lib = _lib.load_library()
    _lib.check(lib.rh_validate_host(_lib.context(), n, m.ctypes.data,
                                    None if e is None else e.ctypes.data, float(threshold),
                                    flag.ctypes.data, sev.ctypes.data), "rh_validate_host")
    return flag.astype(bool), sev


# ------------------------------------------------------------ reference API
def detect_change_point(series: list[float], window: int = 20, kappa: float = 3.0) -> int | None:
    """detector.py:94-108 via rh_screen on the newest point."""
    if len(series) < window + 1:
        return None
    oc, _ = _screen(len(series) - 1, list(series[:-1]), [series[-1]], [0], window, kappa,
                    filter_enabled=False)
    return len(series) - 1 if oc[0] & _lib.RH_SC_CANDIDATE else None


def filter_candidate(observed: float, predicted: float, escalation_factor: float = 1.25) -> str:
    """detector.py:111-116 (scalar rule; the batched form is fused into rh_detect_batch)."""
    if predicted <= 0:
        return ESCALATE
    return ESCALATE if observed > escalation_factor * predicted else BENIGN


def validate(stage_times, link_ratios=None, threshold: float = 1.25,
             cost_s: float = 3.0) -> ValidationResult:
    """detector.py:127-158 via rh_validate."""
    keys = sorted(stage_times)
    flags, sev = _validate_arrays([stage_times[k][0] for k in keys],
                                  [stage_times[k][1] for k in keys], threshold)
    stages = {k: float(v) for k, f, v in zip(keys, flags, sev) if f}
    lkeys = sorted(link_ratios or {})
    lf, lsev = _validate_arrays([link_ratios[k] for k in lkeys], None, threshold)
    links = {k: float(v) for k, f, v in zip(lkeys, lf, lsev) if f}
    return ValidationResult(bool(stages or links), stages, links, cost_s)


@dataclass
class DetectorState:
    """detector.py:182-271; the screen runs on the GPU (rh_screen)."""

    window: int = 20
    kappa: float = 3.0
    escalation_factor: float = 1.25
    filter_enabled: bool = True
    filter_cost_s: float = 0.05
    validation_cost_s: float = 3.0
    series: list[float] = field(default_factory=list)
    stats: DetectorStats = field(default_factory=DetectorStats)

    def reset_series(self) -> None:
        self.series.clear()

    def observe(self, record, predicted: float, reference_stage_cost=None) -> DetectorOutcome:
        out = DetectorOutcome()
        reference = reference_stage_cost or record.stage_cost_reference
        keys = sorted(record.stage_cost)
        # the filter verdict is a host scalar rule; validation (when escalated,
        # or with the filter disabled) and the screen of the new observation
        # run in ONE device call (rh_observe_host: one copy in, one copy out)
        verdict = filter_candidate(record.observed_time, predicted, self.escalation_factor)
        do_val = verdict == ESCALATE or not self.filter_enabled
        lkeys = sorted(record.link_ratio or {})
        ns, nl = len(keys), len(lkeys)
        meas = np.ascontiguousarray([record.stage_cost[k] for k in keys] or [0.0], np.float64)
        expd = np.ascontiguousarray([reference.get(k, 0.0) for k in keys] or [0.0], np.float64)
        lr = np.ascontiguousarray([record.link_ratio[k] for k in lkeys] or [0.0], np.float64)
        sf, ss = np.zeros(max(ns, 1), np.uint8), np.zeros(max(ns, 1))
        lf, ls = np.zeros(max(nl, 1), np.uint8), np.zeros(max(nl, 1))
        h = min(len(self.series), self.window)
        hist = np.ascontiguousarray(self.series[len(self.series) - h:] if h else [0.0], np.float64)
        oc = np.zeros(1, np.uint8)
        new_len = np.zeros(1, np.int64)
        params = _lib.ScreenParams(int(self.window), 1 if self.filter_enabled else 0,
                                   float(self.kappa))
        lib = _lib.load_library()
        _lib.check(lib.rh_observe_host(
            _lib.context(), _lib.C.byref(params), len(self.series), hist.ctypes.data,
            float(record.observed_time), 1 if verdict == ESCALATE else 0, 1 if do_val else 0,
            ns, meas.ctypes.data, expd.ctypes.data, nl, lr.ctypes.data,
            float(self.escalation_factor), sf.ctypes.data, ss.ctypes.data, lf.ctypes.data,
            ls.ctypes.data, oc.ctypes.data, new_len.ctypes.data), "rh_observe_host")
        result = None
        if do_val:
            stages = {k: float(v) for k, f, v in zip(keys, sf, ss) if f}
            links = {k: float(v) for k, f, v in zip(lkeys, lf, ls) if f}
            result = ValidationResult(bool(stages or links), stages, links,
                                      self.validation_cost_s)
        return self._apply(int(oc[0]), record.observed_time, verdict, result, out)

    def _apply(self, oc: int, observed: float, verdict: str, result, out: DetectorOutcome):
        """Replay one outcome code into the reference's stats / series / alarms."""
        self.series.append(observed)
        if not oc:
            return out
        if oc & _lib.RH_SC_CANDIDATE:
            out.candidate = True
            self.stats.candidates += 1
            out.alarms.append("candidate")
        if oc & _lib.RH_SC_FILTERED:
            out.charged_s += self.filter_cost_s
            self.stats.filter_cost_s += self.filter_cost_s
            self.stats.filter_checks += 1
            out.verdict = verdict
            if not oc & _lib.RH_SC_ESCALATED:
                if oc & _lib.RH_SC_POPPED:
                    self.stats.benign_filtered += 1
                    self.series.pop()
                    out.alarms.append("benign")
                return out
        else:
            out.verdict = ESCALATE
        self.stats.escalations += 1
        out.alarms.append("escalate")
        self.stats.validations += 1
        self.stats.validation_cost_s += result.cost_s
        out.charged_s += result.cost_s
        out.validation = result
        if not oc & _lib.RH_SC_CONFIRMED:
            self.stats.false_alarms += 1
            self.series.pop()
            out.alarms.append("unconfirmed")
        else:
            targets = [f"d{d}s{s}" for d, s in sorted(result.degraded_stages)]
            targets += [f"link{a}-{b}" for a, b in sorted(result.degraded_links)]
            out.alarms.append("confirmed:" + "+".join(targets))
        return out
