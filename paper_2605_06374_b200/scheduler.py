"""Progressive TP -> PP -> DP adaptation (mirror of resilsim/scheduler.py).

Plan objects and ``apply_plan`` are host-side descriptions; every number a
plan is judged by comes from the GPU: ``evaluate_plan`` runs the iteration
predictor (simulate_iteration -> rh_pipeline_batch / rh_dag_critical_path).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .cluster import FAIL_SLOW, FAIL_STOP, HEALTHY, STANDBY
from .comm import LinkModel
from .pipeline import SimulationError, simulate_iteration


class GroupUnrecoverable(RuntimeError):
    """A TP group cannot reach the minimum feasible degree (scheduler.py:30)."""


class StrandedWorkload(SimulationError):
    """A fail-stop stage has pending work and no feasible destination (scheduler.py:34)."""


@dataclass
class Migration:
    mb: int
    stage: int
    source: int
    executor: int


@dataclass
class AdaptationPlan:
    """scheduler.py:46-70"""

    tp_subgroups: dict = field(default_factory=dict)
    excluded_groups: list = field(default_factory=list)
    layer_partition: list[int] | None = None
    dp_assignment: list[int] | None = None
    migrations: list[Migration] = field(default_factory=list)
    stage_orders: dict | None = None
    reconfig_cost_s: float = 0.0
    predicted_makespan_s: float | None = None
    reason: str = ""

    def is_empty(self) -> bool:
        return not (self.tp_subgroups or self.excluded_groups or self.layer_partition is not None
                    or self.dp_assignment is not None or self.migrations)


@dataclass
class ProgressTable:
    """scheduler.py:73-98: forward progress per (replica, stage) + delta."""

    counts: list[list[int]]
    delta: int = 0

    @classmethod
    def zeros(cls, dp: int, pp: int, delta: int = 0) -> "ProgressTable":
        return cls(counts=[[0] * pp for _ in range(dp)], delta=delta)

    def bump(self, replica: int, stage: int) -> None:
        self.counts[replica][stage] += 1

    def gap(self, stage: int) -> int:
        col = [row[stage] for row in self.counts]
        return max(col) - min(col)


def migration_decision(progress: ProgressTable, stage: int, dead: set, next_pending,
                       memory_feasible, outstanding=None):
    """scheduler.py:210-251 -- one stage's per-slot migration decision.

    The API form of the rule the native co-simulation (rh_plan_migration,
    csrc/migration.cu) applies per slot, for callers that drive their own
    slots with Python callbacks: source = the stage's least-progressed replica
    (fail-stop first, then index); destination = the most-progressed healthy
    replica (least outstanding work, then index); migrate when the source is
    fail-stop or the progress gap exceeds delta, it has a pending forward
    chunk, and the destination has memory headroom -> (mb, source, executor)."""
    counts = progress.counts
    n = len(counts)
    d_min = min(range(n), key=lambda d: (counts[d][stage], 0 if (d, stage) in dead else 1, d))
    healthy = [d for d in range(n) if (d, stage) not in dead]
    if not healthy:
        return None
    load = outstanding or (lambda d, s: 0)
    top = max(counts[d][stage] for d in healthy)
    d_max = min((d for d in healthy if counts[d][stage] == top), key=lambda d: (load(d, stage), d))
    if d_max == d_min:
        return None
    if (d_min, stage) not in dead and counts[d_max][stage] - counts[d_min][stage] <= progress.delta:
        return None
    j = next_pending(d_min, stage)
    if j is None or not memory_feasible(j, stage, d_max):
        return None
    return j, d_min, d_max


@dataclass
class MigrationPlanResult:
    migrations: list[Migration]
    makespan: float
    stage_orders: dict = field(default_factory=dict)
    slots: list = field(default_factory=list)


_KIND_NAMES = {0: "F", 2: "W"}


def plan_migration(cfg, micro_batches, model, speeds, *, dp_counts=None, delta: int = 0,
                   capacity: int = 8, edge_seconds=None, record_trace: bool = False,
                   preset_executors=None, migrate: bool = True) -> MigrationPlanResult:
    """scheduler.py:272-513 — progress-aware migration co-simulation.

    Runs natively (rh_plan_migration, csrc/migration.cu).  ``edge_seconds`` is
    evaluated into per-stage hop tables first.  ``record_trace`` slot traces
    are a reference debugging aid and are not produced."""
    import ctypes as C

    import numpy as np

    from . import _lib
    from .cluster import SCHEDULE_1F1B
    from .workload import cost_model_c, csr_of

    P, D, M = cfg.pp, cfg.dp, len(micro_batches)
    ids = [mb.id for mb in micro_batches]
    if ids != sorted(ids) or len(set(ids)) != M:
        raise ValueError("micro-batch ids must be unique and ascending in list order")
    pos = {j: k for k, j in enumerate(ids)}
    if len(cfg.layer_partition) != P:
        raise ValueError("layer partition does not match stage count")
    speed = np.array([speeds[(d, s)] for d in range(D) for s in range(P)], dtype=np.float64)
    mb_off, doc_len = csr_of(micro_batches)
    doc_len = doc_len if doc_len.size else np.zeros(1, np.int32)
    layers = np.asarray(cfg.layer_partition, dtype=np.int32)
    counts = None if dp_counts is None else np.asarray(dp_counts, dtype=np.int32)
    preset = None
    if preset_executors:
        preset = np.full(M * P, -1, dtype=np.int32)
        for (j, s), d in preset_executors.items():
            preset[pos[j] * P + s] = d
    tabs = [None, None, None]
    if edge_seconds is not None:
        nxt = np.zeros((P, D, D))
        prv = np.zeros((P, D, D))
        same = np.zeros((P, D, D))
        for s in range(P):
            for a in range(D):
                for b in range(D):
                    if s + 1 < P:
                        nxt[s, a, b] = edge_seconds(s, a, s + 1, b)
                    if s > 0:
                        prv[s, a, b] = edge_seconds(s, a, s - 1, b)
                    same[s, a, b] = edge_seconds(s, a, s, b)
        tabs = [nxt, prv, same]
    desc = _lib.MigrationDesc(
        P, D, 0 if cfg.schedule == SCHEDULE_1F1B else 1, M, micro_batches[0].token_budget,
        cost_model_c(model), mb_off.ctypes.data, doc_len.ctypes.data, layers.ctypes.data,
        speed.ctypes.data,
        None if counts is None else counts.ctypes.data, int(delta), int(capacity),
        1 if migrate else 0, None if preset is None else preset.ctypes.data,
        *[None if t is None else t.ctypes.data for t in tabs])
    c = 2 if cfg.schedule == SCHEDULE_1F1B else 3
    mig = np.zeros(4 * M * P, dtype=np.int32)
    log = np.zeros(4 * M * P * c, dtype=np.int32)
    n_mig, n_log, ms = C.c_int32(), C.c_int32(), C.c_double()
    lib = _lib.load_library()
    rc = lib.rh_plan_migration(C.byref(desc), mig.ctypes.data, C.byref(n_mig), log.ctypes.data,
                               C.byref(n_log), C.byref(ms))
    if rc == _lib.RH_E_STRANDED:
        raise StrandedWorkload(lib.rh_last_error().decode())
    _lib.check(rc, "rh_plan_migration")
    back = "BW" if cfg.schedule == SCHEDULE_1F1B else "B"
    migrations = [Migration(ids[a], s, src, dst) for a, s, src, dst in
                  mig[:4 * n_mig.value].reshape(-1, 4).tolist()]
    orders: dict = {}
    for d, s, k, j in log[:4 * n_log.value].reshape(-1, 4).tolist():
        orders.setdefault((d, s), []).append((_KIND_NAMES.get(k, back), ids[j]))
    return MigrationPlanResult(migrations=migrations, makespan=ms.value, stage_orders=orders)


def apply_plan(state, cfg, plan):
    """scheduler.py:516-540: materialise group / layer changes on copies."""
    out, new_cfg = state.copy(), cfg.copy()
    for (d, s), (members, standby) in plan.tp_subgroups.items():
        out.tp_groups[(d, s)] = tuple(sorted(members))
        for m in standby:
            if out.devices[m].status != FAIL_STOP:
                out.devices[m].status = STANDBY
        for m in members:
            dev = out.devices[m]
            if dev.status == STANDBY:
                dev.status = HEALTHY if dev.speed >= 1.0 else FAIL_SLOW
    for key in plan.excluded_groups:
        for m in out.tp_groups.get(key, ()):
            if out.devices[m].status != FAIL_STOP:
                out.devices[m].status = STANDBY
        out.tp_groups[key] = ()
    if plan.layer_partition is not None:
        new_cfg.layer_partition = list(plan.layer_partition)
    return out, new_cfg


def evaluate_plan(plan, state, cfg, micro_batches, model, *, comm=None,
                  capacity: int | None = None) -> float:
    """scheduler.py:543-559: predicted makespan under the plan (GPU)."""
    new_state, new_cfg = apply_plan(state, cfg, plan)
    return simulate_iteration(new_state, new_cfg, micro_batches, model, plan, comm=comm,
                              capacity=capacity).observed_time


def reconfig_cost(plan, state, cfg, *, layer_bytes: float, group_rebuild_s: float = 2.0) -> float:
    """scheduler.py:562-593: rebuild constant + state transfer at the worst link."""
    rebuild = bool(plan.tp_subgroups or plan.excluded_groups)
    moved = 0
    new = plan.layer_partition
    if new is not None and list(new) != list(cfg.layer_partition):
        rebuild = True
        moved = sum(max(0, a - b) for a, b in zip(new, cfg.layer_partition))
    if not rebuild:
        return 0.0
    part = list(new) if new is not None else list(cfg.layer_partition)
    reshard = 0.0
    for (d, s), (members, _) in plan.tp_subgroups.items():
        if set(members) != set(state.tp_groups.get((d, s), ())):
            reshard += part[s] * layer_bytes
    return group_rebuild_s + (moved * layer_bytes + reshard) / LinkModel.from_cluster(state).worst_inter()


# ------------------------------------------------ scalar rows on the GPU
def _batch(fn_name: str, *host_arrays_and_outputs):
    """Run one rh_*_batch kernel on host numpy arrays (copied in and out)."""
    import torch

    from . import _lib

    dev = torch.device("cuda", torch.cuda.current_device())
    tens = [torch.from_numpy(a).to(dev) if isinstance(a, np.ndarray) else a
            for a in host_arrays_and_outputs]
    lib = _lib.load_library()
    args = [t.data_ptr() if hasattr(t, "data_ptr") else t for t in tens]
    _lib.check(getattr(lib, fn_name)(_lib.context(), *args, _lib.stream_handle()), fn_name)
    return tens


def candidate_tp_degrees(group_size: int, fail_stop_count: int, k_min: int) -> set[int]:
    """scheduler.py:101-111 (Eq. 3): powers of two in [k_min, survivors]."""
    if k_min < 1 or (k_min & (k_min - 1)) != 0:
        raise ValueError("k_min must be a power of two >= 1")
    out, k = set(), k_min
    while k <= group_size - fail_stop_count:
        out.add(k)
        k *= 2
    return out


def select_tp_subgroup(device_speeds: dict, degrees: set[int]):
    """scheduler.py:114-137 (Eq. 4) via rh_select_subgroup_batch."""
    import torch

    if not degrees:
        raise GroupUnrecoverable("no feasible TP degree")
    ids = np.array(list(device_speeds), dtype=np.int32)
    sp = np.array([device_speeds[i] for i in ids], dtype=np.float64)
    mask = 0
    for k in degrees:
        if k >= 1 and (k & (k - 1)) == 0 and k < 2**31:
            mask |= 1 << (k.bit_length() - 1)
    n = len(ids)
    dev = torch.device("cuda", torch.cuda.current_device())
    ranked = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    best = torch.empty(1, dtype=torch.int32, device=dev)
    _batch("rh_select_subgroup_batch", 1, np.array([0, n], np.int32),
           sp if n else np.zeros(1), ids if n else np.zeros(1, np.int32),
           np.array([mask], np.uint32), ranked, best)
    k = int(best.item())
    if k == 0:
        raise GroupUnrecoverable("group smaller than every candidate degree")
    order = ranked.cpu().numpy()[:n].tolist()
    return tuple(sorted(order[:k])), tuple(sorted(order[k:]))


def subgroup_score(device_speeds: dict, members) -> float:
    """scheduler.py:140-143: |members| * slowest member."""
    if not members:
        return 0.0
    return len(members) * min(device_speeds[d] for d in members)


def repartition_layers(stage_speeds: list[float], total_layers: int,
                       min_layers: int = 1) -> list[int]:
    """scheduler.py:146-207 via rh_repartition_batch."""
    import torch

    n = len(stage_speeds)
    if any(s <= 0 for s in stage_speeds):
        raise ValueError("all stage speeds must be positive")
    if total_layers < n * min_layers:
        raise ValueError(f"cannot give {n} stages {min_layers} layers each out of {total_layers}")
    if n > 32:
        raise ValueError("repartition_layers: at most 32 stages on this path")
    dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(n, dtype=torch.int32, device=dev)
    err = torch.empty(1, dtype=torch.int32, device=dev)
    _batch("rh_repartition_batch", 1, np.array([0, n], np.int32),
           np.asarray(stage_speeds, np.float64), np.array([total_layers], np.int32),
           np.array([min_layers], np.int32), out, err)
    if int(err.item()):
        raise ValueError("repartition_layers: infeasible problem")
    return [int(x) for x in out.cpu().numpy()]
