"""Progressive TP -> PP -> DP adaptation (mirror of resilsim/scheduler.py).

Plan objects and ``apply_plan`` are host-side descriptions; every number a
plan is judged by comes from the GPU: ``evaluate_plan`` runs the iteration
predictor (simulate_iteration -> rh_pipeline_batch / rh_dag_critical_path).
"""

from __future__ import annotations

from dataclasses import dataclass, field

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
