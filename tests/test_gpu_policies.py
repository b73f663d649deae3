"""Scheduler rows 17-21 through the drop-in API on the GPU vs the reference:
select_tp_subgroup / repartition_layers / proportional_split unit vectors,
and full resihp_adapt decisions (subgroups, exclusions, partition,
assignment, migrations, predicted makespan) on 40 reference contexts."""

import pytest

from paper_2605_06374_b200 import policies as mp
from paper_2605_06374_b200 import scheduler as ms
from paper_2605_06374_b200.cluster import (FailureEvent, MicroBatch, ParallelismConfig,
                                           apply_failures, build_cluster)
from paper_2605_06374_b200.comm import CommSpec
from paper_2605_06374_b200.detector import ValidationResult
from paper_2605_06374_b200.workload import CostModel
from tests.golden_io import bits, load

pytestmark = pytest.mark.gpu


def test_tp_degrees_and_subgroups(cuda_device):
    u = load("scheduler_units")
    for g, f, k, exp in u["tp_degrees"]:
        assert sorted(ms.candidate_tp_degrees(g, f, k)) == exp
    for speeds, degs, chosen, standby in u["subgroup"]:
        table = dict(enumerate(speeds))
        if chosen is None:
            with pytest.raises(ms.GroupUnrecoverable):
                ms.select_tp_subgroup(table, set(degs))
            continue
        c, s = ms.select_tp_subgroup(table, set(degs))
        assert list(c) == chosen and list(s) == standby


def test_repartition_golden(cuda_device):
    for speeds, L, ml, exp in load("scheduler_units")["repartition"]:
        if exp is None:
            with pytest.raises(ValueError):
                ms.repartition_layers(speeds, L, ml)
        else:
            assert ms.repartition_layers(speeds, L, ml) == exp


def test_proportional_split_golden(cuda_device):
    for total, w, exp in load("scheduler_units")["proportional"]:
        if exp is None:
            with pytest.raises(ValueError):
                mp.proportional_split(total, w)
        else:
            assert mp.proportional_split(total, w) == exp


def _ctx_of(case):
    T, D, P = case["cfg"]["tp"], case["cfg"]["dp"], case["cfg"]["pp"]
    cfg = ParallelismConfig(T, D, P, case["cfg"]["schedule"], case["cfg"]["layer_partition"])
    st = build_cluster(case["nodes"], 8, cfg, 300.0 * 2**30, 25.0 * 2**30)
    evs = [FailureEvent(k, 0.0, device=d, severity=s) for k, d, s in case["events"]]
    st = apply_failures(st, evs, 0.0)
    mbs = [MicroBatch(i, tuple(d), n) for i, d, n in case["mbs"]]
    confirmed = None
    if case["confirmed"]:
        confirmed = ValidationResult(True, {tuple(k): 0.5 for k in case["confirmed"]}, {}, 3.0)
    return mp.PlanningContext(state=st, cfg=cfg, model=CostModel(2e-6, 5e-10),
                              micro_batches=mbs, comm=CommSpec(),
                              known_speeds={k: v for k, v in case["known"]},
                              new_fail_stop=["stop"] * case["new_fail_stop"],
                              confirmed=confirmed, delta=case["delta"],
                              capacity=case["capacity"])


@pytest.mark.parametrize("k", range(40))
def test_resihp_adapt_matches_reference(k, cuda_device):
    case = load("policies")["cases"][k]
    ctx = _ctx_of(case)
    if "error" in case:
        with pytest.raises((ms.StrandedWorkload, ms.GroupUnrecoverable)):
            mp.resihp_adapt(ctx)
        return
    plan = mp.resihp_adapt(ctx)
    exp = case["plan"]
    assert [[d, s, list(m), list(sb)] for (d, s), (m, sb) in sorted(plan.tp_subgroups.items())] \
        == exp["tp_subgroups"]
    assert [list(x) for x in plan.excluded_groups] == exp["excluded"]
    assert plan.layer_partition == exp["layer_partition"]
    assert plan.dp_assignment == exp["dp_assignment"]
    assert [[m.mb, m.stage, m.source, m.executor] for m in plan.migrations] == exp["migrations"]
    assert bits(plan.predicted_makespan_s) == bits(exp["predicted"])


def test_fail_slow_sheds_work_and_improves_makespan(cuda_device):
    """test_policies.py:135-191 behaviours through the GPU path."""
    from paper_2605_06374_b200.pipeline import simulate_iteration
    from paper_2605_06374_b200.workload import pack_sequences

    cfg = ParallelismConfig(4, 2, 2, layer_partition=[4, 4])
    st = build_cluster(2, 8, cfg, 300e9, 25e9)
    st = apply_failures(st, [FailureEvent("fail_slow_compute", 0.0, device=0, severity=0.4)],
                        0.0)
    mbs = pack_sequences([4096] * 16, 4096)
    ctx = mp.PlanningContext(state=st, cfg=cfg, model=CostModel(2e-6, 5e-10), micro_batches=mbs,
                             comm=CommSpec(), known_speeds={0: 0.4})
    ctx.confirmed = ValidationResult(True, {(0, 0): 0.4}, {}, 3.0)
    before = simulate_iteration(st, cfg, mbs, ctx.model, comm=ctx.comm).observed_time
    plan = mp.resihp_adapt(ctx)
    st2, cfg2 = ms.apply_plan(st, cfg, plan)
    after = simulate_iteration(st2, cfg2, mbs, ctx.model, plan, comm=ctx.comm).observed_time
    assert after < before
    assert mp.make_policy("resihp").plan(ctx) is not None
