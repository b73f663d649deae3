"""Fixture JSON -> this package's objects (test infrastructure)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2605_06374_b200.cluster import (ClusterState, Device, MicroBatch,
                                           ParallelismConfig)
from paper_2605_06374_b200.comm import CommSpec
from paper_2605_06374_b200.workload import CostModel

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load(name: str):
    return json.loads((GOLDEN / f"{name}.json").read_text())


def state_of(j) -> ClusterState:
    devs = [Device(id=i, node_id=n, speed=s, status=st) for i, n, s, st in j["devices"]]
    return ClusterState(devices=devs, devices_per_node=j["devices_per_node"],
                        tp_groups={(d, s): tuple(m) for d, s, m in j["tp_groups"]},
                        intra_bw=j["intra_bw"], inter_bw=j["inter_bw"],
                        link_factors={(a, b): f for a, b, f in j["link_factors"]})


def cfg_of(j) -> ParallelismConfig:
    return ParallelismConfig(tp=j["tp"], dp=j["dp"], pp=j["pp"], schedule=j["schedule"],
                             layer_partition=list(j["layer_partition"]))


def model_of(j) -> CostModel:
    return CostModel(alpha=j["alpha"], beta=j["beta"], chunk_ratios=dict(j["chunk_ratios"]))


def mbs_of(j) -> list[MicroBatch]:
    return [MicroBatch(id=i, doc_lengths=tuple(d), token_budget=n) for i, d, n in j]


def comm_of(j):
    return None if j is None else CommSpec(hidden_bytes_per_token=j[0], layer_bytes=j[1],
                                           p2p_optimized=j[2])


def keyed(rows) -> dict:
    return {(a, b): v for a, b, v in rows}


def bits(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def search_problem(case):
    """(state, cfg, micro-batches, model, comm, SearchInputs) of a search fixture."""
    from paper_2605_06374_b200.cluster import FailureEvent, apply_failures, build_cluster
    from paper_2605_06374_b200.search import build_desc

    T, D, P = case["cfg"]
    cfg = ParallelismConfig(T, D, P, case["sched"], [8] * P)
    st = build_cluster(case["nodes"], case["dpn"], cfg, 300.0 * 2**30, 25.0 * 2**30)
    evs = []
    for kind, target, sev in case["events"]:
        if kind == "fail_slow_comm":
            evs.append(FailureEvent(kind, 0.0, link=tuple(target), severity=sev))
        else:
            evs.append(FailureEvent(kind, 0.0, device=target, severity=sev))
    st = apply_failures(st, evs, 0.0)
    mbs = [MicroBatch(i, tuple(d), case["N"]) for i, d in enumerate(case["mbs"])]
    model = CostModel(alpha=2e-6, beta=5e-10)
    comm = CommSpec() if case["comm"] else None
    quad = [sum(x * x for x in mb.doc_lengths) for mb in mbs]
    inputs = build_desc(st, cfg, mbs, model, comm, capacity=case["capacity"] or None, quad=quad,
                        min_utilization=0.6)
    return st, cfg, mbs, model, comm, inputs
