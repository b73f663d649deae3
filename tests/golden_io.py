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
