"""Host-side packing of the predictor's inputs into the C-ABI layout.

A *segment* is a span of iterations with one layout and one view of device
speeds.  ``segment_for_view`` turns the reference's objects
(ClusterState, ParallelismConfig, CommSpec, plan counts) into the per-segment
tables of include/resihp_b200.h: effective stage speeds, directed hop
weights, all-reduce costs, micro-batch ownership and the exercised-link
ratios.  The arithmetic mirrors pipeline.py:323-372 and comm.py:61-107
operation for operation; it is O(D*P) per segment.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .cluster import FAIL_STOP, SCHEDULE_1F1B, SCHEDULE_ZBH, dp_counts_or_even
from .comm import LinkModel, allreduce_cost, p2p_cost

SCHED_CODE = {SCHEDULE_1F1B: 0, SCHEDULE_ZBH: 1}


def stage_speed_maps(state, cfg):
    """pipeline.py:323-333 -> (actual, healthy) speed per (replica, stage)."""
    actual, healthy = {}, {}
    for d in range(cfg.dp):
        for s in range(cfg.pp):
            actual[(d, s)] = state.effective_stage_speed(d, s, cfg.tp)
            members = state.tp_groups.get((d, s), ())
            healthy[(d, s)] = len(members) / cfg.tp if members else 0.0
    return actual, healthy


def edge_cost_fn(state, cfg, comm, links: LinkModel, token_budget: int):
    """pipeline.py:336-353: seconds on a stage-boundary data edge."""
    nbytes = comm.boundary_tensor_bytes(token_budget)

    def cost(s_from: int, d_from: int, s_to: int, d_to: int) -> float:
        a = state.group_node(d_from, s_from)
        b = state.group_node(d_to, s_to)
        if a is None or b is None:
            return 0.0
        if a == b:
            return nbytes / links.intra_bw
        seconds, _ = p2p_cost(nbytes, len(state.tp_groups[(d_from, s_from)]),
                              len(state.tp_groups[(d_to, s_to)]), comm.p2p_optimized, links,
                              nodes=(a, b))
        return seconds

    return cost


def allreduce_map(state, cfg, comm, links: LinkModel) -> dict[int, float]:
    """pipeline.py:356-372: every replica waits for the slowest stage ring."""
    worst = 0.0
    for s in range(cfg.pp):
        nodes = tuple(n for n in (state.group_node(d, s) for d in range(cfg.dp)) if n is not None)
        worst = max(worst, allreduce_cost(cfg.layer_partition[s] * comm.layer_bytes, cfg.dp,
                                          links, nodes))
    return {d: worst for d in range(cfg.dp)}


def used_link_ratios(state, cfg) -> dict[tuple[int, int], float]:
    """pipeline.py:491-513: measured/expected ratio of every exercised link."""
    used: set[tuple[int, int]] = set()
    for d in range(cfg.dp):
        for s in range(cfg.pp - 1):
            a, b = state.group_node(d, s), state.group_node(d, s + 1)
            if a is not None and b is not None and a != b:
                used.add((min(a, b), max(a, b)))
    if cfg.dp > 1:
        for s in range(cfg.pp):
            ring = [n for n in (state.group_node(d, s) for d in range(cfg.dp)) if n is not None]
            for a, b in zip(ring, ring[1:] + ring[:1]):
                if a != b:
                    used.add((min(a, b), max(a, b)))
    return {k: 1.0 / state.link_factors.get(k, 1.0) for k in sorted(used)}


@dataclass
class Segment:
    """One segment's tables (numpy, C-ABI layout)."""

    layers: np.ndarray      # int32 [P]
    mb_start: np.ndarray    # int32 [D+1]
    speed: np.ndarray       # f64 [D*P]
    hop_fwd: np.ndarray     # f64 [D*P]
    hop_bwd: np.ndarray     # f64 [D*P]
    allreduce: np.ndarray   # f64 [D]
    link_ratio: np.ndarray  # f64 [n_links]


def segment_from_tables(cfg, speeds: dict, counts: list[int], edge=None, ar=None,
                        link_ratio=None) -> Segment:
    D, P = cfg.dp, cfg.pp
    speed = np.array([speeds[(d, s)] for d in range(D) for s in range(P)], dtype=np.float64)
    hf = np.zeros(D * P)
    hb = np.zeros(D * P)
    if edge is not None:
        for d in range(D):
            for s in range(P - 1):
                hf[d * P + s] = edge(s, d, s + 1, d)
                hb[d * P + s] = edge(s + 1, d, s, d)
    arr = np.array([ar.get(d, 0.0) if ar else 0.0 for d in range(D)], dtype=np.float64)
    start = np.zeros(D + 1, dtype=np.int32)
    np.cumsum(counts, out=start[1:])
    lr = np.array(list((link_ratio or {}).values()), dtype=np.float64)
    return Segment(np.asarray(cfg.layer_partition, dtype=np.int32), start, speed, hf, hb, arr, lr)


def segment_for_view(state, cfg, n_micro_batches: int, token_budget: int, *, comm=None,
                     dp_counts=None, healthy: bool = False, clean_links: bool = False,
                     with_links: bool = False) -> Segment:
    """Tables of one view of ``state`` (simulate_iteration, pipeline.py:405-427).

    healthy=True uses the healthy speeds |group|/tp; clean_links=True costs the
    comm edges on an undegraded LinkModel (the reference's ``clean``)."""
    counts = dp_counts_or_even(n_micro_batches, cfg.dp, dp_counts)
    actual, ok = stage_speed_maps(state, cfg)
    speeds = ok if healthy else actual
    edge = ar = None
    if comm is not None:
        links = (LinkModel(intra_bw=state.intra_bw, inter_bw=state.inter_bw) if clean_links
                 else LinkModel.from_cluster(state))
        edge = edge_cost_fn(state, cfg, comm, links, token_budget)
        ar = allreduce_map(state, cfg, comm, links)
    lr = used_link_ratios(state, cfg) if (with_links and comm is not None) else None
    return segment_from_tables(cfg, speeds, counts, edge, ar, lr)


class DeviceSegments:
    """Segment tables stacked and resident on the GPU (keeps tensors alive)."""

    def __init__(self, segments: list[Segment], device):
        import torch

        from . import _lib

        def cat(name, dtype):
            arrs = [getattr(s, name) for s in segments]
            a = np.concatenate(arrs).astype(dtype) if arrs else np.zeros(0, dtype)
            if a.size == 0:
                a = np.zeros(1, dtype)
            return torch.from_numpy(np.ascontiguousarray(a)).to(device)

        self.layers = cat("layers", np.int32)
        self.mb_start = cat("mb_start", np.int32)
        self.speed = cat("speed", np.float64)
        self.hop_fwd = cat("hop_fwd", np.float64)
        self.hop_bwd = cat("hop_bwd", np.float64)
        self.allreduce = cat("allreduce", np.float64)
        n_links = [len(s.link_ratio) for s in segments]
        off = np.zeros(len(segments) + 1, dtype=np.int32)
        np.cumsum(n_links, out=off[1:])
        self.link_off = torch.from_numpy(off).to(device)
        self.link_ratio = cat("link_ratio", np.float64)
        # per-segment maximum ratio: the kernels' link test is one compare
        lmax = np.array([float(np.max(s.link_ratio)) if len(s.link_ratio) else 0.0
                         for s in segments] or [0.0], dtype=np.float64)
        self.link_max = torch.from_numpy(lmax).to(device)
        self.n_seg = len(segments)
        self.max_mb = int(max((np.diff(s.mb_start).max() for s in segments), default=0))
        self.c = _lib.Segments(self.n_seg, self.layers.data_ptr(), self.mb_start.data_ptr(),
                               self.speed.data_ptr(), self.hop_fwd.data_ptr(),
                               self.hop_bwd.data_ptr(), self.allreduce.data_ptr(),
                               self.link_off.data_ptr(), self.link_ratio.data_ptr(),
                               self.link_max.data_ptr())


class HostSegments:
    """Segment tables stacked in host memory, C-ABI layout (the per-call
    rh_pipeline_batch_host path; keeps the arrays alive)."""

    def __init__(self, segments: list[Segment]):
        from . import _lib

        def cat(name, dtype):
            arrs = [getattr(s, name) for s in segments]
            a = np.concatenate(arrs).astype(dtype) if arrs else np.zeros(0, dtype)
            return np.ascontiguousarray(a if a.size else np.zeros(1, dtype))

        self.layers = cat("layers", np.int32)
        self.mb_start = cat("mb_start", np.int32)
        self.speed = cat("speed", np.float64)
        self.hop_fwd = cat("hop_fwd", np.float64)
        self.hop_bwd = cat("hop_bwd", np.float64)
        self.allreduce = cat("allreduce", np.float64)
        off = np.zeros(len(segments) + 1, dtype=np.int32)
        np.cumsum([len(s.link_ratio) for s in segments], out=off[1:])
        self.link_off = off
        self.link_ratio = cat("link_ratio", np.float64)
        self.link_max = np.array([float(np.max(s.link_ratio)) if len(s.link_ratio) else 0.0
                                  for s in segments] or [0.0], dtype=np.float64)
        self.n_seg = len(segments)
        self.max_mb = int(max((np.diff(s.mb_start).max() for s in segments), default=0))
        p = lambda a: a.ctypes.data
        self.c = _lib.Segments(self.n_seg, p(self.layers), p(self.mb_start), p(self.speed),
                               p(self.hop_fwd), p(self.hop_bwd), p(self.allreduce),
                               p(self.link_off), p(self.link_ratio), p(self.link_max))


def pipe_shape(cfg, n_micro_batches: int, token_budget: int, *, capacity=None,
               has_allreduce: bool = False, max_mb: int = 0):
    from . import _lib

    if cfg.schedule not in SCHED_CODE:
        raise ValueError(f"unknown schedule {cfg.schedule!r}")
    return _lib.PipeShape(cfg.pp, cfg.dp, cfg.tp, SCHED_CODE[cfg.schedule], n_micro_batches,
                          token_budget, int(capacity or 0), 1 if has_allreduce else 0,
                          int(max_mb))
