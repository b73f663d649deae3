"""Iteration predictor / simulator (mirror of resilsim/pipeline.py).

``simulate_iteration`` keeps the reference signature.  Canonical plans (no
migrated chunks) go through the fused wavefront kernel (rh_pipeline_batch);
plans with migrations build the chunk DAG on the host (its *structure* only)
and evaluate costs and the critical path on the GPU (rh_chunk_time +
rh_dag_critical_path).  ``critical_path`` on a user DAG is rh_dag_critical_path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cluster import (FAIL_STOP, SCHEDULE_1F1B, SCHEDULE_ZBH, IterationRecord,
                      dp_counts_or_even, split_micro_batches, validate_cluster)
from .tables import (DeviceSegments, HostSegments, allreduce_map, edge_cost_fn, pipe_shape,
                     segment_for_view, stage_speed_maps, used_link_ratios)
from .workload import (CHUNK_ALLREDUCE, CHUNK_B, CHUNK_BW, CHUNK_F, CHUNK_W, KIND_CODE,
                       chunk_times, cost_model_c, csr_of)

EDGE_DATA = "data"
EDGE_RESOURCE = "resource"


class SimulationError(RuntimeError):
    pass


class CycleError(SimulationError):
    pass


@dataclass
class ChunkVertex:
    kind: str
    micro_batch: int
    stage: int
    replica: int
    cost: float

    def label(self) -> str:
        if self.kind == CHUNK_ALLREDUCE:
            return f"AR(d{self.replica})"
        return f"{self.kind}(mb{self.micro_batch},s{self.stage},d{self.replica})"


@dataclass
class Edge:
    src: int
    dst: int
    weight: float
    kind: str


@dataclass
class ChunkDag:
    vertices: list[ChunkVertex]
    edges: list[Edge]
    chains: dict[tuple[int, int], list[int]] = field(default_factory=dict)


# ------------------------------------------------------------ chunk orders
def schedule_1f1b(num_stages: int, stage: int, mb_ids: list[int]) -> list[tuple[str, int]]:
    """pipeline.py:92-101: warmup w = min(P-1-s, M) forwards, F/BW pairs, BW drain."""
    m = len(mb_ids)
    w = min(num_stages - 1 - stage, m)
    seq = [(CHUNK_F, j) for j in mb_ids[:w]]
    for k in range(m - w):
        seq += [(CHUNK_F, mb_ids[w + k]), (CHUNK_BW, mb_ids[k])]
    seq += [(CHUNK_BW, j) for j in mb_ids[m - w:]]
    return seq


def schedule_zbh(num_stages: int, stage: int, mb_ids: list[int]) -> list[tuple[str, int]]:
    """pipeline.py:104-118: F warmup, F/B pairs, B/W drain, W tail."""
    m = len(mb_ids)
    w = min(num_stages - 1 - stage, m)
    seq = [(CHUNK_F, j) for j in mb_ids[:w]]
    for k in range(m - w):
        seq += [(CHUNK_F, mb_ids[w + k]), (CHUNK_B, mb_ids[k])]
    for t in range(w):
        seq += [(CHUNK_B, mb_ids[m - w + t]), (CHUNK_W, mb_ids[t])]
    seq += [(CHUNK_W, j) for j in mb_ids[w:]]
    return seq


def stage_sequence(cfg, stage: int, mb_ids: list[int]) -> list[tuple[str, int]]:
    if cfg.schedule == SCHEDULE_1F1B:
        return schedule_1f1b(cfg.pp, stage, mb_ids)
    if cfg.schedule == SCHEDULE_ZBH:
        return schedule_zbh(cfg.pp, stage, mb_ids)
    raise ValueError(f"unknown schedule {cfg.schedule!r}")


# ------------------------------------------------------------- DAG builder
def build_dag(cfg, micro_batches, model, speeds, p2p: float = 0.0, *, executors=None,
              dp_counts=None, edge_seconds=None, allreduce_seconds=None,
              stage_orders=None) -> ChunkDag:
    """pipeline.py:129-256: the chunk DAG (structure on host, costs on GPU)."""
    if not micro_batches:
        raise ValueError("cannot build a DAG for zero micro-batches")
    P, D = cfg.pp, cfg.dp
    if len(cfg.layer_partition) != P:
        raise ValueError("layer partition does not match stage count")
    owned = split_micro_batches(micro_batches, D, dp_counts)
    owner = {mb.id: d for d, mbs in enumerate(owned) for mb in mbs}
    by_id = {mb.id: mb for mb in micro_batches}
    executors = executors or {}

    def executor(j, s):
        return executors.get((j, s), owner[j])

    def speed_of(d, s):
        return speeds[(d, s)] if isinstance(speeds, dict) else float(speeds)

    own_ids = {(d, s): [] for d in range(D) for s in range(P)}
    foreign = {(d, s): [] for d in range(D) for s in range(P)}
    for mb in micro_batches:
        for s in range(P):
            d = executor(mb.id, s)
            (own_ids if d == owner[mb.id] else foreign)[(d, s)].append(mb.id)

    back = CHUNK_BW if cfg.schedule == SCHEDULE_1F1B else CHUNK_B
    verts: list[tuple[str, int, int, int]] = []
    edges: list[Edge] = []
    chains: dict[tuple[int, int], list[int]] = {}
    vid: dict[tuple[str, int, int], int] = {}
    for d in range(D):
        for s in range(P):
            ids = sorted(own_ids[(d, s)]) + sorted(foreign[(d, s)])
            chain: list[int] = []
            if ids:
                if stage_orders and (d, s) in stage_orders:
                    seq = stage_orders[(d, s)]
                    if {j for _, j in seq} != set(ids):
                        raise ValueError(f"stage order for {(d, s)} does not cover its chunks")
                else:
                    seq = stage_sequence(cfg, s, ids)
                for kind, j in seq:
                    v = len(verts)
                    verts.append((kind, j, s, d))
                    vid[(kind, j, s)] = v
                    if chain:
                        edges.append(Edge(chain[-1], v, 0.0, EDGE_RESOURCE))
                    chain.append(v)
            chains[(d, s)] = chain
    # chunk costs: one batched GPU evaluation of predict_chunk_time
    costs = chunk_times(model, [by_id[j] for _, j, _, _ in verts], [k for k, _, _, _ in verts],
                        [cfg.layer_partition[s] for _, _, s, _ in verts],
                        [speed_of(d, s) for _, _, s, d in verts])
    vertices = [ChunkVertex(k, j, s, d, float(c)) for (k, j, s, d), c in zip(verts, costs)]

    def hop(sf, df, st, dt):
        return edge_seconds(sf, df, st, dt) if edge_seconds is not None else float(p2p)

    for mb in micro_batches:
        j = mb.id
        for s in range(1, P):
            a, b = executor(j, s - 1), executor(j, s)
            edges.append(Edge(vid[(CHUNK_F, j, s - 1)], vid[(CHUNK_F, j, s)],
                              hop(s - 1, a, s, b), EDGE_DATA))
        for s in range(P - 1):
            a, b = executor(j, s + 1), executor(j, s)
            edges.append(Edge(vid[(back, j, s + 1)], vid[(back, j, s)],
                              hop(s + 1, a, s, b), EDGE_DATA))
        if back == CHUNK_B:
            for s in range(P):
                edges.append(Edge(vid[(CHUNK_B, j, s)], vid[(CHUNK_W, j, s)], 0.0, EDGE_DATA))
    if D > 1 and allreduce_seconds is not None:
        for d in range(D):
            c = (allreduce_seconds.get(d, 0.0) if isinstance(allreduce_seconds, dict)
                 else float(allreduce_seconds))
            v = len(vertices)
            vertices.append(ChunkVertex(CHUNK_ALLREDUCE, -1, -1, d, c))
            for s in range(P):
                if chains[(d, s)]:
                    edges.append(Edge(chains[(d, s)][-1], v, 0.0, EDGE_DATA))
    return ChunkDag(vertices=vertices, edges=edges, chains=chains)


# --------------------------------------------------------- critical path
def _find_cycle(dag: ChunkDag, blocked: set[int]) -> str:
    """Name one cycle among unprocessed vertices (error path only)."""
    succ = {v: [] for v in blocked}
    for e in dag.edges:
        if e.src in blocked and e.dst in blocked:
            succ[e.src].append(e.dst)
    alive = set(blocked)
    changed = True
    while changed:  # drop vertices that are only downstream of a cycle
        changed = False
        for v in sorted(alive):
            if not any(x in alive for x in succ[v]):
                alive.discard(v)
                changed = True
    node, order, pos = min(alive), [], {}
    while node not in pos:
        pos[node] = len(order)
        order.append(node)
        node = next(x for x in succ[node] if x in alive)
    cyc = order[pos[node]:] + [node]
    return " -> ".join(dag.vertices[i].label() for i in cyc)


def _run_dag(dag: ChunkDag, chain_keys=None, capacity=None):
    """rh_dag_critical_path on a ChunkDag -> (starts, makespan, chain sums, flags)."""
    nv = len(dag.vertices)
    src = np.fromiter((e.src for e in dag.edges), np.int64, len(dag.edges))
    dst = np.fromiter((e.dst for e in dag.edges), np.int64, len(dag.edges))
    w = np.fromiter((e.weight for e in dag.edges), np.float64, len(dag.edges))
    order = np.argsort(src, kind="stable")
    off = np.zeros(nv + 1, dtype=np.int32)
    np.cumsum(np.bincount(src, minlength=nv)[:nv] if nv else [], out=off[1:])
    cost = np.fromiter((v.cost for v in dag.vertices), np.float64, nv)
    kinds = np.fromiter((KIND_CODE.get(v.kind, 4) for v in dag.vertices), np.uint8, nv)
    chain_off = np.zeros(1, dtype=np.int32)
    if chain_keys:
        bounds = [0]
        for k in chain_keys:
            ch = dag.chains[k]
            if ch and (ch[0] != bounds[-1] or ch[-1] != ch[0] + len(ch) - 1):
                raise ValueError("chains must be contiguous vertex ranges in creation order")
            bounds.append(bounds[-1] + len(ch))
        chain_off = np.asarray(bounds, dtype=np.int32)

    # host arrays through rh_dag_critical_path_host: one copy in, one copy out
    def h(a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        return a if a.size else np.zeros(1, dtype)

    h_cost, h_off = h(cost, np.float64), h(off, np.int32)
    h_dst, h_w = h(dst[order], np.int32), h(w[order], np.float64)
    h_kind, h_chain = h(kinds, np.uint8), h(chain_off, np.int32)
    n_chains = len(chain_keys) if chain_keys else 0
    starts = np.zeros(max(nv, 1), dtype=np.float64)
    ms = np.zeros(1, dtype=np.float64)
    sums = np.zeros(max(n_chains, 1), dtype=np.float64)
    flags = np.zeros(2, dtype=np.int32)
    lib = _lib.load_library()
    _lib.check(lib.rh_dag_critical_path_host(
        _lib.context(), nv, h_cost.ctypes.data, h_off.ctypes.data, h_dst.ctypes.data,
        h_w.ctypes.data, n_chains, h_chain.ctypes.data, h_kind.ctypes.data, int(capacity or 0),
        starts.ctypes.data, ms.ctypes.data, sums.ctypes.data, flags.ctypes.data),
        "rh_dag_critical_path_host")
    return starts[:nv], float(ms[0]), sums[:n_chains], flags


def critical_path(dag: ChunkDag) -> tuple[list[float], float]:
    """pipeline.py:259-292 (Eq. 2) on the GPU."""
    starts, makespan, _, flags = _run_dag(dag)
    if flags[0]:
        blocked = _unprocessed(dag)
        raise CycleError("dependency cycle: " + _find_cycle(dag, blocked))
    return [float(x) for x in starts], makespan


def _unprocessed(dag: ChunkDag) -> set[int]:
    indeg = [0] * len(dag.vertices)
    succ = [[] for _ in dag.vertices]
    for e in dag.edges:
        indeg[e.dst] += 1
        succ[e.src].append(e.dst)
    queue = [v for v, k in enumerate(indeg) if k == 0]
    for u in queue:
        for v in succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                queue.append(v)
    return {v for v, k in enumerate(indeg) if k > 0}


# ------------------------------------------------------------- simulate
def _completeness(state, cfg, micro_batches, owner, executors, speeds) -> None:
    for mb in micro_batches:
        for s in range(cfg.pp):
            d = executors.get((mb.id, s), owner[mb.id])
            if speeds[(d, s)] <= 0.0:
                raise SimulationError(
                    f"execution completeness violated: chunk (mb {mb.id}, stage {s}) "
                    f"assigned to stopped stage (d{d}, s{s})")


def _busy_idle(state, stage_cost: dict, observed: float):
    """pipeline.py:455-474: own-shard compute is busy, the rest is idle."""
    busy = {dev.id: 0.0 for dev in state.devices if dev.status != FAIL_STOP}
    for (d, s), total in stage_cost.items():
        members = [m for m in state.tp_groups.get((d, s), ())
                   if state.devices[m].status != FAIL_STOP]
        if not members:
            continue
        slowest = min(state.devices[m].speed for m in members)
        for m in members:
            if m in busy:
                busy[m] += total * slowest / state.devices[m].speed
    return busy, {m: observed - b for m, b in busy.items()}


def _capacity_error(key):
    return SimulationError(f"activation footprint exceeds capacity at {key}")


def simulate_iteration(state, cfg, micro_batches, model, plan=None, *, comm=None,
                       iteration: int = 0, capacity: int | None = None) -> IterationRecord:
    """pipeline.py:375-488 — actual and healthy-reference critical paths."""
    bad = validate_cluster(state, cfg, check_capacity=False)
    if bad:
        raise SimulationError("invalid cluster: " + "; ".join(bad))
    dp_counts = getattr(plan, "dp_assignment", None) if plan is not None else None
    executors = {}
    if plan is not None:
        for m in getattr(plan, "migrations", []) or []:
            executors[(m.mb, m.stage)] = m.executor
    owned = split_micro_batches(micro_batches, cfg.dp, dp_counts)
    owner = {mb.id: d for d, mbs in enumerate(owned) for mb in mbs}
    speeds, healthy = stage_speed_maps(state, cfg)
    _completeness(state, cfg, micro_batches, owner, executors, speeds)
    orders = getattr(plan, "stage_orders", None) if plan is not None else None
    if not executors:
        orders = None
    budgets = {mb.token_budget for mb in micro_batches}
    if executors or len(budgets) != 1 or any(x < 0 for x in cfg.layer_partition) or \
            (capacity is not None and min(cfg.layer_partition, default=1) == 0):
        return _simulate_general(state, cfg, micro_batches, model, executors, dp_counts,
                                 orders, owner, speeds, healthy, comm, iteration, capacity)
    return _simulate_canonical(state, cfg, micro_batches, model, dp_counts, comm, iteration,
                               capacity)


def _stage_dicts(cfg, counts, sc_actual, sc_ref):
    stage_cost, stage_ref = {}, {}
    for d in range(cfg.dp):
        if counts[d] == 0:
            continue
        for s in range(cfg.pp):
            stage_cost[(d, s)] = float(sc_actual[d * cfg.pp + s])
            stage_ref[(d, s)] = float(sc_ref[d * cfg.pp + s])
    return stage_cost, stage_ref


def _simulate_canonical(state, cfg, micro_batches, model, dp_counts, comm, iteration, capacity):
    M = len(micro_batches)
    N = micro_batches[0].token_budget
    counts = dp_counts_or_even(M, cfg.dp, dp_counts)
    seg_a = segment_for_view(state, cfg, M, N, comm=comm, dp_counts=counts)
    seg_h = segment_for_view(state, cfg, M, N, comm=comm, dp_counts=counts, healthy=True,
                             clean_links=True)
    # the two views as a 2-iteration trace, host arrays through
    # rh_pipeline_batch_host (one copy in, one copy out)
    segs = HostSegments([seg_a, seg_h])
    off, docs = csr_of(micro_batches)
    n_docs = int(off[-1])
    off2 = np.ascontiguousarray(np.concatenate([off, off[1:] + n_docs]), dtype=np.int32)
    docs2 = np.ascontiguousarray(np.concatenate([docs, docs]) if n_docs else np.zeros(1),
                                 dtype=np.int32)
    seg2 = np.array([0, 1], dtype=np.int32)
    tr = _lib.Trace(2, seg2.ctypes.data, off2.ctypes.data, docs2.ctypes.data, None, None)
    ms_h = np.zeros(2, dtype=np.float64)
    st_h = np.zeros(2, dtype=np.uint8)
    sc_h = np.zeros(2 * cfg.dp * cfg.pp, dtype=np.float64)
    out = _lib.PassOut(ms_h.ctypes.data, st_h.ctypes.data, sc_h.ctypes.data, None, None)
    shape = pipe_shape(cfg, M, N, capacity=capacity, has_allreduce=comm is not None,
                       max_mb=segs.max_mb)
    lib = _lib.load_library()
    _lib.check(lib.rh_pipeline_batch_host(_lib.context(), _lib.C.byref(shape),
                                          _lib.C.byref(cost_model_c(model)),
                                          _lib.C.byref(segs.c), _lib.C.byref(tr),
                                          _lib.C.byref(out)), "rh_pipeline_batch_host")
    if st_h[0] & _lib.RH_IT_STOPPED:
        raise SimulationError("execution completeness violated")
    if st_h[0] & _lib.RH_IT_CAPACITY:
        raise SimulationError(f"activation footprint exceeds capacity {capacity}")
    observed, predicted = float(ms_h[0]), float(ms_h[1])
    G = cfg.dp * cfg.pp
    stage_cost, stage_ref = _stage_dicts(cfg, counts, sc_h[:G], sc_h[G:])
    busy, idle = _busy_idle(state, stage_cost, observed)
    return IterationRecord(
        iteration=iteration, observed_time=observed, predicted_healthy_time=predicted,
        per_device_busy=busy, per_device_idle=idle, stage_cost=stage_cost,
        stage_cost_reference=stage_ref,
        link_ratio=used_link_ratios(state, cfg) if comm is not None else {}, migrations=0)


def simulate_iteration_batch(items):
    """simulate_iteration for many independent (state, cfg, micro_batches,
    model, plan, comm, iteration, capacity) items: every canonical item (no
    migrations) with the same pipeline shape, cost model and capacity shares
    ONE rh_pipeline_batch launch (each item = two trace iterations: its
    actual and healthy views); migration plans take the general-DAG path one
    by one.  Returns a list of IterationRecord, or the exception an item
    raises (SimulationError / ValueError) in its place."""
    import torch

    out = [None] * len(items)
    groups = {}
    for k, (state, cfg, mbs, model, plan, comm, iteration, capacity) in enumerate(items):
        try:
            bad = validate_cluster(state, cfg, check_capacity=False)
            if bad:
                raise SimulationError("invalid cluster: " + "; ".join(bad))
            executors = {(m.mb, m.stage): m.executor
                         for m in (getattr(plan, "migrations", None) or [])} if plan else {}
            budgets = {mb.token_budget for mb in mbs}
            if executors or len(budgets) != 1 or any(x < 0 for x in cfg.layer_partition) or \
                    (capacity is not None and min(cfg.layer_partition, default=1) == 0):
                out[k] = simulate_iteration(state, cfg, mbs, model, plan, comm=comm,
                                            iteration=iteration, capacity=capacity)
                continue
            dp_counts = getattr(plan, "dp_assignment", None) if plan is not None else None
            owned = split_micro_batches(mbs, cfg.dp, dp_counts)
            owner = {mb.id: d for d, ms in enumerate(owned) for mb in ms}
            speeds, _ = stage_speed_maps(state, cfg)
            _completeness(state, cfg, mbs, owner, {}, speeds)
            key = (cfg.pp, cfg.dp, cfg.tp, cfg.schedule, len(mbs), mbs[0].token_budget,
                   model.alpha, model.beta, tuple(sorted(model.chunk_ratios.items())),
                   comm is not None, capacity)
            groups.setdefault(key, []).append(k)
        except (SimulationError, ValueError) as exc:
            out[k] = exc
    dev = torch.device("cuda", torch.cuda.current_device())
    lib = _lib.load_library()
    for key, ks in groups.items():
        segs, offs, docs, counts_l = [], [], [], []
        base = 0
        for k in ks:
            state, cfg, mbs, model, plan, comm, iteration, capacity = items[k]
            M, N = len(mbs), mbs[0].token_budget
            counts = dp_counts_or_even(M, cfg.dp, getattr(plan, "dp_assignment", None)
                                       if plan is not None else None)
            counts_l.append(counts)
            segs.append(segment_for_view(state, cfg, M, N, comm=comm, dp_counts=counts))
            segs.append(segment_for_view(state, cfg, M, N, comm=comm, dp_counts=counts,
                                         healthy=True, clean_links=True))
            off, d = csr_of(mbs)
            n_docs = int(off[-1])
            offs += [off[:-1] + base, off[:-1] + base + n_docs]
            docs += [d, d]
            base += 2 * n_docs
        offs.append(np.array([base]))
        state, cfg, mbs, model, plan, comm, iteration, capacity = items[ks[0]]
        M, N, G = len(mbs), mbs[0].token_budget, cfg.dp * cfg.pp
        n = 2 * len(ks)
        dsegs = DeviceSegments(segs, dev)
        t_off = torch.from_numpy(np.concatenate(offs).astype(np.int32)).to(dev)
        t_doc = torch.from_numpy(np.concatenate(docs).astype(np.int32)).to(dev)
        t_seg = torch.arange(n, dtype=torch.int32, device=dev)
        tr = _lib.Trace(n, t_seg.data_ptr(), t_off.data_ptr(), t_doc.data_ptr(), None, None)
        ms = torch.empty(n, dtype=torch.float64, device=dev)
        st = torch.empty(n, dtype=torch.uint8, device=dev)
        sc = torch.empty(n * G, dtype=torch.float64, device=dev)
        res = _lib.PassOut(ms.data_ptr(), st.data_ptr(), sc.data_ptr(), None, None)
        shape = pipe_shape(cfg, M, N, capacity=capacity, has_allreduce=comm is not None,
                           max_mb=dsegs.max_mb)
        _lib.check(lib.rh_pipeline_batch(_lib.context(), _lib.C.byref(shape),
                                         _lib.C.byref(cost_model_c(model)),
                                         _lib.C.byref(dsegs.c), _lib.C.byref(tr),
                                         _lib.C.byref(res), _lib.stream_handle()),
                   "rh_pipeline_batch")
        ms_h, st_h, sc_h = ms.cpu().numpy(), st.cpu().numpy(), sc.cpu().numpy().reshape(n, G)
        for q, k in enumerate(ks):
            state, cfg, mbs, model, plan, comm, iteration, capacity = items[k]
            if st_h[2 * q] & _lib.RH_IT_STOPPED:
                out[k] = SimulationError("execution completeness violated")
                continue
            if st_h[2 * q] & _lib.RH_IT_CAPACITY:
                out[k] = SimulationError(f"activation footprint exceeds capacity {capacity}")
                continue
            observed, predicted = float(ms_h[2 * q]), float(ms_h[2 * q + 1])
            stage_cost, stage_ref = _stage_dicts(cfg, counts_l[q], sc_h[2 * q], sc_h[2 * q + 1])
            busy, idle = _busy_idle(state, stage_cost, observed)
            out[k] = IterationRecord(
                iteration=iteration, observed_time=observed, predicted_healthy_time=predicted,
                per_device_busy=busy, per_device_idle=idle, stage_cost=stage_cost,
                stage_cost_reference=stage_ref,
                link_ratio=used_link_ratios(state, cfg) if comm is not None else {}, migrations=0)
    return out


def _simulate_general(state, cfg, micro_batches, model, executors, dp_counts, orders, owner,
                      speeds, healthy, comm, iteration, capacity):
    from .comm import LinkModel

    if comm is not None:
        links = LinkModel.from_cluster(state)
        clean = LinkModel(intra_bw=state.intra_bw, inter_bw=state.inter_bw)
        N = micro_batches[0].token_budget
        e_act, e_ok = edge_cost_fn(state, cfg, comm, links, N), edge_cost_fn(state, cfg, comm,
                                                                              clean, N)
        ar_act, ar_ok = allreduce_map(state, cfg, comm, links), allreduce_map(state, cfg, comm,
                                                                              clean)
    else:
        e_act = e_ok = ar_act = ar_ok = None
    dag = build_dag(cfg, micro_batches, model, speeds, executors=executors,
                    dp_counts=dp_counts, edge_seconds=e_act, allreduce_seconds=ar_act,
                    stage_orders=orders)
    ref = build_dag(cfg, micro_batches, model, healthy, executors=executors,
                    dp_counts=dp_counts, edge_seconds=e_ok, allreduce_seconds=ar_ok,
                    stage_orders=orders)
    keys = [k for k in dag.chains if dag.chains[k]]
    starts, observed, sums, flags = _run_dag(dag, keys, capacity)
    if flags[0]:
        raise CycleError("dependency cycle: " + _find_cycle(dag, _unprocessed(dag)))
    if flags[1]:
        raise SimulationError(f"activation footprint exceeds capacity {capacity}")
    _, predicted, sums_ref, flags_ref = _run_dag(ref, keys, None)
    if flags_ref[0]:
        raise CycleError("dependency cycle: " + _find_cycle(ref, _unprocessed(ref)))
    stage_cost = {k: float(v) for k, v in zip(keys, sums)}
    stage_ref = {k: float(v) for k, v in zip(keys, sums_ref)}
    busy, idle = _busy_idle(state, stage_cost, observed)
    return IterationRecord(
        iteration=iteration, observed_time=observed, predicted_healthy_time=predicted,
        per_device_busy=busy, per_device_idle=idle, stage_cost=stage_cost,
        stage_cost_reference=stage_ref,
        link_ratio=used_link_ratios(state, cfg) if comm is not None else {},
        migrations=sum(1 for (j, s), d in executors.items() if d != owner[j]))
