"""Scheduler re-plan search over (DP, TP, PP) x partition x assignment (GPU).

``ReplanSearch`` turns a PlanningContext-like description (ClusterState with
the scheduler's known speeds, ParallelismConfig, micro-batches, CostModel,
CommSpec) into an rh_search (include/resihp_b200.h) and scores candidate
ranges on the GPU.  ``distributed_best`` shards the index range across the
ranks of a torch.distributed group and finishes with ONE collective: an
all-gather of each rank's 16-byte (score, index) pair, reduced identically
on every rank by the lexicographic (score, index) rule (NCCL has no MINLOC).
The candidate space and the score are defined in DESIGN.md §5.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cluster import FAIL_STOP, STANDBY, ClusterState, Device, ParallelismConfig
from .tables import SCHED_CODE
from .workload import cost_model_c, quad_loads


class SearchDesc(C.Structure):
    _fields_ = [
        ("n_devices", C.c_int32), ("devices_per_node", C.c_int32), ("device_speed", C.c_void_p),
        ("intra_bw", C.c_double), ("inter_bw", C.c_double), ("n_links", C.c_int32),
        ("link_nodes", C.c_void_p), ("link_factor", C.c_void_p), ("model", _lib.CostModelC),
        ("schedule", C.c_int32), ("token_budget", C.c_int32), ("n_micro_batches", C.c_int32),
        ("quad", C.c_void_p), ("total_layers", C.c_int32), ("min_layers", C.c_int32),
        ("capacity", C.c_int32), ("has_comm", C.c_int32), ("hidden_bytes_per_token", C.c_double),
        ("layer_bytes", C.c_double), ("p2p_optimized", C.c_int32), ("nominal_tp", C.c_int32),
        ("max_tp", C.c_int32),
        ("max_pp", C.c_int32), ("max_dp", C.c_int32), ("min_utilization", C.c_double),
        ("cur_tp", C.c_int32), ("cur_dp", C.c_int32), ("cur_pp", C.c_int32),
        ("cur_groups", C.c_void_p), ("cur_partition", C.c_void_p),
        ("group_rebuild_s", C.c_double), ("amortize_iterations", C.c_int32)]


class Candidate(C.Structure):
    _fields_ = [("index", C.c_int64), ("tp", C.c_int32), ("dp", C.c_int32), ("pp", C.c_int32),
                ("layout", C.c_int32), ("partition_variant", C.c_int32),
                ("count_variant", C.c_int32), ("feasible", C.c_int32)]


_SIGS = {
    "rh_search_create": ([C.c_void_p, C.POINTER(SearchDesc), C.POINTER(C.c_void_p), C.c_void_p],
                         C.c_int),
    "rh_search_destroy": ([C.c_void_p], C.c_int),
    "rh_search_set_workload": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "rh_search_size": ([C.c_void_p], C.c_int64),
    "rh_search_shard": ([C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                         C.POINTER(C.c_int64)], C.c_int),
    "rh_search_layouts": ([C.c_void_p], C.c_int32),
    "rh_search_eval": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                        C.c_void_p, C.c_void_p], C.c_int),
    "rh_search_decode": ([C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(Candidate), C.c_void_p,
                          C.c_void_p, C.c_void_p], C.c_int),
}
EXPORTED_SYMBOLS = tuple(_SIGS)


def _declare(lib):
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes, fn.restype = args, res
    return lib


@dataclass
class SearchInputs:
    """Host arrays + scalars of one rh_search_desc (kept alive by the owner)."""

    desc: SearchDesc
    arrays: dict


def build_desc(state: ClusterState, cfg: ParallelismConfig, micro_batches, model, comm=None, *,
               known_speeds: dict | None = None, capacity: int | None = None,
               min_layers: int = 1, max_tp: int | None = None, max_pp: int = 32,
               max_dp: int = 64, min_utilization: float = 0.9, group_rebuild_s: float = 2.0,
               amortize_iterations: int = 25, quad=None, defer_quad: bool = False) -> SearchInputs:
    """Descriptor of a re-plan (PlanningContext fields, policies.py:53-81).

    Device speeds are the scheduler's KNOWN view (PlanningContext.known_state,
    policies.py:73-81); fail-stop devices are not executable."""
    n = len(state.devices)
    speed = np.zeros(n, dtype=np.float64)
    devs = state.devices
    stopped = {dev.id for dev in devs if dev.status == FAIL_STOP}
    if known_speeds is None:
        ids = np.fromiter((dev.id for dev in devs), dtype=np.int64, count=n)
        sp = np.fromiter((dev.speed for dev in devs), dtype=np.float64, count=n)
        speed[ids] = np.minimum(1.0, sp)
    else:
        for dev in devs:
            speed[dev.id] = min(1.0, known_speeds.get(dev.id, 1.0))
    if stopped:
        speed[np.fromiter(stopped, dtype=np.int64, count=len(stopped))] = 0.0
    links = sorted(state.link_factors.items())
    link_nodes = np.array([[a, b] for (a, b), _ in links] or [[0, 0]], dtype=np.int32)
    link_factor = np.array([f for _, f in links] or [1.0], dtype=np.float64)
    N = micro_batches[0].token_budget
    if any(mb.token_budget != N for mb in micro_batches):
        raise ValueError("micro-batches must share one token budget")
    q = (np.zeros(1, np.int64) if defer_quad else
         np.asarray(quad if quad is not None else quad_loads(micro_batches), dtype=np.int64))
    T0, D0, P0 = cfg.tp, cfg.dp, cfg.pp
    groups = []
    full = True
    tg = state.tp_groups
    for d in range(D0):
        for s in range(P0):
            g = tuple(sorted(tg.get((d, s), ())))
            if len(g) != T0 or (stopped and not stopped.isdisjoint(g)):
                full = False
            groups.append(g)
    cur_groups = np.array([m for g in groups for m in g] if full else [-1], dtype=np.int32)
    cur_part = np.asarray(cfg.layer_partition or [0], dtype=np.int32)
    arrays = {"speed": speed, "link_nodes": link_nodes, "link_factor": link_factor, "quad": q,
              "cur_groups": cur_groups, "cur_part": cur_part}
    ptr = lambda a: a.ctypes.data
    desc = SearchDesc(
        n, state.devices_per_node, ptr(speed), float(state.intra_bw), float(state.inter_bw),
        len(links), ptr(link_nodes), ptr(link_factor), cost_model_c(model),
        SCHED_CODE[cfg.schedule], N, len(micro_batches), None if defer_quad else ptr(q),
        int(sum(cfg.layer_partition)),
        int(min_layers), int(capacity or 0), 1 if comm is not None else 0,
        float(comm.hidden_bytes_per_token) if comm is not None else 0.0,
        float(comm.layer_bytes) if comm is not None else 256.0 * 2**20,
        1 if (comm is None or comm.p2p_optimized) else 0, int(cfg.tp),
        int(max_tp or state.devices_per_node), int(max_pp), int(max_dp), float(min_utilization),
        T0 if full else 0, D0 if full else 0, P0, ptr(cur_groups) if full else None,
        ptr(cur_part), float(group_rebuild_s), int(amortize_iterations))
    return SearchInputs(desc, arrays)


@dataclass
class CandidatePlan:
    index: int
    tp: int
    dp: int
    pp: int
    partition: list[int]
    counts: list[int]
    groups: list[tuple[int, ...]]
    partition_variant: int
    count_variant: int
    feasible: bool

    def apply(self, state: ClusterState, schedule: str, nominal_tp: int):
        """(ClusterState, ParallelismConfig, dp_assignment) of this layout.

        The config keeps the NOMINAL TP degree: a T-wide group then runs at
        slowest * T / nominal_tp (cluster.py:155-169), which is how the
        reference prices TP subgroups and what makes layouts of different T
        comparable."""
        out = state.copy()
        out.tp_groups = {}
        members = set()
        for g, mem in enumerate(self.groups):
            out.tp_groups[(g // self.pp, g % self.pp)] = tuple(mem)
            members.update(mem)
        for dev in out.devices:
            if dev.status != FAIL_STOP and dev.id not in members:
                dev.status = STANDBY
            elif dev.id in members:
                dev.status = "fail_slow" if dev.speed < 1.0 else "healthy"
        cfg = ParallelismConfig(tp=nominal_tp, dp=self.dp, pp=self.pp, schedule=schedule,
                                layer_partition=list(self.partition))
        return out, cfg, list(self.counts)


class ReplanSearch:
    """A prepared re-plan on one GPU (owns the device-side rh_search)."""

    def __init__(self, inputs: SearchInputs, device=None):
        import torch

        self.inputs = inputs
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.lib = _declare(_lib.load_library())
        self.ctx = _lib.context(self.dev.index)
        h = C.c_void_p()
        with torch.cuda.device(self.dev):
            _lib.check(self.lib.rh_search_create(self.ctx, C.byref(inputs.desc), C.byref(h),
                                                 _lib.stream_handle()), "rh_search_create")
        self.handle = h.value
        self.size = int(self.lib.rh_search_size(self.handle))
        self.layouts = int(self.lib.rh_search_layouts(self.handle))
        self._best = torch.empty(1, dtype=torch.float64, device=self.dev)
        self._idx = torch.empty(1, dtype=torch.int64, device=self.dev)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.rh_search_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def set_workload(self, quad) -> None:
        """Quad loads of a search created with build_desc(defer_quad=True)
        (rh_search_set_workload)."""
        import torch

        q = np.ascontiguousarray(quad, dtype=np.int64)
        with torch.cuda.device(self.dev):
            _lib.check(self.lib.rh_search_set_workload(self.ctx, self.handle, q.ctypes.data,
                                                       _lib.stream_handle()),
                       "rh_search_set_workload")

    def shard(self, rank: int, world: int) -> tuple[int, int]:
        """Cost-balanced contiguous shard of the candidate range for `rank`
        (rh_search_shard: boundaries between (layout, partition) blocks)."""
        b, e = C.c_int64(), C.c_int64()
        _lib.check(self.lib.rh_search_shard(self.handle, int(rank), int(world), C.byref(b),
                                            C.byref(e)), "rh_search_shard")
        return int(b.value), int(e.value)

    def eval_async(self, begin: int = 0, end: int | None = None, scores=None):
        """Launch scoring of [begin, end); results stay on the device."""
        end = self.size if end is None else int(end)
        _lib.check(self.lib.rh_search_eval(self.ctx, self.handle, int(begin), end,
                                           self._best.data_ptr(), self._idx.data_ptr(),
                                           None if scores is None else scores.data_ptr(),
                                           _lib.stream_handle()), "rh_search_eval")
        return self._best, self._idx

    def best(self, begin: int = 0, end: int | None = None) -> tuple[float, int]:
        b, i = self.eval_async(begin, end)
        return float(b.item()), int(i.item())

    def scores(self, begin: int = 0, end: int | None = None) -> np.ndarray:
        import torch

        end = self.size if end is None else int(end)
        out = torch.empty(max(end - begin, 1), dtype=torch.float64, device=self.dev)
        self.eval_async(begin, end, out)
        return out.cpu().numpy()[:end - begin]

    def decode(self, index: int) -> CandidatePlan:
        c = Candidate()
        # upper bounds for the output arrays
        n_dev = self.inputs.desc.n_devices
        groups = np.zeros(n_dev + 1, dtype=np.int32)
        part = np.zeros(64, dtype=np.int32)
        cnt = np.zeros(128, dtype=np.int32)
        _lib.check(self.lib.rh_search_decode(self.ctx, self.handle, int(index), C.byref(c),
                                             groups.ctypes.data, part.ctypes.data,
                                             cnt.ctypes.data), "rh_search_decode")
        g = list(map(tuple, groups[:c.dp * c.pp * c.tp].reshape(-1, c.tp).tolist()))
        return CandidatePlan(int(c.index), c.tp, c.dp, c.pp, part[:c.pp].tolist(),
                             cnt[:c.dp].tolist(), g, c.partition_variant, c.count_variant,
                             bool(c.feasible))


def lexicographic_min(pairs) -> tuple[float, int]:
    """(score, index) min; infeasible (+inf / -1) entries lose."""
    best, bi = math.inf, -1
    for s, i in pairs:
        i = int(i)
        if i < 0:
            continue
        if bi < 0 or s < best or (s == best and i < bi):
            best, bi = float(s), i
    return best, bi


def shard_range(size: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [size*r/W, size*(r+1)/W) of the candidate index range."""
    return size * rank // world, size * (rank + 1) // world


def minloc_allreduce(score: float, index: int, group=None, device=None) -> tuple[float, int]:
    """One collective: all-gather of 16-byte (score bits, index) pairs, then
    the same lexicographic reduction on every rank (bit-exact fp64)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    mine = torch.tensor([np.float64(score).view(np.int64), int(index)], dtype=torch.int64,
                        device=dev)
    out = torch.empty(2 * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, mine, group=group)
    vals = out.cpu().numpy().reshape(world, 2)
    return lexicographic_min((vals[r, 0].view(np.float64), vals[r, 1]) for r in range(world))


def distributed_best(search: ReplanSearch, group=None, begin: int = 0,
                     end: int | None = None) -> tuple[float, int]:
    """Shard [begin, end) across the ranks of `group`, score locally on each
    rank's GPU, and combine with one NCCL all-gather."""
    import torch.distributed as dist

    end = search.size if end is None else end
    if not dist.is_available() or not dist.is_initialized():
        return search.best(begin, end)
    r, w = dist.get_rank(group), dist.get_world_size(group)
    if begin == 0 and end == search.size:
        a, b = search.shard(r, w)  # cost-balanced over the whole space
    else:
        a, b = shard_range(end - begin, r, w)
        a, b = begin + a, begin + b
    best, idx = search.eval_async(a, b)
    if dist.get_backend(group) == "nccl":
        import torch

        packed = torch.stack([best.view(torch.int64)[0], idx[0]])
        out = torch.empty(2 * w, dtype=torch.int64, device=packed.device)
        dist.all_gather_into_tensor(out, packed, group=group)
        vals = out.cpu().numpy().reshape(w, 2)
        return lexicographic_min((vals[k, 0].view(np.float64), vals[k, 1]) for k in range(w))
    return minloc_allreduce(float(best.item()), int(idx.item()), group)


class NcclComm:
    """An NCCL communicator made through the C ABI (rh_nccl_comm_create); the
    unique id travels over the existing process group (or any channel)."""

    def __init__(self, rank: int, world: int, device=None, group=None):
        import torch
        import torch.distributed as dist

        self.lib = _lib.load_library()
        self.world = world
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.ctx = _lib.context(self.dev.index)
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            _lib.check(self.lib.rh_nccl_unique_id(uid.ctypes.data), "rh_nccl_unique_id")
        t = torch.from_numpy(uid)
        if dist.get_backend(group) == "nccl":
            t = t.to(self.dev)
        dist.broadcast(t, src=0, group=group)
        uid = t.cpu().numpy().astype(np.uint8)
        h = C.c_void_p()
        _lib.check(self.lib.rh_nccl_comm_create(self.ctx, world, rank, uid.ctypes.data,
                                                C.byref(h)), "rh_nccl_comm_create")
        self.handle = h.value

    def minloc(self, best, idx, stream=None):
        """In place: the (score, index) device scalars of this rank -> the
        lexicographic minimum over all ranks (rh_minloc_allreduce)."""
        _lib.check(self.lib.rh_minloc_allreduce(self.ctx, self.handle, self.world,
                                                best.data_ptr(), idx.data_ptr(),
                                                _lib.stream_handle(stream)),
                   "rh_minloc_allreduce")
        return best, idx

    def close(self):
        if getattr(self, "handle", None):
            self.lib.rh_nccl_comm_destroy(self.handle)
            self.handle = None
