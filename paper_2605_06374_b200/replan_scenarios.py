"""Re-plan problems of BASELINE.json configs[2..4] (synthetic, seeded).

C3  256 GPUs  (32 nodes x 8), Llama-70B (80 layers), current TP4 x DP4 x PP16,
    64 micro-batches: one fail-stop, two fail-slow devices.
C4  1024 GPUs (128 nodes x 8), 80 layers, current TP8 x DP16 x PP8,
    128 micro-batches: one fail-stop, four fail-slow devices, one slow link.
C5  4096 GPUs (512 nodes x 8), 80 layers, current TP8 x DP32 x PP16: the
    "10^5-sequence workload-to-replica assignment" of BASELINE configs[4] --
    100,000 lognormal(7.2, 0.8) sequences FFD-packed (workload.py:52-80) into
    512 micro-batches of N tokens (the smallest multiple of 64 at or above
    total / 512 with which FFD fits every sequence into the 512), one
    fail-stop, eight fail-slow
    devices, two slow links.
C3 / C4 draw documents like harness._DocSource (harness.py:235-263):
lognormal(7.2, 0.8) until the iteration's M x 4096 tokens are covered, FFD,
first M bins.  All use alpha=2e-6, beta=5e-10, default CommSpec, capacity P+2
(harness.py:118-120).

``replan_from_sequences`` is the timed C5 entry point: raw sequence lengths
and the cluster's known state in, the decoded plan and every sequence's
replica out (pack, quad loads, descriptor, GPU search, collective, decode).
"""

from __future__ import annotations

import numpy as np

from .cluster import FailureEvent, MicroBatch, ParallelismConfig, apply_failures, build_cluster
from .comm import CommSpec
from .search import build_desc
from .trace import pack_ffd, synth_iterations
from .workload import CostModel

GIB = float(2**30)

# min_utilization / max_dp size the candidate spaces to the configs' scale:
# C3 1.79e6 (exhaustive), C4 1.18e6 (~1e6), C5 ~1e7 candidates
SPECS = {
    "C3": dict(T=4, D=4, P=16, M=64, slow=2, links=0, min_utilization=0.95, max_dp=64),
    "C4": dict(T=8, D=16, P=8, M=128, slow=4, links=1, min_utilization=0.987, max_dp=32),
    "C5": dict(T=8, D=32, P=16, M=512, slow=8, links=2, min_utilization=0.985, max_dp=64,
               n_sequences=100_000),
}


def sequence_workload(n_sequences: int, M: int, seed: int = 0, mean: float = 7.2,
                      sigma: float = 0.8) -> tuple[np.ndarray, int]:
    """n_sequences lognormal lengths (rounded half-to-even, >= 1) and the
    micro-batch token budget N that packs them into M micro-batches."""
    rng = np.random.default_rng([seed, 9])
    docs = np.maximum(1, np.rint(rng.lognormal(mean, sigma, n_sequences))).astype(np.int64)
    # the smallest multiple of 64 tokens at or above the volume bound for
    # which FFD places every sequence within the M micro-batches
    N = -(-int(-(-int(docs.sum()) // M)) // 64) * 64
    while True:
        d = np.minimum(docs, N).astype(np.int32)
        off, _ = pack_ffd(d, N)
        if len(off) - 1 <= M:
            return d, N
        N += 64


def _state(sp, layers, seed):
    T, D, P = sp["T"], sp["D"], sp["P"]
    n_dev = T * D * P
    nodes = n_dev // 8
    part = [layers // P + (1 if i < layers % P else 0) for i in range(P)]
    cfg = ParallelismConfig(T, D, P, "1f1b", part)
    st = build_cluster(nodes, 8, cfg, 300.0 * GIB, 25.0 * GIB)
    rng = np.random.default_rng([seed, 5])
    devs = rng.choice(n_dev, size=sp["slow"] + 1, replace=False)
    evs = [FailureEvent("fail_stop", 0.0, device=int(devs[0]))]
    evs += [FailureEvent("fail_slow_compute", 0.0, device=int(x),
                         severity=float(rng.uniform(0.3, 0.7))) for x in devs[1:]]
    for k in range(sp["links"]):
        a = int(rng.integers(0, nodes - 1))
        evs.append(FailureEvent("fail_slow_comm", 0.0, link=(a, a + 1), severity=0.5))
    return apply_failures(st, evs, 0.0), cfg


def pack_workload(docs: np.ndarray, N: int, M: int):
    """FFD-pack sequences into the first M micro-batches of N tokens ->
    (mb_off[M+1], packed lengths incl. padding, quad loads[M], bin of every
    packed entry)."""
    from . import _lib

    lib = _lib.load_library()
    lengths = np.ascontiguousarray(docs, dtype=np.int32)
    n = len(lengths)
    nb, ne = _lib.C.c_int64(), _lib.C.c_int64()
    off = np.empty(n + 2, dtype=np.int32)
    packed = np.empty(2 * n + 1, dtype=np.int32)
    quad = np.empty(max(M, 1), dtype=np.int64)
    _lib.check(lib.rh_pack_sequences_quad(n, lengths.ctypes.data, int(N), int(M), off.ctypes.data,
                                          packed.ctypes.data, quad.ctypes.data,
                                          _lib.C.byref(nb), _lib.C.byref(ne)),
               "rh_pack_sequences_quad")
    if nb.value < M:
        raise ValueError(f"workload fills only {nb.value} of {M} micro-batches")
    return off[:nb.value + 1], packed[:ne.value], quad[:M]


def replan_problem(name: str, seed: int = 0, *, min_utilization: float | None = None,
                   max_dp: int | None = None, max_pp: int = 32, layers: int = 80):
    sp = SPECS[name]
    min_utilization = sp["min_utilization"] if min_utilization is None else min_utilization
    max_dp = sp["max_dp"] if max_dp is None else max_dp
    P, M = sp["P"], sp["M"]
    st, cfg = _state(sp, layers, seed)
    if "n_sequences" in sp:
        docs, N = sequence_workload(sp["n_sequences"], M, seed)
        off, packed, quad = pack_workload(docs, N, M)
        quad = [int(q) for q in quad]
        mbs = [MicroBatch(j, tuple(int(x) for x in packed[off[j]:off[j + 1]]), N)
               for j in range(M)]
    else:
        off, packed = synth_iterations(1, M, 4096, 7.2, 0.8, seed)
        mbs = [MicroBatch(j, tuple(int(x) for x in packed[off[j]:off[j + 1]]), 4096)
               for j in range(M)]
        quad = [sum(x * x for x in mb.doc_lengths) for mb in mbs]
    inputs = build_desc(st, cfg, mbs, CostModel(2e-6, 5e-10), CommSpec(), capacity=P + 2,
                        quad=quad, min_utilization=min_utilization, max_dp=max_dp,
                        max_pp=max_pp)
    return st, cfg, mbs, inputs


class _Budget:
    """Token budget / count of a packed workload (what build_desc reads when
    the quad loads come precomputed)."""

    __slots__ = ("token_budget",)

    def __init__(self, n):
        self.token_budget = n


def replan_from_sequences(state, cfg, docs: np.ndarray, N: int, M: int, model, comm, *,
                          capacity, min_utilization, max_dp, max_pp=32, device=None,
                          group=None):
    """Failure report -> plan for a workload of raw sequences: FFD-pack them
    into M micro-batches of N tokens (rh_pack_sequences), quad loads,
    re-plan descriptor from the known cluster state, GPU search over every
    (DP, TP, PP) x partition x assignment candidate (sharded over the ranks of
    `group` with one collective when torch.distributed is initialised),
    decode, and the replica of every packed sequence under the chosen
    assignment.  Returns (plan, score, index, entry_replica[packed entries],
    search)."""
    import threading

    from .search import ReplanSearch, distributed_best

    # the FFD runs on a host thread (rh_pack_sequences releases the GIL)
    # while the descriptor is built and the search is created: layouts,
    # placement, repartition, splits and op lists do not depend on the quad
    # loads, which are supplied afterwards (rh_search_set_workload)
    packed_out = {}

    def pack():
        try:
            packed_out["v"] = pack_workload(docs, N, M)
        except Exception as exc:  # re-raised below
            packed_out["e"] = exc

    th = threading.Thread(target=pack)
    th.start()
    mbs = [_Budget(N)] * M
    inputs = build_desc(state, cfg, mbs, model, comm, capacity=capacity, defer_quad=True,
                        min_utilization=min_utilization, max_dp=max_dp, max_pp=max_pp)
    search = ReplanSearch(inputs, device)
    th.join()
    if "e" in packed_out:
        raise packed_out["e"]
    off, packed, quad = packed_out["v"]
    search.set_workload(quad)
    score, idx = distributed_best(search, group)
    plan = search.decode(idx) if idx >= 0 else None
    entry_replica = None
    if plan is not None:
        # every packed entry (sequence or padding) belongs to micro-batch b, and
        # micro-batches are owned contiguously by replica (split_micro_batches,
        # cluster.py:309-328)
        bins = np.repeat(np.arange(M, dtype=np.int32), np.diff(off))
        start = np.cumsum([0] + list(plan.counts))
        entry_replica = np.searchsorted(start, bins, side="right") - 1
    return plan, score, idx, entry_replica, search
