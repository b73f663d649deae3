"""Micro-batch cost model (mirror of resilsim/workload.py).

``quad_load`` and ``predict_chunk_time`` run on the GPU (rh_quad_load /
rh_chunk_time); batch callers should use ``quad_loads`` / ``chunk_times``.
``pack_sequences`` (first-fit decreasing) is host-side workload ingest.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .cluster import MicroBatch

CHUNK_F = "F"
CHUNK_B = "B"
CHUNK_W = "W"
CHUNK_BW = "BW"
CHUNK_ALLREDUCE = "AR"

KIND_CODE = {CHUNK_F: 0, CHUNK_B: 1, CHUNK_W: 2, CHUNK_BW: 3}
DEFAULT_CHUNK_RATIOS = {CHUNK_F: 1.0, CHUNK_B: 1.0, CHUNK_W: 1.0}


@dataclass
class CostModel:
    """workload.py:29-49: t = ratio * L * (alpha*N + beta*sum l^2) / speed."""

    alpha: float
    beta: float
    chunk_ratios: dict[str, float] = field(default_factory=lambda: dict(DEFAULT_CHUNK_RATIOS))

    def __post_init__(self):
        if self.alpha < 0 or self.beta < 0:
            raise ValueError("cost coefficients must be non-negative")
        if self.alpha == 0 and self.beta == 0:
            raise ValueError("cost model needs at least one non-zero coefficient")
        for kind in (CHUNK_F, CHUNK_B, CHUNK_W):
            if self.chunk_ratios.get(kind, 0.0) <= 0:
                raise ValueError(f"chunk ratio for {kind} must be positive")

    def ratio(self, kind: str) -> float:
        if kind == CHUNK_BW:
            return self.chunk_ratios[CHUNK_B] + self.chunk_ratios[CHUNK_W]
        return self.chunk_ratios[kind]


def cost_model_c(model):
    """rh_cost_model struct of any CostModel-like object (duck-typed)."""
    from . import _lib

    r = model.chunk_ratios
    return _lib.CostModelC(float(model.alpha), float(model.beta), float(r[CHUNK_F]),
                           float(r[CHUNK_B]), float(r[CHUNK_W]))


def pack_sequences(doc_lengths, token_budget: int) -> list[MicroBatch]:
    """workload.py:52-80: first-fit decreasing into bins of exactly
    ``token_budget`` tokens; each bin's residual becomes a padding document."""
    lengths = [int(x) for x in doc_lengths]
    for x in lengths:
        if x <= 0:
            raise ValueError(f"document length must be positive, got {x}")
        if x > token_budget:
            raise ValueError(f"document of {x} tokens exceeds budget {token_budget}")
    contents: list[list[int]] = []
    free: list[int] = []
    for x in sorted(lengths, reverse=True):
        slot = next((i for i, room in enumerate(free) if x <= room), None)
        if slot is None:
            contents.append([x])
            free.append(token_budget - x)
        else:
            contents[slot].append(x)
            free[slot] -= x
    return [MicroBatch(id=i, doc_lengths=tuple(docs + ([room] if room > 0 else [])),
                       token_budget=token_budget)
            for i, (docs, room) in enumerate(zip(contents, free))]


def csr_of(micro_batches) -> tuple[np.ndarray, np.ndarray]:
    """(mb_off int32[M+1], doc_len int32[...]) of a list of micro-batches."""
    counts = np.fromiter((len(mb.doc_lengths) for mb in micro_batches), dtype=np.int64,
                         count=len(micro_batches))
    off = np.zeros(len(micro_batches) + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    if off[-1] >= 2**31:
        raise ValueError("too many documents for int32 offsets")
    docs = np.fromiter((x for mb in micro_batches for x in mb.doc_lengths), dtype=np.int64,
                       count=int(off[-1]))
    if docs.size and (docs.min() < 0 or docs.max() >= 2**31):
        raise ValueError("document length outside int32")
    return off.astype(np.int32), docs.astype(np.int32)


def quad_loads(micro_batches) -> np.ndarray:
    """quad_load of every micro-batch, computed by rh_quad_load on the GPU
    (rh_quad_load_host: one copy in, one copy out)."""
    from . import _lib

    n = len(micro_batches)
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    off, docs = csr_of(micro_batches)
    docs = docs if docs.size else np.zeros(1, np.int32)
    out = np.empty(n, dtype=np.int64)
    lib = _lib.load_library()
    _lib.check(lib.rh_quad_load_host(_lib.context(), n, off.ctypes.data, docs.ctypes.data,
                                     out.ctypes.data), "rh_quad_load_host")
    return out


def quad_load(mb: MicroBatch) -> int:
    """workload.py:83-85 — sum of squared document lengths, padding included."""
    return int(quad_loads([mb])[0])


def chunk_times(model, micro_batches, kinds, layers, speeds) -> np.ndarray:
    """predict_chunk_time for n chunks at once (rh_chunk_time on the GPU).

    ``micro_batches``, ``kinds``, ``layers`` and ``speeds`` are parallel
    sequences.  Raises ValueError like the reference when a speed is <= 0.
    """
    from . import _lib

    n = len(kinds)
    if n == 0:
        return np.zeros(0, dtype=np.float64)
    sp = np.ascontiguousarray(speeds, dtype=np.float64)
    if (sp <= 0).any():
        raise ValueError("cannot schedule onto a stopped device (speed <= 0)")
    uniq: dict[int, int] = {}
    mbs = []
    idx = np.empty(n, dtype=np.int64)
    for i, mb in enumerate(micro_batches):
        k = id(mb)
        if k not in uniq:
            uniq[k] = len(mbs)
            mbs.append(mb)
        idx[i] = uniq[k]
    off, docs = csr_of(mbs)
    docs = docs if docs.size else np.zeros(1, np.int32)
    budget = np.fromiter((mbs[j].token_budget for j in idx), np.int32, n)
    kind = np.fromiter((KIND_CODE[k] for k in kinds), np.uint8, n)
    lay = np.ascontiguousarray(layers, dtype=np.int32)
    out = np.empty(n, dtype=np.float64)
    bad = np.zeros(n, dtype=np.uint8)
    lib = _lib.load_library()
    # quad loads + chunk times in one round trip (rh_chunk_time_docs_host)
    _lib.check(lib.rh_chunk_time_docs_host(_lib.context(), _lib.C.byref(cost_model_c(model)),
                                           len(mbs), off.ctypes.data, docs.ctypes.data, n,
                                           idx.ctypes.data, budget.ctypes.data, kind.ctypes.data,
                                           lay.ctypes.data, sp.ctypes.data, out.ctypes.data,
                                           bad.ctypes.data), "rh_chunk_time_docs_host")
    return out


def predict_chunk_time(mb: MicroBatch, kind: str, model: CostModel, layers_on_stage: int,
                       device_speed: float) -> float:
    """workload.py:88-98"""
    if device_speed <= 0:
        raise ValueError("cannot schedule onto a stopped device (speed <= 0)")
    return float(chunk_times(model, [mb], [kind], [layers_on_stage], [device_speed])[0])


def fit_cost_model(samples, chunk_ratios=None):
    """workload.py:101-125 -- offline calibration of (alpha, beta) from
    (micro-batch, measured F time) pairs: least squares on the columns
    (token budget N, quad load Q) -- the quad loads of all samples in one GPU
    batch (quad_loads), the 2-column solve on the host (numpy lstsq, as the
    reference) -- a negative coefficient is clamped to 0 and the other refit
    alone; returns (CostModel, in-sample MAPE)."""
    if len(samples) < 2:
        raise ValueError("need at least two samples to fit the cost model")
    mbs = [mb for mb, _ in samples]
    times = np.array([float(t) for _, t in samples], dtype=np.float64)
    budgets = np.array([float(mb.token_budget) for mb in mbs], dtype=np.float64)
    quads = quad_loads(mbs).astype(np.float64)
    if np.ptp(quads) == 0 and np.ptp(budgets) == 0:
        raise ValueError("unidentifiable beta: all samples share the same quad load")
    sol = np.linalg.lstsq(np.column_stack([budgets, quads]), times, rcond=None)[0]
    alpha, beta = float(sol[0]), float(sol[1])
    if alpha < 0:  # noise pushed one coefficient below zero: refit the other alone
        alpha, beta = 0.0, float(np.dot(quads, times) / np.dot(quads, quads))
    elif beta < 0:
        alpha, beta = float(np.dot(budgets, times) / np.dot(budgets, budgets)), 0.0
    fit = alpha * budgets + beta * quads
    mape = float(np.mean(np.abs(fit - times) / times))
    return CostModel(alpha=alpha, beta=beta,
                     chunk_ratios=dict(chunk_ratios or DEFAULT_CHUNK_RATIOS)), mape
