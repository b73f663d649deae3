"""Seeded random traces for parity tests (test infrastructure)."""

from __future__ import annotations

import numpy as np

from paper_2605_06374_b200.cluster import ParallelismConfig
from paper_2605_06374_b200.tables import Segment
from paper_2605_06374_b200.trace import DetectorTrace, synth_iterations
from paper_2605_06374_b200.workload import CostModel


def random_counts(rng, M, D, allow_zero=True):
    if D == 1:
        return [M]
    cuts = np.sort(rng.integers(0 if allow_zero else 1, M + 1, size=D - 1))
    c = np.diff(np.concatenate([[0], cuts, [M]])).tolist()
    return [int(x) for x in c]


def random_segment(rng, cfg, M, *, slow_p=0.2, hop=True, ar=True, stop=False,
                   counts=None, unit=False) -> Segment:
    D, P = cfg.dp, cfg.pp
    speed = np.ones(D * P)
    if not unit:
        slow = rng.random(D * P) < slow_p
        speed[slow] = rng.choice([0.5, 0.25, 0.75, 0.3, 0.6], size=int(slow.sum()))
        half = rng.random(D * P) < 0.1
        speed[half] *= 0.5  # subgroup |group|/tp
    if stop:
        speed[rng.integers(D * P)] = 0.0
    hf = rng.uniform(0, 2e-3, D * P) if hop else np.zeros(D * P)
    hb = rng.uniform(0, 2e-3, D * P) if hop else np.zeros(D * P)
    hf[P - 1::P] = 0.0
    hb[P - 1::P] = 0.0
    counts = counts if counts is not None else random_counts(rng, M, D)
    start = np.zeros(D + 1, np.int32)
    np.cumsum(counts, out=start[1:])
    arr = np.full(D, rng.uniform(0, 0.05)) if ar else np.zeros(D)
    layers = np.asarray(cfg.layer_partition, np.int32)
    lr = rng.choice([1.0, 1.0, 2.5, 1.1], size=int(rng.integers(0, 4))).astype(np.float64)
    return Segment(layers, start, speed, hf, hb, arr, lr)


def random_trace(seed, *, n_iter=16, tp=None, dp=None, pp=None, schedule=None, M=None, N=None,
                 n_seg=None, comm=None, stop=False, unit=False, mean=7.0, sigma=0.8,
                 ratios=None) -> DetectorTrace:
    rng = np.random.default_rng(seed)
    tp = tp or int(rng.choice([1, 2, 4, 8]))
    dp = dp or int(rng.integers(1, 5))
    pp = pp or int(rng.integers(1, 7))
    schedule = schedule or str(rng.choice(["1f1b", "zbh"]))
    M = M or int(rng.integers(1, 4 * dp + 1))
    N = N or int(rng.choice([1024, 2048, 4096]))
    layers = [int(x) for x in rng.integers(1, 6, size=pp)]
    cfg = ParallelismConfig(tp=tp, dp=dp, pp=pp, schedule=schedule, layer_partition=layers)
    model = CostModel(alpha=float(rng.uniform(1e-6, 4e-6)), beta=float(rng.uniform(1e-10, 9e-10)),
                      chunk_ratios=ratios or {"F": 1.0, "B": float(rng.choice([1.0, 0.5, 1.25])),
                                              "W": float(rng.choice([1.0, 0.5, 0.75]))})
    mb_off, doc_len = synth_iterations(n_iter, M, N, mean, sigma, seed)
    n_seg = n_seg or int(rng.integers(1, 4))
    comm = bool(rng.integers(0, 2)) if comm is None else comm
    known, actual = [], []
    for _ in range(n_seg):
        counts = random_counts(rng, M, dp)
        k = random_segment(rng, cfg, M, hop=comm, ar=comm, counts=counts, unit=unit)
        a = random_segment(rng, cfg, M, hop=comm, ar=comm, counts=counts, stop=stop, unit=unit)
        a.hop_fwd, a.hop_bwd, a.allreduce = k.hop_fwd, k.hop_bwd, k.allreduce
        known.append(k)
        actual.append(a)
    seg = rng.integers(0, n_seg, size=n_iter).astype(np.int32)
    reset = np.zeros(n_iter, np.uint8)
    return DetectorTrace(cfg=cfg, model=model, M=M, N=N, has_allreduce=comm and dp > 1,
                         seg=seg, mb_off=mb_off, doc_len=doc_len, known=known, actual=actual,
                         reset=reset)


def with_measurements(trace: DetectorTrace, oracle, noise=0.01, seed=1) -> DetectorTrace:
    ms, st, sc = oracle.pipeline(trace, view="actual")
    trace.attach_measurements(sc, ms, noise=noise, seed=seed)
    return trace
