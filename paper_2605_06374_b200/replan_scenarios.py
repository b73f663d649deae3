"""Re-plan problems of BASELINE.json configs[2..4] (synthetic, seeded).

C3  256 GPUs  (32 nodes x 8), Llama-70B (80 layers), current TP4 x DP4 x PP16,
    64 micro-batches: one fail-stop, two fail-slow devices.
C4  1024 GPUs (128 nodes x 8), 80 layers, current TP8 x DP16 x PP8,
    128 micro-batches: one fail-stop, four fail-slow devices, one slow link.
C5  4096 GPUs (512 nodes x 8), 80 layers, current TP8 x DP32 x PP16,
    512 micro-batches packed from ~10^5-token-scale lognormal documents
    (see DESIGN.md §6), one fail-stop, eight fail-slow devices, two slow links.
All use alpha=2e-6, beta=5e-10, default CommSpec, capacity P+2 (harness.py:118-120),
lognormal(7.2, 0.8) documents FFD-packed into 4096-token micro-batches.
"""

from __future__ import annotations

import numpy as np

from .cluster import FailureEvent, MicroBatch, ParallelismConfig, apply_failures, build_cluster
from .comm import CommSpec
from .search import build_desc
from .trace import synth_iterations
from .workload import CostModel

GIB = float(2**30)

# min_utilization / max_dp size the candidate spaces to the configs' scale:
# C3 1.79e6 (exhaustive), C4 1.18e6 (~1e6), C5 9.66e6 (~1e7) candidates
SPECS = {
    "C3": dict(T=4, D=4, P=16, M=64, slow=2, links=0, min_utilization=0.95, max_dp=64),
    "C4": dict(T=8, D=16, P=8, M=128, slow=4, links=1, min_utilization=0.987, max_dp=32),
    "C5": dict(T=8, D=32, P=16, M=512, slow=8, links=2, min_utilization=0.985, max_dp=64),
}


def replan_problem(name: str, seed: int = 0, *, min_utilization: float | None = None,
                   max_dp: int | None = None, max_pp: int = 32, layers: int = 80):
    sp = SPECS[name]
    min_utilization = sp["min_utilization"] if min_utilization is None else min_utilization
    max_dp = sp["max_dp"] if max_dp is None else max_dp
    T, D, P, M = sp["T"], sp["D"], sp["P"], sp["M"]
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
    st = apply_failures(st, evs, 0.0)
    off, docs = synth_iterations(1, M, 4096, 7.2, 0.8, seed)
    mbs = [MicroBatch(j, tuple(int(x) for x in docs[off[j]:off[j + 1]]), 4096) for j in range(M)]
    quad = [sum(x * x for x in mb.doc_lengths) for mb in mbs]
    inputs = build_desc(st, cfg, mbs, CostModel(2e-6, 5e-10), CommSpec(), capacity=P + 2,
                        quad=quad, min_utilization=min_utilization, max_dp=max_dp,
                        max_pp=max_pp)
    return st, cfg, mbs, inputs
