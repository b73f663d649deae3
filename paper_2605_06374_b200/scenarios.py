"""Synthetic Detector traces of the BASELINE.json configurations.

C2 (configs[1]): 256 simulated GPUs, Llama-2 13B cost shape (40 layers),
TP4 x DP16 x PP4, 128 micro-batches of 4096 tokens per iteration,
lognormal(7.2, 0.8) document lengths, 10k iterations with mixed faults:

  it 2500  fail-slow compute (device 37, severity 0.5); the predictor learns
           it 2 iterations later (confirmation) and the series resets
  it 4000  fail-slow comm on link (4, 5) (severity 0.5); learned at 4002
  it 6000  fail-stop of device 150; its TP group continues as a 2-wide
           subgroup (resihp_adapt's TP step) from the same iteration
  it 7500  a second fail-slow compute (device 201, severity 0.3), learned at
           7503, then a greyhound-style proportional micro-batch re-split

Each phase is a segment with a KNOWN view (predictor) and an ACTUAL view
(ground truth for the synthetic measurements), built with the same host
table code the drop-in simulate_iteration uses.
"""

from __future__ import annotations

import numpy as np

from .cluster import FailureEvent, ParallelismConfig, apply_failures, build_cluster
from .comm import CommSpec
from .scheduler import AdaptationPlan, apply_plan
from .tables import segment_for_view
from .trace import DetectorTrace, synth_iterations
from .workload import CostModel

GIB = float(2**30)


def _proportional(total: int, weights: list[float]) -> list[int]:
    wsum = sum(weights)
    shares = [total * w / wsum for w in weights]
    counts = [int(q) for q in shares]
    order = sorted(range(len(weights)), key=lambda i: (-(shares[i] - counts[i]), i))
    for i in order[: total - sum(counts)]:
        counts[i] += 1
    return counts


def c2_trace(n_iter: int = 10_000, seed: int = 0, *, tp=4, dp=16, pp=4, layers=40, M=128,
             N=4096, mean=7.2, sigma=0.8, packer=None) -> DetectorTrace:
    cfg = ParallelismConfig(tp=tp, dp=dp, pp=pp, layer_partition=[layers // pp] * pp)
    n_dev = tp * dp * pp
    nodes = -(-n_dev // 8)
    base = build_cluster(nodes, 8, cfg, 300.0 * GIB, 25.0 * GIB)
    model = CostModel(alpha=2e-6, beta=5e-10)
    comm = CommSpec()
    f = lambda i: int(i * n_iter / 10_000)  # phase boundaries scale with n_iter
    slow1 = FailureEvent("fail_slow_compute", 0.0, device=37 % n_dev, severity=0.5)
    link = FailureEvent("fail_slow_comm", 0.0, link=(4 % nodes, 5 % nodes), severity=0.5) \
        if nodes > 1 else None
    stop = FailureEvent("fail_stop", 0.0, device=150 % n_dev)
    slow2 = FailureEvent("fail_slow_compute", 0.0, device=201 % n_dev, severity=0.3)

    def state_with(events, plan=None):
        s = apply_failures(base, [e for e in events if e is not None], 0.0) if events else base.copy()
        c = cfg
        if plan is not None:
            s, c = apply_plan(s, cfg, plan)
        return s, c

    # TP subgroup for the fail-stop: the 2 fastest surviving members
    key = next(k for k, g in base.tp_groups.items() if stop.device in g)
    members = [m for m in base.tp_groups[key] if m != stop.device]
    sub = AdaptationPlan(tp_subgroups={key: (tuple(sorted(members[:2])),
                                             tuple(sorted(members[2:])))})
    phases = []  # (start, actual events, known events, plan, counts, reset)
    phases.append((0, [], [], None, None, False))
    phases.append((f(2500), [slow1], [], None, None, False))
    phases.append((f(2502), [slow1], [slow1], None, None, True))
    phases.append((f(4000), [slow1, link], [slow1], None, None, False))
    phases.append((f(4002), [slow1, link], [slow1, link], None, None, True))
    phases.append((f(6000), [slow1, link, stop], [slow1, link, stop], sub, None, True))
    phases.append((f(7500), [slow1, link, stop, slow2], [slow1, link, stop], sub, None, False))
    phases.append((f(7503), [slow1, link, stop, slow2], [slow1, link, stop, slow2], sub, "prop",
                   True))

    known, actual, sizes = [], [], []
    for start, act_ev, kn_ev, plan, counts, _ in phases:
        sa, ca = state_with(act_ev, plan)
        sk, ck = state_with(kn_ev, plan)
        if counts == "prop":
            rs = [min(sk.effective_stage_speed(d, s, cfg.tp) for s in range(cfg.pp))
                  for d in range(cfg.dp)]
            counts = _proportional(M, rs)
        known.append(segment_for_view(sk, ck, M, N, comm=comm, dp_counts=counts,
                                      with_links=True))
        actual.append(segment_for_view(sa, ca, M, N, comm=comm, dp_counts=counts,
                                       with_links=True))
        # the measured link ratios come from the actual fabric
        known[-1].link_ratio = actual[-1].link_ratio
        sizes.append([len(sa.tp_groups[(d, s)]) for d in range(cfg.dp) for s in range(cfg.pp)])
    seg = np.zeros(n_iter, np.int32)
    reset = np.zeros(n_iter, np.uint8)
    for k, (start, *_rest) in enumerate(phases):
        seg[start:] = k
        if phases[k][5] and start < n_iter:
            reset[start] = 1
    mb_off, doc_len = synth_iterations(n_iter, M, N, mean, sigma, seed, packer=packer)
    tr = DetectorTrace(cfg=cfg, model=model, M=M, N=N, has_allreduce=dp > 1, seg=seg,
                       mb_off=mb_off, doc_len=doc_len, known=known, actual=actual, reset=reset,
                       group_size=np.asarray(sizes, dtype=np.int64))
    tr.meta = {"workload": "C2", "devices": n_dev, "layers": layers, "nodes": nodes}
    return tr
