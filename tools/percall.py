"""Per-call latency of the drop-in API against the reference (baseline/_ref)
on the same C1-shaped inputs (32 GPUs, TP4 x DP4 x PP2, 16 micro-batches,
one fail-slow device): quad_load, predict_chunk_time, build_dag +
critical_path, simulate_iteration, DetectorState.observe, evaluate_plan.
Median of repeated single calls, one process.  Prints one JSON object."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402

import resilsim  # noqa: E402,F401  (the reference, pip-installed into baseline/_ref)
from resilsim import cluster as r_cl, comm as r_cm, detector as r_dt  # noqa: E402
from resilsim import pipeline as r_pl, scheduler as r_sc, workload as r_wl  # noqa: E402

from paper_2605_06374_b200 import cluster as o_cl, comm as o_cm, detector as o_dt  # noqa: E402
from paper_2605_06374_b200 import pipeline as o_pl, scheduler as o_sc, workload as o_wl  # noqa: E402

GIB = float(2**30)


def problem(cl, cm, wl):
    cfg = cl.ParallelismConfig(4, 4, 2, "1f1b", [16, 16])
    st = cl.build_cluster(4, 8, cfg, 300.0 * GIB, 25.0 * GIB)
    st = cl.apply_failures(st, [cl.FailureEvent("fail_slow_compute", 0.0, device=5, severity=0.5)], 0.0)
    rng = np.random.default_rng(3)
    mbs = []
    for j in range(16):
        docs, left = [], 4096
        while left > 0:
            x = int(min(left, max(1, round(rng.lognormal(7.2, 0.8)))))
            docs.append(x)
            left -= x
        mbs.append(wl.MicroBatch(j, tuple(docs), 4096))
    return cfg, st, mbs, wl.CostModel(2e-6, 5e-10), cm.CommSpec()


def timed(fn, n):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


def suite(cl, cm, wl, pl, dt, sc, n):
    cfg, st, mbs, model, comm = problem(cl, cm, wl)
    rec = pl.simulate_iteration(st, cfg, mbs, model, comm=comm, capacity=4)
    speeds = {(d, s): 1.0 for d in range(4) for s in range(2)}
    det = dt.DetectorState()
    plan = sc.AdaptationPlan(dp_assignment=[4, 4, 4, 4])
    out = {
        "quad_load": timed(lambda: wl.quad_load(mbs[0]), n),
        "predict_chunk_time": timed(lambda: wl.predict_chunk_time(mbs[0], "F", model, 16, 0.5), n),
        "build_dag+critical_path": timed(
            lambda: pl.critical_path(pl.build_dag(cfg, mbs, model, speeds)), n),
        "simulate_iteration": timed(
            lambda: pl.simulate_iteration(st, cfg, mbs, model, comm=comm, capacity=4), n),
        "DetectorState.observe": timed(
            lambda: det.observe(rec, rec.predicted_healthy_time, rec.stage_cost_reference), n),
        "evaluate_plan": timed(
            lambda: sc.evaluate_plan(plan, st, cfg, mbs, model, comm=comm, capacity=4), n),
    }
    return out


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    ref = suite(r_cl, r_cm, r_wl, r_pl, r_dt, r_sc, n)
    ours = suite(o_cl, o_cm, o_wl, o_pl, o_dt, o_sc, n)
    print(json.dumps({"unit": "us per call (median)", "shape": "C1: 32 GPUs TP4xDP4xPP2, 16 mbs",
                      "reference": ref, "drop_in": ours,
                      "ratio_ref_over_ours": {k: ref[k] / ours[k] for k in ref}}, indent=1))
