"""Benchmark: batched Detector pass (BASELINE.json configs[1], "C2").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One STEP = one full Detector pass over a 10,000-iteration device x iteration
trace of a 256-GPU cluster (TP4 x DP16 x PP4, Llama-2-13B layer count, 128
micro-batches/iteration, mixed fail-slow / fail-stop / link faults): the
workload-aware predictor (critical path of the canonical 1F1B chunk DAG,
Eq. 2) on the known view, the 1.25x filter, per-(replica,stage) and link
validation, and the median/MAD change-point state machine.
  value  = device-samples/s over all ranks (256 x 10,000 per step per rank),
           inputs resident in HBM, L2 flushed (256 MiB write) before every
           step, each step timed with CUDA events on the launching stream;
  e2e    = the same metric through the reference-facing C-ABI call
           rh_detector_pass_host_packed with pinned host buffers in the packed
           wire form (H2D + kernels + D2H inside the timed region);
  roofline of the dominant kernel (pass_small_kernel<P=4,1F1B,detect>);
  cpu_baseline = the C oracle restatement of the reference on the host cores.
Multi-GPU (torchrun): one trace of N x 10^4 iterations in contiguous shards, one
per rank, cut at series resets (adaptation boundaries: detect_shard.py), so no
data-path collective (weak scaling); the step time is the max over ranks.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Detector samples/s"
UNIT = "device-samples/s"
N_ITER = 10_000


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML SM clock + throttle reasons sampled during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("RESIHP_BACKEND") == "gloo":
            dist.init_process_group("gloo")
        else:
            import torch

            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def build_trace(rank: int, n_iter: int, use_oracle: bool):
    """The C2 trace.  use_oracle (the reference arm): documents packed by the
    oracle's literal FFD and measurements from the oracle's DAG, so that
    process never loads the product library (checked by
    tests/test_bench_contract.py)."""
    from paper_2605_06374_b200.scenarios import c2_trace

    if use_oracle:
        from tests.oracle_bind import Oracle

        o = Oracle()
        tr = c2_trace(n_iter, seed=rank, packer=o.pack_sequences)
        ms, st, sc = o.pipeline(tr, view="actual")
        tr.attach_measurements(sc, ms, seed=rank)
        return tr
    from paper_2605_06374_b200.detect_pass import synthesize_measurements

    tr = c2_trace(n_iter, seed=rank)
    synthesize_measurements(tr, seed=rank)
    return tr


def algorithmic_bytes(tr) -> float:
    """HBM bytes one detect launch must move."""
    return float(sum(tr.nbytes_per_iter().values()) * tr.n_iter)


def cpu_baseline(tr, threads=None):
    from tests.oracle_bind import Oracle

    o = Oracle()
    cores = threads or os.cpu_count() or 1
    reps, t0 = 0, time.perf_counter()
    while True:
        ms, st, *_ = o.detect(tr, threads=cores)
        o.screen(tr.observed, st, reset=tr.reset)
        reps += 1
        if time.perf_counter() - t0 > 10.0 or reps >= 50:
            break
    dt = (time.perf_counter() - t0) / reps
    d = tr.cfg.dp * tr.cfg.pp * tr.cfg.tp
    return {"value": tr.n_iter * d / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"full C2 trace ({tr.n_iter} iterations x {d} devices), {reps} reps, "
                      "oracle/liboracle.so (C restatement of resilsim build_dag+critical_path"
                      "+DetectorState.observe), pthreads over iterations"}


def _py_ref_worker(args):
    """One reference run_scenario (baseline/_ref) at the C2 shape -> (iterations, seconds)."""
    ref_dir, seed, iters = args
    sys.path.insert(0, ref_dir)
    from resilsim.harness import run_scenario, scenario_from_mapping

    m = {"name": "c2", "seed": seed, "iterations": iters, "policy": "resihp",
         "cluster": {"nodes": 32, "devices_per_node": 8},
         "parallelism": {"tp": 4, "dp": 16, "pp": 4, "layers": 40},
         "workload": {"token_budget": 4096, "micro_batches": 128,
                      "doc_lengths": {"kind": "lognormal", "mean": 7.2, "sigma": 0.8}},
         "failures": []}
    sc = scenario_from_mapping(m)
    t0 = time.perf_counter()
    res = run_scenario(sc)
    return len(res.records), time.perf_counter() - t0


def python_reference_baseline(budget_s=20.0):
    """The reference's own Python Detector loop: resilsim
    run_scenario at the C2 shape -- per iteration simulate_iteration (actual +
    known view) and DetectorState.observe -- one scenario per process over
    all host cores (the cli.py:86-92 ProcessPool pattern); device-samples/s =
    iterations x 256 devices / wall time."""
    from concurrent.futures import ProcessPoolExecutor

    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "resilsim").exists():
        return {"unavailable": "baseline/_ref (pip install of /root/reference/pkg) is missing"}
    cores = os.cpu_count() or 1
    # size: one probe run on this core, then a pool round of ~budget_s
    n0, t0 = _py_ref_worker((str(ref_dir), 0, 2))
    per_iter = t0 / max(1, n0)
    iters = max(2, int(budget_s / max(per_iter, 1e-3)))
    wall0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=cores) as ex:
        res = list(ex.map(_py_ref_worker, [(str(ref_dir), 1 + k, iters) for k in range(cores)]))
    wall = time.perf_counter() - wall0
    n = sum(r[0] for r in res)
    return {"value": n * 256 / wall, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{cores} x resilsim run_scenario (C2 shape: 256 GPUs TP4xDP16xPP4, 128 "
                      f"micro-batches, resihp detector on, no re-plan), {iters} iterations each, "
                      "one process per core (cli.py:86-92 pattern); includes scenario setup",
            "per_iteration_ms_one_core": per_iter * 1e3}


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm's CPU restatement on all host cores."""
    if rank != 0:
        return
    tr = build_trace(0, N_ITER, use_oracle=True)
    from tests.oracle_bind import Oracle

    o = Oracle()
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        ms, st, *_ = o.detect(tr, threads=cores)
        o.screen(tr.observed, st, reset=tr.reset)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ms, st, *_ = o.detect(tr, threads=cores)
        o.screen(tr.observed, st, reset=tr.reset)
        times.append(time.perf_counter() - t0)
    step = sum(times) / len(times)
    d = tr.cfg.dp * tr.cfg.pp * tr.cfg.tp
    value = tr.n_iter * d / step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(tr),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"full C2 trace per step ({tr.n_iter} iterations)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of(tr):
    c = tr.cfg
    return {"workload": "C2: 256-GPU Llama-2-13B (40 layers) TP4xDP16xPP4 1F1B, mixed fail-stop"
                        " + fail-slow + link fault, full Detector trace",
            "iterations_per_step": tr.n_iter, "devices": c.tp * c.dp * c.pp,
            "micro_batches": tr.M, "token_budget": tr.N,
            "doc_lengths": "lognormal(7.2, 0.8) FFD-packed", "l2": "flushed (256 MiB write) "
            "before every step; trace ~35 MB per rank",
            "parallelism": "one trace of n_gpus x 10^4 iterations, one contiguous shard per "
                           "rank cut at series resets (detect_shard.py), no data-path "
                           "collective"}


def run_ours(args, world, rank, local):
    import torch

    from paper_2605_06374_b200 import _lib
    from paper_2605_06374_b200.detect_pass import DetectorPass

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tr = build_trace(rank, N_ITER, use_oracle=False)
    if world > 1 and rank > 0:
        # rank r holds iterations [r*10^4, (r+1)*10^4) of ONE trace of world*10^4
        # iterations; its shard starts at a series reset (an adaptation
        # boundary), so its screen needs no state from rank r-1
        # (detect_shard.shard_bounds): no data-path collective
        tr.reset[0] = 1
    p = DetectorPass(tr, dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]

    for _ in range(args.warmup):
        flush.fill_(1)
        p.run()
    torch.cuda.synchronize()
    l0 = _lib.launches(local)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        wall0 = time.perf_counter()
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            ev[k][0].record(stream)
            p.detect()
            ev[k][1].record(stream)
            p.screen()
            ev[k][2].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    launches = _lib.launches(local) - l0
    det_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
    scr_ms = [ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps)]
    step_ms = sum(a + b for a, b in zip(det_ms, scr_ms)) / args.steps
    if world > 1:
        t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        step_ms = float(t.item())
    devices = tr.cfg.tp * tr.cfg.dp * tr.cfg.pp
    value = world * tr.n_iter * devices / (step_ms * 1e-3)

    # sanity: the timed pass produced the checked result shape
    res = p.results()
    assert res["status"].shape == (tr.n_iter,)

    e2e = run_e2e(tr, p, args, dev)
    if world > 1:
        t = torch.tensor([e2e["step_s"]], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e["step_s"] = float(t.item())
    peak, peak_src = _peaks()
    det_avg = sum(det_ms) / len(det_ms)
    nbytes = algorithmic_bytes(tr)
    achieved = nbytes / (det_avg * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "detect_kernel_ncu.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(tr),
        "e2e": {"value": world * tr.n_iter * devices / e2e["step_s"], "unit": UNIT,
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ("pass_small_kernel<P=%d,1F1B,detect>" % tr.cfg.pp
                                if tr.cfg.pp <= 4 else "pass_kernel<1F1B,detect>"),
                     "algorithmic_bytes": nbytes,
                     "kernel_ms": det_avg, "peak_source": peak_src},
        "breakdown_ms": {"detect": det_avg, "screen": sum(scr_ms) / len(scr_ms)},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "wall_s_timed_region": wall,
    }
    return line, tr


def run_e2e(tr, p, args, dev):
    """rh_detector_pass_host_packed with pinned host buffers in the packed wire
    form (uint16 document lengths, uint8 documents per micro-batch, int32
    per-iteration document offsets); H2D + kernels + D2H timed."""
    import torch

    from paper_2605_06374_b200 import _lib
    from paper_2605_06374_b200.tables import pipe_shape

    pin = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).pin_memory()
    segs = tr.known
    cat = lambda name, dt: pin(np.concatenate([getattr(s, name) for s in segs]), dt)
    pk = tr.packed()
    h = {
        "seg": pin(tr.seg, np.int32), "iter_doc": pin(pk["iter_doc"], np.int32),
        "mb_docs": pin(pk["mb_docs"], np.uint8), "doc_len": pin(pk["doc_len"], np.uint16),
        "dt": pin(tr.device_time, np.float32),
        "obs": pin(tr.observed, np.float64), "reset": pin(tr.reset, np.uint8),
        "layers": cat("layers", np.int32), "mb_start": cat("mb_start", np.int32),
        "speed": cat("speed", np.float64), "hf": cat("hop_fwd", np.float64),
        "hb": cat("hop_bwd", np.float64), "ar": cat("allreduce", np.float64),
        "lr": pin(np.concatenate([s.link_ratio for s in segs] + [np.zeros(1)]), np.float64),
    }
    off = np.zeros(len(segs) + 1, np.int32)
    np.cumsum([len(s.link_ratio) for s in segs], out=off[1:])
    h["loff"] = pin(off, np.int32)
    h["lmax"] = pin(np.array([float(np.max(s.link_ratio)) if len(s.link_ratio) else 0.0
                              for s in segs]), np.float64)
    n, G = tr.n_iter, tr.cfg.dp * tr.cfg.pp
    o = {"ms": torch.empty(n, dtype=torch.float64).pin_memory(),
         "st": torch.empty(n, dtype=torch.uint8).pin_memory(),
         "fl": torch.empty(n * G, dtype=torch.uint8).pin_memory(),
         "sv": torch.empty(n * G, dtype=torch.float32).pin_memory(),
         "oc": torch.empty(n, dtype=torch.uint8).pin_memory()}
    seg_c = _lib.Segments(len(segs), h["layers"].data_ptr(), h["mb_start"].data_ptr(),
                          h["speed"].data_ptr(), h["hf"].data_ptr(), h["hb"].data_ptr(),
                          h["ar"].data_ptr(), h["loff"].data_ptr(), h["lr"].data_ptr(),
                          h["lmax"].data_ptr())
    tr_c = _lib.TracePacked(n, h["seg"].data_ptr(), h["iter_doc"].data_ptr(),
                            h["mb_docs"].data_ptr(), h["doc_len"].data_ptr(),
                            h["dt"].data_ptr(), h["obs"].data_ptr())
    out_c = _lib.PassOut(o["ms"].data_ptr(), o["st"].data_ptr(), None, o["fl"].data_ptr(),
                         o["sv"].data_ptr())
    max_mb = int(max(np.diff(s.mb_start).max() for s in segs))
    shape = pipe_shape(tr.cfg, tr.M, tr.N, has_allreduce=tr.has_allreduce, max_mb=max_mb)
    lib = _lib.load_library()
    ctx = _lib.context(dev.index)
    series_len = C.c_int64()
    stream = torch.cuda.current_stream(dev)

    def call():
        _lib.check(lib.rh_detector_pass_host_packed(
            ctx, C.byref(shape), C.byref(p.model_c), C.byref(seg_c), C.byref(tr_c), 1.25,
            C.byref(p.screen_params), 0, None, h["reset"].data_ptr(), C.byref(out_c),
            o["oc"].data_ptr(), C.byref(series_len), stream.cuda_stream),
            "rh_detector_pass_host_packed")

    for _ in range(max(1, args.warmup)):
        call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        call()
    step = (time.perf_counter() - t0) / args.steps
    # e2e results agree with the device-resident pass
    r = p.results()
    assert np.array_equal(o["st"].numpy(), r["status"])
    assert np.array_equal(o["oc"].numpy(), r["outcome"])
    h2d = sum(t.numel() * t.element_size() for k, t in h.items())
    d2h = sum(t.numel() * t.element_size() for t in o.values()) + 8
    return {"step_s": step, "h2d": int(h2d), "d2h": int(d2h)}


def tile_trace(tr, reps: int):
    """The trace repeated `reps` times back to back (documents, offsets,
    segment ids, measurements, resets): SURVEY §8(d)'s 10^5-iteration trace R
    from a 10^4-iteration sample without 10x the host-side generation."""
    import copy

    n, M = tr.n_iter, tr.M
    docs = tr.doc_len.size
    out = copy.copy(tr)
    base = np.asarray(tr.mb_off[:n * M], dtype=np.int64)
    offs = [base + k * docs for k in range(reps)] + [np.array([reps * docs], np.int64)]
    out.mb_off = np.concatenate(offs).astype(np.int32)
    out.doc_len = np.tile(tr.doc_len, reps)
    out.seg = np.tile(tr.seg, reps)
    out.reset = np.tile(tr.reset, reps)
    out.reset[::n] = 1  # each tile is its own series (reset at the tile start)
    out.device_time = np.tile(tr.device_time, (reps, 1, 1, 1))
    out.observed = np.tile(tr.observed, reps)
    return out


def run_trace_r(args, dev, sample=10_000, reps=10):
    """SURVEY §8(d)'s Detector roofline trace R -- the C5 shape (4096 GPUs,
    TP8 x DP32 x PP16, 80 layers, 512 micro-batches, the C2 fault phases) --
    at its specified 10^5 iterations (~2.8 GB): a 10^4-iteration sample
    generated on the host and tiled 10x in HBM.  Far larger than L2: no
    flush needed between steps."""
    import torch

    from paper_2605_06374_b200.detect_pass import DetectorPass, synthesize_measurements
    from paper_2605_06374_b200.scenarios import c2_trace

    tr0 = c2_trace(sample, seed=0, tp=8, dp=32, pp=16, layers=80, M=512)
    synthesize_measurements(tr0, seed=0)
    tr = tile_trace(tr0, reps)
    del tr0
    n_iter = tr.n_iter
    p = DetectorPass(tr, dev)
    for _ in range(args.warmup):
        p.run()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 10))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    stream = torch.cuda.current_stream(dev)
    for k in range(steps):
        ev[k][0].record(stream)
        p.detect()
        ev[k][1].record(stream)
        p.screen()
        ev[k][2].record(stream)
    torch.cuda.synchronize()
    det = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    scr = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    nbytes = algorithmic_bytes(tr)
    peak, _ = _peaks()
    dev_n = 8 * 32 * 16
    res = {"workload": "SURVEY trace R: C5 shape (4096 GPUs, TP8xDP32xPP16, 80 layers, 512 "
                       f"micro-batches), {n_iter} iterations ({sample}-iteration sample tiled "
                       f"{reps}x in HBM)",
           "iterations": n_iter,
           "device_samples_per_s": n_iter * dev_n / ((det + scr) * 1e-3),
           "detect_ms": det, "screen_ms": scr, "algorithmic_bytes": nbytes,
           "achieved_gbs": nbytes / (det * 1e-3) / 1e9,
           "frac_of_hbm": nbytes / (det * 1e-3) / 1e9 / peak,
           "kernel": "pass_wide_kernel<P=16,detect> (thread per replica, segment tables in L1, "
                     "level-ordered warm-up + loop-form 1F1B walk)"}
    prof = ROOT / "profiles" / "trace_r_kernel_ncu.json"
    if prof.exists():  # DRAM bytes of one launch, from the committed ncu capture
        res["traffic"] = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    del p
    torch.cuda.empty_cache()
    return res


def run_scheduler(args, world, rank, local, names=("C3", "C4", "C5")):
    """Re-plan search (BASELINE configs[2..4]): candidates/s and re-plan latency.

    Each rank scores its contiguous shard of the candidate index range; one
    NCCL all-gather of (score, index) pairs finishes the min-loc.  Latency =
    wall clock from the failure report (the scheduler's known cluster state
    and the workload) to the decoded plan: descriptor (build_desc), search
    create + per-layout GPU prep, sharded scoring, the collective, decode --
    and for C5 (10^5 sequences) also the FFD packing of the sequences into
    the 512 micro-batches, their quad loads and every packed sequence's
    replica under the chosen assignment (replan_from_sequences)."""
    import torch

    from paper_2605_06374_b200.comm import CommSpec
    from paper_2605_06374_b200.replan_scenarios import (SPECS, replan_from_sequences,
                                                        replan_problem, sequence_workload)
    from paper_2605_06374_b200.search import ReplanSearch, build_desc, distributed_best
    from paper_2605_06374_b200.workload import CostModel

    dev = torch.device("cuda", local)
    group = torch.distributed.group.WORLD if world > 1 else None
    out = {}
    for name in names:
        sp = SPECS[name]
        st, cfg, mbs, inputs = replan_problem(name)
        s = ReplanSearch(inputs, dev)
        a, b = s.shard(rank, world)
        s.eval_async(a, b)  # warm-up (module load, caches)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.eval_async(a, b)
        e1.record()
        torch.cuda.synchronize()
        eval_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([eval_ms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            eval_ms = float(t.item())
        model, comm = CostModel(2e-6, 5e-10), CommSpec()
        kw = dict(capacity=cfg.pp + 2, min_utilization=sp["min_utilization"],
                  max_dp=sp["max_dp"])
        seqs = None
        if "n_sequences" in sp:
            seqs, N = sequence_workload(sp["n_sequences"], sp["M"])

        def replan():
            if seqs is not None:
                plan, score, idx, entry_rep, srch = replan_from_sequences(
                    st, cfg, seqs, N, sp["M"], model, comm, device=dev, group=group, **kw)
                return plan, score, idx, srch
            inp = build_desc(st, cfg, mbs, model, comm, quad=inputs.arrays["quad"], **kw)
            srch = ReplanSearch(inp, dev)
            score, idx = distributed_best(srch, group)
            return (srch.decode(idx) if idx >= 0 else None), score, idx, srch

        replan()  # warm-up
        lat = []
        for _ in range(5):
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan, score, idx, srch = replan()
            torch.cuda.synchronize()
            lat.append((time.perf_counter() - t0) * 1e3)
            del srch
        lat_ms = float(np.median(lat))
        if world > 1:
            t = torch.tensor([lat_ms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            lat_ms = float(t.item())
        out[name] = {
            "devices": len(st.devices), "candidates": s.size, "layouts": s.layouts,
            "micro_batches": sp["M"], "token_budget": int(mbs[0].token_budget),
            "candidates_per_s": s.size / (eval_ms * 1e-3), "eval_ms": eval_ms,
            "replan_latency_ms": lat_ms, "best_score_s": score, "best_index": idx,
            "best_plan": None if plan is None else {
                "tp": plan.tp, "dp": plan.dp, "pp": plan.pp, "partition": plan.partition,
                "counts": plan.counts},
        }
        if seqs is not None:
            out[name]["n_sequences"] = int(len(seqs))
            out[name]["latency_includes"] = ("FFD pack of the sequences, quad loads, build_desc, "
                                             "search create, sharded eval, collective, decode, "
                                             "sequence -> replica map")
        else:
            out[name]["latency_includes"] = ("build_desc, search create, sharded eval, "
                                             "collective, decode")
        out[name]["roofline"] = search_roofline(s, sp["M"], out[name]["candidates_per_s"], dev)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            out[name]["cpu_baseline"] = search_cpu_baseline(inputs, s.size)
            out[name]["cpu_baseline_python_reference"] = search_python_reference_baseline(
                st, cfg, mbs, s, k={"C5": 100}.get(name, 1000))
        del s
    return out


# ------------------------------------------------- re-plan: drop-in vs reference
REPLAN_CASES = {
    # name: (T, D, P, layers, micro-batches, fail-slow device, severity)
    "C1": (4, 4, 2, 32, 16, 5, 0.5),
    "C3": (4, 4, 16, 80, 64, 37, 0.4),
}


def _replan_ctx(ns, case, docs):
    """A ResiHPPolicy.plan context (policies.py:53-81) built with the modules
    of `ns` (the reference's or this package's): a confirmed fail-slow device
    with its severity known to the scheduler (SURVEY §8(d) re-plan)."""
    T, D, P, L, M, dev, sev = case
    cfg = ns.cluster.ParallelismConfig(tp=T, dp=D, pp=P, layer_partition=[L // P] * P)
    st = ns.cluster.build_cluster(max(1, T * D * P // 8), 8, cfg, 300.0 * 2**30, 25.0 * 2**30)
    st = ns.cluster.apply_failures(
        st, [ns.cluster.FailureEvent(kind="fail_slow_compute", start=0.0, device=dev,
                                     severity=sev)], 0.0)
    key = next(k for k, g in st.tp_groups.items() if dev in g)
    mbs = ns.workload.pack_sequences([int(x) for x in docs], 4096)[:M]
    conf = ns.detector.ValidationResult(confirmed=True, degraded_stages={key: sev},
                                        degraded_links={}, cost_s=3.0)
    return ns.policies.PlanningContext(
        state=st, cfg=cfg, model=ns.workload.CostModel(alpha=2e-6, beta=5e-10), micro_batches=mbs,
        comm=ns.comm.CommSpec(), known_speeds={dev: sev}, confirmed=conf, capacity=P + 2)


def run_percall(reps=30):
    """Per-call latency of the drop-in API against the reference's Python on
    the same C1-shaped inputs (tools/percall.py in a child process: quad_load,
    predict_chunk_time, build_dag + critical_path, simulate_iteration,
    DetectorState.observe, evaluate_plan)."""
    import subprocess

    r = subprocess.run([sys.executable, str(ROOT / "tools" / "percall.py"), str(reps)],
                       capture_output=True, text=True, timeout=600)
    try:
        return json.loads(r.stdout)
    except ValueError:
        return {"unavailable": (r.stderr or r.stdout)[-300:]}


def run_replan_compare():
    """ResiHPPolicy.plan -- the reference's (baseline/_ref, Python, one host
    core) against this package's drop-in (GPU subgroup / repartition /
    proportional kernels, native plan_migration, GPU evaluate_plan) on the
    same C1 and C3 contexts: wall time of one plan() and whether the two plans
    agree (partition, assignment, subgroups, migrations, predicted makespan)."""
    import importlib
    import types

    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "resilsim").exists():
        return {"unavailable": "baseline/_ref (pip install of /root/reference/pkg) is missing"}
    sys.path.insert(0, str(ref_dir))
    try:
        ref = types.SimpleNamespace(**{m: importlib.import_module(f"resilsim.{m}") for m in
                                       ("cluster", "comm", "workload", "detector", "policies")})
    finally:
        sys.path.remove(str(ref_dir))
    import paper_2605_06374_b200 as pkg

    ours = types.SimpleNamespace(**{m: importlib.import_module(f"paper_2605_06374_b200.{m}")
                                    for m in ("cluster", "comm", "workload", "detector",
                                              "policies")})
    del pkg
    out = {}
    for name, case in REPLAN_CASES.items():
        T, D, P, L, M, *_ = case
        rng = np.random.default_rng([7, M])
        docs = np.clip(np.rint(rng.lognormal(7.2, 0.8, M * 4096 // 1500 + 64)), 1, 4096)
        rctx, octx = _replan_ctx(ref, case, docs), _replan_ctx(ours, case, docs)
        t0 = time.perf_counter()
        rplan = ref.policies.ResiHPPolicy().plan(rctx)
        ref_ms = (time.perf_counter() - t0) * 1e3
        ours.policies.ResiHPPolicy().plan(_replan_ctx(ours, case, docs))  # warm-up
        times = []
        for _ in range(3):
            octx = _replan_ctx(ours, case, docs)
            t0 = time.perf_counter()
            oplan = ours.policies.ResiHPPolicy().plan(octx)
            times.append((time.perf_counter() - t0) * 1e3)
        ours_ms = float(np.median(times))
        same = (rplan.layer_partition == oplan.layer_partition and
                rplan.dp_assignment == oplan.dp_assignment and
                sorted(rplan.tp_subgroups.items()) == sorted(oplan.tp_subgroups.items()) and
                [(m.mb, m.stage, m.source, m.executor) for m in rplan.migrations] ==
                [(m.mb, m.stage, m.source, m.executor) for m in oplan.migrations] and
                np.float64(rplan.predicted_makespan_s).view(np.uint64) ==
                np.float64(oplan.predicted_makespan_s).view(np.uint64))
        out[name] = {"devices": T * D * P, "tp_dp_pp": [T, D, P], "micro_batches": M,
                     "reference_ms": ref_ms, "ours_ms": ours_ms, "speedup": ref_ms / ours_ms,
                     "plans_identical": bool(same), "migrations": len(oplan.migrations),
                     "reference": "baseline/_ref resilsim ResiHPPolicy.plan (Python, 1 core)",
                     "ours": "paper_2605_06374_b200 ResiHPPolicy.plan (drop-in, GPU + native)"}
    return out


_FP64_PEAK = {}


def fp64_peak(dev) -> float:
    """Measured FP64 instruction rate of this device (rh_fp64_peak), cached."""
    if dev.index not in _FP64_PEAK:
        from paper_2605_06374_b200 import _lib

        v = C.c_double()
        _lib.check(_lib.load_library().rh_fp64_peak(_lib.context(dev.index), C.byref(v)),
                   "rh_fp64_peak")
        _FP64_PEAK[dev.index] = v.value
    return _FP64_PEAK[dev.index]


def search_roofline(s, M, cand_per_s, dev, sample=2000):
    """FP64 roofline of the re-plan search: the naive algorithm's fp64 work
    per feasible candidate (V + 2E -- a multiply per chunk, an
    add and a max per DAG edge; V = 2MP (+D all-reduce vertices), E = (2MP -
    DP) chain + 2M(P-1) data (+DP all-reduce) edges), averaged over a
    uniform sample of decoded candidates, times candidates/s, against the
    measured FP64 instruction rate.  The kernels evaluate each (layout,
    partition, replica, first micro-batch, count) pipeline once and share it
    across assignment variants, so this naive-equivalent rate can exceed the
    pipe's peak; DESIGN.md §3.4 gives the measured pipe utilisation."""
    rng = np.random.default_rng(11)
    ops, feas = 0.0, 0
    for _ in range(sample):
        c = s.decode(int(rng.integers(0, s.size)))
        if not c.feasible:
            continue
        feas += 1
        D, P = c.dp, c.pp
        ar = D if D > 1 else 0
        V = 2 * M * P + ar
        E = (2 * M * P - D * P) + 2 * M * (P - 1) + (D * P if D > 1 else 0)
        ops += V + 2 * E
    per_cand = ops / max(1, sample)  # infeasible candidates count as 0 work
    achieved = cand_per_s * per_cand
    peak = fp64_peak(dev)
    return {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
            "unit": "T fp64 ops/s", "frac": achieved / peak,
            "ops_per_candidate": per_cand, "feasible_share": feas / max(1, sample),
            "note": "naive-equivalent work (V + 2E per feasible candidate) / measured "
                    "rh_fp64_peak (DFMA chains); work shared across assignment variants "
                    "lets this exceed 1"}


_PYSB = {}  # the re-plan problem the forked reference workers score


def _py_search_worker(cands):
    """Reference evaluate_plan + reconfig_cost (baseline/_ref) of decoded
    candidates -> (scored, seconds).  Mirrors tests/golden/make_golden.py's
    _ref_score: the plan's TP groups replace the state's, non-members stand
    by, the config keeps the nominal TP degree."""
    ref_dir, prob = _PYSB["ref"], _PYSB["problem"]
    sys.path.insert(0, ref_dir)
    from resilsim import cluster as rc
    from resilsim import pipeline as rp
    from resilsim import scheduler as rs
    from resilsim import workload as rw
    from resilsim.comm import CommSpec

    devs, dpn, groups0, intra, inter, links, T, D, P, sched, part0, mbs, cap = prob
    st = rc.ClusterState(devices=[rc.Device(i, nd, sp, stt) for i, nd, sp, stt in devs],
                         devices_per_node=dpn, tp_groups=dict(groups0), intra_bw=intra,
                         inter_bw=inter, link_factors=dict(links))
    mbs_r = [rw.MicroBatch(id=j, doc_lengths=d, token_budget=n) for j, d, n in mbs]
    model, comm = rw.CostModel(alpha=2e-6, beta=5e-10), CommSpec()
    t0 = time.perf_counter()
    done = 0
    for tp, dp, pp, part, counts, groups in cands:
        st2 = st.copy()
        st2.tp_groups = {(g // pp, g % pp): tuple(m) for g, m in enumerate(groups)}
        members = {m for g in groups for m in g}
        for dev in st2.devices:
            if dev.status != rc.FAIL_STOP:
                dev.status = ((rc.FAIL_SLOW if dev.speed < 1.0 else rc.HEALTHY)
                              if dev.id in members else rc.STANDBY)
        cfg2 = rc.ParallelismConfig(tp=T, dp=dp, pp=pp, schedule=sched, layer_partition=list(part))
        try:
            rs.evaluate_plan(rs.AdaptationPlan(dp_assignment=list(counts)), st2, cfg2, mbs_r,
                             model, comm=comm, capacity=cap)
        except rp.SimulationError:
            pass
        if tp == T and dp == D and pp == P:
            rs.reconfig_cost(rs.AdaptationPlan(layer_partition=list(part)), st, rc.ParallelismConfig(
                tp=T, dp=D, pp=P, schedule=sched, layer_partition=list(part0)),
                layer_bytes=256.0 * 2**20)
        done += 1
    return done, time.perf_counter() - t0


def search_python_reference_baseline(st, cfg, mbs, search, k, budget_s=12.0):
    """The reference's own candidate scoring (SURVEY §8(d) CPU baseline (2)):
    resilsim evaluate_plan + reconfig_cost (baseline/_ref) on k uniformly
    sampled feasible candidates of the benchmarked space, decoded by the
    search, one process per host core (fork; the cli.py:86-92 pattern)."""
    import multiprocessing as mp

    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "resilsim").exists():
        return {"unavailable": "baseline/_ref (pip install of /root/reference/pkg) is missing"}
    rng = np.random.default_rng(7)
    cands = []
    tries = 0
    while len(cands) < k and tries < 50 * k:
        tries += 1
        c = search.decode(int(rng.integers(0, search.size)))
        if c.feasible:
            cands.append((c.tp, c.dp, c.pp, list(c.partition), list(c.counts),
                          [tuple(g) for g in c.groups]))
    _PYSB["ref"] = str(ref_dir)
    _PYSB["problem"] = (
        [(d.id, d.node_id, d.speed, d.status) for d in st.devices], st.devices_per_node,
        dict(st.tp_groups), st.intra_bw, st.inter_bw, dict(st.link_factors), cfg.tp, cfg.dp,
        cfg.pp, cfg.schedule, list(cfg.layer_partition),
        [(mb.id, tuple(mb.doc_lengths), mb.token_budget) for mb in mbs], cfg.pp + 2)
    cores = os.cpu_count() or 1
    # size the sample: one candidate on this core first
    n1, t1 = _py_search_worker(cands[:1])
    k = max(cores, min(len(cands), int(budget_s * cores / max(t1, 1e-4))))
    cands = cands[:k]
    parts = [cands[i::cores] for i in range(cores)]
    wall0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_py_search_worker, parts)
    wall = time.perf_counter() - wall0
    n = sum(r[0] for r in res)
    return {"value": n / wall, "unit": "candidates/s", "cores": cores, "kind": "reference",
            "sample": f"{n} uniformly sampled feasible candidates, resilsim evaluate_plan + "
                      "reconfig_cost (baseline/_ref) per candidate, one process per core; "
                      "includes worker start-up",
            "per_candidate_ms_one_core": t1 * 1e3}


def search_cpu_baseline(inputs, size, budget_s=4.0):
    """Oracle re-plan scoring on all host cores over a bounded contiguous sample."""
    from tests.oracle_bind import Oracle

    o = Oracle().search(inputs)
    cores = os.cpu_count() or 1
    k = 256
    while True:  # grow the sample until it costs ~budget_s
        mid = size // 3
        t0 = time.perf_counter()
        o.best(mid, min(size, mid + k), threads=cores)
        dt = time.perf_counter() - t0
        if dt > budget_s / 4 or mid + k >= size:
            break
        k *= 4
    return {"value": k / dt, "unit": "candidates/s", "cores": cores, "kind": "port",
            "sample": f"{k} contiguous candidates from index {size // 3} (oracle: build_dag + "
                      "Kahn per candidate, pthreads)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-scheduler", action="store_true")
    ap.add_argument("--no-replan", action="store_true",
                    help="skip the drop-in vs reference ResiHPPolicy.plan comparison")
    ap.add_argument("--no-trace-r", action="store_true", help="skip the C5-shape trace R sample")
    ap.add_argument("--scheduler-only", default="", help="comma list of C3,C4,C5: only these")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if args.scheduler_only:
        import torch

        torch.cuda.set_device(local)
        res = run_scheduler(args, world, rank, local, tuple(args.scheduler_only.split(",")))
        if rank == 0:
            print(json.dumps({"scheduler": res}), flush=True)
        return
    line, tr = run_ours(args, world, rank, local)
    if world == 1 and not args.no_trace_r:
        import torch

        line["trace_R"] = run_trace_r(args, torch.device("cuda", local))
    if not args.no_scheduler:
        line["scheduler"] = run_scheduler(args, world, rank, local)
    if rank == 0 and world == 1 and not args.no_replan:
        line["replan"] = run_replan_compare()
        line["percall"] = run_percall()
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(tr)
            line["cpu_baseline_python_reference"] = python_reference_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
