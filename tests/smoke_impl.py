"""__graft_entry__.smoke(): one small Detector pass on cuda:0 vs the oracle."""

from __future__ import annotations

import numpy as np


def run_smoke() -> None:
    import torch

    from paper_2605_06374_b200 import _lib
    from paper_2605_06374_b200.detect_pass import DetectorPass
    from tests.helpers import random_trace, with_measurements
    from tests.oracle_bind import Oracle

    assert torch.cuda.is_available(), "smoke() needs cuda:0"
    torch.cuda.set_device(0)
    oracle = Oracle()
    tr = with_measurements(random_trace(7, n_iter=64, tp=4, dp=4, pp=2, M=16, comm=True),
                           oracle, noise=0.02)
    p = DetectorPass(tr)
    p.run()
    torch.cuda.synchronize()
    r = p.results()
    oms, ost, _, ofl, _ = oracle.detect(tr)
    ooc, oln = oracle.screen(tr.observed, ost, reset=tr.reset)
    assert np.array_equal(r["makespan"].view(np.uint64), oms.view(np.uint64)), "makespan"
    assert np.array_equal(r["status"], ost), "status"
    assert np.array_equal(r["stage_flag"], ofl), "flags"
    assert np.array_equal(r["outcome"], ooc) and r["series_len"] == oln, "screen"
    # a long pipeline (the trace-R / C3-C5 kernel, pass_wide_kernel) ...
    tw = with_measurements(random_trace(11, n_iter=40, tp=8, dp=8, pp=16, M=136, comm=True,
                                        schedule="1f1b"), oracle, noise=0.02)
    pw = DetectorPass(tw)
    pw.detect()
    rw = pw.results()
    wms, wst, *_ = oracle.detect(tw)
    assert np.array_equal(rw["makespan"].view(np.uint64), wms.view(np.uint64)), "wide makespan"
    assert np.array_equal(rw["status"], wst), "wide status"
    # ... and one re-plan search (register walks, combine2, min-loc)
    from paper_2605_06374_b200.search import ReplanSearch
    from tests.golden_io import load, search_problem

    case = load("search")["cases"][0]
    *_, inputs = search_problem(case)
    assert list(ReplanSearch(inputs).best()) == case["best"], "search winner"
    print(f"smoke ok: {tr.n_iter} + {tw.n_iter} iterations bit-exact, search winner, "
          f"{_lib.launches()} launches")
