"""Break the re-plan latency of bench.py's scheduler configs into its parts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_06374_b200.replan_scenarios import replan_problem  # noqa: E402
from paper_2605_06374_b200.search import ReplanSearch  # noqa: E402

dev = torch.device("cuda", 0)
for name in ("C3", "C4", "C5"):
    st, cfg, mbs, inputs = replan_problem(name)
    s = ReplanSearch(inputs, dev)
    s.best()
    del s
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = ReplanSearch(inputs, dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        b, i = s.best()
        t2 = time.perf_counter()
        plan = s.decode(i)
        t3 = time.perf_counter()
        del s
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        print(f"{name} rep{rep}: create {1e3*(t1-t0):6.2f} ms  eval+minloc {1e3*(t2-t1):6.2f}"
              f"  decode {1e3*(t3-t2):5.2f}  destroy {1e3*(t4-t3):5.2f}")
