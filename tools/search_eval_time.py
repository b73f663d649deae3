"""Event-timed re-plan search eval on the C3/C4/C5 spaces (A/B of builds; debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_06374_b200.replan_scenarios import replan_problem  # noqa: E402
from paper_2605_06374_b200.search import ReplanSearch  # noqa: E402

out = []
for name in sys.argv[1:] or ["C3", "C4", "C5"]:
    st, cfg, mbs, inputs = replan_problem(name)
    s = ReplanSearch(inputs, torch.device("cuda", 0))
    best = s.best()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.eval_async()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    out.append(f"{name} eval median {ts[3]:.3f} ms min {ts[0]:.3f} best {best}")
print(" | ".join(out))
