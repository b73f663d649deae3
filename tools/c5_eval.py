"""One C5 re-plan eval (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_06374_b200.replan_scenarios import replan_problem  # noqa: E402
from paper_2605_06374_b200.search import ReplanSearch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
st, cfg, mbs, inputs = replan_problem(name)
s = ReplanSearch(inputs, torch.device("cuda", 0))
print(s.best())
