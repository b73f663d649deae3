"""Wall-clock breakdown of the C5 re-plan from 10^5 sequences (GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_06374_b200.comm import CommSpec  # noqa: E402
from paper_2605_06374_b200.replan_scenarios import (SPECS, _Budget, pack_workload,  # noqa: E402
                                                    replan_problem, sequence_workload)
from paper_2605_06374_b200.search import ReplanSearch, build_desc  # noqa: E402
from paper_2605_06374_b200.workload import CostModel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
sp = SPECS[name]
st, cfg, mbs, inputs = replan_problem(name)
docs, N = sequence_workload(sp["n_sequences"], sp["M"])
dev = torch.device("cuda", 0)
model, comm = CostModel(2e-6, 5e-10), CommSpec()
kw = dict(capacity=cfg.pp + 2, min_utilization=sp["min_utilization"], max_dp=sp["max_dp"])
for rep in range(4):
    t = [time.perf_counter()]
    off, packed, quad = pack_workload(docs, N, sp["M"])
    t.append(time.perf_counter())
    inp = build_desc(st, cfg, [_Budget(N)] * sp["M"], model, comm, quad=quad, **kw)
    t.append(time.perf_counter())
    s = ReplanSearch(inp, dev)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    b, i = s.best()
    t.append(time.perf_counter())
    plan = s.decode(i)
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"pack {d[0]:.2f} ms  build_desc {d[1]:.2f}  create {d[2]:.2f}  eval+sync {d[3]:.2f}  "
          f"decode {d[4]:.2f}  total {sum(d):.2f}")
from paper_2605_06374_b200.replan_scenarios import replan_from_sequences  # noqa: E402

for rep in range(4):
    t0 = time.perf_counter()
    plan, score, idx, er, srch = replan_from_sequences(st, cfg, docs, N, sp["M"], model, comm,
                                                        device=dev, **kw)
    torch.cuda.synchronize()
    print(f"replan_from_sequences (FFD overlapped with create): {(time.perf_counter() - t0) * 1e3:.2f} ms")
    del srch
