"""The structural property the shuffle wavefront (csrc/wavefront.cuh) relies on.

In the canonical 1F1B / ZBH chunk DAG (pipeline.py:92-256), process every
vertex at its level (longest path from a source, in vertices) — exactly the
step at which the dynamic wavefront processes it.  Then
  (i)  B(j, s) is always one level after B(j, s+1), and
  (ii) F(j+1, s-1) is never before F(j, s): a producer stage never runs more
       than one forward ahead of its consumer,
so "the last value the neighbour produced" is always the needed one.
Exhaustive over the shapes below (the kernel also detects violations).
"""

import pytest

from paper_2605_06374_b200.pipeline import schedule_1f1b, schedule_zbh


def levels(P, M, zbh):
    seqs = [(schedule_zbh if zbh else schedule_1f1b)(P, s, list(range(M))) for s in range(P)]
    back = "B" if zbh else "BW"
    lev = {}
    ptr = [0] * P
    # process in wavefront order: repeatedly advance every stage whose next
    # vertex has its data dependency levelled
    remaining = sum(len(q) for q in seqs)
    prev = [-1] * P
    while remaining:
        progressed = False
        for s in range(P):
            if ptr[s] == len(seqs[s]):
                continue
            kind, j = seqs[s][ptr[s]]
            dep = None
            if kind == "F" and s > 0:
                dep = ("F", j, s - 1)
            elif kind == back and s < P - 1:
                dep = (back, j, s + 1)
            elif kind == "W":
                dep = ("B", j, s)
            if dep is not None and dep not in lev:
                continue
            lv = max(prev[s] + 1, lev[dep] + 1 if dep is not None else 0)
            lev[(kind, j, s)] = lv
            prev[s] = lv
            ptr[s] += 1
            remaining -= 1
            progressed = True
        assert progressed, "canonical DAG must be acyclic"
    return lev


@pytest.mark.parametrize("zbh", [False, True])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8, 13, 16, 32])
def test_lead_bound(P, zbh):
    back = "B" if zbh else "BW"
    for M in list(range(1, 25)) + [31, 40, 64]:
        lev = levels(P, M, zbh)
        for s in range(P - 1):
            for j in range(M):
                assert lev[(back, j, s)] == lev[(back, j, s + 1)] + 1
        for s in range(1, P):
            for j in range(M - 1):
                assert lev[("F", j + 1, s - 1)] >= lev[("F", j, s)]
