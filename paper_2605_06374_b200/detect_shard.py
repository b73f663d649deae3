"""One Detector trace sharded over the ranks of a process group.

The predictor / residual pass is per iteration, so rank r takes a contiguous
range [a_r, b_r) of the trace's iterations.  The DetectorState.observe state
machine (detector.py:182-271) is sequential along the series, but its whole
state at an iteration is (series length since the last reset, the last
`window` kept observations): that is what crosses a shard boundary.

* Cuts are placed on adaptation boundaries when the trace has them: a series
  reset (harness.py:398) starts an independent series, so a shard that begins
  with a reset screens with no input at all (`shard_bounds`).
* Any other cut hands the state over: rank r screens its range once the rank
  before it has sent (series length, visible tail) -- `screen_handoff`, one
  small point-to-point message per boundary, the chain only as long as the
  run of cuts without a reset.

`screen_fn(observed, status, reset, series_len, hist) -> (outcome, series_len)`
is rh_screen on the GPU (detector._screen); the CPU tests pass the oracle.
"""

from __future__ import annotations

import numpy as np

from ._lib import RH_SC_POPPED


def shard_bounds(n: int, world: int, reset=None, slack: float = 0.25) -> list[tuple[int, int]]:
    """Contiguous shards of [0, n): the even split, each interior cut moved to
    the first reset within `slack` of a shard length after it (an independent
    series start) when there is one."""
    cuts = [0]
    reset = None if reset is None else np.asarray(reset, dtype=bool)
    step = n / max(1, world)
    for r in range(1, world):
        c = int(round(r * step))
        if reset is not None:
            hi = min(n, c + int(slack * step))
            nz = np.flatnonzero(reset[c:hi])
            if nz.size:
                c += int(nz[0])
        cuts.append(max(cuts[-1], min(n, c)))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def tail_state(observed, outcome, reset, series_len: int, hist, window: int):
    """(series length, last `window` kept observations) after a shard, from
    its outcome bits: an observation stays in the series unless popped; a
    reset clears it first (detector.py:198-271, harness.py:398)."""
    tail = list(hist[len(hist) - min(len(hist), series_len, window):]) if series_len else []
    length = int(series_len)
    popped = (np.asarray(outcome) & RH_SC_POPPED) != 0
    rst = np.zeros(len(observed), bool) if reset is None else np.asarray(reset, bool)
    start = 0
    last_reset = np.flatnonzero(rst)
    if last_reset.size:
        start = int(last_reset[-1])
        tail, length = [], 0
    kept = np.asarray(observed[start:], dtype=np.float64)[~popped[start:]]
    length += int(kept.size)
    tail = (tail + kept.tolist())[-window:]
    return length, tail


def screen_handoff(observed, status, reset, bounds, rank: int, screen_fn, *, window: int = 20,
                   group=None, series_len: int = 0, hist=()):
    """Rank `rank`'s outcomes for its shard bounds[rank] of one series.

    A shard that starts with a reset screens from an empty series; otherwise
    it receives (series length, visible tail) from rank - 1.  Every rank sends
    its end state to rank + 1 unless that shard starts with a reset.  The
    result equals screening the whole trace in one pass, bit for bit."""
    import torch
    import torch.distributed as dist

    world = len(bounds)
    a, b = bounds[rank]
    obs = np.asarray(observed[a:b], dtype=np.float64)
    st = np.asarray(status[a:b], dtype=np.uint8)
    rst = None if reset is None else np.asarray(reset[a:b], dtype=np.uint8)
    starts_fresh = rank == 0 or (rst is not None and b > a and rst[0])
    L0, h0 = int(series_len), list(hist)
    if rank > 0 and not starts_fresh:
        msg = torch.zeros(2 + window, dtype=torch.float64)
        dist.recv(msg, src=rank - 1, group=group)
        L0 = int(msg[0].item())
        h0 = msg[2:2 + int(msg[1].item())].tolist()
    if b > a:
        oc, _ = screen_fn(obs, st, rst, L0, h0)
    else:
        oc = np.zeros(0, np.uint8)
    if rank + 1 < world:
        na, nbnd = bounds[rank + 1]
        nxt_fresh = reset is not None and nbnd > na and reset[na]
        if not nxt_fresh:
            L1, t1 = tail_state(obs, oc, rst, L0, h0, window)
            msg = torch.zeros(2 + window, dtype=torch.float64)
            msg[0], msg[1] = float(L1), float(len(t1))
            if t1:
                msg[2:2 + len(t1)] = torch.tensor(t1, dtype=torch.float64)
            dist.send(msg, dst=rank + 1, group=group)
    return oc


class ShardedDetectorPass:
    """This rank's shard of one trace on its GPU: the fused predictor /
    residual pass (rh_detect_batch) over iterations bounds[rank], then the
    screen with the boundary hand-off.  Outcomes of all ranks together equal
    the single-pass DetectorPass."""

    def __init__(self, trace, rank: int, world: int, device=None, *, group=None,
                 window: int = 20, kappa: float = 3.0, filter_enabled: bool = True):
        from .detect_pass import DetectorPass

        self.bounds = shard_bounds(trace.n_iter, world, trace.reset)
        self.rank, self.group = rank, group
        self.window, self.kappa, self.fe = window, kappa, filter_enabled
        a, b = self.bounds[rank]
        self.trace = trace
        self.local = trace.slice(a, b)
        self.pass_ = DetectorPass(self.local, device, window=window, kappa=kappa,
                                  filter_enabled=filter_enabled)

    def detect(self):
        self.pass_.detect(prepare_screen=False)

    def screen(self) -> np.ndarray:
        """This shard's DetectorState.observe outcome bits (rh_screen)."""
        from .detector import _screen

        st = self.pass_.status.cpu().numpy()
        a, b = self.bounds[self.rank]
        n = self.trace.n_iter
        status = np.zeros(n, np.uint8)
        status[a:b] = st

        def fn(obs, s, rst, L, hist):
            return _screen(L, list(hist), obs, s, self.window, self.kappa, self.fe, reset=rst)

        return screen_handoff(self.trace.observed, status, self.trace.reset, self.bounds,
                              self.rank, fn, window=self.window, group=self.group)
