"""Device x iteration traces for the batched Detector pass.

A trace holds, in the C-ABI layout of include/resihp_b200.h:
  * the packed micro-batches of every iteration (int32 CSR of doc lengths),
  * segment tables of the KNOWN view (what the predictor believes) and of
    the ACTUAL view (ground truth used to synthesise measurements),
  * measured per-device stage times (float32 [n, D, P, T]) and observed
    iteration times (float64 [n]),
  * series-reset flags at adaptation boundaries (harness.py:398).

Synthetic workloads follow harness._DocSource (harness.py:235-263):
lognormal(mean, sigma) lengths rounded half-to-even and clipped to [1, N],
drawn until the iteration's token target is met, FFD-packed, first M bins.
Measurements follow harness.py:424-427: stage_cost * (1 + sigma * N(0,1)).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .tables import Segment


def pack_ffd(lengths: np.ndarray, budget: int, max_bins: int = -1):
    """pack_sequences via the native rh_pack_sequences -> (mb_off, doc_len),
    one call (outputs sized for the worst case: a bin per document plus its
    padding entry)."""
    lib = _lib.load_library()
    lengths = np.ascontiguousarray(lengths, dtype=np.int32)
    n = len(lengths)
    nb, ne = C.c_int64(), C.c_int64()
    off = np.empty(n + 2, dtype=np.int32)
    docs = np.empty(2 * n + 1, dtype=np.int32)
    _lib.check(lib.rh_pack_sequences(n, lengths.ctypes.data, int(budget), int(max_bins),
                                     off.ctypes.data, docs.ctypes.data, C.byref(nb),
                                     C.byref(ne)), "rh_pack_sequences")
    return off[:nb.value + 1], docs[:ne.value]


def draw_documents(rng: np.random.Generator, target_tokens: int, budget: int, mean: float,
                   sigma: float) -> np.ndarray:
    """Lengths drawn until their sum reaches target_tokens (harness.py:243-263)."""
    out = []
    total = 0
    est = max(8, int(target_tokens / max(1.0, np.exp(mean + sigma * sigma / 2)) * 1.2) + 8)
    while total < target_tokens:
        raw = rng.lognormal(mean, sigma, size=est)
        x = np.clip(np.rint(raw), 1, budget).astype(np.int64)
        cs = total + np.cumsum(x)
        k = int(np.searchsorted(cs, target_tokens, side="left"))
        if k < len(x):
            out.append(x[:k + 1])
            total = int(cs[k])
        else:
            out.append(x)
            total = int(cs[-1])
    return np.concatenate(out)


def synth_iterations(n_iter: int, M: int, N: int, mean: float, sigma: float, seed: int,
                     packer=None):
    """Packed micro-batches of n_iter iterations -> (mb_off[n*M+1], doc_len).

    `packer(lengths, budget, max_bins) -> (off, docs)` defaults to the native
    pack_ffd; bench.py's reference arm passes the oracle's literal FFD so that
    process never loads the product library."""
    packer = packer or pack_ffd
    rng = np.random.default_rng([seed, 0])
    offs, docs = [np.zeros(1, np.int64)], []
    base = 0
    for _ in range(n_iter):
        lengths = draw_documents(rng, M * N, N, mean, sigma)
        off, d = packer(lengths, N, M)
        if len(off) - 1 < M:
            raise ValueError("workload produced fewer than M micro-batches")
        offs.append(off[1:].astype(np.int64) + base)
        docs.append(d)
        base += int(off[-1])
    mb_off = np.concatenate(offs)
    if mb_off[-1] >= 2**31:
        raise ValueError("trace too large for int32 document offsets")
    return mb_off.astype(np.int32), np.concatenate(docs).astype(np.int32)


@dataclass
class DetectorTrace:
    cfg: object
    model: object
    M: int
    N: int
    has_allreduce: bool
    seg: np.ndarray
    mb_off: np.ndarray
    doc_len: np.ndarray
    known: list[Segment]
    actual: list[Segment]
    reset: np.ndarray
    device_time: np.ndarray | None = None
    observed: np.ndarray | None = None
    group_size: np.ndarray | None = None   # [n_seg, D*P] members per group
    meta: dict = field(default_factory=dict)

    @property
    def n_iter(self) -> int:
        return len(self.seg)

    def nbytes_per_iter(self) -> dict:
        """Algorithmic HBM bytes of one Detector-pass iteration."""
        D, P, T = self.cfg.dp, self.cfg.pp, self.cfg.tp
        G = D * P
        n = self.n_iter
        docs = self.doc_len.size * 4 / n
        return {
            "doc_len": docs,
            "mb_off": 4.0 * self.M,
            "seg": 4.0,
            "device_time": 4.0 * G * T,
            "observed": 8.0,
            "out_makespan_status": 9.0,
            "out_flag_severity": 5.0 * G,
        }

    def slice(self, a: int, b: int) -> "DetectorTrace":
        """Iterations [a, b) as a trace of their own (offsets rebased; the
        segment tables are shared) -- one rank's shard (detect_shard.py)."""
        import copy

        M = self.M
        out = copy.copy(self)
        off = np.asarray(self.mb_off[a * M:b * M + 1], dtype=np.int64)
        lo, hi = int(off[0]), int(off[-1])
        out.mb_off = (off - lo).astype(np.int32)
        out.doc_len = np.ascontiguousarray(self.doc_len[lo:hi])
        out.seg = np.ascontiguousarray(self.seg[a:b])
        out.reset = np.ascontiguousarray(self.reset[a:b])
        if self.device_time is not None:
            out.device_time = np.ascontiguousarray(self.device_time[a:b])
        if self.observed is not None:
            out.observed = np.ascontiguousarray(self.observed[a:b])
        return out

    def packed(self) -> dict:
        """The packed wire form (rh_trace_packed): per-iteration document
        offsets (int32), documents per micro-batch (uint8) and document
        lengths (uint16).  Raises ValueError when the trace does not fit it."""
        n, M = self.n_iter, self.M
        off = np.asarray(self.mb_off, dtype=np.int64)
        counts = np.diff(off)
        if counts.size and (counts.max() > 255 or counts.min() < 0):
            raise ValueError("packed trace: a micro-batch holds more than 255 documents")
        if self.doc_len.size and (self.doc_len.max() > 65535 or self.doc_len.min() < 0):
            raise ValueError("packed trace: a document is longer than 65535 tokens")
        return {
            "iter_doc": np.ascontiguousarray(off[::M][:n + 1], dtype=np.int32),
            "mb_docs": np.ascontiguousarray(counts, dtype=np.uint8),
            "doc_len": np.ascontiguousarray(self.doc_len, dtype=np.uint16),
        }

    def attach_measurements(self, stage_cost_actual: np.ndarray, observed: np.ndarray,
                            noise: float = 0.01, seed: int = 1) -> None:
        """device_time from the ground-truth stage costs (harness.py:424-427):
        the group's slowest member reports stage_cost*(1+noise*N(0,1)) rounded
        to float32; the other members report a random 90-100% of it."""
        D, P, T = self.cfg.dp, self.cfg.pp, self.cfg.tp
        n, G = self.n_iter, D * P
        rng = np.random.default_rng([seed, 1])
        sc = np.asarray(stage_cost_actual, dtype=np.float64).reshape(n, G)
        noisy = (sc * (1.0 + noise * rng.standard_normal((n, G)))).astype(np.float32)
        dt = noisy[:, :, None] * rng.uniform(0.9, 1.0, (n, G, T)).astype(np.float32)
        gsz = (self.group_size[self.seg] if self.group_size is not None
               else np.full((n, G), T, dtype=np.int64))
        slowest = (rng.random((n, G)) * gsz).astype(np.int64)
        np.put_along_axis(dt, slowest[:, :, None], noisy[:, :, None], axis=2)
        dt[np.arange(T)[None, None, :] >= gsz[:, :, None]] = 0.0
        dt[sc <= 0.0] = 0.0
        self.device_time = np.ascontiguousarray(dt.reshape(n, D, P, T))
        self.observed = np.asarray(observed, dtype=np.float64).copy()
