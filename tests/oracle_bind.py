"""ctypes binding of the CPU oracle (oracle/liboracle.so) — test infrastructure.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use it.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2605_06374_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
ORACLE_LIB = ROOT / "oracle" / "liboracle.so"


def _ptr(a):
    return None if a is None else a.ctypes.data


class HostSegments:
    """Segment tables stacked in host memory (C-ABI layout)."""

    def __init__(self, segments):
        def cat(name, dtype):
            arrs = [getattr(s, name) for s in segments]
            a = np.concatenate(arrs).astype(dtype) if arrs else np.zeros(0, dtype)
            return np.ascontiguousarray(a if a.size else np.zeros(1, dtype))

        self.layers = cat("layers", np.int32)
        self.mb_start = cat("mb_start", np.int32)
        self.speed = cat("speed", np.float64)
        self.hop_fwd = cat("hop_fwd", np.float64)
        self.hop_bwd = cat("hop_bwd", np.float64)
        self.allreduce = cat("allreduce", np.float64)
        off = np.zeros(len(segments) + 1, dtype=np.int32)
        np.cumsum([len(s.link_ratio) for s in segments], out=off[1:])
        self.link_off = off
        self.link_ratio = cat("link_ratio", np.float64)
        self.max_mb = int(max((np.diff(s.mb_start).max() for s in segments), default=0))
        self.c = _lib.Segments(len(segments), _ptr(self.layers), _ptr(self.mb_start),
                               _ptr(self.speed), _ptr(self.hop_fwd), _ptr(self.hop_bwd),
                               _ptr(self.allreduce), _ptr(self.link_off),
                               _ptr(self.link_ratio))


class Oracle:
    def __init__(self):
        if not ORACLE_LIB.exists():
            import __graft_entry__ as g

            g.build_oracle()
        self.lib = C.CDLL(str(ORACLE_LIB))
        p = C.c_void_p
        L = self.lib
        L.orc_pack_sequences.argtypes = [C.c_int64, p, C.c_int32, C.c_int64, p, p,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_pack_sequences.restype = C.c_int
        L.orc_quad_load.argtypes = [C.c_int32, p]
        L.orc_quad_load.restype = C.c_int64
        L.orc_chunk_time.argtypes = [C.POINTER(_lib.CostModelC), C.c_int, C.c_int64, C.c_int32,
                                     C.c_int32, C.c_double, C.POINTER(C.c_int)]
        L.orc_chunk_time.restype = C.c_double
        L.orc_critical_path.argtypes = [C.c_int32, p, C.c_int32, p, p, p, p, p]
        L.orc_critical_path.restype = C.c_int
        for name in ("orc_pipeline_batch",):
            f = getattr(L, name)
            f.argtypes = [C.POINTER(_lib.PipeShape), C.POINTER(_lib.CostModelC),
                          C.POINTER(_lib.Segments), C.POINTER(_lib.Trace),
                          C.POINTER(_lib.PassOut), C.c_int]
            f.restype = C.c_int
        L.orc_detect_batch.argtypes = [C.POINTER(_lib.PipeShape), C.POINTER(_lib.CostModelC),
                                       C.POINTER(_lib.Segments), C.POINTER(_lib.Trace),
                                       C.c_double, C.POINTER(_lib.PassOut), C.c_int]
        L.orc_detect_batch.restype = C.c_int
        L.orc_validate.argtypes = [C.c_int64, p, p, C.c_double, p, p]
        L.orc_validate.restype = C.c_int
        L.orc_change_point.argtypes = [C.c_int64, p, C.c_int, C.c_double]
        L.orc_change_point.restype = C.c_int
        L.orc_screen.argtypes = [C.POINTER(_lib.ScreenParams), C.c_int64, p, C.c_int64, p, p,
                                 p, p, C.POINTER(C.c_int64)]
        L.orc_screen.restype = C.c_int
        from paper_2605_06374_b200.search import Candidate, SearchDesc

        L.orc_search_create.argtypes = [C.POINTER(SearchDesc)]
        L.orc_search_create.restype = p
        L.orc_search_destroy.argtypes = [p]
        L.orc_search_size.argtypes = [p]
        L.orc_search_size.restype = C.c_int64
        L.orc_search_score.argtypes = [p, C.c_int64]
        L.orc_search_score.restype = C.c_double
        L.orc_search_eval.argtypes = [p, C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_double),
                                      C.POINTER(C.c_int64), p]
        L.orc_search_eval_memo.argtypes = L.orc_search_eval.argtypes
        L.orc_search_decode.argtypes = [p, C.c_int64, C.POINTER(Candidate), p, p, p]

    # ------------------------------------------------------------ search
    def search(self, inputs):
        return OracleSearch(self, inputs)

    # ------------------------------------------------------------ scalar
    def quad_load(self, docs) -> int:
        a = np.ascontiguousarray(docs, dtype=np.int32)
        return int(self.lib.orc_quad_load(len(a), _ptr(a)))

    def chunk_time(self, model_c, kind: int, quad: int, budget: int, layers: int,
                   speed: float) -> float:
        bad = C.c_int(0)
        t = self.lib.orc_chunk_time(C.byref(model_c), kind, quad, budget, layers, speed,
                                    C.byref(bad))
        if bad.value:
            raise ValueError("speed <= 0")
        return t

    def critical_path(self, cost, src, dst, w):
        cost = np.ascontiguousarray(cost, np.float64)
        src = np.ascontiguousarray(src, np.int32)
        dst = np.ascontiguousarray(dst, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        starts = np.zeros(max(len(cost), 1))
        ms = C.c_double()
        cyc = self.lib.orc_critical_path(len(cost), _ptr(cost), len(src), _ptr(src), _ptr(dst),
                                         _ptr(w), _ptr(starts), C.byref(ms))
        return starts[:len(cost)], ms.value, bool(cyc)

    # ------------------------------------------------------------ batches
    def _trace_c(self, trace, detect):
        keep = []

        def a(x, dt):
            if x is None:
                return None
            x = np.ascontiguousarray(x, dtype=dt)
            keep.append(x)
            return x.ctypes.data

        tr = _lib.Trace(trace.n_iter, a(trace.seg, np.int32), a(trace.mb_off, np.int32),
                        a(trace.doc_len if trace.doc_len.size else np.zeros(1), np.int32),
                        a(trace.device_time, np.float32) if detect else None,
                        a(trace.observed, np.float64) if detect else None)
        return tr, keep

    def pack_sequences(self, lengths, budget, max_bins=-1):
        """workload.py:52-80 (literal FFD) -> (mb_off, doc_len), the
        rh_pack_sequences contract: a drop-in `packer` for synth_iterations."""
        v = np.ascontiguousarray(lengths, dtype=np.int32)
        nb, ne = C.c_int64(), C.c_int64()
        if self.lib.orc_pack_sequences(len(v), _ptr(v), int(budget), int(max_bins), None, None,
                                       C.byref(nb), C.byref(ne)):
            raise ValueError("orc_pack_sequences: document length outside [1, budget]")
        off = np.zeros(nb.value + 1, np.int32)
        docs = np.zeros(max(ne.value, 1), np.int32)
        self.lib.orc_pack_sequences(len(v), _ptr(v), int(budget), int(max_bins), _ptr(off),
                                    _ptr(docs), C.byref(nb), C.byref(ne))
        return off, docs[:ne.value]

    def pipeline(self, trace, view="known", capacity=None, threads=0):
        segs = HostSegments(trace.known if view == "known" else trace.actual)
        shape = pipe_shape_of(trace, capacity, segs.max_mb)
        tr, keep = self._trace_c(trace, False)
        n, G = trace.n_iter, trace.cfg.dp * trace.cfg.pp
        ms = np.zeros(n)
        st = np.zeros(n, np.uint8)
        sc = np.zeros(n * G)
        out = _lib.PassOut(_ptr(ms), _ptr(st), _ptr(sc), None, None)
        self.lib.orc_pipeline_batch(C.byref(shape), C.byref(model_c_of(trace.model)),
                                    C.byref(segs.c), C.byref(tr), C.byref(out), threads)
        return ms, st, sc.reshape(n, G)

    def detect(self, trace, threshold=1.25, threads=0):
        segs = HostSegments(trace.known)
        shape = pipe_shape_of(trace, None, segs.max_mb)
        tr, keep = self._trace_c(trace, True)
        n, G = trace.n_iter, trace.cfg.dp * trace.cfg.pp
        ms = np.zeros(n)
        st = np.zeros(n, np.uint8)
        sc = np.zeros(n * G)
        fl = np.zeros(n * G, np.uint8)
        sv = np.zeros(n * G, np.float32)
        out = _lib.PassOut(_ptr(ms), _ptr(st), _ptr(sc), _ptr(fl), _ptr(sv))
        self.lib.orc_detect_batch(C.byref(shape), C.byref(model_c_of(trace.model)),
                                  C.byref(segs.c), C.byref(tr), threshold, C.byref(out), threads)
        return ms, st, sc.reshape(n, G), fl.reshape(n, G), sv.reshape(n, G)

    def screen(self, observed, it_status, window=20, kappa=3.0, filter_enabled=True,
               series_len=0, hist=None, reset=None):
        obs = np.ascontiguousarray(observed, np.float64)
        st = np.ascontiguousarray(it_status, np.uint8)
        h = np.ascontiguousarray(hist if hist is not None and len(hist) else [0.0], np.float64)
        rs = None if reset is None else np.ascontiguousarray(reset, np.uint8)
        oc = np.zeros(max(len(obs), 1), np.uint8)
        ln = C.c_int64()
        params = _lib.ScreenParams(window, 1 if filter_enabled else 0, kappa)
        self.lib.orc_screen(C.byref(params), series_len, _ptr(h), len(obs), _ptr(obs), _ptr(st),
                            _ptr(rs), _ptr(oc), C.byref(ln))
        return oc[:len(obs)], ln.value

    def change_point(self, series, window=20, kappa=3.0):
        s = np.ascontiguousarray(series, np.float64)
        return bool(self.lib.orc_change_point(len(s), _ptr(s), window, kappa))


def model_c_of(model):
    from paper_2605_06374_b200.workload import cost_model_c

    return cost_model_c(model)


def pipe_shape_of(trace, capacity, max_mb):
    from paper_2605_06374_b200.tables import pipe_shape

    return pipe_shape(trace.cfg, trace.M, trace.N, capacity=capacity,
                      has_allreduce=trace.has_allreduce, max_mb=max_mb)


class OracleSearch:
    """CPU restatement of the re-plan search (oracle/search_oracle.c)."""

    def __init__(self, oracle: Oracle, inputs):
        self.o, self.inputs = oracle, inputs
        self.h = oracle.lib.orc_search_create(C.byref(inputs.desc))
        self.size = int(oracle.lib.orc_search_size(self.h))

    def __del__(self):
        try:
            self.o.lib.orc_search_destroy(self.h)
        except Exception:
            pass

    def score(self, index: int) -> float:
        return float(self.o.lib.orc_search_score(self.h, int(index)))

    def best(self, begin=0, end=None, threads=0, with_scores=False):
        end = self.size if end is None else end
        b, i = C.c_double(), C.c_int64()
        sc = np.zeros(max(end - begin, 1)) if with_scores else None
        self.o.lib.orc_search_eval(self.h, begin, end, threads, C.byref(b), C.byref(i),
                                   None if sc is None else sc.ctypes.data)
        return (b.value, i.value, sc[:end - begin]) if with_scores else (b.value, i.value)

    def best_memo(self, begin=0, end=None, threads=0, with_scores=False):
        """orc_search_eval_memo: the same scores / winner, replica pipelines
        memoised across assignment variants (full-space scans at C3-C5)."""
        end = self.size if end is None else end
        b, i = C.c_double(), C.c_int64()
        sc = np.zeros(max(end - begin, 1)) if with_scores else None
        self.o.lib.orc_search_eval_memo(self.h, begin, end, threads, C.byref(b), C.byref(i),
                                        None if sc is None else sc.ctypes.data)
        return (b.value, i.value, sc[:end - begin]) if with_scores else (b.value, i.value)

    def decode(self, index: int):
        from paper_2605_06374_b200.search import Candidate, CandidatePlan

        c = Candidate()
        groups = np.zeros(self.inputs.desc.n_devices + 1, np.int32)
        part = np.zeros(64, np.int32)
        cnt = np.zeros(128, np.int32)
        self.o.lib.orc_search_decode(self.h, int(index), C.byref(c), groups.ctypes.data,
                                     part.ctypes.data, cnt.ctypes.data)
        g = [tuple(int(x) for x in groups[k * c.tp:(k + 1) * c.tp]) for k in range(c.dp * c.pp)]
        return CandidatePlan(int(c.index), c.tp, c.dp, c.pp, part[:c.pp].tolist(),
                             cnt[:c.dp].tolist(), g, c.partition_variant, c.count_variant,
                             bool(c.feasible))
