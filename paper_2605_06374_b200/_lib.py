"""ctypes binding of libresihp_b200.so (the C ABI in include/resihp_b200.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
fallback: if the shared object is missing, or no sm_100 GPU is visible, every
GPU-backed entry point raises ``BackendUnavailable`` immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("RESIHP_B200_LIB", _HERE / "libresihp_b200.so"))

RH_OK, RH_E_INVALID, RH_E_CUDA, RH_E_NOMEM, RH_E_SHAPE, RH_E_STRANDED = 0, -1, -2, -3, -4, -5

RH_IT_ESCALATE = 1
RH_IT_STAGE_FLAG = 2
RH_IT_LINK_FLAG = 4
RH_IT_STOPPED = 8
RH_IT_CAPACITY = 16
RH_IT_OVERFLOW = 32

RH_SC_CANDIDATE = 1
RH_SC_FILTERED = 2
RH_SC_ESCALATED = 4
RH_SC_CONFIRMED = 8
RH_SC_POPPED = 16

RH_SCHED_1F1B = 0
RH_SCHED_ZBH = 1

_p = C.c_void_p


class BackendUnavailable(RuntimeError):
    """The CUDA library or an sm_100 device is missing (no CPU fallback exists)."""


class LibraryError(RuntimeError):
    pass


class CostModelC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("ratio_f", C.c_double),
                ("ratio_b", C.c_double), ("ratio_w", C.c_double)]


class PipeShape(C.Structure):
    _fields_ = [("pp", C.c_int32), ("dp", C.c_int32), ("tp", C.c_int32),
                ("schedule", C.c_int32), ("micro_batches", C.c_int32),
                ("token_budget", C.c_int32), ("capacity", C.c_int32),
                ("has_allreduce", C.c_int32), ("max_mb_per_replica", C.c_int32)]


class Segments(C.Structure):
    _fields_ = [("n_seg", C.c_int32), ("layers", _p), ("mb_start", _p), ("speed", _p),
                ("hop_fwd", _p), ("hop_bwd", _p), ("allreduce", _p), ("link_off", _p),
                ("link_ratio", _p), ("link_max", _p)]


class Trace(C.Structure):
    _fields_ = [("n_iter", C.c_int64), ("seg", _p), ("mb_off", _p), ("doc_len", _p),
                ("device_time", _p), ("observed", _p)]


class TracePacked(C.Structure):
    _fields_ = [("n_iter", C.c_int64), ("seg", _p), ("iter_doc", _p), ("mb_docs", _p),
                ("doc_len", _p), ("device_time", _p), ("observed", _p)]


class PassOut(C.Structure):
    _fields_ = [("makespan", _p), ("status", _p), ("stage_cost", _p),
                ("stage_flag", _p), ("severity", _p)]


class MigrationDesc(C.Structure):
    _fields_ = [("pp", C.c_int32), ("dp", C.c_int32), ("schedule", C.c_int32),
                ("n_mb", C.c_int32), ("token_budget", C.c_int32), ("model", CostModelC),
                ("mb_off", _p), ("doc_len", _p), ("layers", _p), ("speed", _p),
                ("dp_counts", _p),
                ("delta", C.c_int32), ("capacity", C.c_int32), ("migrate", C.c_int32),
                ("preset", _p), ("hop_next", _p), ("hop_prev", _p), ("hop_same", _p)]


class ScreenParams(C.Structure):
    _fields_ = [("window", C.c_int32), ("filter_enabled", C.c_int32), ("kappa", C.c_double)]


_SIGS = {
    "rh_abi_version": ([], C.c_int),
    "rh_last_error": ([], C.c_char_p),
    "rh_ctx_create": ([C.c_int, C.POINTER(_p)], C.c_int),
    "rh_ctx_destroy": ([_p], C.c_int),
    "rh_ctx_launches": ([_p], C.c_int64),
    "rh_selftest_division": ([_p, C.c_int64, C.c_uint64, C.POINTER(C.c_int64)], C.c_int),
    "rh_quad_load_host": ([_p, C.c_int64, _p, _p, _p], C.c_int),
    "rh_chunk_time_host": ([_p, C.POINTER(CostModelC), C.c_int64, _p, _p, _p, _p, _p, _p, _p],
                           C.c_int),
    "rh_validate_host": ([_p, C.c_int64, _p, _p, C.c_double, _p, _p], C.c_int),
    "rh_screen_host": ([_p, C.POINTER(ScreenParams), C.c_int64, _p, C.c_int64, _p, _p, _p, _p,
                        _p], C.c_int),
    "rh_dag_critical_path_host": ([_p, C.c_int32, _p, _p, _p, _p, C.c_int32, _p, _p, C.c_int32,
                                   _p, _p, _p, _p], C.c_int),
    "rh_pipeline_batch_host": ([_p, C.POINTER(PipeShape), C.POINTER(CostModelC),
                                C.POINTER(Segments), C.POINTER(Trace), C.POINTER(PassOut)], C.c_int),
    "rh_chunk_time_docs_host": ([_p, C.POINTER(CostModelC), C.c_int64, _p, _p, C.c_int64, _p, _p,
                                 _p, _p, _p, _p, _p], C.c_int),
    "rh_observe_host": ([_p, C.POINTER(ScreenParams), C.c_int64, _p, C.c_double, C.c_int32,
                         C.c_int32, C.c_int32, _p, _p, C.c_int32, _p, C.c_double, _p, _p, _p, _p,
                         _p, _p], C.c_int),
    "rh_fp64_peak": ([_p, C.POINTER(C.c_double)], C.c_int),
    "rh_quad_load": ([_p, C.c_int64, _p, _p, _p, _p], C.c_int),
    "rh_chunk_time": ([_p, C.POINTER(CostModelC), C.c_int64, _p, _p, _p, _p, _p, _p, _p, _p],
                      C.c_int),
    "rh_pipeline_batch": ([_p, C.POINTER(PipeShape), C.POINTER(CostModelC),
                           C.POINTER(Segments), C.POINTER(Trace), C.POINTER(PassOut), _p],
                          C.c_int),
    "rh_detect_batch": ([_p, C.POINTER(PipeShape), C.POINTER(CostModelC), C.POINTER(Segments),
                         C.POINTER(Trace), C.c_double, C.POINTER(PassOut), _p], C.c_int),
    "rh_detector_pass_host": ([_p, C.POINTER(PipeShape), C.POINTER(CostModelC),
                               C.POINTER(Segments), C.POINTER(Trace), C.c_double,
                               C.POINTER(ScreenParams), C.c_int64, _p, _p, C.POINTER(PassOut),
                               _p, C.POINTER(C.c_int64), _p], C.c_int),
    "rh_detector_pass_host_packed": ([_p, C.POINTER(PipeShape), C.POINTER(CostModelC),
                                      C.POINTER(Segments), C.POINTER(TracePacked), C.c_double,
                                      C.POINTER(ScreenParams), C.c_int64, _p, _p,
                                      C.POINTER(PassOut), _p, C.POINTER(C.c_int64), _p],
                                     C.c_int),
    "rh_pack_sequences_quad": ([C.c_int64, _p, C.c_int32, C.c_int64, _p, _p, _p,
                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "rh_pack_sequences": ([C.c_int64, _p, C.c_int32, C.c_int64, _p, _p, C.POINTER(C.c_int64),
                           C.POINTER(C.c_int64)], C.c_int),
    "rh_repartition_batch": ([_p, C.c_int32, _p, _p, _p, _p, _p, _p, _p], C.c_int),
    "rh_proportional_split_batch": ([_p, C.c_int32, _p, _p, _p, _p, _p, _p], C.c_int),
    "rh_select_subgroup_batch": ([_p, C.c_int32, _p, _p, _p, _p, _p, _p, _p], C.c_int),
    "rh_plan_migration": ([C.POINTER(MigrationDesc), _p, C.POINTER(C.c_int32), _p,
                           C.POINTER(C.c_int32), C.POINTER(C.c_double)], C.c_int),
    "rh_validate": ([_p, C.c_int64, _p, _p, C.c_double, _p, _p, _p], C.c_int),
    "rh_screen": ([_p, C.POINTER(ScreenParams), C.c_int64, _p, C.c_int64, _p, _p, _p, _p, _p,
                   _p], C.c_int),
    "rh_screen_prepare": ([_p, C.POINTER(ScreenParams), C.c_int64, _p, C.c_int64, _p, _p, _p],
                          C.c_int),
    "rh_nccl_unique_id": ([_p], C.c_int),
    "rh_nccl_comm_create": ([_p, C.c_int32, C.c_int32, _p, C.POINTER(_p)], C.c_int),
    "rh_nccl_comm_destroy": ([_p], C.c_int),
    "rh_minloc_allreduce": ([_p, _p, C.c_int32, _p, _p, _p], C.c_int),
    "rh_dag_critical_path": ([_p, C.c_int32, _p, _p, _p, _p, C.c_int32, _p, _p, C.c_int32,
                              _p, _p, _p, _p, _p], C.c_int),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lock = threading.Lock()
_lib: C.CDLL | None = None
_ctx: dict[int, int] = {}


def load_library() -> C.CDLL:
    """dlopen the library and declare every prototype (no GPU required)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise BackendUnavailable(
                    f"{LIB_PATH} is missing: run `python __graft_entry__.py` to build it")
            lib = C.CDLL(str(LIB_PATH))
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == RH_OK:
        return
    msg = (load_library().rh_last_error() or b"").decode(errors="replace")
    if rc == RH_E_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise LibraryError(f"{what} failed ({rc}): {msg}")


def context(device: int | None = None) -> int:
    """Per-device library context (created once, lives for the process)."""
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device visible; the B200 path has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    with _lock:
        handle = _ctx.get(dev)
    if handle is None:
        lib = load_library()
        out = _p()
        check(lib.rh_ctx_create(dev, C.byref(out)), "rh_ctx_create")
        with _lock:
            handle = _ctx.setdefault(dev, out.value)
    return handle


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    """Raw address of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def launches(device: int | None = None) -> int:
    return load_library().rh_ctx_launches(context(device))
