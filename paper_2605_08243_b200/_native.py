"""ctypes binding of libsimba.so (include/simba.h).

The library is built in-tree (``python __graft_entry__.py`` or
``python -m paper_2605_08243_b200._build``).  There is no CPU fallback: if the
library is missing this module raises ImportError, and if no CUDA device is
present every device call fails with DeviceError.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SIMBA_LIB", PKG / "_lib" / "libsimba.so"))

OK, EINVAL, ERANGE, ECAPACITY, ECUDA, ENOMEM = 0, 1, 2, 3, 4, 5
MAX_SIZE = 24
TABLE_MAX = 64
MODE_SEARCH, MODE_COUNT = 0, 1
STATUS_FOUND, STATUS_NOT_FOUND, STATUS_TIMED_OUT = 0, 1, 2
NO_RANK = (1 << 64) - 1
XBEST_HANDLE_BYTES = 64


class Options(C.Structure):
    _fields_ = [
        ("device", C.c_int),
        ("r0", C.c_int),
        ("rg", C.c_int),
        ("table_examples", C.c_int),
        ("block_threads", C.c_int),
        ("blocks_per_sm", C.c_int),
        ("kernel", C.c_int),
    ]


class Result(C.Structure):
    _fields_ = [
        ("visited", C.c_uint64),
        ("count", C.c_uint64),
        ("best_rank", C.c_uint64),
        ("found", C.c_int32),
        ("completed", C.c_int32),
        ("size", C.c_int32),
        ("tokens", C.c_int32 * MAX_SIZE),
        ("kernel_ms", C.c_double),
        ("launches", C.c_uint64),
        ("units", C.c_uint64),
        ("rank_units", C.c_uint64),
        ("ex0_hits", C.c_uint64),
    ]


class Range(C.Structure):
    _fields_ = [
        ("size", C.c_int),
        ("mode", C.c_int),
        ("lo", C.c_uint64),
        ("hi", C.c_uint64),
        ("chunk", C.c_uint64),
        ("shard", C.c_uint64),
        ("nshards", C.c_uint64),
        ("stop_above", C.c_uint64),
        ("time_budget_s", C.c_double),
    ]


class Level(C.Structure):
    _fields_ = [
        ("size", C.c_int32),
        ("count", C.c_uint64),
        ("first_rank", C.c_uint64),
        ("visited", C.c_uint64),
    ]


class Outcome(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("size", C.c_int32),
        ("rank", C.c_uint64),
        ("tokens", C.c_int32 * MAX_SIZE),
        ("nsizes", C.c_int32),
        ("visited", C.c_uint64 * MAX_SIZE),
        ("millis", C.c_double * MAX_SIZE),
        ("kernel_ms", C.c_double),
        ("launches", C.c_uint64),
    ]


VFB_NONE, VFB_FOUND, VFB_OOM, VFB_TIMED_OUT = 0, 1, 2, 3


class VfbRow(C.Structure):
    _fields_ = [
        ("candidates", C.c_uint64),
        ("stored", C.c_uint64),
        ("stored_cum", C.c_uint64),
        ("event_index", C.c_uint64),
        ("event", C.c_int32),
        ("millis", C.c_double),
    ]


# every symbol include/simba.h declares, with its ctypes signature
SIGNATURES = {
    "simba_table_build": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "simba_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                   C.c_int, C.POINTER(Options), C.POINTER(C.c_void_p)]),
    "simba_ctx_destroy": (None, [C.c_void_p]),
    "simba_scan_range": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                   C.c_int, C.POINTER(Result)]),
    "simba_run": (C.c_int, [C.c_void_p, C.POINTER(Range), C.POINTER(Result)]),
    "simba_run_levels": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_double,
                                   C.POINTER(Level), C.POINTER(Result)]),
    "simba_synthesize": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_double, C.POINTER(Outcome)]),
    "simba_decode": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_int32)]),
    "simba_decode_batch": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_int32)]),
    "simba_ctx_info": (C.c_int, [C.c_void_p] + [C.POINTER(C.c_int)] * 7),
    "simba_ctx_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "simba_ctx_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "simba_ctx_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int]),
    "simba_int32_peak": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "simba_int32_pipe_peak": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "simba_vfb_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                   C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]),
    "simba_vfb_level": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.POINTER(VfbRow)]),
    "simba_vfb_tokens": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_int)]),
    "simba_vfb_destroy": (None, [C.c_void_p]),
    "simba_xbest_create": (C.c_int, [C.c_int, C.POINTER(C.c_ubyte), C.POINTER(C.c_void_p)]),
    "simba_xbest_open": (C.c_int, [C.c_int, C.POINTER(C.c_ubyte), C.POINTER(C.c_void_p)]),
    "simba_xbest_reset": (C.c_int, [C.c_void_p]),
    "simba_xbest_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "simba_xbest_destroy": (None, [C.c_void_p]),
    "simba_ctx_set_xbest": (C.c_int, [C.c_void_p, C.c_void_p]),
    "simba_last_error": (C.c_char_p, []),
    "simba_device_count": (C.c_int, []),
    "simba_launch_count": (C.c_uint64, []),
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is not built; run `python __graft_entry__.py` or `python paper_2605_08243_b200/_build.py` (nvcc, sm_100a). "
            "The SIMBA device path has no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class DeviceError(RuntimeError):
    """CUDA failure or missing device (SIMBA_ECUDA)."""


def last_error() -> str:
    msg = lib.simba_last_error()
    return msg.decode() if msg else ""


def check_rc(rc: int, what: str = "") -> None:
    """Map a SIMBA_* status code to the exception the reference raises."""
    if rc == OK:
        return
    msg = last_error() or what
    if rc in (EINVAL, ERANGE):
        raise ValueError(msg)
    if rc == ECAPACITY:
        raise OverflowError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)


def device_count() -> int:
    return lib.simba_device_count()


def launch_count() -> int:
    return lib.simba_launch_count()
