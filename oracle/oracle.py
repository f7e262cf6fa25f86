"""ctypes wrapper of the CPU oracle (oracle/simba_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg, never by the product package.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
MAXS = 64


class _Res(C.Structure):
    _fields_ = [
        ("visited", C.c_uint64),
        ("count", C.c_uint64),
        ("best_rank", C.c_uint64),
        ("has_best", C.c_int32),
        ("best_tokens", C.c_int32 * MAXS),
    ]


def build() -> Path:
    """Compile liboracle.so from simba_oracle.c (make; gcc only)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < (HERE / "simba_oracle.c").stat().st_mtime:
            build()
        L = C.CDLL(str(LIB_PATH))
        L.oracle_table_new.restype = C.c_void_p
        L.oracle_table_free.argtypes = [C.c_void_p]
        L.oracle_build.argtypes = [C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.oracle_table_max_size64.argtypes = [C.c_void_p]
        L.oracle_table_entry.argtypes = [C.c_void_p, C.c_int, C.c_int,
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.oracle_decode_into.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_int32)]
        L.oracle_eval_tokens.argtypes = [C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_uint64), C.c_uint64]
        L.oracle_eval_tokens.restype = C.c_uint64
        spec_args = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.oracle_scan_range.argtypes = spec_args + [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                                    C.c_uint64, C.c_int, C.POINTER(_Res)]
        L.oracle_scan_range_mt.argtypes = spec_args + [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                                       C.c_uint64, C.c_int, C.c_int, C.POINTER(_Res)]
        L.oracle_synthesize.argtypes = spec_args + [
            C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
            C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
        _lib = L
    return _lib


class CapacityError(OverflowError):
    def __init__(self, s, op):
        super().__init__(f"count T[{s}][{op}] exceeds 128-bit capacity")
        self.s, self.op = s, op


class OracleTable:
    """counting.build restated in C (counting.py:88-128)."""

    def __init__(self, k: int, max_size: int):
        L = lib()
        self._p = C.c_void_p(L.oracle_table_new())
        es, eo = C.c_int(0), C.c_int(0)
        rc = L.oracle_build(k, max_size, self._p, C.byref(es), C.byref(eo))
        if rc == 1:
            raise CapacityError(es.value, eo.value)
        if rc != 0:
            raise ValueError("bad table arguments")
        self.k, self.max_size = k, max_size
        self.max_size64 = L.oracle_table_max_size64(self._p)

    def __del__(self):
        if getattr(self, "_p", None) and _lib is not None:
            _lib.oracle_table_free(self._p)
            self._p = None

    def entry(self, s: int, op: int) -> int:
        lo, hi = C.c_uint64(), C.c_uint64()
        lib().oracle_table_entry(self._p, s, op, C.byref(lo), C.byref(hi))
        return lo.value | (hi.value << 64)

    def rows(self):
        return [[self.entry(s, op) for op in range(9)] for s in range(self.max_size + 1)]

    def total(self, s: int) -> int:
        return self.entry(s, 8)

    def cumulative(self, s: int) -> int:
        return self.entry(s, 9)

    def operator_offset(self, s: int, op: int) -> int:
        return sum(self.entry(s, o) for o in range(op))


def decode(table: OracleTable, rank: int, size: int) -> tuple[int, ...]:
    buf = (C.c_int32 * MAXS)()
    lib().oracle_decode_into(table._p, rank, size, buf)
    return tuple(buf[:size])


def eval_tokens(tokens, inputs, w: int) -> int:
    toks = (C.c_int32 * MAXS)(*tokens)
    ins = (C.c_uint64 * max(1, len(inputs)))(*inputs)
    mask = (1 << w) - 1
    return lib().oracle_eval_tokens(toks, len(tokens), ins, mask)


def _spec_arrays(k, pairs):
    n = len(pairs)
    ins = (C.c_uint64 * (n * k))(*[v for i, _ in pairs for v in i])
    outs = (C.c_uint64 * n)(*[o for _, o in pairs])
    return n, ins, outs


def scan_range(table, k, w, pairs, size, offset, block_total, start, stop, shuffled=False, threads=1):
    """engine._scan_range (engine.py:128-156) + exhaustive count.
    Returns (visited, count, best_rank|None, best_tokens|None)."""
    n, ins, outs = _spec_arrays(k, pairs)
    r = _Res()
    if threads <= 1:
        rc = lib().oracle_scan_range(table._p, k, w, n, ins, outs, size, offset, block_total,
                                     start, stop, int(shuffled), C.byref(r))
    else:
        rc = lib().oracle_scan_range_mt(table._p, k, w, n, ins, outs, size, offset, block_total,
                                        start, stop, int(shuffled), threads, C.byref(r))
    if rc:
        raise ValueError("oracle scan rejected its arguments")
    best = r.best_rank if r.has_best else None
    toks = tuple(r.best_tokens[:size]) if r.has_best else None
    return r.visited, r.count, best, toks


def synthesize(table, k, w, pairs, size_bound, chunk=1 << 16, shuffled=False):
    """engine.synthesize (engine.py:190-276), workers=1, no time budget.
    Returns dict(status, size, rank, tokens, per_size=[[s, visited], ...])."""
    n, ins, outs = _spec_arrays(k, pairs)
    st, fs, reached = C.c_int(), C.c_int(), C.c_int()
    fr = C.c_uint64()
    toks = (C.c_int32 * MAXS)()
    vis = (C.c_uint64 * MAXS)()
    rc = lib().oracle_synthesize(table._p, k, w, n, ins, outs, size_bound, chunk, int(shuffled),
                                 C.byref(st), C.byref(fs), C.byref(fr), toks, vis, C.byref(reached))
    if rc:
        raise ValueError("oracle synthesize rejected its arguments")
    per = [[s + 1, vis[s]] for s in range(reached.value)]
    if st.value == 0:
        return {"status": "found", "size": fs.value, "rank": fr.value,
                "tokens": list(toks[:fs.value]), "per_size": per}
    return {"status": "not_found", "size": None, "rank": None, "tokens": None, "per_size": per}


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
