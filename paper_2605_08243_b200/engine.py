"""Cache-free bottom-up synthesis on B200 (drop-in for mbasynth.engine).

Same public surface as the reference (engine.py:31-113, 190-316):
``Specification``, ``EngineConfig``, ``Status``, ``SizeStats``,
``SynthesisOutcome``, ``synthesize(spec, table, cfg)`` and ``run_stats``,
with the same validation errors, status values and result format.  The
search itself runs in libsimba.so (hand-written sm_100a kernels behind the C
ABI of include/simba.h): Algorithm 1 visits sizes 1..C in order, each size
level's rank space in ascending chunks with early exit above the best hit,
and returns (minimum size with a hit, minimum in-size rank at that size) --
the result the reference returns in both local and shuffled mode.  The host
re-verifies the winner with ``check`` exactly like engine.py:264-269.

Additions (not in the reference): ``DeviceContext`` (a Specification bound to
one GPU, reusable across calls), ``count_solutions`` (exhaustive
satisfying-candidate counts per size) and
``scan_range`` (the ``_scan_range`` seam of engine.py:128-156).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from enum import Enum

from . import _native as N
from .counting import CountTable
from .expr import DEFAULT_WIDTH, RpnExpr, check, validate_width

DEFAULT_CHUNK = 1 << 16
_KERNELS = {"unit": 0, "direct": 1}


class Status(Enum):
    FOUND = "found"
    NOT_FOUND = "not_found"
    TIMED_OUT = "timed_out"
    OOM_ABORTED = "oom_aborted"


@dataclass(frozen=True)
class Specification:
    """n input-output pairs over k variables of w-bit words (engine.py:40-78)."""

    k: int
    w: int
    pairs: tuple[tuple[tuple[int, ...], int], ...]

    def __post_init__(self):
        if self.k < 1:
            raise ValueError(f"variable count must be >= 1, got {self.k}")
        validate_width(self.w)
        if not self.pairs:
            raise ValueError("specification needs at least one pair")
        limit = 1 << self.w
        seen = set()
        for inputs, output in self.pairs:
            if len(inputs) != self.k:
                raise ValueError(f"input tuple {inputs} has {len(inputs)} components, expected {self.k}")
            for v in (*inputs, output):
                if not 0 <= v < limit:
                    raise ValueError(f"value {v} does not fit in {self.w} bits")
            if inputs in seen:
                raise ValueError(f"duplicate input tuple {inputs}")
            seen.add(inputs)

    @property
    def n(self) -> int:
        return len(self.pairs)

    @classmethod
    def of(cls, pairs, k: int, w: int = DEFAULT_WIDTH) -> "Specification":
        return cls(k=k, w=w, pairs=tuple((tuple(i), o) for i, o in pairs))


@dataclass(frozen=True)
class EngineConfig:
    """engine.py:81-97.  ``chunk`` and ``workers`` are accepted for drop-in
    compatibility; like in the reference they never change results (the device
    picks its own chunking).  ``device``/``r0``/``table_examples``/``kernel``
    select the GPU and the kernel configuration (0 = automatic)."""

    size_bound: int
    mode: str = "local"
    chunk: int = DEFAULT_CHUNK
    workers: int = 1
    time_budget: float | None = None
    device: int = 0
    r0: int = 0
    rg: int = 0
    table_examples: int = 0
    kernel: str = "unit"

    def __post_init__(self):
        if self.size_bound < 1:
            raise ValueError(f"size bound must be >= 1, got {self.size_bound}")
        if self.chunk < 1:
            raise ValueError(f"chunk must be >= 1, got {self.chunk}")
        if self.mode not in ("local", "shuffled"):
            raise ValueError(f"mode must be 'local' or 'shuffled', got {self.mode!r}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.kernel not in _KERNELS:
            raise ValueError(f"kernel must be one of {sorted(_KERNELS)}, got {self.kernel!r}")


@dataclass(frozen=True)
class SizeStats:
    size: int
    candidates: int
    millis: float


@dataclass(frozen=True)
class SynthesisOutcome:
    status: Status
    expr: RpnExpr | None = None
    size: int | None = None
    rank: int | None = None
    stats: tuple[SizeStats, ...] = field(default_factory=tuple)


@dataclass(frozen=True)
class RangeResult:
    """One device scan of a rank range."""

    visited: int
    count: int
    best_rank: int | None
    tokens: tuple[int, ...] | None
    completed: bool
    kernel_ms: float
    launches: int
    units: int = 0
    rank_units: int = 0
    ex0_hits: int = 0
    size: int = 0  # the level of best_rank (multi-level requests)


@dataclass(frozen=True)
class SizeCount:
    """Exhaustive-mode result for one size level."""

    size: int
    count: int
    first_rank: int | None
    candidates: int
    millis: float


def _spec_arrays(spec: Specification):
    flat = [v for inputs, _ in spec.pairs for v in inputs]
    xs = (C.c_uint64 * len(flat))(*flat)
    ys = (C.c_uint64 * spec.n)(*[o for _, o in spec.pairs])
    return xs, ys


class DeviceContext:
    """A Specification bound to one GPU: tables, examples and the per-spec
    super-leaf value tables staged in device memory (simba_ctx_create)."""

    def __init__(self, spec: Specification, max_size: int, device: int = 0, r0: int = 0, rg: int = 0,
                 table_examples: int = 0, kernel: str = "unit", block_threads: int = 0,
                 blocks_per_sm: int = 0):
        self.spec = spec
        self.max_size = max_size
        opts = N.Options(device=device, r0=r0, rg=rg, table_examples=table_examples,
                         block_threads=block_threads, blocks_per_sm=blocks_per_sm,
                         kernel=_KERNELS[kernel])
        xs, ys = _spec_arrays(spec)
        ptr = C.c_void_p()
        rc = N.lib.simba_ctx_create(spec.k, spec.w, spec.n, xs, ys, max_size, C.byref(opts), C.byref(ptr))
        N.check_rc(rc, "simba_ctx_create")
        self._ptr = ptr
        from .counting import build
        self.table = build(spec.k, max_size)

    def close(self):
        ptr = getattr(self, "_ptr", None)
        if ptr:
            self._ptr = None
            lib = getattr(N, "lib", None)  # None during interpreter shutdown
            if lib is not None:
                lib.simba_ctx_destroy(ptr)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        self.close()

    def info(self) -> dict:
        vals = [C.c_int() for _ in range(7)]
        N.check_rc(N.lib.simba_ctx_info(self._ptr, *[C.byref(v) for v in vals]))
        keys = ("r0", "rg", "table_examples", "word_bytes", "grid_blocks", "block_threads", "smem_bytes")
        return dict(zip(keys, (v.value for v in vals)))

    @staticmethod
    def _result(r: N.Result, size: int) -> RangeResult:
        found = bool(r.found)
        return RangeResult(
            visited=r.visited, count=r.count,
            best_rank=r.best_rank if found else None,
            tokens=tuple(r.tokens[:size]) if found else None,
            completed=bool(r.completed), kernel_ms=r.kernel_ms, launches=r.launches,
            units=r.units, rank_units=r.rank_units, ex0_hits=r.ex0_hits, size=r.size)

    def scan_range(self, size, offset, block_total, start, stop, shuffled=False):
        """engine._scan_range (engine.py:128-156) -> (visited, best_rank, best_tokens)."""
        r = N.Result()
        N.check_rc(N.lib.simba_scan_range(self._ptr, size, offset, block_total, start, stop,
                                          int(bool(shuffled)), C.byref(r)))
        res = self._result(r, size)
        return res.visited, res.best_rank, res.tokens

    def run(self, size: int, lo: int, hi: int, mode: str = "search", chunk: int = 0, shard: int = 0,
            nshards: int = 1, stop_above: int | None = None, time_budget: float | None = None) -> RangeResult:
        req = N.Range(size=size, mode=N.MODE_SEARCH if mode == "search" else N.MODE_COUNT,
                      lo=lo, hi=hi, chunk=chunk, shard=shard, nshards=nshards,
                      stop_above=N.NO_RANK if stop_above is None else stop_above,
                      time_budget_s=-1.0 if time_budget is None else float(time_budget))
        r = N.Result()
        N.check_rc(N.lib.simba_run(self._ptr, C.byref(req), C.byref(r)))
        return self._result(r, size)

    def run_levels(self, size_lo: int, size_hi: int, mode: str = "count", shard: int = 0, nshards: int = 1,
                   time_budget: float | None = None):
        """Levels size_lo..size_hi in one launch (simba_run_levels): returns
        (RangeResult of the whole request -- its best_rank/tokens/size are the
        minimum (size, rank) --, [(size, count, first_rank | None, visited)])."""
        n = size_hi - size_lo + 1
        lv = (N.Level * n)()
        r = N.Result()
        N.check_rc(N.lib.simba_run_levels(self._ptr, size_lo, size_hi,
                                          N.MODE_SEARCH if mode == "search" else N.MODE_COUNT, shard, nshards,
                                          -1.0 if time_budget is None else float(time_budget), lv, C.byref(r)))
        levels = [(x.size, x.count, None if x.first_rank == N.NO_RANK else x.first_rank, x.visited) for x in lv]
        return self._result(r, r.size), levels

    def count(self, size: int, lo: int = 0, hi: int | None = None, **kw) -> RangeResult:
        if hi is None:
            hi = self.total(size)
        return self.run(size, lo, hi, mode="count", **kw)

    def synthesize_raw(self, size_bound: int, shuffled: bool = False, time_budget: float | None = None):
        out = N.Outcome()
        N.check_rc(N.lib.simba_synthesize(self._ptr, size_bound, int(shuffled),
                                          -1.0 if time_budget is None else float(time_budget),
                                          C.byref(out)))
        return out

    def copied_bytes(self) -> tuple[int, int]:
        """(host->device, device->host) bytes this context has copied."""
        h, d = C.c_uint64(), C.c_uint64()
        N.check_rc(N.lib.simba_ctx_bytes(self._ptr, C.byref(h), C.byref(d)))
        return h.value, d.value

    def stream_handle(self) -> int:
        """cudaStream_t of this context (wrap with torch.cuda.ExternalStream)."""
        h = C.c_void_p()
        N.check_rc(N.lib.simba_ctx_stream(self._ptr, C.byref(h)))
        return h.value or 0

    PATHS = ("rf_fold", "rf_gen", "rf_row", "cf_fold", "cf_gen", "cyc_outer", "cyc_x", "cyc_tile", "direct",
             "ph_plan", "ph_exec", "ph_verify", "w_plan", "w_exec", "row_none", "gen_nt1", "gen_nt2", "gen_nt3",
             "gen_arith", "gen_res_aff", "gen_res_bw")

    def path_stats(self) -> dict:
        """Per-path (calls, candidates) of the unit kernel since creation;
        empty unless libsimba was built with -DSIMBA_STATS (diagnostics)."""
        buf = (C.c_uint64 * (2 * len(self.PATHS)))()
        n = N.lib.simba_ctx_stats(self._ptr, buf, len(buf))
        if n < 0:
            N.check_rc(n)
        return {name: (buf[2 * i], buf[2 * i + 1]) for i, name in enumerate(self.PATHS) if 2 * i + 1 < n}

    def decode(self, rank: int, size: int) -> tuple[int, ...]:
        buf = (C.c_int32 * N.MAX_SIZE)()
        N.check_rc(N.lib.simba_decode(self._ptr, rank, size, buf))
        return tuple(buf[:size])

    def decode_batch(self, rank0: int, count: int, size: int):
        """Tokens of the ranks [rank0, rank0 + count), as a (count, size) int32 array."""
        import numpy as np

        out = np.empty((count, size), dtype=np.int32)
        N.check_rc(N.lib.simba_decode_batch(self._ptr, rank0, count, size,
                                            out.ctypes.data_as(C.POINTER(C.c_int32))))
        return out

    def total(self, size: int) -> int:
        return self.table.total(size)

    def set_shared_minimum(self, shared: "SharedMinimum | None") -> None:
        """Attach (or, with None, detach) the shared minimum of a sharded
        search: sharded SEARCH requests of this context publish their hits to
        it and skip ranks above any shard's hit (simba_ctx_set_xbest)."""
        N.check_rc(N.lib.simba_ctx_set_xbest(self._ptr, shared._ptr if shared is not None else None))
        self._shared = shared  # the word must outlive the attachment


class SharedMinimum:
    """The 8-byte minimum (virtual rank) every shard of a sharded search
    publishes its hits to and polls (SURVEY.md 8(e) early exit; simba_xbest).
    Created on one process's GPU; the other processes open it from its CUDA
    IPC handle (``handle``), over NVLink when their GPU differs."""

    def __init__(self, device: int = 0, handle: bytes | None = None):
        ptr = C.c_void_p()
        if handle is None:
            buf = (C.c_ubyte * N.XBEST_HANDLE_BYTES)()
            N.check_rc(N.lib.simba_xbest_create(device, buf, C.byref(ptr)), "simba_xbest_create")
            self.handle = bytes(buf)
        else:
            if len(handle) != N.XBEST_HANDLE_BYTES:
                raise ValueError("shared-minimum handle must be 64 bytes")
            buf = (C.c_ubyte * N.XBEST_HANDLE_BYTES).from_buffer_copy(handle)
            N.check_rc(N.lib.simba_xbest_open(device, buf, C.byref(ptr)), "simba_xbest_open")
            self.handle = bytes(handle)
        self._ptr = ptr

    def reset(self) -> None:
        N.check_rc(N.lib.simba_xbest_reset(self._ptr))

    def read(self) -> int | None:
        v = C.c_uint64()
        N.check_rc(N.lib.simba_xbest_read(self._ptr, C.byref(v)))
        return None if v.value == N.NO_RANK else v.value

    def close(self) -> None:
        ptr = getattr(self, "_ptr", None)
        if ptr:
            self._ptr = None
            lib = getattr(N, "lib", None)
            if lib is not None:
                lib.simba_xbest_destroy(ptr)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        self.close()


def _check_args(spec: Specification, table: CountTable, cfg: EngineConfig):
    if spec.k != table.k:
        raise ValueError(f"spec has k={spec.k} but table was built for k={table.k}")
    if cfg.size_bound > table.max_size:
        raise ValueError(f"size bound {cfg.size_bound} exceeds table extent {table.max_size}")


def synthesize(spec: Specification, table: CountTable, cfg: EngineConfig) -> SynthesisOutcome:
    """engine.synthesize (engine.py:190-276) on the device."""
    _check_args(spec, table, cfg)
    with DeviceContext(spec, cfg.size_bound, device=cfg.device, r0=cfg.r0, rg=cfg.rg,
                       table_examples=cfg.table_examples, kernel=cfg.kernel) as ctx:
        out = ctx.synthesize_raw(cfg.size_bound, shuffled=(cfg.mode == "shuffled"),
                                 time_budget=cfg.time_budget)
    stats = tuple(SizeStats(s + 1, out.visited[s], out.millis[s]) for s in range(out.nsizes))
    if out.status == N.STATUS_FOUND:
        expr = RpnExpr(tuple(out.tokens[:out.size]))
        if not check(expr, spec):  # re-verify outside the parallel path (engine.py:264-269)
            raise RuntimeError(f"internal error: candidate rank {out.rank} failed re-verification")
        return SynthesisOutcome(Status.FOUND, expr, out.size, out.rank, stats)
    if out.status == N.STATUS_TIMED_OUT:
        return SynthesisOutcome(Status.TIMED_OUT, stats=stats)
    return SynthesisOutcome(Status.NOT_FOUND, stats=stats)


def count_solutions(spec: Specification, table: CountTable, cfg: EngineConfig) -> tuple[SizeCount, ...]:
    """Exhaustive mode: #{n < T[s][8] : check(decode(n, s), spec)} and the
    smallest such n for every s in 1..C (oracle: enumerate_all + check,
    engine.py:279-293, expr.py:201-218)."""
    _check_args(spec, table, cfg)
    out = []
    with DeviceContext(spec, cfg.size_bound, device=cfg.device, r0=cfg.r0, rg=cfg.rg,
                       table_examples=cfg.table_examples, kernel=cfg.kernel) as ctx:
        if cfg.kernel == "direct":  # the per-rank kernel runs one level per launch
            for s in range(1, cfg.size_bound + 1):
                t0 = time.perf_counter()
                r = ctx.run(s, 0, table.total(s), mode="count")
                out.append(SizeCount(s, r.count, r.best_rank, r.visited, (time.perf_counter() - t0) * 1e3))
        else:  # every level in one launch; its time apportioned by candidates
            t0 = time.perf_counter()
            _, levels = ctx.run_levels(1, cfg.size_bound, mode="count")
            ms = (time.perf_counter() - t0) * 1e3
            tot = sum(v for *_, v in levels) or 1
            out = [SizeCount(s, c, f, v, ms * v / tot) for s, c, f, v in levels]
    return tuple(out)


def enumerate_all(size: int, table: CountTable, visitor=None, batch: int = 1 << 20) -> int:
    """engine.enumerate_all (engine.py:279-293): decode every rank of ``size``
    once (on the device, in batches) and hand each expression to ``visitor``
    in rank order; returns the number of ranks."""
    from .codec import _decoder

    total = table.total(size)
    dec = _decoder(table)
    for r0 in range(0, total, batch):
        toks = dec.decode_batch(r0, min(batch, total - r0), size)
        if visitor is not None:
            for row in toks.tolist():
                visitor(RpnExpr(tuple(row)))
    return total


def run_stats(outcome: SynthesisOutcome) -> dict:
    """engine.run_stats (engine.py:296-316)."""
    total_candidates = sum(s.candidates for s in outcome.stats)
    total_millis = sum(s.millis for s in outcome.stats)
    per_second = total_candidates / (total_millis / 1e3) if total_millis > 0 else 0.0
    return {
        "status": outcome.status.value,
        "expr": str(outcome.expr) if outcome.expr is not None else None,
        "size": outcome.size,
        "rank": str(outcome.rank) if outcome.rank is not None else None,
        "per_size": [
            {"size": s.size, "candidates": s.candidates, "millis": round(s.millis, 3)}
            for s in outcome.stats
        ],
        "total_candidates": total_candidates,
        "total_millis": round(total_millis, 3),
        "candidates_per_second": round(per_second, 1),
    }
