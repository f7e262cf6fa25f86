"""The cache-based comparison baseline ("VFB") on the GPU.

Mirror of the reference module ``mbasynth.baseline`` (baseline.py): the same
names, arguments, dataclasses and report layout, with the enumeration itself
running on the device (csrc/vfb_impl.cuh, C ABI ``simba_vfb_*`` in
include/simba.h).  This is SURVEY.md 8(f) row 4: the paper's comparison point
(PAPER.md:290-318), a different algorithm from SIMBA that stores one
behaviour vector per distinct candidate and therefore runs out of (modeled)
memory where the cache-free search keeps going.

Semantics follow run_baseline (baseline.py:88-249): candidates of size s in
slot order over the cached representatives of smaller sizes, a match ends the
run FOUND (checked before the cache), a behaviour already cached is dropped,
a new one is stored unless the modeled storage would exceed the budget (then
OOM_ABORTED at that size).  The time budget is polled between device batches
and between sizes, never mid-candidate (baseline.py:99-101).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

from . import _native as N
from . import counting
from .engine import SizeStats, Specification, Status, SynthesisOutcome
from .expr import RpnExpr, check

DEFAULT_MEMORY_BUDGET = 2_500_000_000  # bytes (baseline.py:22)
_UNBOUNDED = (1 << 64) - 1


def entry_bytes(n: int, w: int) -> int:
    """Modeled bytes of one cache entry: n words of w bits (baseline.py:25-27)."""
    return (n * w) // 8


def modeled_bytes(entries: int, n: int, w: int) -> int:
    """Modeled storage of `entries` cache entries (baseline.py:30-31)."""
    return entry_bytes(n, w) * entries


def format_mem(nbytes: int) -> str:
    """Decimal MB/GB with one digit, '<1 MB' below a megabyte (baseline.py:34-42)."""
    if nbytes >= 1_000_000_000:
        return "%.1f GB" % (nbytes / 1e9)
    if nbytes >= 1_000_000:
        return "%.1f MB" % (nbytes / 1e6)
    return "<1 MB"


@dataclass(frozen=True)
class CacheSizeRow:
    """Per-size cache growth (baseline.py:45-52)."""

    size: int
    stored: int
    stored_cum: int
    candidates: int
    modeled_bytes: int
    millis: float


@dataclass(frozen=True)
class CacheStats:
    """A run's cache growth (baseline.py:55-67)."""

    k: int
    n: int
    w: int
    rows: tuple[CacheSizeRow, ...]
    oom_at: int | None = None
    expr_tokens_total: int = 0

    def stored_cum(self) -> int:
        return self.rows[-1].stored_cum if self.rows else 0


class _Run:
    """One simba_vfb object (device cache of one run)."""

    def __init__(self, spec: Specification, max_entries: int, device: int):
        xs = [v for inputs, _ in spec.pairs for v in inputs]
        ys = [out for _, out in spec.pairs]
        x = (C.c_uint64 * len(xs))(*xs)
        y = (C.c_uint64 * len(ys))(*ys)
        h = C.c_void_p()
        N.check_rc(N.lib.simba_vfb_create(spec.k, spec.w, spec.n, x, y, max_entries, device, C.byref(h)),
                   "simba_vfb_create")
        self.h = h

    def level(self, size: int, budget_s: float | None) -> N.VfbRow:
        row = N.VfbRow()
        N.check_rc(N.lib.simba_vfb_level(self.h, size, -1.0 if budget_s is None else max(budget_s, 0.0),
                                         C.byref(row)), "simba_vfb_level")
        return row

    def tokens(self, cand: int) -> tuple[int, ...]:
        buf = (C.c_int32 * N.MAX_SIZE)()
        n = C.c_int()
        N.check_rc(N.lib.simba_vfb_tokens(self.h, cand, buf, N.MAX_SIZE, C.byref(n)), "simba_vfb_tokens")
        return tuple(buf[: n.value])

    def close(self) -> None:
        if self.h:
            N.lib.simba_vfb_destroy(self.h)
            self.h = None


def run_baseline(
    spec: Specification,
    size_bound: int,
    memory_budget: int = DEFAULT_MEMORY_BUDGET,
    time_budget: float | None = None,
    device: int = 0,
) -> tuple[SynthesisOutcome, CacheStats]:
    """Bottom-up enumeration with behaviour-vector deduplication on the device
    (baseline.run_baseline, baseline.py:88-249).

    FOUND at the first size with a candidate matching the outputs, NOT_FOUND
    once the bound is exhausted, OOM_ABORTED (``oom_at`` set) when the modeled
    storage would exceed ``memory_budget``, TIMED_OUT when ``time_budget``
    seconds pass (polled between device batches and sizes).
    """
    if size_bound < 1:
        raise ValueError(f"size bound must be >= 1, got {size_bound}")
    if size_bound > N.MAX_SIZE:
        raise ValueError(f"size bound {size_bound} above the device limit {N.MAX_SIZE}")
    per = entry_bytes(spec.n, spec.w)
    # (stored + 1) * per > budget  <=>  stored >= budget // per
    cap = _UNBOUNDED if per == 0 else max(0, memory_budget // per)
    cap = min(cap, _UNBOUNDED)
    deadline = None if time_budget is None else time.monotonic() + time_budget
    rows: list[CacheSizeRow] = []
    tokens_total = 0
    oom_at = None
    found: tuple[tuple[int, ...], int] | None = None
    timed_out = False
    run = _Run(spec, cap, device)
    try:
        for s in range(1, size_bound + 1):
            left = None if deadline is None else deadline - time.monotonic()
            r = run.level(s, left)
            tokens_total += r.stored * s
            rows.append(CacheSizeRow(s, r.stored, r.stored_cum, r.candidates,
                                     modeled_bytes(r.stored_cum, spec.n, spec.w), r.millis))
            if r.event == N.VFB_FOUND:
                found = (run.tokens(r.event_index), s)
                break
            if r.event == N.VFB_OOM:
                oom_at = s
                break
            if r.event == N.VFB_TIMED_OUT or (deadline is not None and time.monotonic() > deadline):
                timed_out = True
                break
    finally:
        run.close()
    stats = CacheStats(k=spec.k, n=spec.n, w=spec.w, rows=tuple(rows), oom_at=oom_at,
                       expr_tokens_total=tokens_total)
    per_size = tuple(SizeStats(r.size, r.candidates, r.millis) for r in rows)
    if found is not None:
        expr = RpnExpr(found[0])
        if not check(expr, spec):
            raise RuntimeError("internal error: cached solution failed re-verification")
        return SynthesisOutcome(Status.FOUND, expr, found[1], None, per_size), stats
    if oom_at is not None:
        return SynthesisOutcome(Status.OOM_ABORTED, stats=per_size), stats
    if timed_out:
        return SynthesisOutcome(Status.TIMED_OUT, stats=per_size), stats
    return SynthesisOutcome(Status.NOT_FOUND, stats=per_size), stats


def project_oom_size(cum_entries_by_size: list[tuple[int, int]], n: int, w: int, budget: int,
                     horizon: int = 64) -> int | None:
    """First size whose modeled cumulative storage exceeds ``budget``
    (baseline.py:252-286): an observed size if one does, else the per-size
    growth of the last two observations extended geometrically up to
    ``horizon`` (needs two consecutive, growing observations)."""
    if not cum_entries_by_size:
        return None
    over = [s for s, cum in cum_entries_by_size if modeled_bytes(cum, n, w) > budget]
    if over:
        return over[0]
    if len(cum_entries_by_size) < 2:
        return None
    (s_prev, c_prev), (s_last, c_last) = cum_entries_by_size[-2], cum_entries_by_size[-1]
    if s_last != s_prev + 1 or c_last <= c_prev:
        return None
    c_before = cum_entries_by_size[-3][1] if len(cum_entries_by_size) > 2 else 0
    step = c_last - c_prev
    ratio = step / max(c_prev - c_before, 1)
    cum, s = c_last, s_last
    while s < horizon:
        s += 1
        step = max(int(step * ratio), 1)
        cum += step
        if modeled_bytes(cum, n, w) > budget:
            return s
    return None


_HEADER = ("Size", "#MBA", "#VFB cache", "VFB mem", "% cached", "VFB cum. time (s; hardware-dependent)")


def cache_report(stats: CacheStats, fmt: str = "table") -> str:
    """Per-size cache growth table (baseline.py:289-334): size, all canonical
    expressions up to the size, cached entries, modeled memory, share cached
    and cumulative time; the OOM size's row reads OOM.  ``fmt="csv"`` gives
    the same cells comma-separated without digit grouping."""
    if not stats.rows:
        return ""
    tab = counting.build(stats.k, stats.rows[-1].size)
    body = []
    elapsed = 0.0
    for row in stats.rows:
        elapsed += row.millis
        mba = tab.cumulative_total(row.size)
        if stats.oom_at == row.size:
            body.append([str(row.size), f"{mba:,}"] + ["OOM"] * 4)
            continue
        share = 100.0 * row.stored_cum / mba if mba else 0.0
        body.append([str(row.size), f"{mba:,}", f"{row.stored_cum:,}", format_mem(row.modeled_bytes),
                     f"{share:.1f}%", f"{elapsed / 1e3:.1f}"])
    if fmt == "csv":
        return "\n".join([",".join(_HEADER)] + [",".join(c.replace(",", "") for c in cells) for cells in body])
    widths = [max(len(h), *(len(cells[i]) for cells in body)) for i, h in enumerate(_HEADER)]
    out = ["  ".join(h.rjust(widths[i]) for i, h in enumerate(_HEADER))]
    out += ["  ".join(c.rjust(widths[i]) for i, c in enumerate(cells)) for cells in body]
    return "\n".join(out)
