"""Reference-side plugin: run the UNMODIFIED reference's search on libsimba.

``install(engine)`` takes the reference's loaded ``mbasynth.engine`` module
and swaps its data-parallel backend -- the seam SPEC.md:311 names ("a
pluggable data-parallel map over an index range whose body is pure") -- for
the device path, leaving Algorithm 1 itself (blocks, chunks, waves, the
local-mode break, timeouts, the host re-verification; engine.py:190-276)
the reference's own code:

  _EvalContext   engine.py:116-125 (built at engine.py:215 and in the worker
                 initializer engine.py:164-167) -> a context that binds the
                 spec to the GPU (simba_ctx_create) on first use
  _scan_range    engine.py:128-156 (called at engine.py:241) -> simba_scan_range:
                 same (visited, best_rank, best_tokens) for the same chunk
  _init_worker / _scan_task   engine.py:159-172 -> the same over the device
                 context, importable by name so that spawned workers run them
  ProcessPoolExecutor         engine.py:208-214 -> a spawn-context pool: a
                 CUDA context must never cross a fork

This is the two-line change of INTEGRATION.md applied from outside, so the
reference's own tests can run through the device (tests/test_reference_backend.py).
Nothing here imports the reference; there is no CPU path behind it.
"""

from __future__ import annotations

import functools
import multiprocessing

from .engine import DeviceContext, Specification
from .suite import device_size_bound


class DeviceEvalContext:
    """Stands in for engine._EvalContext: the table and spec of one search,
    bound to the GPU lazily (the parent of a spawn pool never needs a device
    context of its own)."""

    def __init__(self, table, spec):
        self.table = table
        self.spec = spec
        self._dev = None

    def device(self) -> DeviceContext:
        if self._dev is None:
            spec = Specification(k=self.spec.k, w=self.spec.w, pairs=tuple(self.spec.pairs))
            self._dev = DeviceContext(spec, device_size_bound(self.spec.k, self.table.max_size))
        return self._dev


def scan_range(ctx: DeviceEvalContext, size: int, offset: int, block_total: int, start: int, stop: int,
               shuffled: bool):
    """engine._scan_range (engine.py:128-156) on the device: decode-evaluate-
    discard local indices [start, stop) of one operator block."""
    return ctx.device().scan_range(size, offset, block_total, start, stop, shuffled)


_WORKER_CTX: DeviceEvalContext | None = None


def init_worker(k: int, max_size: int, w: int, pairs) -> None:
    """engine._init_worker (engine.py:164-167) for spawn workers."""
    global _WORKER_CTX
    from .counting import build

    _WORKER_CTX = DeviceEvalContext(build(k, max_size), Specification(k=k, w=w, pairs=tuple(pairs)))


def scan_task(task):
    """engine._scan_task (engine.py:170-172)."""
    size, offset, block_total, start, stop, shuffled = task
    return scan_range(_WORKER_CTX, size, offset, block_total, start, stop, shuffled)


def install(engine) -> None:
    """Route a loaded reference ``engine`` module through libsimba (idempotent)."""
    from concurrent.futures import ProcessPoolExecutor

    engine._EvalContext = DeviceEvalContext
    engine._scan_range = scan_range
    engine._init_worker = init_worker
    engine._scan_task = scan_task
    engine.ProcessPoolExecutor = functools.partial(ProcessPoolExecutor,
                                                   mp_context=multiprocessing.get_context("spawn"))
    engine.SIMBA_BACKEND = True
