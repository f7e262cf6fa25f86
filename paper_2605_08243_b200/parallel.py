"""Multi-GPU sharding of the search: one process per GPU.

Each size level's rank space [0, T[s][8]) is cut into super-chunks dealt
round-robin to the ranks (super-chunk c -> rank c mod world), so every GPU
advances through the level in ascending rank order together.  The only
exchange is one MIN (first satisfying rank) and one SUM (count, visited) per
size level -- 24 bytes, done with ``torch.distributed.all_reduce`` (NCCL on
GPUs, gloo in the CPU tests).  The result equals the single-device one:

* count mode: every rank is visited by exactly one shard, so the SUM is the
  exhaustive count and the MIN the first satisfying rank;
* search mode: a shard skips only ranks above its own best hit, so its result
  is the exact minimum of its shard and the MIN over shards is the level's
  minimum -- the (size, rank) the reference returns (engine.py:244-262).
* early exit across GPUs (``search_fused(..., shared=...)``): the shards also
  publish every hit to one shared 8-byte minimum (``SharedMinimum``: a word
  on rank 0's GPU, mapped into the other ranks over NVLink by its CUDA IPC
  handle) and fold it into their own bound at every claim and CTA phase, so
  a shard stops claiming above ANY shard's hit -- the reference's break after
  the first wave with a hit (engine.py:248-250).  Still exact: a chunk is
  skipped only when its start is above a verified hit, which is >= the job's
  minimum, so every chunk at or below the minimum is scanned by its owner.

The device work is a ``scan(size, lo, hi, mode, shard, nshards, chunk)``
callable (``DeviceContext.run`` on a GPU); the tests plug in the CPU oracle
with the same chunk ownership to check the protocol on CPU with gloo.
"""

from __future__ import annotations

from dataclasses import dataclass

NO_RANK = (1 << 64) - 1
_I64_MAX = (1 << 63) - 1


@dataclass(frozen=True)
class LevelResult:
    size: int
    count: int
    first_rank: int | None
    visited: int


def _reduce(count: int, first: int | None, visited: int, device=None, group=None):
    import torch
    import torch.distributed as dist

    if first is not None and first > _I64_MAX:
        raise OverflowError("rank beyond int64 in the distributed reduction")
    sums = torch.tensor([count, visited], dtype=torch.int64, device=device)
    mins = torch.tensor([_I64_MAX if first is None else first], dtype=torch.int64, device=device)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mins, op=dist.ReduceOp.MIN, group=group)
    f = int(mins.item())
    return int(sums[0].item()), (None if f == _I64_MAX else f), int(sums[1].item())


def run_level(scan, size: int, total: int, mode: str, rank: int, world: int, chunk: int = 0,
              device=None, group=None) -> LevelResult:
    """Scan size level `size` across `world` ranks and reduce.  `scan` returns
    an object with .count, .best_rank (None if no hit) and .visited."""
    r = scan(size, 0, total, mode, rank, world, chunk)
    if world == 1:
        return LevelResult(size, r.count, r.best_rank, r.visited)
    count, first, visited = _reduce(r.count, r.best_rank, r.visited, device=device, group=group)
    return LevelResult(size, count, first, visited)


def count_levels(scan, totals, rank: int, world: int, chunk: int = 0, device=None, group=None):
    """Exhaustive count of sizes 1..len(totals) (totals[s-1] = T[s][8])."""
    return [run_level(scan, s, t, "count", rank, world, chunk, device, group)
            for s, t in enumerate(totals, start=1)]


def search(scan, totals, rank: int, world: int, chunk: int = 0, device=None, group=None):
    """Algorithm 1 across ranks: sizes ascending, stop at the first size with a
    hit.  Returns (found_size | None, rank | None, per-level results)."""
    levels = []
    for s, t in enumerate(totals, start=1):
        lv = run_level(scan, s, t, "search", rank, world, chunk, device, group)
        levels.append(lv)
        if lv.first_rank is not None:
            return s, lv.first_rank, levels
    return None, None, levels


def count_fused(scan_levels, size_bound: int, rank: int, world: int, device=None, group=None):
    """Every level 1..size_bound in ONE device request per rank (simba_run_levels:
    the levels' concatenated rank space sharded round-robin), then one SUM and
    one MIN reduction for all levels together."""
    _, levels = scan_levels(1, size_bound, "count", rank, world)
    if world == 1:
        return [LevelResult(s, c, f, v) for s, c, f, v in levels]
    import torch
    import torch.distributed as dist

    sums = torch.tensor([[c, v] for _, c, _, v in levels], dtype=torch.int64, device=device)
    mins = torch.tensor([_I64_MAX if f is None else f for _, _, f, _ in levels], dtype=torch.int64, device=device)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mins, op=dist.ReduceOp.MIN, group=group)
    return [LevelResult(s, int(sums[i, 0].item()), None if int(mins[i].item()) == _I64_MAX else int(mins[i].item()),
                        int(sums[i, 1].item())) for i, (s, *_) in enumerate(levels)]


def shared_minimum(rank: int, world: int, device: int = 0, group=None):
    """One SharedMinimum for the job: created on rank 0's GPU, its IPC handle
    broadcast once (the only setup exchange), opened by every other rank."""
    import torch.distributed as dist

    from .engine import SharedMinimum

    obj = [None]
    mine = None
    if rank == 0:
        mine = SharedMinimum(device)
        obj[0] = mine.handle
    if world > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    if rank != 0:
        mine = SharedMinimum(device, handle=obj[0])
    return mine


def search_fused(scan_levels, size_bound: int, rank: int, world: int, device=None, group=None, shared=None):
    """Algorithm 1 in one device request per rank: each shard returns its
    minimum (size, rank); the job's answer is the lexicographic minimum over
    shards (MIN of the size, then MIN of the rank among shards at that size).
    With `shared` (a SharedMinimum attached to every rank's context) the
    shards stop above any shard's hit; rank 0 resets it and a barrier orders
    the reset before every launch (the previous search's reductions already
    ordered every launch before the reset)."""
    if shared is not None and world > 1:
        import torch.distributed as dist

        if rank == 0:
            shared.reset()
        dist.barrier(group=group)
    r, levels = scan_levels(1, size_bound, "search", rank, world)
    size = r.size if r.best_rank is not None else None
    first = r.best_rank
    if world > 1:
        import torch
        import torch.distributed as dist

        t = torch.tensor([_I64_MAX if size is None else size], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        best_size = int(t.item())
        t = torch.tensor([first if size is not None and size == best_size else _I64_MAX], dtype=torch.int64,
                         device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        size = None if best_size == _I64_MAX else best_size
        first = None if size is None else int(t.item())
    return size, first, levels


def device_levels(ctx):
    """Adapter: DeviceContext.run_levels as a `scan_levels` callable."""
    def scan_levels(size_lo, size_hi, mode, shard, nshards):
        return ctx.run_levels(size_lo, size_hi, mode=mode, shard=shard, nshards=nshards)
    return scan_levels


def device_scan(ctx):
    """Adapter: DeviceContext.run as a `scan` callable."""
    def scan(size, lo, hi, mode, shard, nshards, chunk):
        return ctx.run(size, lo, hi, mode=mode, chunk=chunk, shard=shard, nshards=nshards)
    return scan
