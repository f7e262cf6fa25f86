"""Multi-rank protocol (paper_2605_08243_b200/parallel.py) on CPU with gloo,
world_size 2: the shard ownership of the device ABI (round-robin chunks,
simba_run with nshards > 1) emulated with the CPU oracle as the scanner.
The reduced results must equal the single-process reference results."""

import os
import socket
from types import SimpleNamespace

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from conftest import load_golden
from paper_2605_08243_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_scan(table, k, w, pairs):
    """Same chunk ownership as the kernel when chunk is given and nshards > 1:
    chunk c of [lo, hi) belongs to shard c % nshards."""
    def scan(size, lo, hi, mode, shard, nshards, chunk):
        chunk = chunk or 997
        count, best, visited = 0, None, 0
        c = shard
        while lo + c * chunk < hi:
            a = lo + c * chunk
            b = min(hi, a + chunk)
            if mode == "search" and best is not None and a > best:
                break
            _, cnt, first, _ = O.scan_range(table, k, w, pairs, size, 0, table.total(size), a, b)
            count += cnt
            visited += b - a
            if first is not None and (best is None or first < best):
                best = first
            c += nshards
        return SimpleNamespace(count=count, best_rank=best, visited=visited)
    return scan


def oracle_levels(table, k, w, pairs, chunk):
    """Fused request emulated level by level with the same per-level shard
    ownership (the reduction is what is under test)."""
    scan = oracle_scan(table, k, w, pairs)

    def scan_levels(size_lo, size_hi, mode, shard, nshards):
        levels, found = [], None
        for s in range(size_lo, size_hi + 1):
            r = scan(s, 0, table.total(s), mode, shard, nshards, chunk)
            levels.append((s, r.count, r.best_rank, r.visited))
            if mode == "search" and r.best_rank is not None and found is None:
                found = (s, r.best_rank)
                break
        res = SimpleNamespace(size=found[0] if found else size_hi, best_rank=found[1] if found else None)
        return res, levels
    return scan_levels


def _worker(rank, world, port, cases, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for kind, spec, C, arg in cases:
            pairs = [(tuple(i), o) for i, o in spec["pairs"]]
            table = O.OracleTable(spec["k"], C)
            scan = oracle_scan(table, spec["k"], spec["w"], pairs)
            totals = [table.total(s) for s in range(1, C + 1)]
            if kind == "count":
                lv = parallel.count_levels(scan, totals, rank, world, chunk=arg)
                res.append([[x.size, x.count, x.first_rank, x.visited] for x in lv])
                fused = parallel.count_fused(oracle_levels(table, spec["k"], spec["w"], pairs, arg), C, rank, world)
                assert [[x.size, x.count, x.first_rank, x.visited] for x in fused] == res[-1]
            else:
                size, first, lv = parallel.search(scan, totals, rank, world, chunk=arg)
                res.append([size, first])
                fs, ff, _ = parallel.search_fused(oracle_levels(table, spec["k"], spec["w"], pairs, arg), C, rank,
                                                  world)
                assert [fs, ff] == [size, first]
                # with a shared minimum: rank 0 resets it, a barrier orders the reset
                # before every rank's request (the device word is exercised in
                # tests/test_xbest.py)
                shared = _FakeShared()
                fs, ff, _ = parallel.search_fused(oracle_levels(table, spec["k"], spec["w"], pairs, arg), C, rank,
                                                  world, shared=shared)
                assert [fs, ff] == [size, first]
                assert shared.resets == (1 if rank == 0 else 0)
        out[rank] = res
    finally:
        dist.destroy_process_group()


class _FakeShared:
    def __init__(self):
        self.resets = 0

    def reset(self):
        self.resets += 1


@pytest.mark.parametrize("world", [2])
def test_two_rank_protocol_matches_reference(world):
    counts = [r for r in load_golden("counts") if r["name"] in ("C1_seed3", "C2_s5_i0", "C2_s7_i1")]
    search = [r for r in load_golden("search") if r["meta"].get("config") in ("C1", "C2")][::9]
    cases = [("count", r["spec"], r["size_bound"], 313) for r in counts]
    cases += [("search", r["spec"], r["size_bound"], 129) for r in search]
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, cases, out), nprocs=world, join=True, start_method="spawn")
    for rank in range(world):
        got = out[rank]
        for (kind, spec, C, _), g, ref in zip(cases, got, counts + search):
            if kind == "count":
                table = O.OracleTable(spec["k"], C)
                assert [[a, b, c] for a, b, c, _ in g] == ref["per_size"]
                assert [v for *_, v in g] == [table.total(s) for s in range(1, C + 1)]
            else:
                assert g == [ref["size"], ref["rank"]], ref["name"]
