"""Cross-GPU early exit of a sharded search (the reference's
break after the first wave with a hit, engine.py:248-250): every shard
publishes its hits to one shared 8-byte minimum (simba_xbest) and stops
claiming above any shard's hit.  The answer must stay the exact minimum
(size, rank) -- the oracle's and the single launch's -- while shards scan
less.  The multi-process test maps the word into other processes through its
CUDA IPC handle, as the ranks of a multi-GPU job do (here all on cuda:0)."""

import os
import random
import socket

import pytest

import oracle as O

pytestmark = pytest.mark.gpu

S = pytest.importorskip("paper_2605_08243_b200")
from paper_2605_08243_b200 import _native as N  # noqa: E402
from paper_2605_08243_b200 import codec, expr, parallel  # noqa: E402
from paper_2605_08243_b200.engine import DeviceContext, SharedMinimum  # noqa: E402

SIZE = 11


@pytest.fixture(scope="module", autouse=True)
def need_device():
    if N.device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU tests must run on a B200")


def planted(seed, target_size):
    """k=4 w=32 n=10 spec labelled by a uniform expression of target_size."""
    rng = random.Random(seed)
    table = S.build(4, SIZE)
    e = codec.sample_uniform(target_size, table, rng)
    pairs, seen = [], set()
    while len(pairs) < 10:
        x = tuple(rng.getrandbits(32) for _ in range(4))
        if x not in seen:
            seen.add(x)
            pairs.append((x, expr.evaluate(e, x, 32)))
    return tuple(pairs)


CASES = [(31, 9), (32, 10), (33, 10), (34, 11), (35, 11)]


def oracle_answer(pairs, bound=SIZE):
    tab = O.OracleTable(4, bound)
    for s in range(1, bound + 1):
        _, _, first, toks = O.scan_range(tab, 4, 32, list(pairs), s, 0, tab.total(s), 0, tab.total(s),
                                         threads=O.cpu_count())
        if first is not None:
            return s, first, toks
    return None, None, None


def test_shared_minimum_in_process_exact_and_shorter():
    for seed, ts in CASES:
        pairs = tuple(planted(seed, ts))
        spec = S.Specification(k=4, w=32, pairs=pairs)
        want = oracle_answer(pairs)
        assert want[0] is not None
        table = S.build(4, SIZE)
        vrank = sum(table.total(s) for s in range(1, want[0])) + want[1]
        with DeviceContext(spec, SIZE) as ctx, SharedMinimum(0) as shared:
            one, _ = ctx.run_levels(1, SIZE, mode="search")
            assert (one.size, one.best_rank, one.tokens) == want
            for nsh in (2, 8):
                alone = [ctx.run_levels(1, SIZE, mode="search", shard=i, nshards=nsh)[0] for i in range(nsh)]
                ctx.set_shared_minimum(shared)
                shared.reset()
                together = [ctx.run_levels(1, SIZE, mode="search", shard=i, nshards=nsh)[0] for i in range(nsh)]
                ctx.set_shared_minimum(None)
                for runs in (alone, together):
                    hits = [(r.size, r.best_rank, r.tokens) for r in runs if r.best_rank is not None]
                    assert min(hits) == want, (seed, nsh)
                assert shared.read() == vrank
                # later shards start from the published minimum: no more work than
                # alone (up to the piece granularity at which a stop is counted)
                slack = nsh << 20
                assert sum(r.visited for r in together) <= sum(r.visited for r in alone) + slack, (seed, nsh)


def test_shared_minimum_detached_contexts_ignore_it():
    pairs = tuple(planted(31, 9))
    spec = S.Specification(k=4, w=32, pairs=pairs)
    with DeviceContext(spec, SIZE) as ctx, SharedMinimum(0) as shared:
        shared.reset()
        # a single-shard or count request never touches the word
        ctx.set_shared_minimum(shared)
        ctx.run_levels(1, SIZE, mode="search")
        ctx.run_levels(1, 9, mode="count", shard=0, nshards=2)
        assert shared.read() is None
        ctx.set_shared_minimum(None)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, cases, count_bound, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shared = parallel.shared_minimum(rank, world, device=0)
        res, counts = [], []
        for pairs in cases:
            spec = S.Specification(k=4, w=32, pairs=tuple(pairs))
            with DeviceContext(spec, SIZE, device=0) as ctx:
                ctx.set_shared_minimum(shared)
                size, first, levels = parallel.search_fused(parallel.device_levels(ctx), SIZE, rank, world,
                                                            shared=shared)
                ctx.set_shared_minimum(None)
                lv = parallel.count_fused(parallel.device_levels(ctx), count_bound, rank, world)
            res.append([size, first, sum(v for *_, v in levels)])
            counts.append([[x.size, x.count, x.first_rank, x.visited] for x in lv])
        dist.barrier()  # the creator's word outlives every rank's searches
        shared.close()
        out[rank] = (res, counts)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [3, 8])
def test_sharded_device_path_across_processes(world):
    """The multi-GPU protocol with the real device path: `world` processes
    (gloo; all on cuda:0 here, one GPU each on a multi-GPU node) shard the
    fused search with the shared minimum and the fused count; every rank gets
    the oracle's (size, rank) and the oracle's per-level counts."""
    import torch.multiprocessing as mp

    cases = [planted(seed, ts) for seed, ts in CASES]
    want = [oracle_answer(p)[:2] for p in cases]
    count_bound = 10
    tab = O.OracleTable(4, count_bound)
    want_counts = []
    for p in cases:
        rows = []
        for s in range(1, count_bound + 1):
            _, c, f, _ = O.scan_range(tab, 4, 32, list(p), s, 0, tab.total(s), 0, tab.total(s),
                                      threads=O.cpu_count())
            rows.append([s, c, f, tab.total(s)])
        want_counts.append(rows)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_rank_main, args=(world, _free_port(), cases, count_bound, out), nprocs=world, join=True,
                       start_method="spawn")
    for rank in range(world):
        got, counts = out[rank]
        assert [tuple(g[:2]) for g in got] == [tuple(w) for w in want], rank
        assert counts == want_counts, rank


def test_shared_minimum_stops_a_shard_above_another_shards_hit():
    """The planted size-9 spec of the C5 golden (first hits: level 9 at rank
    12435603, level 10 at 73124301): over levels 1..11 in 2 shards, the answer
    lies in shard 0's first super-chunk while shard 1's own first hit is a
    level-10 rank far above it.  Alone, shard 1 sweeps up to its own hit;
    attached to the minimum shard 0 published, it stops at once, and it
    reports the job's answer."""
    from conftest import load_golden

    p = next(x for x in load_golden("c5")["planted"] if x["name"] == "sparse_size9")
    spec = S.Specification(k=4, w=32, pairs=tuple((tuple(i), o) for i, o in p["spec"]["pairs"]))
    lv9 = next(x for x in p["levels"] if x["size"] == 9)
    want = (9, lv9["first"])
    with DeviceContext(spec, SIZE) as ctx, SharedMinimum(0) as shared:
        alone1, _ = ctx.run_levels(1, SIZE, mode="search", shard=1, nshards=2)
        ctx.set_shared_minimum(shared)
        shared.reset()
        r0, _ = ctx.run_levels(1, SIZE, mode="search", shard=0, nshards=2)
        r1, _ = ctx.run_levels(1, SIZE, mode="search", shard=1, nshards=2)
        ctx.set_shared_minimum(None)
    assert (r0.size, r0.best_rank) == want
    assert alone1.best_rank is not None and (alone1.size, alone1.best_rank) > want
    assert (r1.size, r1.best_rank) == want  # the pulled minimum
    assert r1.visited + (1 << 20) < alone1.visited, (r1.visited, alone1.visited)


def _tts_rank_main(rank, world, port, specs, bound, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shared = parallel.shared_minimum(rank, world, device=0)
        res = []
        for pairs in specs:
            dist.barrier()
            spec = S.Specification(k=4, w=32, pairs=tuple(tuple(x) if isinstance(x, list) else x for x in pairs))
            with DeviceContext(spec, bound, device=0) as ctx:
                ctx.set_shared_minimum(shared)
                size, first, _ = parallel.search_fused(parallel.device_levels(ctx), bound, rank, world, shared=shared)
                ctx.set_shared_minimum(None)
            res.append([size, first])
        dist.barrier()
        shared.close()
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_consecutive_searches_never_see_the_previous_minimum():
    """Consecutive C5 time-to-solve targets on 8 processes sharing one minimum,
    each right after a target with a smaller answer, two of them dense
    (per-example tables, examples reordered at context creation).  The word's
    reset must land before any rank launches: with a reset that returned once
    its value was staged, 8 ranks on one GPU reported the previous target's
    answer for s12_k4_i08 and s12_k4_i37."""
    import torch.multiprocessing as mp
    from conftest import load_golden

    g = load_golden("c5")
    recs = {r["id"]: r for recs in g["tts"].values() for r in recs}
    order = ["s11_k4_i40", "s12_k4_i08", "s12_k4_i32", "s12_k4_i37", "s11_k4_i16", "s12_k4_i08"]
    specs = [[(tuple(i), o) for i, o in recs[x]["spec"]["pairs"]] for x in order]
    want = [[recs[x]["oracle"]["size"], recs[x]["oracle"]["rank"]] for x in order]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_tts_rank_main, args=(8, _free_port(), specs, 12, out), nprocs=8, join=True,
                       start_method="spawn")
    for rank in range(8):
        assert out[rank] == want, rank
