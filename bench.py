#!/usr/bin/env python
"""bench.py -- SIMBA hot path on B200: candidate expressions evaluated per second.

Workload (BASELINE.json configs[4], "C5"): k=4 variables, w=32, n=10 examples,
random outputs (unsatisfiable; the reference's full-sweep spec style,
test_acceptance.py:278-289), exhaustive-count sweep of every size level 1..13
(111,946,005,116 candidates per step) in ONE launch per step and rank: the
levels' concatenated rank space (simba_run_levels) is sharded round-robin over
the ranks (torchrun for N>1, one process per GPU) and reduced with one
all_reduce per step -- the only exchange.

value   device-timed whole-job candidates/s (CUDA events on the library
        stream, inputs resident, max over ranks)
e2e     same metric through the public API with host buffers each step
        (context creation = H2D of spec + tables, per-spec value tables,
        scans, D2H of the results)
roofline  INT32 issue roofline of the step's launch: algorithmic integer ops
        (sum_s T[s] * s * e-bar) / its CUDA-event duration,
        against the INT32 peak measured on this box by simba_int32_peak
        (MEASURED_PEAKS.json has no integer figure)
cpu_baseline  the CPU oracle (oracle/simba_oracle.c, restatement of the
        reference path) on all host threads over a bounded size-13 sample

`--impl reference` times that CPU implementation as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "candidate exprs evaluated/sec"
UNIT = "candidates/s"
K, W_BITS, N_PAIRS, SEED = 4, 32, 10, 31337


def unsat_pairs(k=K, w=W_BITS, n=N_PAIRS, seed=SEED):
    rng = random.Random(seed)
    pairs, seen = [], set()
    while len(pairs) < n:
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x in seen:
            continue
        seen.add(x)
        pairs.append((x, rng.getrandbits(w)))
    return tuple(pairs)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [r for r in rows if r[0] > 0.5 * r[1]] or rows
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU oracle


def cpu_sample(size_bound, budget_s=10.0, seed_offset=0):
    """The CPU oracle (reference restatement) on all host threads over a bounded
    rank window of the largest size level, sized to ~budget_s."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O

    pairs = list(unsat_pairs())
    tab = O.OracleTable(K, size_bound)
    threads = O.cpu_count()
    total = tab.total(size_bound)
    lo = total // 3 + seed_offset
    n = 1 << 20
    t0 = time.perf_counter()
    O.scan_range(tab, K, W_BITS, pairs, size_bound, 0, total, lo, lo + n, threads=threads)
    rate = n / (time.perf_counter() - t0)
    n2 = int(min(total - lo, max(n, rate * budget_s)))
    t0 = time.perf_counter()
    v, cnt, _, _ = O.scan_range(tab, K, W_BITS, pairs, size_bound, 0, total, lo, lo + n2, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": v / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{v} consecutive size-{size_bound} ranks from {lo} (k=4 w=32 n=10 unsat spec), "
                      f"oracle/simba_oracle.c with {threads} threads, {dt:.1f}s"}


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        cpu_sample(args.size_bound, budget_s=args.ref_step_s)
    samples = [cpu_sample(args.size_bound, budget_s=args.ref_step_s, seed_offset=i) for i in range(args.steps)]
    value = statistics.mean(s["value"] for s in samples)
    cb = dict(samples[0])
    cb["value"] = value
    cb["sample"] = f"{args.steps} steps of: " + samples[0]["sample"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": config_dict(args),
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args):
    return {"workload": f"C5 exhaustive-count sweep, sizes 1..{args.size_bound}, k=4 w=32 n=10, "
                        "random-output (unsat) spec; all levels in one launch, sharded round-robin across ranks",
            "k": K, "w": W_BITS, "n_examples": N_PAIRS, "size_bound": args.size_bound,
            "parallelism": f"rank-space shards x{args.gpus}",
            "l2": "no flush needed: ~0 HBM bytes per candidate; value tables <= 80 MB built once per spec"}


# ---------------------------------------------------------------- our arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size-bound", type=int, default=13)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tts", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2605_08243_b200 as S
    from paper_2605_08243_b200 import _native as N
    from paper_2605_08243_b200 import parallel
    from paper_2605_08243_b200.engine import DeviceContext

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    # SIMBA_BENCH_DEVICE / SIMBA_BENCH_BACKEND=gloo: exercise the multi-rank
    # path with several ranks on one GPU (testing only; NCCL needs distinct GPUs)
    local = env_int("SIMBA_BENCH_DEVICE", local)
    backend = os.environ.get("SIMBA_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    rdev = dev if backend == "nccl" else torch.device("cpu")  # reduction tensors

    C = args.size_bound
    spec = S.Specification(k=K, w=W_BITS, pairs=unsat_pairs())
    table = S.build(K, C)
    totals = [table.total(s) for s in range(1, C + 1)]
    cands_per_step = sum(totals)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = DeviceContext(spec, C, device=local)
    info = ctx.info()
    scan_levels = parallel.device_levels(ctx)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev)
    launch = {}

    def step():
        # every size level 1..C in ONE launch per rank (this rank's round-robin
        # shard of the levels' concatenated rank space), one reduction per step
        r, levels = scan_levels(1, C, "count", rank, world)
        launch["ms"] = r.kernel_ms
        launch["ex0"] = r.ex0_hits
        if world > 1:
            tot = torch.tensor([sum(v for *_, v in levels), sum(c for _, c, _, _ in levels)], dtype=torch.int64,
                               device=rdev)
            dist.all_reduce(tot, op=dist.ReduceOp.SUM)
            return int(tot[0].item())
        return sum(v for *_, v in levels)

    for _ in range(args.warmup):
        step()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    launches0 = N.launch_count()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    klaunch = []
    visited = 0
    for _ in range(args.steps):
        visited = step()
        klaunch.append(launch["ms"])
    torch.cuda.synchronize()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = N.launch_count() - launches0
    clocks = sampler.stop()
    dev_ms = e0.elapsed_time(e1)
    dev_ms = allmax(dev_ms)
    assert visited == cands_per_step, (visited, cands_per_step)
    value = cands_per_step * args.steps / (dev_ms * 1e-3)

    # roofline of the (only) launch of a step: all levels, INT32 issue peak
    peak_ops, peak_ms = C_double_pair(N, local)
    ebar = 1.0 + launch["ex0"] / max(1, cands_per_step // world)
    k_ms = statistics.mean(klaunch)
    algo_ops = sum(t * s for s, t in enumerate(totals, start=1)) / world * ebar  # sum over levels of T[s] * s
    achieved = algo_ops / (k_ms * 1e-3)
    prof = profile_summary()
    cand_s = (cands_per_step / world) / (k_ms * 1e-3)
    roofline = {"bound": "int32", "achieved": achieved / 1e9, "peak": peak_ops / 1e9, "unit": "Gop/s",
                "frac": achieved / peak_ops, "traffic": prof.get("dram_bytes_per_launch"),
                "note": f"the step's unit_kernel launch (levels 1..{C}): sum_s T[s]/N x s tokens x e-bar={ebar:.6f} "
                        f"integer ops (SURVEY.md 8(d)) / {k_ms:.3f} ms (CUDA events); peak = simba_int32_peak "
                        "LOP3+IMAD issue rate measured on this GPU (no integer figure in MEASURED_PEAKS.json). "
                        "frac > 1 because shared subtrees are evaluated once per row/column, so the kernel spends "
                        "~1 LOP3 per candidate instead of s*e-bar ops (DESIGN.md 2); see 'per_candidate' for the "
                        "instruction-level view",
                "per_candidate": {
                    "test_ops_per_s": cand_s * ebar / 1e9,
                    "frac_of_peak": cand_s * ebar / peak_ops,
                    "warp_inst_per_candidate": prof.get("warp_inst_per_candidate"),
                    "issue_active_pct": prof.get("issue_active_pct"),
                    "note": "one masked-compare (LOP3.PAND) test per candidate and example evaluated: "
                            "the floor of this algorithm; ncu fields from the committed profile "
                            "(profiles/ncu_unit_kernel.json: this step's fused launch, C5 sizes 1..13)"}}

    # e2e through the public API: host spec -> context (H2D) -> scans -> D2H
    e2e = None
    if args.e2e_steps > 0:
        def e2e_step():
            c2 = DeviceContext(spec, C, device=local)
            parallel.count_fused(parallel.device_levels(c2), C, rank, world, device=rdev)
            hb, db = c2.copied_bytes()
            c2.close()
            return hb, db

        e2e_step()  # untimed warm-up: the first context of a process also allocates its pooled arena
        h2d = d2h = 0
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            hb, db = e2e_step()
            h2d += hb
            d2h += db
        torch.cuda.synchronize()
        barrier()
        e2e_s = allmax(time.perf_counter() - t0)
        e2e = {"value": cands_per_step * args.e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d // args.e2e_steps, "d2h_bytes_per_step": d2h // args.e2e_steps}

    tts = None
    if not args.no_tts:
        if world == 1:
            tts = time_to_solve(S, C)
        else:  # every rank takes part: sharded fused search + MIN exchange
            tts = time_to_solve_ranks(S, C, rank, world, local, rdev, allmax, barrier)

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_sample(C, budget_s=args.cpu_budget)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config_dict(argparse.Namespace(size_bound=C, gpus=world)),
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "time_to_solve": tts,
            "kernel": {"launch_ms": k_ms, "launches_per_step": 1, "e_bar": ebar, **info},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def C_double_pair(N, device):
    import ctypes as C

    ops, ms = C.c_double(), C.c_double()
    N.check_rc(N.lib.simba_int32_peak(device, 4096, C.byref(ops), C.byref(ms)))
    return ops.value, ms.value


def profile_summary():
    """Per-launch figures of the step's unit-kernel launch from the committed
    ncu summary (profiles/ncu_unit_kernel.json, a copy of the fused-sweep
    capture): DRAM bytes, warp instructions per candidate, issue-active %."""
    p = ROOT / "profiles" / "ncu_unit_kernel.json"
    out = {}
    try:
        d = json.loads(p.read_text())
    except (OSError, ValueError):
        return out
    out["dram_bytes_per_launch"] = d.get("dram_bytes_per_launch")
    m = d.get("metrics", {})
    try:
        out["warp_inst_per_candidate"] = float(m["smsp__inst_executed.sum"][0]) / d["candidates_per_launch"]
    except (KeyError, ValueError, TypeError, ZeroDivisionError):
        pass
    try:
        out["issue_active_pct"] = float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0])
    except (KeyError, ValueError, TypeError):
        pass
    return out


def time_to_solve(S, C):
    """Time-to-solution (synthesize, sizes 1..C, early exit) for the C5
    targets of sizes 11..13 whose specs are pinned in tests/golden/windows.json."""
    wins = json.loads((ROOT / "tests" / "golden" / "windows.json").read_text())
    out = []
    # one untimed search first: module load / first-context costs are per process
    S.synthesize(S.Specification(k=K, w=W_BITS, pairs=unsat_pairs()), S.build(K, 5), S.EngineConfig(size_bound=5))
    for r in wins:
        if r.get("meta", {}).get("config") != "C5" or "target_rank" not in r.get("meta", {}):
            continue
        sp = r["spec"]
        spec = S.Specification(k=sp["k"], w=sp["w"], pairs=tuple((tuple(i), o) for i, o in sp["pairs"]))
        t0 = time.perf_counter()
        o = S.synthesize(spec, S.build(sp["k"], C), S.EngineConfig(size_bound=C))
        ms = (time.perf_counter() - t0) * 1e3
        out.append({"target_size": r["size"], "found_size": o.size, "rank": o.rank, "ms": round(ms, 2)})
    return out


def c5_targets(S):
    wins = json.loads((ROOT / "tests" / "golden" / "windows.json").read_text())
    for r in wins:
        if r.get("meta", {}).get("config") != "C5" or "target_rank" not in r.get("meta", {}):
            continue
        sp = r["spec"]
        yield r["size"], S.Specification(k=sp["k"], w=sp["w"], pairs=tuple((tuple(i), o) for i, o in sp["pairs"]))


def time_to_solve_ranks(S, C, rank, world, local, rdev, allmax, barrier):
    """time_to_solve on N ranks: each rank binds the spec to
    its GPU and runs its shard of sizes 1..C as one fused search launch; one
    MIN exchange gives the (size, rank) answer (parallel.search_fused).  The
    time is the max over ranks, context creation included like synthesize's."""
    from paper_2605_08243_b200 import parallel as P
    from paper_2605_08243_b200.engine import DeviceContext

    with DeviceContext(S.Specification(k=K, w=W_BITS, pairs=unsat_pairs()), 5, device=local) as ctx:
        P.search_fused(P.device_levels(ctx), 5, rank, world, device=rdev)  # untimed first search
    out = []
    for target, spec in c5_targets(S):
        barrier()
        t0 = time.perf_counter()
        with DeviceContext(spec, C, device=local) as ctx:
            size, first, _ = P.search_fused(P.device_levels(ctx), C, rank, world, device=rdev)
        ms = allmax(time.perf_counter() - t0) * 1e3
        out.append({"target_size": target, "found_size": size, "rank": first, "ms": round(ms, 2), "ranks": world})
    return out


if __name__ == "__main__":
    sys.exit(main())
