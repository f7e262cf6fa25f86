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
roofline  INT32 roofline of the step's launch: algorithmic integer ops
        (sum_s T[s] * s * e-bar) / its CUDA-event duration,
        against P_int32 = the LOP3-only ALU-pipe rate measured in this run
        (simba_int32_pipe_peak; MEASURED_PEAKS.json has no integer figure).
        That frac exceeds 1 by construction; roofline.hw holds
        the hardware fractions: the mandatory test op per candidate against
        the ALU-pipe peak, and issued instructions against the issue limit
cpu_baseline  the CPU oracle (oracle/simba_oracle.c, restatement of the
        reference path) on all host threads over a bounded size-13 sample;
        cpu_baseline.python_reference = the unmodified Python reference
        (baseline/_ref) through its own synthesize() with workers = all
        host threads, on the same spec
time_to_solve  synthesize on the 30-target suite (ten per size 11/12/13,
        minimal size = target size), every answer asserted against the
        oracle's (tests/golden/c5.json); with N ranks, a sharded fused search
        with the cross-GPU shared minimum

`--impl reference` times the CPU oracle as the reference arm.
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


_PY_REF = r"""
import json, os, sys, time
from mbasynth import counting
from mbasynth.engine import EngineConfig, Specification, synthesize, run_stats
pairs, budget = json.loads(sys.argv[1]), float(sys.argv[2])
spec = Specification(k=4, w=32, pairs=tuple((tuple(i), o) for i, o in pairs))
workers = len(os.sched_getaffinity(0))
t0 = time.perf_counter()
out = synthesize(spec, counting.build(4, 13), EngineConfig(size_bound=13, workers=workers, time_budget=budget))
wall = time.perf_counter() - t0
st = run_stats(out)
print(json.dumps({"status": out.status.value, "workers": workers, "wall_s": wall,
                  "visited": st["total_candidates"], "rate_stats": st["candidates_per_second"],
                  "sizes": [[x.size, x.candidates] for x in out.stats]}))
"""


def python_reference_sample(budget_s=20.0):
    """The UNMODIFIED reference (Python, installed in baseline/_ref) through its
    public synthesize() on the C5 unsat spec with workers = all host threads
    and a time budget: its own per-size stats give candidates/s (the rate
    SURVEY.md 6 quotes), measured on this host in this run."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "mbasynth").is_dir():
        return {"unavailable": "reference not installed in baseline/_ref (DESIGN.md: reference install)"}
    env = dict(os.environ, PYTHONPATH=str(ref))
    try:
        p = subprocess.run([sys.executable, "-c", _PY_REF, json.dumps([[list(i), o] for i, o in unsat_pairs()]),
                            str(budget_s)], cwd=str(ref), env=env, capture_output=True, text=True,
                           timeout=budget_s * 4 + 120)
        d = json.loads(p.stdout.strip().splitlines()[-1])
    except (subprocess.TimeoutExpired, ValueError, IndexError) as exc:
        return {"unavailable": f"reference run failed: {exc!r}"[:200]}
    return {"value": d["visited"] / d["wall_s"], "unit": UNIT, "cores": d["workers"], "kind": "reference",
            "rate_per_size_stats": d["rate_stats"],
            "sample": f"mbasynth.synthesize (unmodified, baseline/_ref) on the C5 unsat spec, workers={d['workers']}, "
                      f"time_budget={budget_s:g}s: {d['status']}, {d['visited']} candidates in {d['wall_s']:.1f}s "
                      f"wall (sizes swept {d['sizes']})"}


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
    # the reference's own Python path on the same host, for context
    cb["python_reference"] = python_reference_sample(args.py_ref_s)
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
    ap.add_argument("--py-ref-s", type=float, default=15.0, help="time budget of the Python reference sample")
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

    # roofline of the (only) launch of a step: all levels, INT32 pipe peaks
    peaks = int_peaks(N, local)
    ebar = 1.0 + launch["ex0"] / max(1, cands_per_step // world)
    k_ms = statistics.mean(klaunch)
    algo_ops = sum(t * s for s, t in enumerate(totals, start=1)) / world * ebar  # sum over levels of T[s] * s
    achieved = algo_ops / (k_ms * 1e-3)
    cand_s = (cands_per_step / world) / (k_ms * 1e-3)
    sha = lib_sha16()
    prof = profile_summary(sha)
    sms = info.get("grid_blocks", 148)  # one CTA per SM
    clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
    issue_peak = sms * 4 * clk  # warp instructions/s: 1 per SMSP and cycle
    hw = {
        "test_op_frac": cand_s * ebar / peaks["alu"],
        "test_op_note": "the one masked compare (LOP3.PAND) per candidate and example evaluated -- the "
                        "algorithm's floor -- against the LOP3-only ALU-pipe peak measured in this run",
        "warp_inst_per_candidate": prof.get("warp_inst_per_candidate"),
        "issue_frac": (prof["warp_inst_per_candidate"] * cand_s / issue_peak
                       if prof.get("warp_inst_per_candidate") else None),
        "issue_note": "issued warp instructions/s (this run's candidates/s x the ncu instructions per candidate of "
                      "this build) / (SMs x 4 schedulers x the SM clock sampled in this run)",
        "alu_pipe_pct": prof.get("alu_pipe_pct"),
        "issue_active_pct": prof.get("issue_active_pct"),
        "profile": prof.get("file"), "profile_build": prof.get("build"), "build": sha,
        "profile_matches_build": prof.get("build") == sha,
    }
    roofline = {"bound": "int32", "achieved": achieved / 1e9, "peak": peaks["alu"] / 1e9, "unit": "Gop/s",
                "frac": achieved / peaks["alu"], "traffic": prof.get("dram_bytes_per_launch"),
                "peak_dual": peaks["dual"] / 1e9,
                "note": f"SURVEY.md 8(d): the step's unit_kernel launch (levels 1..{C}), sum_s T[s]/N x s tokens "
                        f"x e-bar={ebar:.6f} integer ops / {k_ms:.3f} ms (CUDA events) against P_int32 = the "
                        "LOP3-only ALU-pipe rate measured in this run (simba_int32_pipe_peak; peak_dual = LOP3+IMAD, "
                        "the issue limit; MEASURED_PEAKS.json has no integer figure).  frac > 1 by construction: "
                        "subtrees shared by a row or column are evaluated once and the ancestors are folded into "
                        "the test, so the kernel spends ~1 LOP3 per candidate, not s*e-bar ops (DESIGN.md 2).  "
                        "Efficiency is in 'hw'.",
                "hw": hw}

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
        cpu["python_reference"] = python_reference_sample(args.py_ref_s)

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


def int_peaks(N, device):
    """Integer pipe peaks measured on this GPU (simba_int32_pipe_peak):
    LOP3-only (ALU pipe = SURVEY.md 8(d)'s P_int32) and LOP3+IMAD (ALU + FMA
    pipes, the issue limit); best of three launches each."""
    import ctypes as C

    out = {}
    for name, mode in (("alu", 0), ("dual", 1)):
        best = 0.0
        for _ in range(3):
            ops, ms = C.c_double(), C.c_double()
            N.check_rc(N.lib.simba_int32_pipe_peak(device, 8192, mode, C.byref(ops), C.byref(ms)))
            best = max(best, ops.value)
        out[name] = best
    return out


def lib_sha16():
    """Identity of the libsimba build: sha256 of its CUDA sources and header
    (what a rebuild with the same nvcc reproduces; the binary itself is not
    byte-stable across rebuilds)."""
    import hashlib

    h = hashlib.sha256()
    for f in ("paper_2605_08243_b200/csrc/simba.cu", "paper_2605_08243_b200/csrc/simba_device.cuh",
              "paper_2605_08243_b200/csrc/vfb_impl.cuh", "include/simba.h"):
        h.update((ROOT / f).read_bytes())
    return h.hexdigest()[:16]


def profile_summary(sha):
    """Per-launch figures of the step's unit-kernel launch from the committed
    ncu summary (profiles/ncu_unit_kernel.json: the bench-step launch of a
    given libsimba build, its sha recorded as "build"): DRAM bytes, warp
    instructions per candidate, ALU-pipe and issue-active %.  The bench line
    says whether that build is the one running (profile_matches_build)."""
    p = ROOT / "profiles" / "ncu_unit_kernel.json"
    out = {"file": str(p.relative_to(ROOT))}
    try:
        d = json.loads(p.read_text())
    except (OSError, ValueError):
        return out
    out["build"] = d.get("libsimba_sha16")
    out["dram_bytes_per_launch"] = d.get("dram_bytes_per_launch")
    m = d.get("metrics", {})

    def f(name):
        try:
            return float(m[name][0])
        except (KeyError, ValueError, TypeError, IndexError):
            return None

    try:
        out["warp_inst_per_candidate"] = f("smsp__inst_executed.sum") / d["candidates_per_launch"]
    except (KeyError, TypeError, ZeroDivisionError):
        pass
    out["issue_active_pct"] = f("smsp__issue_active.avg.pct_of_peak_sustained_active")
    out["alu_pipe_pct"] = f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")
    return out


def c5_targets(S):
    """The time-to-solve suite (BASELINE configs[4]): ten targets per size
    11, 12, 13 drawn by the reference's own suite generator whose MINIMAL
    solution size is that size, each with the oracle's answer pinned in
    tests/golden/c5.json (make_c5_golden.py)."""
    g = json.loads((ROOT / "tests" / "golden" / "c5.json").read_text())
    for size in sorted(g["tts"], key=int):
        for rec in g["tts"][size]:
            sp = rec["spec"]
            spec = S.Specification(k=sp["k"], w=sp["w"], pairs=tuple((tuple(i), o) for i, o in sp["pairs"]))
            yield int(size), spec, rec


def tts_summary(out):
    by = {}
    for r in out:
        by.setdefault(r["target_size"], []).append(r)
    return {str(s): {"n": len(rs), "median_ms": round(statistics.median(r["ms"] for r in rs), 2),
                     "max_ms": round(max(r["ms"] for r in rs), 2),
                     "cpu_oracle_median_s": round(statistics.median(r["cpu_oracle_s"] for r in rs), 1)}
            for s, rs in sorted(by.items())}


def _tts_record(target, rec, size, first, ms, **extra):
    want = rec["oracle"]
    if (size, first) != (want["size"], want["rank"]):
        raise AssertionError(f"time-to-solve {rec['id']}: device ({size}, {first}) != oracle "
                             f"({want['size']}, {want['rank']})")
    return {"id": rec["id"], "target_size": target, "found_size": size, "rank": first, "ms": round(ms, 2),
            "cpu_oracle_s": rec["oracle_s"], **extra}


def time_to_solve(S, C):
    """Time-to-solution of synthesize (sizes 1..C, early exit; context
    creation included) on the 30-target suite, every answer asserted equal to
    the oracle's."""
    out = []
    # one untimed search first: module load / first-context costs are per process
    S.synthesize(S.Specification(k=K, w=W_BITS, pairs=unsat_pairs()), S.build(K, 5), S.EngineConfig(size_bound=5))
    table = S.build(K, C)
    for target, spec, rec in c5_targets(S):
        t0 = time.perf_counter()
        o = S.synthesize(spec, table, S.EngineConfig(size_bound=C))
        ms = (time.perf_counter() - t0) * 1e3
        out.append(_tts_record(target, rec, o.size, o.rank, ms))
    return {"targets": out, "by_size": tts_summary(out),
            "verified": "every (size, rank) equals the oracle's (tests/golden/c5.json)",
            "cpu_oracle": "cpu_oracle_s: the multithreaded C oracle's Alg. 1 on the GPU box host (recorded when the "
                          "golden was made, make_c5_golden.py)"}


def time_to_solve_ranks(S, C, rank, world, local, rdev, allmax, barrier):
    """time_to_solve on N ranks: each rank binds the spec to
    its GPU and runs its shard of sizes 1..C as one fused search launch, all
    shards publishing hits to one shared minimum on rank 0's GPU (early exit
    across GPUs); one MIN exchange gives the (size, rank) answer
    (parallel.search_fused).  The time is the max over ranks, context
    creation included like synthesize's."""
    from paper_2605_08243_b200 import parallel as P
    from paper_2605_08243_b200.engine import DeviceContext

    shared = P.shared_minimum(rank, world, device=local)
    with DeviceContext(S.Specification(k=K, w=W_BITS, pairs=unsat_pairs()), 5, device=local) as ctx:
        ctx.set_shared_minimum(shared)
        P.search_fused(P.device_levels(ctx), 5, rank, world, device=rdev, shared=shared)  # untimed first search
        ctx.set_shared_minimum(None)
    out = []
    for target, spec, rec in c5_targets(S):
        barrier()
        t0 = time.perf_counter()
        with DeviceContext(spec, C, device=local) as ctx:
            ctx.set_shared_minimum(shared)
            size, first, _ = P.search_fused(P.device_levels(ctx), C, rank, world, device=rdev, shared=shared)
            ctx.set_shared_minimum(None)
        ms = allmax(time.perf_counter() - t0) * 1e3
        out.append(_tts_record(target, rec, size, first, ms, ranks=world))
    barrier()  # rank 0's word outlives every rank's searches
    shared.close()
    return {"targets": out, "by_size": tts_summary(out),
            "verified": "every (size, rank) equals the oracle's (tests/golden/c5.json)"}


if __name__ == "__main__":
    sys.exit(main())
