"""Summarise an ncu --set full report into profiles/<name>.json (run here, no GPU).

usage: python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/name.json [label] [candidates/launch]
"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, dst, label="", candidates=None):
    raw = page(rep, "--page", "raw")
    h, units, vals = raw[0], raw[1], raw[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__block_size", "launch__grid_size", "sm__cycles_active.avg",
            "smsp__average_warp_latency_per_inst_issued.ratio", "lts__t_bytes.sum"]
    metrics = {k: (d.get(k), u.get(k)) for k in keep if k in d}

    def num(k, scale=1.0):
        try:
            return float(d[k].replace(",", "")) * scale
        except (KeyError, ValueError):
            return None

    def bytes_(k):
        unit = u.get(k, "")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        return num(k, mult)

    src = page(rep, "--page", "source", "--print-source", "sass")
    sh, rows = src[1], src[2:]
    stalls = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    agg = {c[6:]: sum(f(r[sh.index(c)]) for r in rows) for c in stalls}
    tot = sum(agg.values()) or 1.0
    ie, isrc = sh.index("Instructions Executed"), sh.index("Source")
    top = sorted(rows, key=lambda r: -f(r[ie]))[:24]
    summary = {
        "label": label, "report": rep, "metrics": metrics,
        "candidates_per_launch": int(candidates) if candidates else None,
        "dram_bytes_per_launch": (bytes_("dram__bytes_read.sum") or 0) + (bytes_("dram__bytes_write.sum") or 0),
        "stall_share": {k: round(v / tot, 4) for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v},
        "top_sass_by_executions": [{"sass": r[isrc], "executed": int(f(r[ie]))} for r in top],
        "opcode_executions": dict(Counter({(r[isrc].split()[1] if r[isrc].startswith("@") else r[isrc].split()[0]):
                                           0 for r in rows if r[isrc]})) and None,
    }
    ops = Counter()
    for r in rows:
        parts = r[isrc].split()
        if parts:
            ops[parts[1] if parts[0].startswith("@") else parts[0]] += f(r[ie])
    summary["opcode_executions"] = dict(ops.most_common(20))
    with open(dst, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({k: summary[k] for k in ("label", "dram_bytes_per_launch", "stall_share")}, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
