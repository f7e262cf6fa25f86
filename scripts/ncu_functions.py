"""Per-function totals of an ncu source page (cuda lines of libsimba's own
files): samples, instructions and no-instruction stalls, by the enclosing
function of each source line.  usage: ncu_functions.py rep [top]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def function_starts(path):
    starts = []
    head = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:__device__|__global__|static|inline|[A-Za-z_][\w:<>,\s\*&]*\s)"
                      r"[^;=]*?\b(\w+)\s*\(")
    for i, line in enumerate(path.read_text().splitlines(), start=1):
        if not line or line[0] in " \t#/}{" or line.rstrip().endswith(";"):
            continue
        m = head.match(line)
        if m and m.group(1) not in ("if", "for", "while", "switch", "return"):
            starts.append((i, m.group(1)))
    return starts


files = {p.name: function_starts(p) for p in (ROOT / "paper_2605_08243_b200" / "csrc").glob("*.cu*")}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
fname, hdr = None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or fname not in files:
        continue
    d = dict(zip(hdr, r))

    def f(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    ln = int(r[0])
    fn = "?"
    for start, name in files[fname]:
        if start > ln:
            break
        fn = name
    a = agg[f"{fname}:{fn}"]
    a[0] += f("Warp Stall Sampling (All Samples)")
    a[1] += f("Instructions Executed")
    a[2] += f("stall_no_inst")
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"{'function':40s} {'samples':>8s} {'instr':>8s} {'no_inst':>8s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k:40s} {100 * v[0] / ts:7.1f}% {100 * v[1] / ti:7.1f}% {100 * v[2] / ts:7.1f}%")
