"""Which CUDA source lines emit a given SASS opcode (executions, samples).

usage: python scripts/ncu_ops.py rep.ncu-rep OPCODE_PREFIX[,OPCODE_PREFIX...] [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, ops = sys.argv[1], sys.argv[2].split(",")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, line, text = None, None, ""
ex, sm = collections.Counter(), collections.Counter()
src = {}


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0].isdigit():
        line, text = int(r[0]), r[1][:80]
        continue
    if len(r) < 8 or not r[3].strip():
        continue
    p = r[3].split()
    o = p[1] if p[0].startswith("@") else p[0]
    if any(o.startswith(x) for x in ops):
        k = (fname, line, o)
        ex[k] += num(r[7])
        sm[k] += num(r[4])
        src[k] = text
for k, v in sorted(ex.items(), key=lambda kv: -sm[kv[0]])[:top]:
    print(f"{k[0][:12]:12s}{k[1]:5d} {k[2]:18s} ex={v:.2e} samp={int(sm[k]):7d}  {src[k]}")
