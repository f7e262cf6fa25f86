"""Per-source-line breakdown (warp samples, instructions) of an ncu report.

usage: python scripts/ncu_lines.py rep.ncu-rep [top]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    def f(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    rows.append((fname, int(r[0]), r[1][:90], f("Warp Stall Sampling (All Samples)"), f("Instructions Executed")))
ts = sum(x[3] for x in rows) or 1
ti = sum(x[4] for x in rows) or 1
print(f"total samples {ts:.0f}  warp-instructions {ti:.3e}")
for fn, ln, src, s, i in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{fn:18s}{ln:5d} samp {100*s/ts:5.1f}%  inst {100*i/ti:5.1f}%  {src}")

# optional range aggregation: python scripts/ncu_lines.py rep N name:file:lo-hi ...
ranges = [a.split(":") for a in sys.argv[3:]]
if ranges:
    print("--- ranges")
    for name, fn, lohi in ranges:
        lo, hi = map(int, lohi.split("-"))
        s = sum(x[3] for x in rows if x[0] == fn and lo <= x[1] <= hi)
        i = sum(x[4] for x in rows if x[0] == fn and lo <= x[1] <= hi)
        print(f"{name:14s} samp {100*s/ts:5.1f}%  inst {100*i/ti:5.1f}%")
