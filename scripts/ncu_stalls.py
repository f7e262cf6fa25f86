"""Per-source-line stall breakdown of an ncu report (cuda lines only):
top lines by a stall reason.  usage: ncu_stalls.py rep [reason] [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
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
    rows.append((fname, int(r[0]), r[1][:80], f(reason), f("Warp Stall Sampling (All Samples)")))
tot = sum(x[4] for x in rows) or 1
tr = sum(x[3] for x in rows) or 1
print(f"{reason}: {100 * tr / tot:.1f}% of all samples")
for fn, ln, src, s, a in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{fn:18s}{ln:5d} {100 * s / tot:5.1f}% of samples  {src}")
