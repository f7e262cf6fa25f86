"""Per-function breakdown (warp samples, instructions) of an ncu report.

usage: python scripts/ncu_funcs.py rep.ncu-rep
"""
import collections, csv, io, re, subprocess, sys


def f(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def byfunc(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    S, I = collections.Counter(), collections.Counter()
    fn, hdr = None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "Kernel Name":
            continue
        if r[0] == "Address":
            hdr = r
            continue
        if hdr is None:
            continue
        d = dict(zip(hdr, r))
        src = d.get("Source", "")
        # function boundaries are not marked on the sass page; use the address order
        S[fn] += f(d.get("Warp Stall Sampling (All Samples)"))
        I[fn] += f(d.get("Instructions Executed"))
    return S, I


if __name__ == "__main__":
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    S, I = collections.Counter(), collections.Counter()
    fn, hdr = None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "Function Name":
            fn = re.sub(r"\(.*", "", r[1]).replace("simba::", "")
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        S[fn] += f(d.get("Warp Stall Sampling (All Samples)"))
        I[fn] += f(d.get("Instructions Executed"))
    ts, ti = sum(S.values()) or 1, sum(I.values()) or 1
    for k, v in S.most_common(30):
        print(f"{100 * v / ts:5.1f}% samples {100 * I[k] / ti:5.1f}% inst  {k}")
