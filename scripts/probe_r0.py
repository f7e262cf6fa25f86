"""C5 sweep time per size for explicit r0[:block_threads] values (diagnostics).
usage: probe_r0.py 6 7:512 ...  [--sizes 11,12,13]"""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from probe import run, unsat  # noqa: E402

sizes = [12, 13]
args = sys.argv[1:]
if "--sizes" in args:
    i = args.index("--sizes")
    sizes = [int(x) for x in args[i + 1].split(",")]
    args = args[:i] + args[i + 2:]
spec4 = unsat(4, 32, 10, 31337)
for a in args:
    r0, _, bt = a.partition(":")
    kw = {"r0": int(r0)}
    if bt:
        kw["block_threads"] = int(bt)
    run(f"C5 {a}", spec4, sizes, **kw)
