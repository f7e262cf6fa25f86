"""Quick throughput probe of the device kernels (diagnostics, not the bench)."""
import random, sys, time
sys.path.insert(0, ".")
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

def unsat(k, w, n, seed):
    rng = random.Random(seed); pairs = []; seen = set()
    while len(pairs) < n:
        x = tuple(rng.getrandbits(w) for _ in range(k))
        if x in seen: continue
        seen.add(x); pairs.append((x, rng.getrandbits(w)))
    return S.Specification(k=k, w=w, pairs=tuple(pairs))

def run(label, spec, sizes, **kw):
    with DeviceContext(spec, max(sizes), **kw) as ctx:
        info = ctx.info()
        for s in sizes:
            r = ctx.count(s)  # warm
            r = ctx.count(s)
            print(f"{label:28s} s={s:2d} T={r.visited:.3e} kernel={r.kernel_ms:9.3f} ms  "
                  f"{r.visited / (r.kernel_ms * 1e-3):.3e} cand/s  count={r.count} units={r.units} rank_units={r.rank_units} {info}", flush=True)

spec4 = unsat(4, 32, 10, 31337)
if len(sys.argv) > 1:
    run("C5 unit", spec4, [int(sys.argv[1])]); sys.exit()
run("C5 unit", spec4, [9, 10, 11, 12])
run("C5 direct", spec4, [9, 10], kernel="direct")
run("C5 unit r0=4", spec4, [11], r0=4)
run("C5 unit r0=3", spec4, [11], r0=3)
spec3 = unsat(3, 32, 10, 777)
run("C3 unit", spec3, [9, 10, 11])
spec4w = unsat(3, 64, 100, 4242)
run("C4 unit", spec4w, [9, 10])
