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
    t0 = time.perf_counter()
    with DeviceContext(spec, max(sizes), **kw) as ctx:
        info = ctx.info()
        tc = time.perf_counter() - t0
        for s in sizes:
            r = ctx.count(s)  # warm
            r = ctx.count(s)
            st = ctx.path_stats()
            if st:
                cyc = {k: v for k, v in st.items() if k.startswith(("cyc", "w_"))}
                ph = {k: v for k, v in st.items() if k.startswith("ph_")}
                paths = {k: v for k, v in st.items() if not k.startswith(("cyc", "w_", "ph_"))}
                ctas = info["grid_blocks"]
                print("   phases per CTA:", {k: (round(v[0] / ctas, 1), round(v[1] / ctas / 1e6, 2)) for k, v in ph.items()},
                      "Mcyc (ph_verify count = descriptors)")
                tot = sum(v[1] for v in paths.values()) or 1
                print("   paths:", {k: (v[0], round(100 * v[1] / tot, 2)) for k, v in paths.items() if v[0]})
                warps = info["grid_blocks"] * info["block_threads"] // 32
                print("   cycles per warp:", {k: (v[0], round(v[1] / warps / 1e6, 2)) for k, v in cyc.items()},
                      "Mcyc; kernel", round(r.kernel_ms * 1.965e3 / 1e3, 2), "Mcyc at 1965 MHz")
            print(f"{label:22s} s={s:2d} T={r.visited:.3e} {r.kernel_ms:9.3f} ms "
                  f"{r.visited / (r.kernel_ms * 1e-3):.3e} cand/s cnt={r.count} units={r.units} "
                  f"rank_units={r.rank_units} ctx={tc*1e3:.0f}ms {info}", flush=True)

if __name__ == "__main__":
    spec4 = unsat(4, 32, 10, 31337)
    if len(sys.argv) > 1 and sys.argv[1] == "r0":
        run("C5 r0=5 256x2", spec4, [11, 12, 13])
        run("C5 r0=5 512x1", spec4, [11, 12, 13], block_threads=512)
        run("C5 r0=6 512x1", spec4, [11, 12, 13], r0=6, block_threads=512)
        run("C3 r0=6 256x2", unsat(3, 32, 10, 777), [11, 12])
        run("C3 r0=7 512x1", unsat(3, 32, 10, 777), [11, 12], r0=7, block_threads=512)
        sys.exit()
    if len(sys.argv) > 1:
        run("C5 unit", spec4, [int(a) for a in sys.argv[1:]]); sys.exit()
    run("C5 unit", spec4, [9, 10, 11, 12, 13])
    run("C5 unit rg=8", spec4, [12, 13], rg=8)
    run("C5 direct", spec4, [9, 10], kernel="direct")
    run("C5 unit r0=4", spec4, [11], r0=4)
    spec3 = unsat(3, 32, 10, 777)
    run("C3 unit", spec3, [9, 10, 11, 12])
    spec4w = unsat(3, 64, 100, 4242)
    run("C4 unit", spec4w, [9, 10, 11])
    spec2 = unsat(2, 32, 10, 99)
    run("C2 unit", spec2, [7, 10, 13])
