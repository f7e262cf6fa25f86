"""CTA start/end spread of one fused-sweep shard launch (libsimba built with
-DSIMBA_CTA_TIMES prints one line per CTA).  usage: probe_cta_times.py N shard"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2605_08243_b200 as S
from paper_2605_08243_b200.engine import DeviceContext

N, i = int(sys.argv[1]), int(sys.argv[2])
spec = S.Specification(k=4, w=32, pairs=bench.unsat_pairs())
with DeviceContext(spec, 13) as ctx:
    r = ctx.run_levels(1, 13, shard=i, nshards=N)[0]
    print("KERNEL_MS", r.kernel_ms, flush=True)
