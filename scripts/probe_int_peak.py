"""The integer roofline probes (simba_int32_pipe_peak, modes 0 = LOP3 only,
1 = LOP3 + IMAD): ops/s on this GPU; run under ncu to read the pipe
utilisation (profiles/r02_ncu_int_peak.txt)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_08243_b200 import _native as N  # noqa: E402

for mode, name in ((0, "ALU (LOP3)"), (1, "ALU+FMA (LOP3+IMAD)")):
    ops, ms = C.c_double(), C.c_double()
    N.check_rc(N.lib.simba_int32_pipe_peak(0, 8192, mode, C.byref(ops), C.byref(ms)))
    print(f"{name}: {ops.value / 1e12:.2f} T int-ops/s ({ms.value:.2f} ms)", flush=True)
