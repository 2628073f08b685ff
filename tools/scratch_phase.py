"""Dev helper: phase timers of the scratch-phase kernel on the pure accept path (A = 0)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["QAPSA_LIB"] = os.path.join(ROOT, "paper_1208_2675_b200", "libqapsa_timers.so")
import numpy as np  # noqa: E402

from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config, start_perm, taixxa  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "zero"
if mode == "zero":
    n, I = 100, 100000
    _, B = taixxa(n, 7)
    A = np.zeros((n, n), np.int32)
    p0 = start_perm(n, 1, 0)
    sch = Q.make_schedule(0, 10.0, 1.0, I)
else:
    A, B, p0, cfg = config(3)
    I = int(float(mode))
s = Q.Solver(A, B, p0)
s.delta_init()
if mode != "zero":
    t0, tf = s.schedule_bounds()
    sch = Q.make_schedule(0, t0, tf, 10**8)
L = Q.lib()
buf = (C.c_ulonglong * 128)()
L.qapsa_debug_phase_cycles(buf)
g = s.run(0, I, sch, 1 if mode == "zero" else SA_SEED)
ms, _ = s.last_kernel_time()
L.qapsa_debug_phase_cycles(buf)
na = max(1, buf[127])
print(f"{ms*1e-3*1.965e9/na:.0f} clk per accept ({na} accepts in the first kernel)")
names = ["window values ready", "tests done (from loop top)", "stage done (from decision)",
         "staging barrier passed (from decision)", "non-accepting windows (total)", "accept read (from decision)",
         "next rows' p (from decision)", "previous MMA waited (from decision)", "tensor loads done (from decision)",
         "shared loads done (from decision)", "decision (from loop top)"]
for w in (0,):
    b = buf[16 * w: 16 * w + 12]
    print(f"warp {w}:\n  " + "\n  ".join(f"{nm} {b[i]/na:.0f}" for i, nm in enumerate(names) if b[i]))
