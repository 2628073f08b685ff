"""Dev helper: phase timers (libqapsa_timers.so) on the pure accept path (A = 0, every iteration
accepts)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["QAPSA_LIB"] = os.path.join(ROOT, "paper_1208_2675_b200", "libqapsa_timers.so")
import numpy as np  # noqa: E402

from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import start_perm, taixxa  # noqa: E402

n, I = 100, 100000
_, B = taixxa(n, 7)
A = np.zeros((n, n), np.int32)
s = Q.Solver(A, B, start_perm(n, 1, 0))
s.delta_init()
L = Q.lib()
buf = (C.c_ulonglong * 128)()
L.qapsa_debug_phase_cycles(buf)
g = s.run(0, I, Q.make_schedule(0, 10.0, 1.0, I), 1)
ms, _ = s.last_kernel_time()
L.qapsa_debug_phase_cycles(buf)
na = max(1, buf[127])
print(f"{ms*1e-3*1.965e9/na:.0f} clk per accept ({na} accepts)")
names = ["window (top->decision)", "", "stage barrier", "epilogue math", "mbar_d", "barrier 2", "RMW done",
         "stage loads", "operands stored", "touching reads", "ballot (from top)", "wait::st+fence"]
for w in range(8):
    b = buf[16 * w: 16 * w + 12]
    print(f"warp {w}: " + ", ".join(f"{nm} {b[i]/na:.0f}" for i, nm in enumerate(names) if nm and b[i]))
