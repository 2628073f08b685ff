"""Per-phase cycle breakdown of the tensor-memory single-chain kernel (debug build
libqapsa_timers.so, -DQAPSA_PHASE_TIMERS; register-accumulated timers of thread 0 (lane warp 0)
and thread 128 (helper warp 4))."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["QAPSA_LIB"] = os.path.join(ROOT, "paper_1208_2675_b200", "libqapsa_timers.so")
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

iters = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**6
k0 = int(float(sys.argv[2])) if len(sys.argv) > 2 else 0
A, B, p0, cfg = config(3)
s = Q.Solver(A, B, p0)
assert s.uses_tensor_core()
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, cfg["iters"])
L = Q.lib()
buf = (C.c_ulonglong * 128)()
if k0:
    s.run(0, k0, sch, SA_SEED)
L.qapsa_debug_phase_cycles(buf)
g = s.run(k0, iters, sch, SA_SEED)
ms, _ = s.last_kernel_time()
L.qapsa_debug_phase_cycles(buf)
na = max(1, buf[127])
clk = ms * 1e-3 * 1.965e9
print(f"k0 {k0:.0e} iters {iters:.0e}: {ms:.1f} ms (~{clk:.3e} clk), accepts {g['accepted']}, "
      f"{clk/max(1,g['accepted']):.0f} clk/accept")
print(f"  windows: accepting {buf[0]/na:.0f} clk/accept; non-accepting total {buf[1]/1e6:.2f} Mclk "
      f"({buf[1]/max(1,clk)*100:.1f}% of the kernel)")
print(f"  lane t0 after decision: stage barrier {buf[2]/na:.0f}, Z done {buf[3]/na:.0f}, MMA done {buf[4]/na:.0f}, "
      f"epilogue barrier {buf[5]/na:.0f}, RMW done {buf[6]/na:.0f}")
print(f"  lane t0 stage: loads {buf[7]/na:.0f}, operands stored {buf[8]/na:.0f}, touching reads {buf[9]/na:.0f}, "
      f"proxy fence {buf[10]/na:.0f}, wait::st+fence {buf[11]/na:.0f}")
print(f"  helper t128 after decision: thresholds {buf[18]/na:.0f}")
for w in range(8):
    b = buf[16 * w: 16 * w + 12]
    print(f"  warp {w}: loop top -> ballot {b[10]/max(1, na):.0f} (per accept, incl. non-accepting windows), "
          f"barrier2 at {b[5]/na:.0f}, RMW done {b[6]/na:.0f}")
