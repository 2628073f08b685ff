"""Profiling driver: one config-3 qap_sa_run over iterations [0, ITERS) (default 1e7,
the high-acceptance first decile), preceded by reset + delta_init.  Used under
ncu; prints the kernel time when run plain."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

iters = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**7
k0 = int(float(sys.argv[2])) if len(sys.argv) > 2 else 0
A, B, p0, cfg = config(3)
s = Q.Solver(A, B, p0)
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, cfg["iters"])
g = s.run(k0, iters, sch, SA_SEED)
ms, _ = s.last_kernel_time()
print(f"iters [{k0},{k0+iters}) kernel {ms:.2f} ms accepted {g['accepted']} "
      f"-> {ms*1e6/max(1,g['accepted']):.0f} ns/accept, {iters/(ms/1e3):.3e} it/s")
