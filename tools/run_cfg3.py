"""Run config 3 (single chain) for `iters` iterations from k0 on the chosen engine (dev helper
for profiling): python tools/run_cfg3.py iters [k0] [tmem|smem]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

iters = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**6
k0 = int(float(sys.argv[2])) if len(sys.argv) > 2 else 0
eng = sys.argv[3] if len(sys.argv) > 3 else "tmem"
A, B, p0, cfg = config(3)
s = Q.Solver(A, B, p0)
s.set_option(Q.QAP_OPT_TENSOR_CORE, 1 if eng == "tmem" else 0)
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, cfg["iters"])
if k0:
    s.run(0, k0, sch, SA_SEED)
g = s.run(k0, iters, sch, SA_SEED)
ms, _ = s.last_kernel_time()
print(f"{eng} k0={k0:.0e} iters={iters:.0e}: {ms:.1f} ms, accepted {g['accepted']}, "
      f"{ms*1e6/max(1, g['accepted']):.0f} ns/accept")
