"""Run a BASELINE config (single chain) for `iters` iterations from k0 (dev helper):
python tools/run_cfg.py cfg iters [k0] [tmem|smem]; prints time, accepts and ns/accept."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

cfgi = int(sys.argv[1])
iters = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**6
k0 = int(float(sys.argv[3])) if len(sys.argv) > 3 else 0
eng = sys.argv[4] if len(sys.argv) > 4 else "tmem"
A, B, p0, cfg = config(cfgi)
s = Q.Solver(A, B, p0)
s.set_option(Q.QAP_OPT_TENSOR_CORE, 1 if eng == "tmem" else 0)
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, cfg["iters"])
pos = 0
while pos < k0:                     # advance to k0 in chunks (same trajectory as one call)
    step = min(k0 - pos, 10**8)
    s.run(pos, step, sch, SA_SEED)
    pos += step
g = s.run(k0, iters, sch, SA_SEED)
ms, _ = s.last_kernel_time()
print(f"cfg{cfgi} {eng} tc={s.uses_tensor_core()} k0={k0:.0e} iters={iters:.0e}: {ms:.1f} ms, "
      f"{iters / ms * 1e3:.3e} it/s, accepted {g['accepted']}, "
      f"{ms*1e6/max(1, g['accepted']):.0f} ns/accept, cost {g['cost']}")
