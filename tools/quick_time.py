"""Quick GPU timing of config 3 (single chain) and a reduced ensemble (dev helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config, start_perms  # noqa: E402

A, B, p0, cfg = config(3)
I = cfg["iters"]
s = Q.Solver(A, B, p0)
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, I)
for eng, thr in ((1, 0), (0, 512)):
    s.set_option(Q.QAP_OPT_TENSOR_CORE, eng)
    s.set_option(Q.QAP_OPT_THREADS, thr)
    for frac in (10, 1):
        s.reset(); s.delta_init()
        n = I // frac
        t = time.time()
        g = s.run(0, n, sch, SA_SEED)
        dt = time.time() - t
        ms, _ = s.last_kernel_time()
        print(f"engine={'tmem' if s.uses_tensor_core() else 'smem'} threads={thr} iters={n:.0e} kernel {ms:.1f} ms wall {dt*1e3:.1f} ms "
              f"{n/(ms/1e3):.3e} it/s acc={g['accepted']} best={g['best_cost']}", flush=True)
if "--no-ens" in sys.argv:
    sys.exit(0)
A5, B5, _, c5 = config(5)
for chains, iters in ((1036, 10**6), (8192, 10**6)):
    p0s = start_perms(100, SA_SEED, 0, chains)
    sch5 = Q.make_schedule(0, t0, tf, iters)
    t = time.time()
    r = s.ensemble(0, p0s, iters, sch5, SA_SEED)
    dt = time.time() - t
    ms, _ = s.last_kernel_time()
    print(f"ensemble chains={chains} iters={iters:.0e}: kernel {ms:.1f} ms "
          f"{chains*iters/(ms/1e3):.3e} chain-it/s best={r['best_cost']} acc={r['stats']['accepted']}",
          flush=True)
