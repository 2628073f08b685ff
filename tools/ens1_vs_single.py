"""Latency of one chain on the ensemble scratch kernel (k_ens_scratch, or the 2-per-SM kernel with
e4 = 0) vs the single-chain scratch kernel, over config 3's hot start (dev helper):
python tools/ens1_vs_single.py [iters]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

I = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200000
A, B, p0, cfg = config(3)
for e4 in (1, 0):
    s = Q.Solver(A, B, p0)
    s.set_option(Q.QAP_OPT_SWITCH_GAP, 0x7FFFFFFF)
    s.set_option(Q.QAP_OPT_ENSEMBLE_SCRATCH4, e4)
    s.delta_init()
    t0, tf = s.schedule_bounds()
    sch = Q.make_schedule(0, t0, tf, cfg["iters"])
    for _ in range(2):
        r = s.ensemble(0, p0[None, :].copy(), I, sch, SA_SEED)
        ms, _ = s.last_kernel_time()
    print(f"1-chain ensemble e4={e4}: {ms:.2f} ms for {I} iterations, accepted {r['stats']['accepted']}")
s = Q.Solver(A, B, p0)
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, cfg["iters"])
for _ in range(2):
    g = s.run(0, I, sch, SA_SEED)
    ms, _ = s.last_kernel_time()
    s.reset(p0)
    s.delta_init()
print(f"single chain: {ms:.2f} ms for {I} iterations, accepted {g['accepted']}")
