"""Fig. 1/2-shaped sweep (§5): for a BASELINE instance, run the chain
with an I-iteration schedule for several I and record the device time, the acceptance rate
P = accepted / I and the best cost -- the quantities the paper plots against I.  The paper's
absolute values are unrecoverable (other hardware, QAPLIB data not present); this reproduces
the shape on the synthetic instances.  Usage: python tools/fig_grid.py [cfg] [Imax] > out.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 3
imax = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**8
A, B, p0, cfg = config(cfgi)
rows = []
I = 10**4
while I <= imax:
    with Q.Solver(A, B, p0) as s:
        s.delta_init()
        t0, tf = s.schedule_bounds()
        g = s.run(0, I, Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, I), SA_SEED)
        ms, _ = s.last_kernel_time()
        rows.append({"I": I, "device_ms": ms, "it_per_s": I / (ms / 1e3), "P": g["accepted"] / I,
                     "best_cost": g["best_cost"], "final_cost": g["cost"], "engine": s.engine()})
    print(json.dumps(rows[-1]), file=sys.stderr)
    I *= 10
print(json.dumps({"config": cfgi, "instance": cfg["name"], "seed": SA_SEED, "rows": rows}))
