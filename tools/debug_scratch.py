"""Dev helper: first divergence of the scratch-phase engine from the oracle (config 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

A, B, p0, cfg = config(1)
sch = O.geometric_schedule_for(A, B, p0, cfg["iters"])
qs = Q.make_schedule(sch.kind, sch.t0, sch.tf, sch.total_iters)
ref = O.Run(A, B, p0)
prev = 0
for I in list(range(128, 193)):
    with Q.Solver(A, B, p0) as s:
        s.delta_init()
        g = s.run(0, I, qs, SA_SEED)
        p, bp, D = s.state()
    r = O.Run(A, B, p0).run(0, I, sch, SA_SEED)
    ok = g["accepted"] == r["accepted"] and g["cost"] == r["cost"]
    print(I, "gpu acc", g["accepted"], "cost", g["cost"], "| oracle acc", r["accepted"], "cost", r["cost"], "OK" if ok else "MISMATCH")
    if not ok:
        break

# state just before the divergence
I0 = I - 1
r = O.Run(A, B, p0)
o = r.run(0, I0, sch, SA_SEED)
print("oracle p at", I0, list(r.p))
with Q.Solver(A, B, p0) as s:
    s.delta_init()
    g = s.run(0, I0, qs, SA_SEED)
    p, bp, D = s.state()
print("gpu    p at", I0, list(p))
o1 = O.Run(A, B, p0); oo = o1.run(0, I, sch, SA_SEED)
print("oracle after", I, "p", list(o1.p), "acc", oo["accepted"])
n = len(p0); M = n * (n - 1) // 2
q = I0 % M
rr = 0
while (rr + 1) * n - (rr + 1) * (rr + 2) // 2 <= q: rr += 1
ss = q - (rr * n - rr * (rr + 1) // 2) + rr + 1
print("iteration", I0, "pair", (rr, ss), "oracle delta", int(r.D[q]))
