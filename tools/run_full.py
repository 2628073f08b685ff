"""A whole BASELINE single-chain run in chunks of 1e8 iterations (same trajectory as one call):
python tools/run_full.py cfg; prints the device time per chunk and in total."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 4
A, B, p0, cfg = config(cfgi)
I = cfg["iters"]
s = Q.Solver(A, B, p0)
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(Q.QAP_COOL_GEOMETRIC, t0, tf, I)
tot_ms, acc, k, chunks = 0.0, 0, 0, []
while k < I:
    step = min(10**8, I - k)
    g = s.run(k, step, sch, SA_SEED)
    ms, _ = s.last_kernel_time()
    tot_ms += ms
    acc += g["accepted"]
    chunks.append({"k0": k, "iters": step, "ms": ms, "accepted": g["accepted"]})
    print(json.dumps(chunks[-1]), file=sys.stderr, flush=True)
    k += step
print(json.dumps({"config": cfgi, "instance": cfg["name"], "iters": I, "engine": s.engine(),
                  "device_ms": tot_ms, "it_per_s": I / (tot_ms / 1e3), "accepted": acc,
                  "cost": g["cost"], "best_cost": g["best_cost"], "near_ties": g["near_ties"],
                  "chunks": chunks}))
