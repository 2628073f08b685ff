"""Host-clock breakdown of one end-to-end config-3 call (create, delta_init, run, state, destroy)
(dev helper): python tools/e2e_breakdown.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
A, B, p0, cfg = config(3)
stream = torch.cuda.Stream()
mode = sys.argv[2] if len(sys.argv) > 2 else "bench"
kw = dict(stream=stream.cuda_stream) if mode == "bench" else {}
s0 = Q.Solver(A, B, p0, **kw)
s0.delta_init()
t0, tf = s0.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, cfg["iters"])
s0.run(0, cfg["iters"] if mode == "bench" else 10**6, sch, SA_SEED)
flush = torch.empty(64 << 20, device="cuda") if mode == "bench" else None
if mode != "bench":
    s0.close()
for _ in range(reps):
    torch.cuda.synchronize()
    ts = [time.perf_counter()]
    s = Q.Solver(A, B, p0, **kw)
    ts.append(time.perf_counter())
    s.delta_init()
    ts.append(time.perf_counter())
    g = s.run(0, cfg["iters"], sch, SA_SEED)
    ts.append(time.perf_counter())
    s.state(want_delta=False)
    ts.append(time.perf_counter())
    dev_ms, _ = s.last_kernel_time()
    s.close()
    ts.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(ts, ts[1:])]
    print(f"create {d[0]:.1f} ms, delta_init {d[1]:.1f}, run {d[2]:.1f} (device {dev_ms:.1f}), state {d[3]:.1f}, "
          f"destroy {d[4]:.1f}; total {sum(d):.1f} ms")
