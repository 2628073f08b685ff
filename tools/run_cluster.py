"""Run the cluster engine on a tai-shaped instance of size n (dev helper for profiling):
python tools/run_cluster.py n iters"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, start_perm, taixxa  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
iters = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**6
A, B = taixxa(n, 4000 + n)
p0 = start_perm(n, 13, 0)
s = Q.Solver(A, B, p0)
assert s.engine() == Q.QAP_ENGINE_CLUSTER
s.delta_init()
t0, tf = s.schedule_bounds()
g = s.run(0, iters, Q.make_schedule(0, t0, tf, iters), SA_SEED)
ms, _ = s.last_kernel_time()
print(f"cluster engine n={n} iters={iters:.0e}: {ms:.1f} ms, {iters / ms * 1e3:.3e} it/s, accepted {g['accepted']}, "
      f"{ms * 1e6 / max(1, g['accepted']):.0f} ns/accept")
