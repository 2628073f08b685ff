"""Time one taixxa-shaped instance on a chosen engine option: python tools/run_inst.py n iters
[relabel(0/1)] [cluster(1/8)]; schedule = iters."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, start_perm, taixxa  # noqa: E402

n = int(sys.argv[1])
I = int(float(sys.argv[2]))
rl = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cl = int(sys.argv[4]) if len(sys.argv) > 4 else 8
A, B = taixxa(n, n)
with Q.Solver(A, B, start_perm(n, SA_SEED, 0)) as s:
    s.set_option(Q.QAP_OPT_RELABEL, rl)
    s.set_option(Q.QAP_OPT_RELABEL_CLUSTER, cl)
    s.delta_init()
    t0, tf = s.schedule_bounds()
    g = s.run(0, I, Q.make_schedule(0, t0, tf, I), SA_SEED)
    ms, _ = s.last_kernel_time()
    print(f"n={n} I={I:.0e} engine={s.engine()} relabel={rl} cluster={cl}: {ms:.1f} ms, "
          f"{I/(ms/1e3):.3e} it/s, accepted {g['accepted']}, {ms*1e6/max(1,g['accepted']):.0f} ns/accept")
