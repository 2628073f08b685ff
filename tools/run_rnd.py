"""Config 3 with random proposals (R22) on the tensor-memory and shared-memory engines (dev
helper): python tools/run_rnd.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

I = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**7
A, B, p0, cfg = config(3)
for tc in (2, 0):
    s = Q.Solver(A, B, p0)
    s.set_option(Q.QAP_OPT_PROPOSAL, 1)
    s.set_option(Q.QAP_OPT_TENSOR_CORE, tc)
    s.delta_init()
    t0, tf = s.schedule_bounds()
    g = s.run(0, I, Q.make_schedule(0, t0, tf, I), SA_SEED)
    ms, _ = s.last_kernel_time()
    print(f"random proposals, config 3, I={I:.0e}, engine {s.engine()}: {ms:.1f} ms, {I / ms * 1e3:.3e} it/s, "
          f"accepted {g['accepted']}, best {g['best_cost']}")
