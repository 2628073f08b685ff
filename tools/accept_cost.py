"""Dev helper: pure accept-path cost.  A = 0 makes every δ = 0, so every iteration is an accepted
swap (window of one candidate); prints ns and cycles per accept for each engine."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import start_perm, taixxa  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
I = 200000
_, B = taixxa(n, 7)
A = np.zeros((n, n), np.int32)
for eng in (1, 0):
    s = Q.Solver(A, B, start_perm(n, 1, 0))
    s.set_option(Q.QAP_OPT_TENSOR_CORE, eng)
    s.delta_init()
    sch = Q.make_schedule(0, 10.0, 1.0, I)
    g = s.run(0, I, sch, 1)
    ms, _ = s.last_kernel_time()
    print(f"{'tmem' if s.uses_tensor_core() else 'smem'} n={n}: {g['accepted']} accepts, "
          f"{ms*1e6/g['accepted']:.0f} ns = {ms*1e-3*1.965e9/g['accepted']:.0f} clk per accept")
