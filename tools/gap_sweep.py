"""Config 3 single chain for several scratch -> Δ switch gaps (QAP_OPT_SWITCH_GAP; the trajectory is
the same for every gap): python tools/gap_sweep.py gap ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

A, B, p0, cfg = config(3)
gaps = [int(float(x)) for x in sys.argv[1:]] or [256, 1024, 4096, 16384]
for gap in gaps:
    s = Q.Solver(A, B, p0)
    s.set_option(Q.QAP_OPT_SWITCH_GAP, gap)
    s.delta_init()
    t0, tf = s.schedule_bounds()
    sch = Q.make_schedule(0, t0, tf, cfg["iters"])
    best = None
    for rep in range(3):
        s.reset(p0)
        s.delta_init()
        g = s.run(0, cfg["iters"], sch, SA_SEED)
        ms, _ = s.last_kernel_time()
        best = ms if best is None else min(best, ms)
    print(f"gap {gap}: {best:.1f} ms ({cfg['iters'] / best * 1e3:.3e} it/s), best cost {g['best_cost']}")
