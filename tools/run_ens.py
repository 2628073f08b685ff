"""Run part of BASELINE config 5 (ensemble) for profiling: python tools/run_ens.py chains iters [group] [gap] [e4]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config, start_perms  # noqa: E402

C = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1024
I = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**5
grp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
gap = int(float(sys.argv[4])) if len(sys.argv) > 4 else 0
e4 = int(sys.argv[5]) if len(sys.argv) > 5 else 1
A, B, p0, cfg = config(5)
s = Q.Solver(A, B, p0)
if grp:
    s.set_option(Q.QAP_OPT_ENSEMBLE_GROUP, grp)
s.set_option(Q.QAP_OPT_SWITCH_GAP, gap)
s.set_option(Q.QAP_OPT_ENSEMBLE_SCRATCH4, e4)
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, cfg["iters"])
p0s = start_perms(cfg["n"], SA_SEED, 0, C)
res = s.ensemble(0, p0s, I, sch, SA_SEED)
ms, _ = s.last_kernel_time()
print(f"ensemble C={C} I={I:.0e} group={grp or 'default'} gap={gap} e4={e4}: {ms:.1f} ms, {C*I/(ms/1e3):.3e} chain-it/s")
