"""Small runs of every engine for compute-sanitizer (racecheck / synccheck / memcheck), S:279:
python tools/sanitize_run.py [case ...]; cases: tmem tmem_delta smem relabel relabel_1sm ens_tmem ens_smem."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config, start_perms  # noqa: E402

CASES = ["tmem", "tmem_delta", "smem", "relabel", "relabel_1sm", "ens_tmem", "ens_smem"]
todo = sys.argv[1:] or CASES


def single(cfgi, iters, opts):
    A, B, p0, cfg = config(cfgi)
    with Q.Solver(A, B, p0) as s:
        for k, v in opts:
            s.set_option(k, v)
        s.delta_init()
        t0, tf = s.schedule_bounds()
        g = s.run(0, iters, Q.make_schedule(0, t0, tf, cfg["iters"]), SA_SEED)
        return s.engine(), g["accepted"], g["best_cost"]


def ens(chains, iters, opts):
    A, B, p0, cfg = config(5)
    with Q.Solver(A, B, p0) as s:
        for k, v in opts:
            s.set_option(k, v)
        s.delta_init()
        t0, tf = s.schedule_bounds()
        r = s.ensemble(0, None, iters, Q.make_schedule(0, t0, tf, cfg["iters"]), SA_SEED, count=chains)
        return r["best_cost"], r["best_chain"]


for c in todo:
    for cfgi, iters in ((1, 20000), (2, 20000)):
        if c == "tmem":
            print(c, cfgi, single(cfgi, iters, []), flush=True)
        elif c == "tmem_delta":
            print(c, cfgi, single(cfgi, iters, [(Q.QAP_OPT_SCRATCH_PHASE, 0)]), flush=True)
        elif c == "smem":
            print(c, cfgi, single(cfgi, iters, [(Q.QAP_OPT_TENSOR_CORE, 0)]), flush=True)
    if c in ("relabel", "relabel_1sm"):
        opts = [] if c == "relabel" else [(Q.QAP_OPT_RELABEL_CLUSTER, 1)]
        print(c, 4, single(4, 5000, opts), flush=True)
    elif c == "ens_tmem":
        print(c, ens(16, 20000, []), flush=True)
    elif c == "ens_smem":
        print(c, ens(16, 20000, [(Q.QAP_OPT_TENSOR_CORE, 0)]), flush=True)
