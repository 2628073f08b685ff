#!/usr/bin/env python
"""Writes the oracle goldens of the long BASELINE configurations (calls only oracle/ and the
seeded input generators of qap_inputs/; nothing here comes from the CUDA path).

  python tests/golden/make_goldens.py config4 [--threads 1]   # ~25-30 min on one core
  python tests/golden/make_goldens.py config5 [--threads T]   # ~4 core-hours, thread-pooled

config4_full.json  BASELINE config 4 (N=256 grey density, 1 chain, 1e9 iterations), oracle SCRATCH
                   mode (the same trajectory as DELTA, pinned by the EQ1 == SCRATCH == DELTA tests),
                   state after every 1e8 iterations: p, best_p, C, best, accepted, near ties (k,
                   decision), digest (R18).
config5_chains.npz BASELINE config 5 (8192 independent N=100 chains x 1e7 iterations, chain-keyed
                   Fisher-Yates start permutations R14b), per chain: cost, best_cost, accepted,
                   near_ties, digest, iterations, and each chain's near-tie log (k, decision).
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from qap_inputs import CONFIGS, SA_SEED, config  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CHUNK = 10**8


def config4(args):
    A, B, p0, cfg = config(4)
    I = cfg["iters"]
    sch = O.geometric_schedule_for(A, B, p0, I)
    run = O.Run(A, B, p0, mode=O.MODE_SCRATCH)
    rec = {"config": 4, "instance": cfg["name"], "n": cfg["n"], "iters": I, "seed": SA_SEED,
           "schedule": {"kind": sch.kind, "t0": sch.t0, "tf": sch.tf, "total_iters": I},
           "oracle_mode": "SCRATCH", "chunk": CHUNK, "checkpoints": []}
    k = 0
    t_all = time.time()
    while k < I:
        step = min(CHUNK, I - k)
        t = time.time()
        st = run.run(k, step, sch, SA_SEED)
        k += step
        cp = {"k": k, "cost": int(st["cost"]), "best_cost": int(st["best_cost"]),
              "accepted": int(st["accepted"]), "near_ties": int(st["near_ties"]),
              "near_log": [list(x) for x in run.near_log],
              "digest": str(int(st["digest"])), "p": run.p.tolist(), "best_p": run.best_p.tolist(),
              "oracle_s": round(time.time() - t, 1)}
        rec["checkpoints"].append(cp)
        print(json.dumps({kk: v for kk, v in cp.items() if kk not in ("p", "best_p")}), flush=True)
    rec["oracle_total_s"] = round(time.time() - t_all, 1)
    with open(os.path.join(HERE, "config4_full.json"), "w") as f:
        json.dump(rec, f, indent=0)


def config5(args):
    cfg = CONFIGS[5]
    A, B, _, _ = config(5)
    n, C, I = cfg["n"], cfg["chains"], cfg["iters"]
    p00 = O.start_perm(n, SA_SEED, 0)
    sch = O.geometric_schedule_for(A, B, p00, I)
    cap = 8
    t = time.time()
    out, logs = O.ensemble_run(A, B, None, 0, I, sch, SA_SEED, threads=args.threads,
                               mode=O.MODE_SCRATCH, count=C, near_cap=cap)
    dt = time.time() - t
    nk = np.zeros((C, cap), np.uint64)
    nd = np.zeros((C, cap), np.uint8)
    for c, lg in enumerate(logs):
        for i, (kk, d) in enumerate(lg):
            nk[c, i], nd[c, i] = kk, d
    np.savez_compressed(os.path.join(HERE, "config5_chains.npz"), out=out, near_k=nk, near_d=nd,
                        schedule=np.array([sch.kind, sch.t0, sch.tf, I], np.float64),
                        meta=np.array(json.dumps({
                            "config": 5, "chains": C, "iters": I, "n": n, "seed": SA_SEED,
                            "start_perm": "oracle.start_perm (R14b)", "oracle_mode": "SCRATCH",
                            "threads": args.threads, "oracle_s": round(dt, 1),
                            "p0_chain0_sha": hashlib.sha256(p00.tobytes()).hexdigest()[:16]})))
    print(json.dumps({"chains": C, "oracle_s": dt, "near_ties": int(out[:, 3].sum()),
                      "best": int(out[:, 1].min())}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["config4", "config5"])
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    {"config4": config4, "config5": config5}[a.which](a)
