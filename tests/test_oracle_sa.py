"""Whole-trajectory pins of the oracle's sequential SA, no GPU.

Pins: EQ1 (δ from Eq.(1) by definition) == SCRATCH == DELTA trajectories
(AC4); invariants after every accept (AC1/AC2); brute-force optimum hit
rate (AC5); acceptance-rate trend (AC6); determinism and resume.
"""
import numpy as np
import pytest

import oracle as O
from qap_inputs import taixxa, start_perm


def _sched(A, B, p0, I):
    return O.geometric_schedule_for(A, B, p0, I)


@pytest.mark.parametrize("n,I,seed", [(6, 3000, 1), (10, 20000, 2), (15, 20000, 3),
                                      (20, 30000, 4), (13, 50000, 5)])
def test_mode_equivalence_eq1_scratch_delta(n, I, seed):
    A, B = taixxa(n, 300 + seed)
    p0 = start_perm(n, seed, 0)
    sch = _sched(A, B, p0, I)
    res = {}
    for mode in (O.MODE_EQ1, O.MODE_SCRATCH, O.MODE_DELTA):
        if mode == O.MODE_EQ1 and n > 15:
            continue
        run = O.Run(A, B, p0, mode=mode)
        st = run.run(0, I, sch, seed=seed)
        res[mode] = (st, run.p.copy(), run.best_p.copy())
    ref = res[O.MODE_DELTA]
    assert ref[0]["accepted"] > 0
    for mode, (st, p, bp) in res.items():
        assert st == ref[0], mode
        np.testing.assert_array_equal(p, ref[1])
        np.testing.assert_array_equal(bp, ref[2])


def test_invariants_after_every_accept():
    for n, seed in [(7, 1), (16, 2), (30, 3)]:
        A, B = taixxa(n, seed)
        p0 = start_perm(n, seed, 0)
        sch = _sched(A, B, p0, 20000)
        run = O.Run(A, B, p0, mode=O.MODE_DELTA)
        st = run.run(0, 20000, sch, seed=seed, check_every=1)   # raises on mismatch
        assert st["accepted"] > 100
        assert st["best_cost"] <= st["cost"]
        assert O.cost(A, B, run.best_p) == st["best_cost"]


def test_bruteforce_optimum_hit_rate():
    """AC5: 5 instances N=8, 20 runs each at I=1e5: optimum found in >= 90%."""
    hits = total = 0
    for inst in range(5):
        A, B = taixxa(8, 800 + inst)
        opt, _ = O.bruteforce(A, B)
        for run_id in range(20):
            p0 = start_perm(8, 1000 + run_id, inst)
            sch = _sched(A, B, p0, 10**5)
            run = O.Run(A, B, p0)
            st = run.run(0, 10**5, sch, seed=run_id)
            assert st["best_cost"] >= opt
            hits += st["best_cost"] == opt
            total += 1
    assert hits / total >= 0.9, (hits, total)


def test_acceptance_rate_non_increasing_in_I():
    """AC6: a(I) non-increasing over I in {1e3,1e4,1e5,1e6} (mean over seeds, N=50)."""
    A, B = taixxa(50, 5050)
    rates = []
    for I in (10**3, 10**4, 10**5, 10**6):
        acc = []
        for seed in range(4 if I < 10**6 else 2):
            p0 = start_perm(50, seed, 0)
            sch = _sched(A, B, p0, I)
            st = O.Run(A, B, p0).run(0, I, sch, seed=seed)
            acc.append(st["accepted"] / I)
        rates.append(np.mean(acc))
    for a, b in zip(rates, rates[1:]):
        assert b <= a + 0.02, rates


def test_determinism_and_resume():
    """S:207 determinism; resume: [0,I) in one call == split at arbitrary k."""
    A, B = taixxa(25, 77)
    p0 = start_perm(25, 9, 0)
    I = 60000
    sch = _sched(A, B, p0, I)
    one = O.Run(A, B, p0)
    s1 = one.run(0, I, sch, seed=5)
    two = O.Run(A, B, p0)
    for k0, k1 in [(0, 1), (1, 777), (777, 30001), (30001, I)]:
        s2 = two.run(k0, k1 - k0, sch, seed=5)
    assert s1 == s2
    np.testing.assert_array_equal(one.p, two.p)
    np.testing.assert_array_equal(one.D, two.D)
    again = O.Run(A, B, p0).run(0, I, sch, seed=5)
    assert again == s1


def test_seed_and_chain_change_trajectory():
    A, B = taixxa(20, 1)
    p0 = start_perm(20, 1, 0)
    sch = _sched(A, B, p0, 20000)
    a = O.Run(A, B, p0).run(0, 20000, sch, seed=1)
    b = O.Run(A, B, p0).run(0, 20000, sch, seed=2)
    c = O.Run(A, B, p0, chain=7).run(0, 20000, sch, seed=1)
    assert a["digest"] != b["digest"] and a["digest"] != c["digest"]


def near_tie_schedule(A, B, p0, seed, chain=0, I=5000):
    """A constant schedule (t0 = tf = T) that makes iteration 0 a near tie (R16): iteration 0
    proposes pair (0, 1) (R4) with δ = Δ_01 at p0 > 0, and T = δ / (-ln r_0) puts
    δ + T ln r_0 within rounding of 0."""
    import math
    d = int(O.delta_init(A, O.bprime(B, p0))[0])
    assert d > 0
    T = d / -math.log(O.uniform(seed, 0, chain, 0))
    return O.Schedule(O.COOL_GEOMETRIC, T, T, I)


def test_constructed_near_tie_is_flagged_and_followed():
    """R16 on a constructed near tie: the oracle flags iteration 0 (and only it, at the start),
    logs its own decision, adopts a listed decision at a flagged k in either direction, and
    ignores listed decisions at k that are not near ties."""
    A, B = taixxa(12, 3)
    for c in range(40):
        p0 = start_perm(12, 3, c)
        if O.delta_init(A, O.bprime(B, p0))[0] > 0:
            break
    sch = near_tie_schedule(A, B, p0, seed=3)
    one = O.Run(A, B, p0)
    st = one.run(0, 1, sch, seed=3)
    assert st["near_ties"] == 1 and one.near_log == [(0, st["accepted"])]
    for d in (0, 1):                              # the follow entry decides iteration 0
        r = O.Run(A, B, p0)
        assert r.run(0, 1, sch, seed=3, follow=[(0, d)])["accepted"] == d
        assert r.near_log == [(0, d)]
    base = O.Run(A, B, p0)
    b = base.run(0, 5000, sch, seed=3)
    bogus = [(k, 1 - (k % 2)) for k in range(1, 5000, 7) if k not in [x for x, _ in base.near_log]]
    other = O.Run(A, B, p0).run(0, 5000, sch, seed=3, follow=bogus)
    assert other == b


def test_all_zero_flow_accepts_everything():
    """all-zero A -> δ = 0 always -> every proposal accepted (Eq.(2), R5)."""
    n = 9
    _, B = taixxa(n, 2)
    A = np.zeros((n, n), np.int32)
    p0 = start_perm(n, 1, 0)
    st = O.Run(A, B, p0).run(0, 1000, O.Schedule(O.COOL_GEOMETRIC, 1.0, 0.1, 1000), seed=1)
    assert st["accepted"] == 1000 and st["cost"] == 0 and st["best_cost"] == 0


def test_ensemble_matches_single_chains():
    A, B = taixxa(14, 4)
    p0s = np.stack([start_perm(14, 42, c) for c in range(6)])
    sch = _sched(A, B, p0s[0], 3000)
    out = O.ensemble_run(A, B, p0s, 10, 3000, sch, seed=42, threads=3)
    for i in range(6):
        st = O.Run(A, B, p0s[i], chain=10 + i).run(0, 3000, sch, seed=42)
        assert tuple(out[i]) == (st["cost"], st["best_cost"], st["accepted"], st["near_ties"],
                                 np.int64(np.uint64(st["digest"]).view(np.int64)),
                                 st["iterations"])


def test_random_proposals_r22():
    """R22 (random proposals): the pair of iteration k is drawn by Philox tag 3.  Pins:
    the three δ evaluations (Eq.(1) difference, scratch formula, maintained Δ with full
    recomputation checks) give the same trajectory; over many iterations every pair is proposed
    with frequency close to 1/M (within 5 sigma); a brute-force optimum is reached on a tiny
    instance; and the sequence differs from the sequential enumeration."""
    import itertools
    A, B = taixxa(7, 71)
    p0 = start_perm(7, 3, 0)
    I = 20000
    sch = O.geometric_schedule_for(A, B, p0, I)
    outs = []
    for mode in (O.MODE_EQ1, O.MODE_SCRATCH, O.MODE_DELTA):
        r = O.Run(A, B, p0, mode=mode, proposal=1)
        outs.append(r.run(0, I, sch, 5, check_every=1 if mode == O.MODE_DELTA else 0))
    for key in ("cost", "best_cost", "digest", "accepted"):
        assert outs[0][key] == outs[1][key] == outs[2][key], key
    seq = O.Run(A, B, p0, mode=O.MODE_DELTA).run(0, I, sch, 5)
    assert seq["digest"] != outs[2]["digest"]
    opt = min(O.cost(A, B, np.array(q, np.int32)) for q in itertools.permutations(range(7)))
    assert outs[2]["best_cost"] == opt
    # frequencies: with an all-zero flow every proposal is accepted (δ = 0, R5), so the pair of
    # iteration k is read off the permutation change of a one-iteration call
    n6, K = 6, 6000
    Z = np.zeros((n6, n6), np.int32)
    Bz = taixxa(n6, 1)[1]
    rz = O.Run(Z, Bz, np.arange(n6, dtype=np.int32), mode=O.MODE_DELTA, proposal=1)
    sz = O.Schedule(O.COOL_GEOMETRIC, 1.0, 0.5, K)
    counts = {}
    for k in range(K):
        before = rz.p.copy()
        rz.run(k, 1, sz, 9)
        r_, s_ = np.nonzero(before != rz.p)[0]
        counts[(r_, s_)] = counts.get((r_, s_), 0) + 1
    M6 = n6 * (n6 - 1) // 2
    assert len(counts) == M6
    exp = K / M6                                  # 400 per pair; 5 sigma = 5 * sqrt(400) = 100
    assert all(abs(c - exp) < 100 for c in counts.values()), counts
