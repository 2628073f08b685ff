"""Pins of the CPU oracle against things other than itself (no GPU).

Each test names what it pins to: a value printed in SPEC.md (tests/golden/),
a published known-answer vector, a closed form, a library routine
(numpy matmul), brute force, or an invariant the mathematics fixes.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from qap_inputs import taixxa, start_perm

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


SPEC = _gold("spec_examples.json")
A3 = np.array(SPEC["instance_n3"]["A"], np.int32)
B3 = np.array(SPEC["instance_n3"]["B"], np.int32)


# ---- SPEC worked examples (golden/spec_examples.json, each with its line) ----

def test_spec_cost():
    assert O.cost(A3, B3, SPEC["cost_identity"]["p"]) == SPEC["cost_identity"]["value"]
    assert O.cost(A3, B3, SPEC["cost_210"]["p"]) == SPEC["cost_210"]["value"]
    assert O.cost(np.zeros((3, 3)), B3, [0, 1, 2]) == 0


def test_spec_bprime():
    np.testing.assert_array_equal(O.bprime(B3, SPEC["bprime_210"]["p"]),
                                  SPEC["bprime_210"]["value"])
    np.testing.assert_array_equal(O.bprime(B3, [0, 1, 2]), B3)


def test_spec_delta_scratch_and_eq1():
    for key in ("delta_01", "delta_02"):
        e = SPEC[key]
        assert O.delta_scratch(A3, B3, e["r"], e["s"]) == e["value"]
        assert O.delta_eq1(A3, B3, [0, 1, 2], e["r"], e["s"]) == e["value"]


def test_spec_delta_init():
    np.testing.assert_array_equal(O.delta_init(A3, B3), SPEC["delta_init_identity"]["value"])


def test_spec_apply_and_update():
    p = np.arange(3, dtype=np.int32)
    Bp = O.bprime(B3, p)
    D = O.delta_init(A3, Bp)
    pre = Bp.copy()
    O.apply_swap(p, Bp, 0, 2)
    O.update_delta(A3, pre, Bp, 0, 2, D)
    e = SPEC["apply_02"]
    np.testing.assert_array_equal(p, e["p_after"])
    np.testing.assert_array_equal(Bp, e["bprime_after"])
    assert O.cost(A3, B3, p) == e["cost_after"]
    assert D[O.index(3, 0, 1)] == SPEC["update_after_02"]["delta01_after"]


def test_spec_lundy_mees():
    e = SPEC["lundy_mees"]
    T = lambda k: O.temperature(O.COOL_LUNDY_MEES, e["t0"], e["tf"], e["total"], k)
    assert T(0) == e["t0"]
    assert T(10) == pytest.approx(e["T10"], rel=1e-12)
    assert T(5) == pytest.approx(e["T5"], rel=1e-12)


def test_spec_next_candidate():
    for n, q, rs in SPEC["next_candidate"]["cases"]:
        assert O.pair(n, q) == tuple(rs)
        assert O.index(n, *rs) == q


def test_spec_init_temperature():
    D = O.delta_init(A3, B3)
    t0, tf = O.temperature_bounds(D, 3)
    assert t0 == pytest.approx(SPEC["init_temperature_n3"]["t0"], rel=1e-15)
    assert tf == SPEC["init_temperature_n3"]["tf"]
    assert O.temperature_bounds(np.zeros(3, np.int64), 3) == (1.0, 0.1)


def test_spec_anneal_forced_first_candidate():
    """first candidate (0,1) has δ=-2 < 0 so it is accepted: cost 62."""
    run = O.Run(A3, B3, np.arange(3, dtype=np.int32))
    st = run.run(0, 1, O.Schedule(O.COOL_GEOMETRIC, 1.0, 1.0, 1), seed=1)
    assert st["accepted"] == 1 and st["cost"] == SPEC["anneal_forced_01"]["cost_after"]


def test_spec_accept_examples():
    """Eq.(2) (S:175-177 cases) as decided inside orc_sa_run.  State p=(2,1,0)
    of the N=3 instance has Δ_01 = +2; iteration k=0 proposes (0,1)
    (S:184).  With T held constant (t0 = tf) the run must accept exactly when
    exp(-2/T) > r_0, r_0 = the oracle's uniform for (seed, k=0)."""
    for delta, T, u, expect in SPEC["accept"]["cases"]:       # the printed numbers
        assert (delta < 0 or math.exp(-delta / T) > u) == expect
    p1 = np.array([2, 1, 0], np.int32)
    seen = set()
    for T in (10.0, 1.0, 3.0):
        for seed in range(40):
            run = O.Run(A3, B3, p1)
            st = run.run(0, 1, O.Schedule(O.COOL_GEOMETRIC, T, T, 1), seed=seed)
            u = O.uniform(seed, 0, 0, 0)
            expect = math.exp(-2.0 / T) > u
            seen.add(expect)
            assert st["accepted"] == int(expect)
            assert st["cost"] == (58 if expect else 56)
    assert seen == {True, False}


# ---- Philox4x32-10 known-answer vectors (golden/philox_kat.json) ----

def test_philox_kat():
    for v in _gold("philox_kat.json")["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        out = [int(x, 16) for x in v["out"]]
        np.testing.assert_array_equal(O.philox4x32_10(ctr, key), np.array(out, np.uint32))


def test_uniform_map_from_kat():
    """R3: U = ((x1:x0 >> 11) + 0.5) 2^-53 with (x0,x1) the KAT output at ctr=0,key=0."""
    x0, x1 = 0x6627E8D5, 0xE169C58D
    expect = (((x1 << 32 | x0) >> 11) + 0.5) / 2.0**53
    assert O.uniform(0, 0, 0, 0) == expect


def test_uniform_range_and_mean():
    us = np.array([O.uniform(7, k, 3, 0) for k in range(200000)])
    assert us.min() > 0.0 and us.max() < 1.0
    assert abs(us.mean() - 0.5) < 0.005          # S:151 asks 0.5 +- 0.01 over 1e6
    assert abs(us.var() - 1 / 12) < 0.002


# ---- closed forms ----

def test_geometric_schedule_endpoints():
    for t0, tf, I in [(1000.0, 2.0, 10**8), (10.0, 10.0, 5), (3.5, 0.25, 2)]:
        assert O.temperature(O.COOL_GEOMETRIC, t0, tf, I, 0) == t0
        assert O.temperature(O.COOL_GEOMETRIC, t0, tf, I, I - 1) == pytest.approx(tf, rel=1e-12)
        Ts = [O.temperature(O.COOL_GEOMETRIC, t0, tf, I, k) for k in range(0, I, max(1, I // 97))]
        assert all(a >= b for a, b in zip(Ts, Ts[1:]))


def test_lundy_mees_endpoints_and_recurrence():
    t0, tf, I = 50.0, 0.5, 1000
    beta = (t0 - tf) / ((I - 1) * t0 * tf)
    T = O.temperature(O.COOL_LUNDY_MEES, t0, tf, I, 0)
    for k in range(1, I):
        T = T / (1 + beta * T)                    # S:168 iterative form
        assert O.temperature(O.COOL_LUNDY_MEES, t0, tf, I, k) == pytest.approx(T, rel=1e-12)
    assert T == pytest.approx(tf, rel=1e-12)


def test_path_graph_linear_arrangement_bruteforce():
    """Closed form: A = path graph (unit flows i~i+1), B_ij = |i-j| on a line.
    Optimal linear arrangement of a path puts neighbours adjacent: C* = 2(n-1)."""
    for n in range(3, 9):
        A = np.zeros((n, n), np.int32)
        for i in range(n - 1):
            A[i, i + 1] = A[i + 1, i] = 1
        idx = np.arange(n)
        B = np.abs(idx[:, None] - idx[None, :]).astype(np.int32)
        c, bp = O.bruteforce(A, B)
        assert c == 2 * (n - 1)
        assert O.cost(A, B, bp) == c


def test_bruteforce_all_equivalent_facilities():
    """A = J - I (every facility identical): every permutation costs sum(B)."""
    n = 6
    A = (np.ones((n, n)) - np.eye(n)).astype(np.int32)
    _, B = taixxa(n, 3)
    c, _ = O.bruteforce(A, B)
    assert c == int(B.sum())


# ---- library routine / definition pins ----

def test_delta_init_matches_matmul_identity():
    """F6: δ(r,s) = 2[M_rs + M_sr - M_rr - M_ss + 2 a_rs B'_rs], M = A B' (numpy int64 matmul)."""
    for n, seed in [(5, 1), (12, 2), (31, 3), (64, 4)]:
        A, B = taixxa(n, seed)
        p = start_perm(n, 42, seed)
        Bp = B[np.ix_(p, p)]
        M = A.astype(np.int64) @ Bp.astype(np.int64)
        D = O.delta_init(A, Bp)
        for q in range(len(D)):
            r, s = O.pair(n, q)
            ref = 2 * (M[r, s] + M[s, r] - M[r, r] - M[s, s] + 2 * A[r, s] * Bp[r, s])
            assert D[q] == ref


def test_scratch_delta_equals_cost_difference():
    """δ (S:76 formula) == Eq.(1)(p∘(r s)) - Eq.(1)(p), Eq.(1) evaluated by numpy indexing."""
    rng = np.random.default_rng(0)
    for trial in range(60):
        n = int(rng.integers(3, 21))
        A, B = taixxa(n, 1000 + trial)
        p = rng.permutation(n).astype(np.int32)
        Bp = B[np.ix_(p, p)]
        c0 = int((A.astype(np.int64) * Bp).sum())
        for r in range(n):
            for s in range(r + 1, n):
                q = p.copy()
                q[r], q[s] = q[s], q[r]
                c1 = int((A.astype(np.int64) * B[np.ix_(q, q)]).sum())
                assert O.delta_scratch(A, Bp, r, s) == c1 - c0
                if trial < 5:
                    assert O.delta_eq1(A, B, p, r, s) == c1 - c0


def test_bprime_is_fancy_index():
    A, B = taixxa(17, 5)
    p = start_perm(17, 1, 0)
    np.testing.assert_array_equal(O.bprime(B, p), B[np.ix_(p, p)])


def test_pair_index_enumeration_is_row_major_triangle():
    for n in (2, 3, 7, 12, 100):
        expect = [(r, s) for r in range(n) for s in range(r + 1, n)]
        got = [O.pair(n, q) for q in range(len(expect))]
        assert got == expect
        assert [O.index(n, r, s) for r, s in expect] == list(range(len(expect)))


# ---- invariants ----

def test_update_equals_scratch_recompute_random_sequences():
    """AC1/AC2: after every accepted swap Δ == from-scratch Δ, B' == B[p][p]."""
    rng = np.random.default_rng(1)
    for trial in range(100):
        n = int(rng.integers(3, 21))
        A, B = taixxa(n, 2000 + trial)
        p = rng.permutation(n).astype(np.int32)
        Bp = O.bprime(B, p)
        D = O.delta_init(A, Bp)
        c = O.cost(A, B, p)
        for _ in range(20):
            r, s = sorted(rng.choice(n, 2, replace=False).tolist())
            d = D[O.index(n, r, s)]
            pre = Bp.copy()
            O.apply_swap(p, Bp, r, s)
            O.update_delta(A, pre, Bp, r, s, D)
            c += d
            assert c == O.cost(A, B, p)
            np.testing.assert_array_equal(Bp, B[np.ix_(p, p)])
            np.testing.assert_array_equal(D, O.delta_init(A, Bp))


def test_swap_is_involution():
    A, B = taixxa(9, 9)
    p = start_perm(9, 3, 0)
    Bp = O.bprime(B, p)
    p2, Bp2 = p.copy(), Bp.copy()
    O.apply_swap(p2, Bp2, 2, 7)
    O.apply_swap(p2, Bp2, 2, 7)
    np.testing.assert_array_equal(p2, p)
    np.testing.assert_array_equal(Bp2, Bp)


def test_swap_then_delta_is_negated():
    """Swapping (r,s) twice returns to the same cost, so Δ'_rs = -Δ_rs."""
    A, B = taixxa(11, 4)
    p = start_perm(11, 2, 0)
    Bp = O.bprime(B, p)
    D = O.delta_init(A, Bp)
    pre = Bp.copy()
    d = D[O.index(11, 3, 8)]
    O.apply_swap(p, Bp, 3, 8)
    O.update_delta(A, pre, Bp, 3, 8, D)
    assert D[O.index(11, 3, 8)] == -d


def test_twin_swaps_are_cost_neutral():
    """R21 (relabel engine): if rows x and y of A agree off the pair (twins), exchanging the
    facilities of x and y leaves Eq.(1) unchanged for EVERY permutation, so δ(x,y) = 0 in every
    state and the oracle's Δ holds 0 there.  Checked by direct Eq.(1) sums (numpy) on random
    permutations of an instance with twin classes, and on config 4's grey-density A."""
    from qap_inputs import block_classes, grey_density
    for A, B in (block_classes(24, [5, 4, 2], 7), grey_density(16, 6, 4)):
        n = A.shape[0]
        twins = [(x, y) for x in range(n) for y in range(x + 1, n)
                 if all(A[x, z] == A[y, z] for z in range(n) if z not in (x, y))]
        assert len(twins) >= 10
        rng = np.random.default_rng(3)

        def eq1(p):
            return int((A.astype(np.int64) * B[np.ix_(p, p)]).sum())

        nonzero = 0
        for _ in range(20):
            p = rng.permutation(n)
            c0 = eq1(p)
            for x, y in twins:
                q = p.copy()
                q[x], q[y] = q[y], q[x]
                assert eq1(q) == c0
            D = O.delta_init(A, O.bprime(B, p.astype(np.int32)))
            for x, y in twins:
                assert D[x * n - x * (x + 1) // 2 + y - x - 1] == 0
            nonzero += int(np.count_nonzero(D))
        assert nonzero > 0                      # the other swaps do change the cost


def test_start_perm_is_a_uniform_shuffle():
    """R14b: the chain-keyed Fisher-Yates start permutation.  Pins that do
    not restate the definition: every output is a bijection; over 36000 chains all 24
    permutations of 4 elements occur with frequency 1/24 (chi-square, 23 dof, < 60 ~ p 5e-5);
    Sattolo's variant (j < i, a plausible off-by-one) would produce only the 6 cyclic ones and
    an identity-biased variant (j <= i-1 shifts) would fail the test; different chains and seeds
    give different permutations."""
    import collections
    for n in (2, 5, 100, 256):
        for c in range(5):
            p = O.start_perm(n, 42, c)
            assert sorted(p.tolist()) == list(range(n))
    cnt = collections.Counter(tuple(O.start_perm(4, 7, c).tolist()) for c in range(36000))
    assert len(cnt) == 24
    e = 36000 / 24
    chi2 = sum((v - e) ** 2 / e for v in cnt.values())
    assert chi2 < 60, chi2
    assert not np.array_equal(O.start_perm(100, 42, 0), O.start_perm(100, 42, 1))
    assert not np.array_equal(O.start_perm(100, 42, 0), O.start_perm(100, 43, 0))
