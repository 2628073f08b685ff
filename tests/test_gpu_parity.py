"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Integers (Δ, p, C, counters, digest) must be bit-exact;
Eq.(2) decisions may differ only at flagged near ties (R16), which the oracle
then follows.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_1208_2675_b200 import qapsa as Q
from qap_inputs import SA_SEED, block_classes, config, grey_density, start_perm, start_perms, taixxa

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


TC = Q.QAP_OPT_TENSOR_CORE
SCR = Q.QAP_OPT_SCRATCH_PHASE
# the single-chain engines: tensor memory with the Δ-free high-acceptance phase (default where
# eligible), tensor memory with Δ throughout, shared memory
ENGINES = [pytest.param([(TC, 1), (SCR, 1)], id="tmem"), pytest.param([(TC, 1), (SCR, 0)], id="tmem_delta"),
           pytest.param([(TC, 0)], id="smem")]
RLB = Q.QAP_OPT_RELABEL
# instances with 8-bit A and 16-bit B (config 4): the relabel engine, the same engine with the
# twin relabels off, the shared-memory engine
RLBC = Q.QAP_OPT_RELABEL_CLUSTER
RELABEL_ENGINES = [pytest.param([(RLB, 1)], id="relabel"), pytest.param([(RLB, 2)], id="wide"),
                   pytest.param([(RLB, 1), (RLBC, 1)], id="relabel_1sm"),
                   pytest.param([(RLB, 0)], id="smem")]


def _sched(s: O.Schedule):
    return Q.make_schedule(s.kind, s.t0, s.tf, s.total_iters)


def _compare_run(A, B, p0, I, sched: O.Schedule, seed=SA_SEED, opts=(), k_splits=None,
                 mode=O.MODE_DELTA, proposal=0):
    """GPU run of iterations [0, I) vs the oracle; returns the GPU stats."""
    with Q.Solver(A, B, p0) as s:
        for k, v in opts:
            s.set_option(k, v)
        s.delta_init()
        bounds = k_splits or [0, I]
        tot_acc = 0
        for a, b in zip(bounds, bounds[1:]):
            g = s.run(a, b - a, _sched(sched), seed)
            tot_acc += g["accepted"]
        p, bp, D = s.state()
        n_near, near = s.near_ties()
        gcost = s.cost()
    ref = O.Run(A, B, p0, mode=mode, proposal=proposal)
    o = ref.run(0, I, sched, seed, follow=near)
    assert n_near == o["near_ties"]
    assert tot_acc == o["accepted"]
    for key in ("cost", "best_cost", "digest"):
        assert g[key] == o[key], key
    np.testing.assert_array_equal(p, ref.p)
    np.testing.assert_array_equal(bp, ref.best_p)
    assert gcost == O.cost(A, B, p) == o["cost"]
    if mode == O.MODE_DELTA:
        np.testing.assert_array_equal(D.astype(np.int64), ref.D)
    else:
        np.testing.assert_array_equal(D.astype(np.int64), O.delta_init(A, O.bprime(B, p)))
    return g, tot_acc


def _ens_follow(s):
    """{global chain: [(k, decision), ...]} from the last ensemble's near-tie log (R16)."""
    cnt, log = s.ensemble_near_ties()
    assert cnt == len(log)
    out = {}
    for c, k, d in log:
        out.setdefault(c, []).append((k, d))
    return out


def _check_chain(r, A, B, p0, chain, I, sch, seed, follow, proposal=0, mode=O.MODE_DELTA):
    """One ensemble chain's result against the oracle's single chain with the same global id,
    following the device's decisions at that chain's flagged near ties (R16)."""
    o = O.Run(A, B, p0, chain=chain, proposal=proposal, mode=mode).run(0, I, sch, seed,
                                                                       follow=follow.get(chain))
    assert (r["cost"], r["best_cost"], r["accepted"], r["near_ties"]) == (
        o["cost"], o["best_cost"], o["accepted"], o["near_ties"]), chain
    assert np.uint64(r["digest"]) == np.uint64(o["digest"]), chain
    assert len(follow.get(chain, [])) == r["near_ties"]


# ---------------- a1: Δ-init, Eq.(1), schedule bounds ----------------

@pytest.mark.parametrize("n,seed", [(2, 1), (3, 2), (5, 3), (12, 12), (33, 4), (50, 50), (64, 5),
                                    (100, 100), (129, 6), (200, 7), (256, 8)])
def test_delta_init_bit_exact(n, seed):
    A, B = taixxa(n, seed)
    p0 = start_perm(n, seed, 3)
    with Q.Solver(A, B, p0) as s:
        s.delta_init()
        _, _, D = s.state()
        assert s.cost() == O.cost(A, B, p0)
        q = start_perm(n, seed, 4)
        assert s.cost(q) == O.cost(A, B, q)
        ref = O.delta_init(A, O.bprime(B, p0))
        np.testing.assert_array_equal(D.astype(np.int64), ref)
        t0, tf = s.schedule_bounds()
        assert (t0, tf) == O.temperature_bounds(ref, n)


def test_delta_init_uint16_grey_density():
    A, B = grey_density(256)
    p0 = start_perm(256, SA_SEED, 0)
    with Q.Solver(A, B, p0) as s:
        s.delta_init()
        _, _, D = s.state()
        np.testing.assert_array_equal(D.astype(np.int64), O.delta_init(A, O.bprime(B, p0)))
        assert s.cost() == O.cost(A, B, p0)


def test_reset_restores_p0_and_perm():
    A, B = taixxa(20, 1)
    p0 = start_perm(20, 1, 0)
    with Q.Solver(A, B, p0) as s:
        s.delta_init()
        sch = O.geometric_schedule_for(A, B, p0, 5000)
        s.run(0, 5000, _sched(sch), 1)
        s.reset()
        p, bp, _ = s.state(want_delta=False)
        np.testing.assert_array_equal(p, p0)
        np.testing.assert_array_equal(bp, p0)
        with pytest.raises(Q.QapError):          # Δ invalid after reset
            s.run(0, 10, _sched(sch), 1)
        q = start_perm(20, 2, 0)
        s.reset(q)
        assert s.cost() == O.cost(A, B, q)


# ---------------- a2-a7: full trajectories ----------------

@pytest.mark.parametrize("engine", ENGINES)
def test_config1_full_bit_exact(engine):
    A, B, p0, cfg = config(1)
    sch = O.geometric_schedule_for(A, B, p0, cfg["iters"])
    g, acc = _compare_run(A, B, p0, cfg["iters"], sch, opts=engine)
    assert acc > 100


@pytest.mark.parametrize("engine", ENGINES)
def test_config2_full_bit_exact(engine):
    A, B, p0, cfg = config(2)
    sch = O.geometric_schedule_for(A, B, p0, cfg["iters"])
    _compare_run(A, B, p0, cfg["iters"], sch, mode=O.MODE_SCRATCH, opts=engine)


def test_engine_selection():
    """The tensor-memory engine runs exactly on the eligible instances (n <= 128, entries <= 127)."""
    cases = [(taixxa(100, 1), True), (taixxa(128, 2), True), (taixxa(129, 3), False),
             (taixxa(3, 4), False), (grey_density(256), False)]
    for (A, B), want in cases:
        with Q.Solver(A, B, start_perm(A.shape[0], 1, 0)) as s:
            assert s.uses_tensor_core() == want
            s.set_option(TC, 0)
            assert not s.uses_tensor_core()
    A, B = taixxa(20, 5)
    B2 = B.copy()
    B2[0, 1] = B2[1, 0] = 128
    with Q.Solver(A, B2, start_perm(20, 1, 0)) as s:
        assert not s.uses_tensor_core()


@pytest.mark.parametrize("n,seed", [(4, 1), (31, 2), (32, 3), (33, 4), (64, 5), (97, 6), (127, 7),
                                    (128, 8)])
def test_tmem_engine_full_range_values(n, seed):
    """Entries spanning the whole eligible range [0, 127] (the 8-bit digit encoding of the
    rank update at its limits) and sizes around the 32-lane TMEM quadrants."""
    rng = np.random.default_rng(seed)
    A = rng.integers(0, 128, size=(n, n)).astype(np.int32)
    B = rng.integers(0, 128, size=(n, n)).astype(np.int32)
    A = np.triu(A, 1); A = A + A.T
    B = np.triu(B, 1); B = B + B.T
    A[0, n - 1] = A[n - 1, 0] = 127
    B[0, n - 1] = B[n - 1, 0] = 127
    p0 = start_perm(n, seed, 0)
    sch = O.geometric_schedule_for(A, B, p0, 60000)
    with Q.Solver(A, B, p0) as s:
        assert s.uses_tensor_core()
    g, acc = _compare_run(A, B, p0, 60000, sch)
    assert acc > 100


@pytest.mark.parametrize("scratch", [1, 0])
@pytest.mark.parametrize("wmax", [32, 64, 256, 1024, 4096, 8192])
def test_tmem_window_invariance(wmax, scratch):
    A, B = taixxa(100, 77)
    p0 = start_perm(100, 5, 0)
    sch = O.geometric_schedule_for(A, B, p0, 200000)
    _compare_run(A, B, p0, 200000, sch, opts=[(Q.QAP_OPT_WINDOW_MAX, wmax), (SCR, scratch)])


@pytest.mark.parametrize("threads,wmax", [(256, 32), (512, 128), (1024, 1024), (1024, 64),
                                          (256, 256)])
def test_window_and_cta_shape_invariance(threads, wmax):
    """result independent of window size and CTA shape."""
    A, B = taixxa(50, 77)
    p0 = start_perm(50, 5, 0)
    sch = O.geometric_schedule_for(A, B, p0, 200000)
    _compare_run(A, B, p0, 200000, sch, opts=[(TC, 0), (Q.QAP_OPT_THREADS, threads),
                                                (Q.QAP_OPT_WINDOW_MAX, wmax)])


@pytest.mark.parametrize("engine", ENGINES)
def test_resume_split_calls(engine):
    A, B = taixxa(37, 9)
    p0 = start_perm(37, 9, 0)
    I = 300000
    sch = O.geometric_schedule_for(A, B, p0, I)
    _compare_run(A, B, p0, I, sch, k_splits=[0, 1, 999, 1000, 123457, I], opts=engine)


def test_global_delta_variant():
    """Δ kept in global memory / L2 (the spill path) gives the same trajectory."""
    A, B = taixxa(64, 3)
    p0 = start_perm(64, 3, 0)
    sch = O.geometric_schedule_for(A, B, p0, 200000)
    _compare_run(A, B, p0, 200000, sch, opts=[(Q.QAP_OPT_FORCE_GLOBAL_DELTA, 1)])


@pytest.mark.parametrize("engine", ENGINES)
def test_lundy_mees_schedule(engine):
    A, B = taixxa(30, 30)
    p0 = start_perm(30, 1, 0)
    g = O.geometric_schedule_for(A, B, p0, 100000)
    sch = O.Schedule(O.COOL_LUNDY_MEES, g.t0, g.tf, 100000)
    _compare_run(A, B, p0, 100000, sch, opts=engine)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("n", [2, 3, 4, 5, 7])
def test_tiny_instances_window_wraps(n, engine):
    """M < window: candidates wrap around the triangle many times per window."""
    A, B = taixxa(n, 40 + n)
    p0 = start_perm(n, n, 0)
    sch = O.geometric_schedule_for(A, B, p0, 20000)
    _compare_run(A, B, p0, 20000, sch, opts=engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_all_zero_flow_every_iteration_accepts(engine):
    n = 16
    _, B = taixxa(n, 2)
    A = np.zeros((n, n), np.int32)
    p0 = start_perm(n, 1, 0)
    sch = O.Schedule(O.COOL_GEOMETRIC, 1.0, 0.1, 5000)
    g, acc = _compare_run(A, B, p0, 5000, sch, opts=engine)
    assert acc == 5000 and g["cost"] == 0


@pytest.mark.parametrize("engine", ENGINES)
def test_single_iteration_and_tail_of_schedule(engine):
    A, B = taixxa(25, 2)
    p0 = start_perm(25, 2, 0)
    sch = O.geometric_schedule_for(A, B, p0, 10**6)
    with Q.Solver(A, B, p0) as s:
        for kv in engine:
            s.set_option(*kv)
        s.delta_init()
        g = s.run(10**6 - 1, 1, _sched(sch), 7)
        _, _, D = s.state()
    ref = O.Run(A, B, p0)
    o = ref.run(10**6 - 1, 1, sch, 7)
    assert g["cost"] == o["cost"] and g["digest"] == o["digest"]
    np.testing.assert_array_equal(D.astype(np.int64), ref.D)


def test_schedule_errors():
    A, B = taixxa(10, 1)
    p0 = start_perm(10, 1, 0)
    with Q.Solver(A, B, p0) as s:
        with pytest.raises(Q.QapError) as e:
            s.run(0, 10, Q.make_schedule(0, 1.0, 0.5, 100), 1)     # Δ not initialised
        assert e.value.status == 6
        s.delta_init()
        for bad in [Q.make_schedule(0, 1.0, 2.0, 100), Q.make_schedule(0, 1.0, 0.0, 100),
                    Q.make_schedule(5, 1.0, 0.5, 100), Q.make_schedule(0, 1.0, 0.5, 5)]:
            with pytest.raises(Q.QapError) as e:
                s.run(0, 10, bad, 1)
            assert e.value.status == 5


@pytest.mark.parametrize("engine", RELABEL_ENGINES)
def test_grey_density_uint16_prefix(engine):
    """Config-4-shaped instance (uint16 B, δ≡0 plateau): the first 1e6 iterations (3e5 on the
    slow shared-memory engine) of its 1e9-iteration schedule, in two calls."""
    A, B = grey_density(256)
    p0 = start_perm(256, SA_SEED, 0)
    sch = O.geometric_schedule_for(A, B, p0, 10**9)
    I = 300000 if engine == [(RLB, 0)] else 10**6       # the shared-memory engine is slow here
    g, acc = _compare_run(A, B, p0, I, sch, mode=O.MODE_SCRATCH, opts=engine,
                          k_splits=[0, I // 3, I])
    assert acc > I // 3


def test_relabel_engine_selection():
    for (A, B), want in [(grey_density(256), Q.QAP_ENGINE_RELABEL),
                         (block_classes(40, [6, 3], 1), Q.QAP_ENGINE_RELABEL),
                         (block_classes(40, [6, 3], 1, hi_b=99), Q.QAP_ENGINE_TENSOR_MEMORY),
                         (taixxa(150, 1), Q.QAP_ENGINE_SHARED_MEMORY),    # 8-bit, Δ fits on chip
                         (taixxa(256, 1), Q.QAP_ENGINE_RELABEL),          # 8-bit, Δ would spill
                         (taixxa(100, 1, hi=200), Q.QAP_ENGINE_SHARED_MEMORY)]:
        n = A.shape[0]
        with Q.Solver(A, B, start_perm(n, 1, 0)) as s:
            assert s.engine() == want
            s.set_option(RLB, 0)
            if want == Q.QAP_ENGINE_RELABEL:
                assert s.engine() == Q.QAP_ENGINE_SHARED_MEMORY


@pytest.mark.parametrize("n,sizes,seed,iters", [(4, [2], 1, 3000), (9, [3, 2], 2, 20000),
                                                (33, [8, 5, 3], 3, 50000),
                                                (64, [20, 10, 6, 3], 4, 100000),
                                                (130, [40, 30, 2], 5, 60000),
                                                (256, [92, 100, 3], 6, 60000),
                                                (90, [9, 8, 7, 6, 5, 4], 7, 60000)])   # > RLB_MAXCLS classes
@pytest.mark.parametrize("engine", RELABEL_ENGINES[:3])
def test_relabel_engine_twin_classes(n, sizes, seed, iters, engine):
    """Instances with twin classes (R21) and 16-bit B: Δ, p, best_p, C, digest and every
    counter bit-exact against the oracle in DELTA mode, relabels on and off."""
    A, B = block_classes(n, sizes, seed, hi_b=20000)     # 4 n maxA maxB < 2^31 (R13)
    p0 = start_perm(n, seed, 0)
    sch = O.geometric_schedule_for(A, B, p0, iters)
    _compare_run(A, B, p0, iters, sch, opts=engine)


@pytest.mark.parametrize("engine", RELABEL_ENGINES[:3])
def test_relabel_engine_no_twins_and_resume(engine):
    """A 16-bit instance without twins (the wide engine's ordinary path), and a twin instance
    split into uneven calls (σ is folded back into p and Δ at every exit)."""
    A, _ = taixxa(77, 77)
    _, B = taixxa(77, 78, hi=3000)
    p0 = start_perm(77, 7, 0)
    with Q.Solver(A, B, p0) as s:
        for k, v in engine:
            s.set_option(k, v)
        assert s.engine() == Q.QAP_ENGINE_RELABEL
    _compare_run(A, B, p0, 40000, O.geometric_schedule_for(A, B, p0, 40000), opts=engine)
    A, B = block_classes(101, [30, 20, 10], 8, hi_b=20000)
    p0 = start_perm(101, 8, 0)
    I = 50000
    _compare_run(A, B, p0, I, O.geometric_schedule_for(A, B, p0, I), opts=engine,
                 k_splits=[0, 1, 77, 5000, 5001, 23456, I])


# ---------------- a8: ensemble ----------------

def test_ensemble_per_chain_bit_exact():
    A, B = taixxa(40, 40)
    p0s = start_perms(40, SA_SEED, 100, 50)
    sch = O.geometric_schedule_for(A, B, p0s[0], 30000)
    with Q.Solver(A, B, p0s[0]) as s:
        res = s.ensemble(100, p0s, 30000, _sched(sch), SA_SEED, per_chain=True)
        follow = _ens_follow(s)
    ref = O.ensemble_run(A, B, p0s, 100, 30000, sch, SA_SEED)
    for i, r in enumerate(res["per_chain"]):
        if 100 + i in follow:                   # flagged: replay with the device's decisions
            _check_chain(r, A, B, p0s[i], 100 + i, 30000, sch, SA_SEED, follow)
            continue
        assert (r["cost"], r["best_cost"], r["accepted"], r["iterations"], r["near_ties"]) == tuple(
            int(x) for x in ref[i, [0, 1, 2, 5, 3]])
        assert np.uint64(r["digest"]) == np.int64(ref[i, 4]).astype(np.uint64)
    bi = int(np.lexsort((np.arange(50), ref[:, 1]))[0])
    assert res["best_chain"] == 100 + bi and res["best_cost"] == ref[bi, 1]
    assert O.cost(A, B, res["best_perm"]) == res["best_cost"]


@pytest.mark.parametrize("group", [64, 128, 256])
def test_ensemble_group_shape_invariance(group):
    A, B = taixxa(24, 24)
    p0s = start_perms(24, 3, 0, 20)
    sch = O.geometric_schedule_for(A, B, p0s[0], 20000)
    with Q.Solver(A, B, p0s[0]) as s:
        s.set_option(Q.QAP_OPT_ENSEMBLE_GROUP, group)
        res = s.ensemble(0, p0s, 20000, _sched(sch), 3, per_chain=True)
    ref = O.ensemble_run(A, B, p0s, 0, 20000, sch, 3)
    got = np.array([[r["cost"], r["best_cost"], r["accepted"]] for r in res["per_chain"]])
    np.testing.assert_array_equal(got, ref[:, :3])


# ---------------- full-size configs (launch configuration of bench.py) ----------------

@pytest.mark.slow
def test_config3_full_size():
    """BASELINE config 3 (N=100, 1e8) end to end vs the oracle (SCRATCH δ source)."""
    A, B, p0, cfg = config(3)
    sch = O.geometric_schedule_for(A, B, p0, cfg["iters"])
    _compare_run(A, B, p0, cfg["iters"], sch, mode=O.MODE_SCRATCH)


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.slow
def test_config5_all_chains_vs_oracle_goldens():
    """BASELINE config 5 at full size, as bench.py runs it (8192 x N=100 x 1e7 on one GPU, start
    permutations generated on the device, R14b): EVERY chain's cost, best cost, accepted count,
    near ties and digest against the oracle's (tests/golden/config5_chains.npz, written by
    tests/golden/make_goldens.py from oracle/ only).  A chain whose device decision at a flagged
    near tie differs from the oracle's own is replayed by the oracle following the device (R16).
    Also the argmin and Eq.(1) of the returned best permutation."""
    g = np.load(os.path.join(GOLDEN, "config5_chains.npz"))
    ref, nk, nd = g["out"], g["near_k"], g["near_d"]
    kind, t0, tf, I = g["schedule"]
    A, B, _, cfg = config(5)
    n, C = cfg["n"], cfg["chains"]
    assert (C, int(I)) == (ref.shape[0], cfg["iters"])
    with Q.Solver(A, B, np.arange(n, dtype=np.int32)) as s:
        p00 = s.start_perms(SA_SEED, 0, 1)[0]
        np.testing.assert_array_equal(p00, O.start_perm(n, SA_SEED, 0))
        s.reset(p00)
        s.delta_init()
        assert s.schedule_bounds() == (t0, tf)          # R2 at chain 0's start permutation
        sch = O.Schedule(int(kind), t0, tf, int(I))
        res = s.ensemble(0, None, int(I), _sched(sch), SA_SEED, per_chain=True, count=C)
        follow = _ens_follow(s)
    per = res["per_chain"]
    got = np.array([[r["cost"], r["best_cost"], r["accepted"], r["near_ties"], r["iterations"]]
                    for r in per], np.int64)
    dig = np.array([r["digest"] for r in per], np.uint64)
    replay = []
    for c in range(C):
        m = int(ref[c, 3])
        oracle_log = [(int(nk[c, i]), int(nd[c, i])) for i in range(min(m, nk.shape[1]))]
        if follow.get(c, []) != oracle_log:      # a near tie decided differently: replay
            replay.append(c)
            continue
        assert tuple(got[c]) == tuple(int(x) for x in ref[c, [0, 1, 2, 3, 5]]), c
        assert dig[c] == np.int64(ref[c, 4]).astype(np.uint64), c
    assert len(replay) <= 8, replay             # near ties are rare (< 1 per 1e8 iterations)
    for c in replay:
        _check_chain(per[c], A, B, O.start_perm(n, SA_SEED, c), c, int(I), sch, SA_SEED, follow,
                     mode=O.MODE_SCRATCH)
    best = min(range(C), key=lambda i: (per[i]["best_cost"], i))
    assert res["best_chain"] == best and res["best_cost"] == per[best]["best_cost"]
    assert O.cost(A, B, res["best_perm"]) == res["best_cost"]
    assert int(got[:, 3].sum()) < C * int(I) / 1e8 + 3       # BASELINE: < 1 near tie per 1e8


@pytest.mark.slow
def test_config4_full_run_vs_oracle_goldens():
    """BASELINE config 4 at full length (N=256 grey density, 1e9 iterations) on the relabel
    engine (cluster of 8), in ten calls of 1e8: after every call p, best_p, C, best, accepted,
    digest and the near ties equal the oracle's checkpoints (tests/golden/config4_full.json,
    written by tests/golden/make_goldens.py from oracle/ only)."""
    import json
    with open(os.path.join(GOLDEN, "config4_full.json")) as f:
        gold = json.load(f)
    A, B, p0, cfg = config(4)
    sc = gold["schedule"]
    sch = O.Schedule(sc["kind"], sc["t0"], sc["tf"], sc["total_iters"])
    with Q.Solver(A, B, p0) as s:
        assert s.engine() == Q.QAP_ENGINE_RELABEL
        s.delta_init()
        assert s.schedule_bounds() == (sch.t0, sch.tf)
        k, acc = 0, 0
        for cp in gold["checkpoints"]:
            g = s.run(k, cp["k"] - k, _sched(sch), SA_SEED)
            k = cp["k"]
            acc += g["accepted"]
            p, bp, _ = s.state(want_delta=False)
            n_near, near = s.near_ties()
            assert near == [tuple(x) for x in cp["near_log"]], k
            assert (g["cost"], g["best_cost"], acc, n_near) == (
                cp["cost"], cp["best_cost"], cp["accepted"], cp["near_ties"]), k
            assert g["digest"] == int(cp["digest"]), k
            np.testing.assert_array_equal(p, cp["p"])
            np.testing.assert_array_equal(bp, cp["best_p"])
        _, _, D = s.state()
    np.testing.assert_array_equal(D.astype(np.int64), O.delta_init(A, O.bprime(B, p)))
    assert k == cfg["iters"]


# ---------------- f1: the cluster engine (cluster_chain.cuh): rows of A, B' and Δ over 8 SMs ----------------

CLU = Q.QAP_OPT_CLUSTER_ENGINE


@pytest.mark.parametrize("n,I", [(12, 50000), (50, 100000), (100, 100000), (129, 60000)])
def test_cluster_engine_forced_small(n, I):
    """QAP_OPT_CLUSTER_ENGINE = 2 runs the cluster engine on instances other engines also take:
    bit-exact against the oracle (Δ after the run included), in three calls (resume by k0)."""
    A, B = taixxa(n, 900 + n)
    p0 = start_perm(n, 11, 0)
    sch = O.geometric_schedule_for(A, B, p0, I)
    with Q.Solver(A, B, p0) as s:
        s.set_option(CLU, 2)
        assert s.engine() == Q.QAP_ENGINE_CLUSTER
    _compare_run(A, B, p0, I, sch, opts=[(CLU, 2)], k_splits=[0, I // 3, I // 2, I])


@pytest.mark.parametrize("n", [384, 512])
def test_cluster_engine_large_n(n):
    """N beyond one SM (up to QAP_MAX_N = 512) is accepted and runs on the cluster engine: Δ-init
    against the oracle's, then a 1e5-iteration trajectory bit-exact against the oracle (SCRATCH
    mode: δ from its definition, Δ compared with a from-scratch rebuild at the end)."""
    A, B = taixxa(n, 4000 + n)
    p0 = start_perm(n, 13, 0)
    I = 100000
    with Q.Solver(A, B, p0) as s:
        assert s.engine() == Q.QAP_ENGINE_CLUSTER
        s.delta_init()
        _, _, D = s.state()
        np.testing.assert_array_equal(D.astype(np.int64), O.delta_init(A, O.bprime(B, p0)))
    sch = O.geometric_schedule_for(A, B, p0, I)
    g, acc = _compare_run(A, B, p0, I, sch, mode=O.MODE_SCRATCH)
    assert acc > 1000


@pytest.mark.parametrize("n", [257, 263])
def test_cluster_engine_ragged_n(n):
    """N not a multiple of the cluster (rows of the last CTAs shorter), 8-bit B, five calls."""
    A, B = taixxa(n, 500 + n)
    p0 = start_perm(n, 21, 0)
    I = 50000
    with Q.Solver(A, B, p0) as s:
        assert s.engine() == Q.QAP_ENGINE_CLUSTER
    sch = O.geometric_schedule_for(A, B, p0, I)
    _compare_run(A, B, p0, I, sch, mode=O.MODE_SCRATCH, k_splits=[0, 1, 999, 20000, 33333, I])


def test_cluster_engine_uint16_b():
    """16-bit B on the cluster engine (N = 300 > 256, entries up to 2000)."""
    n = 300
    A, _ = taixxa(n, 301)
    _, B = taixxa(n, 302, 0, 2000)
    p0 = start_perm(n, 17, 0)
    I = 60000
    with Q.Solver(A, B, p0) as s:
        assert s.engine() == Q.QAP_ENGINE_CLUSTER
    sch = O.geometric_schedule_for(A, B, p0, I)
    _compare_run(A, B, p0, I, sch, mode=O.MODE_SCRATCH, k_splits=[0, 25000, I])


def test_qaplib_fixture_through_the_abi():
    """f4: a QAPLIB-format instance read from tests/golden goes through qap_create like any
    other; the run is bit-exact against the oracle and reaches the brute-force optimum."""
    import os
    from paper_1208_2675_b200 import qaplib
    gold = os.path.join(os.path.dirname(__file__), "golden")
    A, B = qaplib.read_dat(os.path.join(gold, "qaplib_tiny4.dat"))
    _, opt, _ = qaplib.read_sln(os.path.join(gold, "qaplib_tiny4.sln"))
    p0 = start_perm(4, SA_SEED, 0)
    I = 20000
    g, _ = _compare_run(A, B, p0, I, O.geometric_schedule_for(A, B, p0, I))
    assert g["best_cost"] == opt


# ---------------- f4: random proposals (R22) ----------------

@pytest.mark.parametrize("tc", [2, 1, 0])
@pytest.mark.parametrize("n,I", [(5, 20000), (12, 100000), (50, 300000), (100, 200000), (128, 100000)])
def test_random_proposals_single_chain(n, I, tc):
    """R22 random proposals (QAP_OPT_PROPOSAL = 1) on the tensor-memory Δ engine (QAP_OPT_TENSOR_CORE
    = 2: windows of random candidates gathered from their TMEM lanes) and on the shared-memory
    engine (the default for random proposals, 1, and 0): bit-exact
    against the oracle's random-proposal mode, split into uneven calls."""
    if n == 128:
        rng = np.random.default_rng(9)
        A = np.triu(rng.integers(0, 128, size=(n, n)), 1).astype(np.int32)
        B = np.triu(rng.integers(0, 128, size=(n, n)), 1).astype(np.int32)
        A, B = A + A.T, B + B.T
    else:
        A, B = taixxa(n, 1000 + n)
    p0 = start_perm(n, SA_SEED, 0)
    opts = [(Q.QAP_OPT_PROPOSAL, 1), (TC, tc)]
    with Q.Solver(A, B, p0) as s:
        for k_, v_ in opts:
            s.set_option(k_, v_)
        assert s.engine() == (Q.QAP_ENGINE_TENSOR_MEMORY if tc == 2 else Q.QAP_ENGINE_SHARED_MEMORY)
    _compare_run(A, B, p0, I, O.geometric_schedule_for(A, B, p0, I), opts=opts,
                 k_splits=[0, 7, I // 3, I], proposal=1)


def test_random_proposals_ensemble_chains():
    """Random proposals in qap_ensemble_run: every chain equals the oracle's single chain with
    the same global chain id (the proposal stream is keyed by it)."""
    A, B = taixxa(30, 31)
    C, I = 12, 20000
    p0s = start_perms(30, SA_SEED, 40, C)
    sch = O.geometric_schedule_for(A, B, p0s[0], I)
    with Q.Solver(A, B, p0s[0]) as s:
        s.set_option(Q.QAP_OPT_PROPOSAL, 1)
        res = s.ensemble(40, p0s, I, _sched(sch), SA_SEED, per_chain=True)
        follow = _ens_follow(s)
    for i, r in enumerate(res["per_chain"]):
        _check_chain(r, A, B, p0s[i], 40 + i, I, sch, SA_SEED, follow, proposal=1)


@pytest.mark.parametrize("engine", [pytest.param([(RLB, 3)], id="relabel"),
                                    pytest.param([(RLB, 3), (RLBC, 1)], id="relabel_1sm"),
                                    pytest.param([(RLB, 0)], id="smem")])
@pytest.mark.parametrize("n", [129, 200, 256])
def test_relabel_engine_8bit_large_n(n, engine):
    """8-bit instances with 128 < N <= 256 (beyond the tensor-memory engine) on the relabel
    engine (forced by QAP_OPT_RELABEL = 3 below N = 256), with and without twins, against the
    oracle."""
    with Q.Solver(*taixxa(n, 1), start_perm(n, 1, 0)) as s:
        for k, v in engine:
            s.set_option(k, v)
        if engine[0] == (RLB, 3):
            assert s.engine() == Q.QAP_ENGINE_RELABEL
    A, B = taixxa(n, 500 + n)
    p0 = start_perm(n, SA_SEED, 0)
    I = 60000
    _compare_run(A, B, p0, I, O.geometric_schedule_for(A, B, p0, I), opts=engine, k_splits=[0, I // 2, I])
    A, B = block_classes(n, [40, 30], 600 + n, hi_b=255)
    _compare_run(A, B, p0, I, O.geometric_schedule_for(A, B, p0, I), opts=engine)


def test_ensemble_tensor_memory_vs_shared_memory():
    """qap_ensemble_run on the tensor-memory engine (default where eligible: one SM per chain,
    scratch phase, Δ rebuild, Δ engine) and on the shared-memory kernel give the same result
    for every chain, and both match the oracle's single chains."""
    A, B = taixxa(60, 61)
    C, I = 40, 50000
    p0s = start_perms(60, SA_SEED, 7, C)
    sch = O.geometric_schedule_for(A, B, p0s[0], I)
    out, fol = {}, {}
    for tcv in (1, 0):
        with Q.Solver(A, B, p0s[0]) as s:
            s.set_option(TC, tcv)
            out[tcv] = s.ensemble(7, p0s, I, _sched(sch), SA_SEED, per_chain=True)
            fol[tcv] = _ens_follow(s)
    assert out[1]["best_cost"] == out[0]["best_cost"] and out[1]["best_chain"] == out[0]["best_chain"]
    np.testing.assert_array_equal(out[1]["best_perm"], out[0]["best_perm"])
    assert fol[1] == fol[0]
    for i, (r1, r0) in enumerate(zip(out[1]["per_chain"], out[0]["per_chain"])):
        assert r1 == r0, i
        if i < 6 or 7 + i in fol[1]:
            _check_chain(r1, A, B, p0s[i], 7 + i, I, sch, SA_SEED, fol[1])


# ---------------- R16: constructed near ties through every engine ----------------

def _near_tie_setup(n=12, inst=3, seed=SA_SEED, chain=0, I=5000):
    """Instance, p0 and a constant schedule T = δ/(-ln r_0) that make iteration 0 (pair (0,1),
    δ = Δ_01(p0) > 0) a near tie for `chain` (R16)."""
    import math
    A, B = taixxa(n, inst)
    for c in range(64):
        p0 = start_perm(n, inst, c)
        d = int(O.delta_init(A, O.bprime(B, p0))[0])
        if d > 0:
            break
    T = d / -math.log(O.uniform(seed, 0, chain, 0))
    return A, B, p0, O.Schedule(O.COOL_GEOMETRIC, T, T, I)


NEAR_ENGINES = ENGINES + [pytest.param([(TC, 0), (RLB, 3)], id="relabel"),
                          pytest.param([(TC, 0), (RLB, 3), (RLBC, 1)], id="relabel_1sm"),
                          pytest.param([(Q.QAP_OPT_CLUSTER_ENGINE, 2)], id="cluster")]


@pytest.mark.parametrize("engine", NEAR_ENGINES)
def test_constructed_near_tie_single_chain(engine):
    """A flagged near tie at k = 0 on every single-chain engine: the device flags it, logs its
    decision, and the oracle following that decision reproduces the whole run bit-exactly."""
    A, B, p0, sch = _near_tie_setup()
    with Q.Solver(A, B, p0) as s:
        for kv in engine:
            s.set_option(*kv)
        if engine[-1] == (RLB, 3) or engine[-1] == (RLBC, 1):
            assert s.engine() == Q.QAP_ENGINE_RELABEL
    g, _ = _compare_run(A, B, p0, sch.total_iters, sch, opts=engine)
    with Q.Solver(A, B, p0) as s:
        for kv in engine:
            s.set_option(*kv)
        s.delta_init()
        s.run(0, sch.total_iters, _sched(sch), SA_SEED)
        n_near, near = s.near_ties()
    assert n_near >= 1 and near[0][0] == 0


@pytest.mark.parametrize("tc", [1, 0])
def test_constructed_near_tie_ensemble_chain(tc):
    """An ensemble in which chain 5 (global id) has a near tie at k = 0: the device logs (5, 0,
    decision) in the ensemble near-tie log, and the oracle's single chain 5 following it matches;
    every other chain matches the oracle too (tensor-memory and shared-memory ensembles)."""
    C, I = 8, 4000
    A, B, _, _ = _near_tie_setup()
    import math
    p0s = start_perms(12, 3, 0, C)
    d = int(O.delta_init(A, O.bprime(B, p0s[5]))[0])
    if d <= 0:
        p0s[5] = p0s[5][[1, 0] + list(range(2, 12))]
        d = int(O.delta_init(A, O.bprime(B, p0s[5]))[0])
    assert d > 0
    T = d / -math.log(O.uniform(SA_SEED, 0, 5, 0))
    sch = O.Schedule(O.COOL_GEOMETRIC, T, T, I)
    with Q.Solver(A, B, p0s[0]) as s:
        s.set_option(TC, tc)
        res = s.ensemble(0, p0s, I, _sched(sch), SA_SEED, per_chain=True)
        follow = _ens_follow(s)
    assert 5 in follow and follow[5][0][0] == 0
    for i, r in enumerate(res["per_chain"]):
        _check_chain(r, A, B, p0s[i], i, I, sch, SA_SEED, follow)


# ---------------- R14b: chain-keyed start permutations on the device ----------------

@pytest.mark.parametrize("n", [2, 3, 12, 100, 256])
def test_start_perms_match_oracle(n):
    A, B = taixxa(n, 1)
    with Q.Solver(A, B, np.arange(n, dtype=np.int32)) as s:
        got = s.start_perms(SA_SEED, 1000, 17)
    for i in range(17):
        np.testing.assert_array_equal(got[i], O.start_perm(n, SA_SEED, 1000 + i))


@pytest.mark.parametrize("tc", [1, 0])
def test_ensemble_device_start_perms(tc):
    """qap_ensemble_run with p0s = NULL: chains start from the device's chain-keyed permutations
    and equal the oracle's chains started from O.start_perm (no host start array)."""
    A, B = taixxa(30, 9)
    C, I = 20, 30000
    sch = O.geometric_schedule_for(A, B, O.start_perm(30, SA_SEED, 0), I)
    with Q.Solver(A, B, np.arange(30, dtype=np.int32)) as s:
        s.set_option(TC, tc)
        res = s.ensemble(300, None, I, _sched(sch), SA_SEED, per_chain=True, count=C)
        follow = _ens_follow(s)
    p0s = np.stack([O.start_perm(30, SA_SEED, 300 + i) for i in range(C)])
    ref = O.ensemble_run(A, B, p0s, 300, I, sch, SA_SEED)
    for i, r in enumerate(res["per_chain"]):
        if 300 + i in follow:
            _check_chain(r, A, B, p0s[i], 300 + i, I, sch, SA_SEED, follow)
            continue
        assert (r["cost"], r["best_cost"], r["accepted"]) == tuple(int(x) for x in ref[i, :3])
    bi = int(np.lexsort((np.arange(C), ref[:, 1]))[0])
    assert res["best_chain"] == 300 + bi


@pytest.mark.parametrize("n", [127, 128])
def test_tmem_ensemble_at_the_lane_limit(n):
    """Tensor-memory ensemble at N = 127, 128 (H columns of the last window rows stay inside a
    chain's 256 TMEM columns; two chains per SM)."""
    rng = np.random.default_rng(n)
    A = np.triu(rng.integers(0, 128, size=(n, n)), 1).astype(np.int32)
    B = np.triu(rng.integers(0, 128, size=(n, n)), 1).astype(np.int32)
    A, B = A + A.T, B + B.T
    C, I = 6, 40000
    p0s = start_perms(n, 2, 0, C)
    sch = O.geometric_schedule_for(A, B, p0s[0], I)
    with Q.Solver(A, B, p0s[0]) as s:
        assert s.uses_tensor_core()
        res = s.ensemble(0, p0s, I, _sched(sch), SA_SEED, per_chain=True)
        follow = _ens_follow(s)
    for i, r in enumerate(res["per_chain"]):
        _check_chain(r, A, B, p0s[i], i, I, sch, SA_SEED, follow)


def test_tmem_ensemble_more_chains_than_grid_y():
    """65537 chains (more than gridDim.y allows in one Δ-rebuild launch): every sampled chain
    equals the oracle's."""
    A, B = taixxa(8, 8)
    C, I = 65537, 300
    sch = O.geometric_schedule_for(A, B, O.start_perm(8, SA_SEED, 0), I)
    with Q.Solver(A, B, np.arange(8, dtype=np.int32)) as s:
        assert s.uses_tensor_core()
        res = s.ensemble(0, None, I, _sched(sch), SA_SEED, per_chain=True, count=C)
        follow = _ens_follow(s)
    per = res["per_chain"]
    for c in [0, 1, 65534, 65535, 65536]:
        _check_chain(per[c], A, B, O.start_perm(8, SA_SEED, c), c, I, sch, SA_SEED, follow)


# ---------------- ensemble scratch phase, four chains per SM (ens_chain.cuh) ----------------

@pytest.mark.parametrize("n,C,I", [(12, 64, 30000), (60, 40, 50000), (100, 24, 60000), (128, 10, 40000)])
def test_ensemble_four_chains_per_sm_vs_two(n, C, I):
    """QAP_OPT_ENSEMBLE_SCRATCH4 = 1 (default: G only in tensor memory, four chains per SM) and 0
    (G and H, two chains per SM) give identical per-chain results, argmin and best permutation;
    chains sampled against the oracle (followed at flagged near ties)."""
    if n == 128:
        rng = np.random.default_rng(5)
        A = np.triu(rng.integers(0, 128, size=(n, n)), 1).astype(np.int32)
        B = np.triu(rng.integers(0, 128, size=(n, n)), 1).astype(np.int32)
        A, B = A + A.T, B + B.T
    else:
        A, B = taixxa(n, 70 + n)
    p0s = start_perms(n, SA_SEED, 11, C)
    sch = O.geometric_schedule_for(A, B, p0s[0], I)
    out, fol = {}, {}
    for e4 in (1, 0):
        with Q.Solver(A, B, p0s[0]) as s:
            assert s.uses_tensor_core()
            s.set_option(Q.QAP_OPT_ENSEMBLE_SCRATCH4, e4)
            out[e4] = s.ensemble(11, p0s, I, _sched(sch), SA_SEED, per_chain=True)
            fol[e4] = _ens_follow(s)
    assert fol[1] == fol[0]
    assert (out[1]["best_cost"], out[1]["best_chain"]) == (out[0]["best_cost"], out[0]["best_chain"])
    np.testing.assert_array_equal(out[1]["best_perm"], out[0]["best_perm"])
    for i, (r1, r0) in enumerate(zip(out[1]["per_chain"], out[0]["per_chain"])):
        assert r1 == r0, i
    for i in sorted({0, 1, C - 1} | {c - 11 for c in fol[1]}):
        _check_chain(out[1]["per_chain"][i], A, B, p0s[i], 11 + i, I, sch, SA_SEED, fol[1])


@pytest.mark.parametrize("gap", [1, 64, 100000, 2**31 - 1])
def test_switch_gap_invariance(gap):
    """QAP_OPT_SWITCH_GAP moves the scratch -> Δ hand-over (f2) without changing the trajectory:
    bit-exact against the oracle for a gap of 1 (hand over at once), 64, 1e5 and never."""
    A, B = taixxa(60, 66)
    p0 = start_perm(60, 6, 0)
    I = 150000
    sch = O.geometric_schedule_for(A, B, p0, I)
    _compare_run(A, B, p0, I, sch, opts=[(Q.QAP_OPT_SWITCH_GAP, gap)], k_splits=[0, 50001, I])


def test_device_pool_reuse_across_contexts_and_streams():
    """Device buffers come from the library's stream-ordered pool (qapsa.cu dev_pool): contexts
    created, run and destroyed back to back on two streams, with a larger context (N = 256,
    relabel engine, bigger buffers) in between, reuse released buffers and every run still
    reproduces the oracle's trajectory; qap_trim_memory hands the pool back."""
    A, B, p0, cfg = config(1)
    I = cfg["iters"]
    sch = O.geometric_schedule_for(A, B, p0, I)
    o = None
    Ab, Bb = grey_density(256)
    pb = start_perm(256, 5, 0)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for rep in range(6):
        st = streams[rep % 2]
        with Q.Solver(A, B, p0, stream=st.cuda_stream) as s:
            s.delta_init()
            g = s.run(0, I, _sched(sch), SA_SEED)
            n_near, near = s.near_ties()
            if o is None:
                o = O.Run(A, B, p0).run(0, I, sch, SA_SEED, follow=near)
            assert (g["cost"], g["best_cost"], g["accepted"], g["digest"]) == (
                o["cost"], o["best_cost"], o["accepted"], o["digest"]), rep
        if rep == 2:
            with Q.Solver(Ab, Bb, pb, stream=st.cuda_stream) as s:
                s.delta_init()
                s.run(0, 20000, _sched(O.geometric_schedule_for(Ab, Bb, pb, 20000)), SA_SEED)
                assert s.cost() == O.cost(Ab, Bb, s.state()[0])
    Q.qap_trim_memory(0)
    with pytest.raises(Q.QapError):
        Q.qap_trim_memory(-1)
