"""Multi-process (gloo, world_size 2, CPU) tests of the ensemble driver's host
logic: chain partition, min-reduce of (cost, chain), owner broadcast of the
permutation, summed statistics, and independence from the number of ranks.
The per-rank chain runner is the oracle here (no GPU in this container)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from paper_1208_2675_b200.dist import chain_range, ensemble_distributed
from qap_inputs import start_perms, taixxa

N, CHAINS, ITERS, SEED = 12, 9, 4000, 7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_runner(A, B, begin, p0s, iters, sched, seed, count):
    if p0s is None:                       # chain-keyed start permutations (R14b)
        p0s = np.stack([O.start_perm(len(A), seed, begin + i) for i in range(count)])
    out = O.ensemble_run(A, B, p0s, begin, iters, sched, seed, threads=2)
    i = int(np.lexsort((np.arange(len(out)), out[:, 1]))[0])
    st = O.Run(A, B, p0s[i], chain=begin + i)
    st.run(0, iters, sched, seed)
    return dict(best_cost=int(out[i, 1]), best_chain=begin + i, best_perm=st.best_p.copy(),
                stats=dict(iterations=int(out[:, 5].sum()), accepted=int(out[:, 2].sum()),
                           near_ties=int(out[:, 3].sum())))


def _worker(rank, world, port, q, keyed=False):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, B = taixxa(N, 3)
    sch = O.geometric_schedule_for(A, B, start_perms(N, SEED, 0, 1)[0], ITERS)
    res = ensemble_distributed(A, B, CHAINS, ITERS, sch, SEED,
                               p0_fn=None if keyed else (lambda b, c: start_perms(N, SEED, b, c)),
                               local_runner=oracle_runner, device="cpu")
    q.put((rank, res.best_cost, res.best_chain, res.best_perm.tolist(), res.iterations,
           res.accepted, res.near_ties))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, keyed=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, keyed)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_chain_range_partitions():
    for chains in (1, 5, 9, 8192):
        for world in (1, 2, 3, 4, 8, 16):
            got = [chain_range(r, world, chains) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == chains
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [e - b for b, e in got]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_matches_single_process():
    A, B = taixxa(N, 3)
    p0s = start_perms(N, SEED, 0, CHAINS)
    sch = O.geometric_schedule_for(A, B, p0s[0], ITERS)
    ref = O.ensemble_run(A, B, p0s, 0, ITERS, sch, SEED, threads=2)
    best = int(np.lexsort((np.arange(CHAINS), ref[:, 1]))[0])
    out = _run(2)
    for rank, cost, chain, perm, its, acc, near in out:
        assert cost == ref[best, 1] and chain == best
        assert O.cost(A, B, perm) == cost
        assert its == CHAINS * ITERS and acc == int(ref[:, 2].sum()) and near == int(ref[:, 3].sum())
    # every rank holds the same (broadcast) permutation
    assert out[0][3] == out[1][3]


def test_gloo_world3_more_ranks_than_share():
    out2 = _run(2)
    out3 = _run(3)
    assert [o[1:] for o in out2][0] == [o[1:] for o in out3][0]


def test_gloo_world2_chain_keyed_start_perms():
    """p0_fn = None: every rank's chains start from the chain-keyed permutations (R14b), so the
    result equals one process running all chains from O.start_perm."""
    A, B = taixxa(N, 3)
    p0s = np.stack([O.start_perm(N, SEED, c) for c in range(CHAINS)])
    sch = O.geometric_schedule_for(A, B, start_perms(N, SEED, 0, 1)[0], ITERS)
    ref = O.ensemble_run(A, B, p0s, 0, ITERS, sch, SEED, threads=2)
    best = int(np.lexsort((np.arange(CHAINS), ref[:, 1]))[0])
    out = _run(2, keyed=True)
    for rank, cost, chain, perm, its, acc, near in out:
        assert cost == ref[best, 1] and chain == best and O.cost(A, B, perm) == cost
        assert acc == int(ref[:, 2].sum())


def test_overflow_is_rejected_before_any_work():
    """The reduction-key bound is checked identically on every rank before the local run (so no
    rank can raise alone and leave the others in a collective)."""
    A = np.full((4, 4), 60000, np.int64) - np.diag([60000] * 4)
    called = []
    with pytest.raises(OverflowError):
        ensemble_distributed(A, A, 2**40, 10, None, 1, local_runner=lambda *a: called.append(1),
                             device="cpu")
    assert not called


def test_bench_self_launches_two_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun relaunches itself with two ranks (torch.distributed.run,
    127.0.0.1 rendezvous); --dry-run drives the host path (rank environment, chain partition,
    the ensemble driver's gloo collectives) without a GPU and rank 0 prints one JSON line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run",
                          "--ens-chains", "9"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["rank0_chains"] == [0, 5] and d["chains"] == 9
