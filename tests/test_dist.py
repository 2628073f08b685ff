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


def oracle_runner(A, B, begin, p0s, iters, sched, seed):
    out = O.ensemble_run(A, B, p0s, begin, iters, sched, seed, threads=2)
    i = int(np.lexsort((np.arange(len(out)), out[:, 1]))[0])
    st = O.Run(A, B, p0s[i], chain=begin + i)
    st.run(0, iters, sched, seed)
    return dict(best_cost=int(out[i, 1]), best_chain=begin + i, best_perm=st.best_p.copy(),
                stats=dict(iterations=int(out[:, 5].sum()), accepted=int(out[:, 2].sum()),
                           near_ties=int(out[:, 3].sum())))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, B = taixxa(N, 3)
    sch = O.geometric_schedule_for(A, B, start_perms(N, SEED, 0, 1)[0], ITERS)
    res = ensemble_distributed(A, B, CHAINS, ITERS, sch, SEED,
                               p0_fn=lambda b, c: start_perms(N, SEED, b, c),
                               local_runner=oracle_runner, device="cpu")
    q.put((rank, res.best_cost, res.best_chain, res.best_perm.tolist(), res.iterations,
           res.accepted, res.near_ties))
    dist.barrier()
    dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
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
