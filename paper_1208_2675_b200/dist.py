"""Multi-GPU ensemble driver: independent chains split over ranks, one NCCL
min-reduce of the best cost and permutation (BASELINE config 5; "run
copies of the heuristic independently on each processor").

One process per GPU (torchrun).  Rank g of G runs the chains with GLOBAL ids
[g*C/G, (g+1)*C/G) through qap_ensemble_run on its own device; chain c's start
permutation and random stream depend only on c, so the result does not depend
on G.  The only collectives are, once per run:
  1. all_reduce(MIN) of key = best_cost * C + chain            (8 bytes)
  2. broadcast of the winning permutation from its owner rank   (4 N bytes)
  3. all_reduce(SUM) of (iterations, accepted, near_ties)        (24 bytes)
There is no data-path collective: chains never exchange state.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


def chain_range(rank: int, world: int, chains: int):
    """Global chain ids [begin, end) of a rank: contiguous, balanced, covering 0..chains-1."""
    per, extra = divmod(chains, world)
    begin = rank * per + min(rank, extra)
    return begin, begin + per + (1 if rank < extra else 0)


@dataclass
class EnsembleResult:
    best_cost: int
    best_chain: int
    best_perm: np.ndarray
    iterations: int
    accepted: int
    near_ties: int
    local: dict


def ensemble_distributed(A, B, chains: int, iters: int, schedule, seed: int,
                         p0_fn: Optional[Callable[[int, int], np.ndarray]] = None,
                         local_runner: Optional[Callable] = None,
                         group=None, device=None) -> EnsembleResult:
    """Run `chains` independent chains of `iters` iterations across the ranks of `group`.

    p0_fn(begin, count) -> (count, n) int32 start permutations of global chains
    [begin, begin+count); None = the chain-keyed start permutations (R14b), which
    qap_ensemble_run generates on the device.  local_runner(A, B, begin, p0s, iters, schedule,
    seed, count) -> dict with best_cost, best_chain (global id), best_perm,
    stats{iterations, accepted, near_ties}; defaults to qap_ensemble_run on this rank's device.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    begin, end = chain_range(rank, world, chains)
    n = int(np.asarray(A).shape[0])
    if local_runner is None:
        local_runner = _gpu_runner(device)
    INT64_MAX = (1 << 63) - 1
    # Eq.(1) <= sum(A) * max(B) for every permutation: checked identically on every rank before
    # any work, so no rank can fail alone and leave the others waiting in a collective
    bound = int(np.asarray(A, np.int64).sum()) * int(np.asarray(B, np.int64).max(initial=0))
    if bound * chains + chains > INT64_MAX:
        raise OverflowError("best_cost * chains could overflow the int64 reduction key")
    if end > begin:
        p0s = p0_fn(begin, end - begin) if p0_fn is not None else None
        res = local_runner(A, B, begin, p0s, iters, schedule, seed, end - begin)
        key0 = int(res["best_cost"]) * chains + int(res["best_chain"])
    else:                                   # more ranks than chains: this rank is idle
        res = dict(best_cost=None, best_chain=-1, best_perm=np.zeros(n, np.int32),
                   stats=dict(iterations=0, accepted=0, near_ties=0))
        key0 = INT64_MAX
    if device is None:
        dev = torch.device("cuda", torch.cuda.current_device()) if (
            dist.is_initialized() and dist.get_backend(group) == "nccl") else torch.device("cpu")
    else:
        dev = torch.device(device)
    key = torch.tensor([key0], dtype=torch.int64, device=dev)
    perm = torch.as_tensor(np.asarray(res["best_perm"], np.int32), device=dev)
    st = res["stats"]
    sums = torch.tensor([int(st["iterations"]), int(st["accepted"]), int(st["near_ties"])],
                        dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
        best_chain = int(key.item()) % chains
        owner = torch.tensor([rank if int(res["best_chain"]) == best_chain else world],
                             dtype=torch.int64, device=dev)
        dist.all_reduce(owner, op=dist.ReduceOp.MIN, group=group)
        src = int(owner.item())
        dist.broadcast(perm, src=dist.get_global_rank(group, src) if group is not None else src,
                       group=group)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    best_cost, best_chain = divmod(int(key.item()), chains)
    s = sums.cpu().tolist()
    return EnsembleResult(best_cost, best_chain, perm.cpu().numpy().astype(np.int32), s[0], s[1],
                          s[2], res)


def _gpu_runner(device):
    def run(A, B, begin, p0s, iters, schedule, seed, count):
        import torch
        from . import qapsa as Q
        dev = torch.cuda.current_device() if device is None else torch.device(device).index
        n = int(np.asarray(A).shape[0])
        ctx_p0 = p0s[0] if p0s is not None else np.arange(n, dtype=np.int32)   # not used by the ensemble
        with Q.Solver(A, B, ctx_p0, device=dev,
                      stream=torch.cuda.current_stream().cuda_stream) as s:
            return s.ensemble(begin, p0s, iters, schedule, seed, count=count)
    return run
