"""Seeded synthetic inputs shared by the oracle tests, the CUDA tests and bench.py.

This module holds NO arithmetic of the method (no cost, no delta, no acceptance,
no schedule, no random stream the annealer draws).  It only builds the
*inputs* of a run: an instance (A, B) and a start permutation p0.

Instance family (§4): "the A and B matrices are symmetric with
zero diagonal; the matrix elements are chosen from independent uniform
distributions" -- the Taixxa family of QAPLIB.  BASELINE.json configs 1-3 and 5
fix the support to 0..99.  Config 4 is the "tai256c-shaped" grey-density
instance (sparse 0/1 flow A, large distances B), see DESIGN.md "Input recipe".

Start permutations are keyed by (seed, chain id) so an ensemble's chains do not
depend on how they are split across GPUs.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "taixxa", "grey_density", "block_classes", "start_perm", "start_perms", "config",
    "CONFIGS",
]


def taixxa(n: int, seed: int, lo: int = 0, hi: int = 99):
    """Random symmetric zero-diagonal instance, entries iid uniform on [lo, hi].

    PAPER.md line 105 (§4).  A's strict upper triangle is drawn first, then B's,
    from numpy's PCG64 seeded with `seed`; both are mirrored.
    """
    if n < 2:
        raise ValueError("n >= 2 required")
    rng = np.random.Generator(np.random.PCG64(seed))
    iu = np.triu_indices(n, 1)
    mats = []
    for _ in range(2):
        m = np.zeros((n, n), dtype=np.int32)
        m[iu] = rng.integers(lo, hi + 1, size=iu[0].size, dtype=np.int64).astype(np.int32)
        m = m + m.T
        mats.append(np.ascontiguousarray(m, dtype=np.int32))
    return mats[0], mats[1]


def grey_density(n: int = 256, m: int = 92, side: int = 16):
    """tai256c-shaped instance (BASELINE.json config 4), no randomness.

    A_ij = 1 iff i != j and i < m and j < m (a dense block of ones: the
    grey-density flow pattern, 13% dense at n=256, m=92).
    B_ij = 255 * (side - d_ij)^2 for i != j, d = Manhattan distance of cells i, j
    on a side x side torus (values up to 57375, so B needs 16 bits).
    """
    if side * side != n:
        raise ValueError("n must be side*side")
    A = np.zeros((n, n), dtype=np.int32)
    A[:m, :m] = 1
    np.fill_diagonal(A, 0)
    ij = np.arange(n)
    x, y = ij // side, ij % side
    dx = np.abs(x[:, None] - x[None, :])
    dy = np.abs(y[:, None] - y[None, :])
    dx = np.minimum(dx, side - dx)
    dy = np.minimum(dy, side - dy)
    d = dx + dy
    B = (255 * (side - d) ** 2).astype(np.int32)
    np.fill_diagonal(B, 0)
    return np.ascontiguousarray(A), np.ascontiguousarray(B)


def block_classes(n: int, sizes, seed: int, hi_a: int = 99, hi_b: int = 60000):
    """Instance whose flow matrix A has twin locations (R21), like config 4.

    Locations are labelled: the first sizes[0] locations class 0, the next sizes[1] class 1, ...,
    every remaining location its own label; the labels are then shuffled over the locations.
    A_xy = V[label x][label y] (x != y) for a random symmetric V uniform on 0..hi_a, so all
    members of a class have equal rows off the pair.  B is symmetric, zero diagonal, uniform
    on 0..hi_b (16-bit when hi_b > 255).  numpy PCG64(seed).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    labels = []
    for c, m in enumerate(sizes):
        labels += [c] * m
    nl = len(sizes)
    labels += list(range(nl, nl + n - len(labels)))
    labels = rng.permutation(np.array(labels, dtype=np.int64))
    L = int(labels.max()) + 1
    V = rng.integers(0, hi_a + 1, size=(L, L), dtype=np.int64)
    V = np.triu(V) + np.triu(V, 1).T
    A = V[labels[:, None], labels[None, :]].astype(np.int32)
    np.fill_diagonal(A, 0)
    iu = np.triu_indices(n, 1)
    B = np.zeros((n, n), dtype=np.int32)
    B[iu] = rng.integers(0, hi_b + 1, size=iu[0].size, dtype=np.int64).astype(np.int32)
    B = B + B.T
    return np.ascontiguousarray(A), np.ascontiguousarray(B)


def start_perm(n: int, seed: int, chain: int = 0) -> np.ndarray:
    """Start permutation p0 of chain `chain`: a uniform shuffle keyed by (seed, chain)."""
    rng = np.random.Generator(np.random.PCG64([seed, chain]))
    return rng.permutation(n).astype(np.int32)


def start_perms(n: int, seed: int, chain_begin: int, count: int) -> np.ndarray:
    """Start permutations of global chains [chain_begin, chain_begin+count), shape (count, n)."""
    out = np.empty((count, n), dtype=np.int32)
    for i in range(count):
        out[i] = start_perm(n, seed, chain_begin + i)
    return out


# BASELINE.json "configs", in order.  iters = SA iterations per chain.
CONFIGS = {
    1: dict(name="tai12a-shaped", kind="taixxa", n=12, inst_seed=12, iters=10**5, chains=1),
    2: dict(name="tai50a-shaped", kind="taixxa", n=50, inst_seed=50, iters=10**7, chains=1),
    3: dict(name="tai100a-shaped", kind="taixxa", n=100, inst_seed=100, iters=10**8, chains=1),
    4: dict(name="tai256c-shaped", kind="grey", n=256, inst_seed=0, iters=10**9, chains=1),
    5: dict(name="ensemble-tai100a-shaped", kind="taixxa", n=100, inst_seed=100, iters=10**7,
            chains=8192),
}
SA_SEED = 42


def config(c: int):
    """(A, B, p0 of chain 0, cfg dict) for BASELINE.json config number c (1-based)."""
    cfg = dict(CONFIGS[c])
    if cfg["kind"] == "taixxa":
        A, B = taixxa(cfg["n"], cfg["inst_seed"])
    else:
        A, B = grey_density(cfg["n"])
    p0 = start_perm(cfg["n"], SA_SEED, 0)
    return A, B, p0, cfg
