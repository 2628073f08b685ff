"""QAPLIB instance and solution files: plain-text readers / writers.

QAPLIB's .dat format is whitespace-separated integers: n, then the n x n matrix A (row-major),
then the n x n matrix B; Eq.(1) is sum_ij a_ij b_p(i)p(j).  A .sln file holds
n, the optimal / best known cost and the permutation, 1-based.  Host-side I/O only: the
instance goes to the device through qap_create like any other (no data path here).
"""
from __future__ import annotations

import numpy as np

__all__ = ["read_dat", "write_dat", "read_sln", "write_sln"]


class QaplibError(ValueError):
    """Malformed QAPLIB file; `kind` is SPEC's error class: "parse" (with the token
    position), "size" (n < 2) or "domain" (negative entries)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind} error: {msg}")
        self.kind = kind


def _ints(text: str, path: str) -> list[int]:
    out = []
    for pos, tok in enumerate(text.split()):
        try:
            out.append(int(tok))
        except ValueError:
            raise QaplibError("parse", f"{path}: token {pos} ({tok!r}) is not an integer") from None
    return out


def read_dat(path: str):
    """(A, B) as int32 arrays from a QAPLIB .dat file.  Raises QaplibError (a ValueError) on a
    malformed file: parse errors with the token position, n < 2, negative entries."""
    with open(path) as f:
        vals = _ints(f.read(), path)
    if not vals:
        raise QaplibError("parse", f"{path}: empty file")
    n = vals[0]
    if n < 2:
        raise QaplibError("size", f"{path}: n = {n} < 2")
    if len(vals) != 1 + 2 * n * n:
        raise QaplibError("parse", f"{path}: expected 1 + 2*{n}^2 integers, found {len(vals)}")
    if min(vals[1:]) < 0:
        raise QaplibError("domain", f"{path}: negative entry")
    A = np.array(vals[1:1 + n * n], dtype=np.int64).reshape(n, n)
    B = np.array(vals[1 + n * n:], dtype=np.int64).reshape(n, n)
    if A.min() < np.iinfo(np.int32).min or A.max() > np.iinfo(np.int32).max or \
            B.min() < np.iinfo(np.int32).min or B.max() > np.iinfo(np.int32).max:
        raise ValueError(f"{path}: entries outside int32")
    return np.ascontiguousarray(A, dtype=np.int32), np.ascontiguousarray(B, dtype=np.int32)


def write_dat(path: str, A, B) -> None:
    A = np.asarray(A)
    B = np.asarray(B)
    n = A.shape[0]
    if A.shape != (n, n) or B.shape != (n, n):
        raise ValueError("A and B must be n x n")
    with open(path, "w") as f:
        f.write(f"{n}\n\n")
        for M in (A, B):
            for row in M:
                f.write(" ".join(str(int(x)) for x in row) + "\n")
            f.write("\n")


def read_sln(path: str):
    """(n, cost, p) from a QAPLIB .sln file; p is returned 0-based (int32)."""
    with open(path) as f:
        vals = _ints(f.read(), path)
    if len(vals) < 2:
        raise ValueError(f"{path}: expected n and the cost")
    n, cost = vals[0], vals[1]
    perm = vals[2:]
    if len(perm) != n or sorted(perm) != list(range(1, n + 1)):
        raise ValueError(f"{path}: not a 1-based permutation of 1..{n}")
    return n, cost, np.array(perm, dtype=np.int32) - 1


def write_sln(path: str, cost: int, p) -> None:
    p = np.asarray(p)
    with open(path, "w") as f:
        f.write(f"{len(p)} {int(cost)}\n")
        f.write(" ".join(str(int(x) + 1) for x in p) + "\n")
