"""ctypes wrapper of the C oracle (oracle/qap_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_1208_2675_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

MODE_EQ1, MODE_SCRATCH, MODE_DELTA = 0, 1, 2
COOL_GEOMETRIC, COOL_LUNDY_MEES = 0, 1

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (make) if missing or stale."""
    src = os.path.join(_HERE, "qap_oracle.c")
    hdr = os.path.join(_HERE, "qap_oracle.h")
    stale = (not os.path.exists(_LIB_PATH)) or any(
        os.path.getmtime(f) > os.path.getmtime(_LIB_PATH) for f in (src, hdr))
    if force or stale:
        subprocess.run(["make", "-s", "-C", _HERE, "-B" if force else "liboracle.so"], check=True)
    return _LIB_PATH


class _State(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("mode", C.c_int32),
        ("A", C.c_void_p), ("B", C.c_void_p), ("p", C.c_void_p), ("best_p", C.c_void_p),
        ("Bp", C.c_void_p), ("D", C.c_void_p),
        ("cost", C.c_int64), ("best_cost", C.c_int64),
        ("digest", C.c_uint64), ("accepted", C.c_uint64), ("near_ties", C.c_uint64),
        ("iterations", C.c_uint64), ("proposal", C.c_int32), ("pad", C.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.orc_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.orc_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_uniform.restype = C.c_double
        L.orc_temperature.argtypes = [C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_uint64]
        L.orc_temperature.restype = C.c_double
        L.orc_cost.argtypes = [C.c_int, _i32p, _i32p, _i32p]
        L.orc_cost.restype = C.c_int64
        L.orc_bprime.argtypes = [C.c_int, _i32p, _i32p, _i32p]
        L.orc_delta_eq1.argtypes = [C.c_int, _i32p, _i32p, _i32p, C.c_int, C.c_int]
        L.orc_delta_eq1.restype = C.c_int64
        L.orc_delta_scratch.argtypes = [C.c_int, _i32p, _i32p, C.c_int, C.c_int]
        L.orc_delta_scratch.restype = C.c_int64
        L.orc_delta_init.argtypes = [C.c_int, _i32p, _i32p, _i64p]
        L.orc_pair.argtypes = [C.c_int, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.orc_index.argtypes = [C.c_int, C.c_int, C.c_int]
        L.orc_index.restype = C.c_int64
        L.orc_apply_swap.argtypes = [C.c_int, _i32p, _i32p, C.c_int, C.c_int]
        L.orc_update_delta.argtypes = [C.c_int, _i32p, _i32p, _i32p, C.c_int, C.c_int, _i64p]
        L.orc_temperature_bounds.argtypes = [C.c_int, _i64p, C.POINTER(C.c_double),
                                             C.POINTER(C.c_double)]
        L.orc_bruteforce.argtypes = [C.c_int, _i32p, _i32p, _i32p]
        L.orc_bruteforce.restype = C.c_int64
        L.orc_state_reset.argtypes = [C.POINTER(_State), _i32p]
        L.orc_sa_run.argtypes = [
            C.POINTER(_State), C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double,
            C.c_uint64, C.c_uint64, C.c_uint32,
            C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int64]
        L.orc_sa_run.restype = C.c_int
        L.orc_ensemble_run.argtypes = [C.c_int, _i32p, _i32p, C.c_void_p, C.c_int64, C.c_uint32,
                                       C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                       C.c_int, C.c_int, _i64p, C.c_void_p, C.c_void_p, C.c_int]
        L.orc_start_perm.argtypes = [C.c_int, C.c_uint64, C.c_uint32, _i32p]
        L.orc_ensemble_run.restype = C.c_int
        _lib = L
    return _lib


def _i32(x):
    return np.ascontiguousarray(x, dtype=np.int32)


# ---- qap-core -------------------------------------------------------------

def philox4x32_10(ctr, key):
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def uniform(seed, k, chain=0, tag=0):
    return lib().orc_uniform(seed, k, chain, tag)


def temperature(kind, t0, tf, total, k):
    return lib().orc_temperature(kind, t0, tf, total, k)


def cost(A, B, p):
    A = _i32(A)
    return int(lib().orc_cost(A.shape[0], A, _i32(B), _i32(p)))


def bprime(B, p):
    B = _i32(B)
    out = np.zeros_like(B)
    lib().orc_bprime(B.shape[0], B, _i32(p), out)
    return out


def delta_eq1(A, B, p, r, s):
    A = _i32(A)
    return int(lib().orc_delta_eq1(A.shape[0], A, _i32(B), _i32(p), r, s))


def delta_scratch(A, Bp, r, s):
    A = _i32(A)
    return int(lib().orc_delta_scratch(A.shape[0], A, _i32(Bp), r, s))


def delta_init(A, Bp):
    A = _i32(A)
    n = A.shape[0]
    D = np.zeros(n * (n - 1) // 2, np.int64)
    lib().orc_delta_init(n, A, _i32(Bp), D)
    return D


def pair(n, q):
    r, s = C.c_int32(), C.c_int32()
    lib().orc_pair(n, q, C.byref(r), C.byref(s))
    return r.value, s.value


def index(n, r, s):
    return int(lib().orc_index(n, r, s))


def apply_swap(p, Bp, r, s):
    """In place on int32 arrays p (n) and Bp (n,n)."""
    lib().orc_apply_swap(p.shape[0], p, Bp, r, s)


def update_delta(A, Bp_pre, Bp_post, r, s, D):
    A = _i32(A)
    lib().orc_update_delta(A.shape[0], A, _i32(Bp_pre), _i32(Bp_post), r, s, D)


def temperature_bounds(D, n):
    t0, tf = C.c_double(), C.c_double()
    lib().orc_temperature_bounds(n, np.ascontiguousarray(D, np.int64), C.byref(t0), C.byref(tf))
    return t0.value, tf.value


def bruteforce(A, B):
    A = _i32(A)
    bp = np.zeros(A.shape[0], np.int32)
    c = lib().orc_bruteforce(A.shape[0], A, _i32(B), bp)
    return int(c), bp


# ---- annealer -------------------------------------------------------------

@dataclass
class Schedule:
    kind: int
    t0: float
    tf: float
    total_iters: int


@dataclass
class Run:
    """Sequential SA chain with owned buffers."""
    A: np.ndarray
    B: np.ndarray
    p0: np.ndarray
    mode: int = MODE_DELTA
    chain: int = 0
    near_log: list = field(default_factory=list)
    proposal: int = 0          # 0 sequential enumeration (R4), 1 random pairs (R22)

    def __post_init__(self):
        self.A = _i32(self.A)
        self.B = _i32(self.B)
        n = self.A.shape[0]
        self.n = n
        self.p = np.zeros(n, np.int32)
        self.best_p = np.zeros(n, np.int32)
        self.Bp = np.zeros((n, n), np.int32)
        self.D = np.zeros(max(1, n * (n - 1) // 2), np.int64)
        self.st = _State()
        self.st.n, self.st.mode, self.st.proposal = n, self.mode, self.proposal
        for name, arr in (("A", self.A), ("B", self.B), ("p", self.p), ("best_p", self.best_p),
                          ("Bp", self.Bp), ("D", self.D)):
            setattr(self.st, name, arr.ctypes.data)
        lib().orc_state_reset(C.byref(self.st), _i32(self.p0))

    def run(self, k0, iters, sched: Schedule, seed, follow=None, check_every=0, near_cap=1024):
        fk = fd = None
        nf = 0
        if follow:
            fk = np.array([k for k, _ in follow], np.uint64)
            fd = np.array([int(d) for _, d in follow], np.uint8)
            nf = len(follow)
        nk = np.zeros(near_cap, np.uint64)
        nd = np.zeros(near_cap, np.uint8)
        rc = lib().orc_sa_run(
            C.byref(self.st), k0, iters, sched.kind, sched.t0, sched.tf, sched.total_iters,
            seed, self.chain,
            fk.ctypes.data if fk is not None else None, fd.ctypes.data if fd is not None else None,
            nf, nk.ctypes.data, nd.ctypes.data, near_cap, check_every)
        if rc < 0:
            raise AssertionError("oracle invariant check failed (B', C or Δ)")
        self.near_log += [(int(nk[i]), int(nd[i])) for i in range(rc)]
        return self.stats()

    def stats(self):
        s = self.st
        return dict(cost=s.cost, best_cost=s.best_cost, digest=s.digest, accepted=s.accepted,
                    near_ties=s.near_ties, iterations=s.iterations)


def start_perm(n, seed, chain):
    """Chain-keyed Fisher-Yates start permutation (R14b)."""
    p = np.zeros(n, np.int32)
    lib().orc_start_perm(n, seed, chain, p)
    return p


def ensemble_run(A, B, p0s, chain_base, iters, sched: Schedule, seed, threads=None,
                 mode=MODE_DELTA, count=None, near_cap=0):
    """Per-chain results (count, 6): cost, best_cost, accepted, near_ties, digest, iterations.
    p0s None: chain c starts from start_perm(n, seed, c) (then `count` is required).
    near_cap > 0: also returns the per-chain near-tie logs, a list of [(k, decision), ...]."""
    A = _i32(A)
    n = A.shape[0]
    if p0s is not None:
        p0s = _i32(p0s)
        count = p0s.shape[0]
    out = np.zeros((count, 6), np.int64)
    nk = np.zeros(max(1, count * near_cap), np.uint64)
    nd = np.zeros(max(1, count * near_cap), np.uint8)
    threads = threads or os.cpu_count() or 1
    lib().orc_ensemble_run(n, A, _i32(B), p0s.ctypes.data if p0s is not None else None, count,
                           chain_base, iters, sched.kind, sched.t0, sched.tf, seed, threads, mode,
                           out, nk.ctypes.data if near_cap else None,
                           nd.ctypes.data if near_cap else None, near_cap)
    if not near_cap:
        return out
    logs = []
    for c in range(count):
        m = min(int(out[c, 3]), near_cap)
        logs.append([(int(nk[c * near_cap + i]), int(nd[c * near_cap + i])) for i in range(m)])
    return out, logs


def geometric_schedule_for(A, B, p0, total_iters):
    """DESIGN.md R1 + R2: geometric schedule with T0/Tf from Δ at p0 (all pairs)."""
    D = delta_init(A, bprime(B, p0))
    t0, tf = temperature_bounds(D, np.asarray(A).shape[0])
    return Schedule(COOL_GEOMETRIC, t0, tf, total_iters)
