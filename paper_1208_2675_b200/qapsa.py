"""Thin ctypes binding of libqapsa (include/qapsa.h), same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  There is no CPU fallback; if the shared library is
missing or no sm_100 device is present the calls raise QapError.
PyTorch is used only to pass the current CUDA stream (plumbing).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QAPSA_LIB") or os.path.join(_PKG, "libqapsa.so")

QAP_OK = 0
STATUS = {0: "QAP_OK", 1: "QAP_E_INVALID_ARG", 2: "QAP_E_DIMENSION", 3: "QAP_E_UNSUPPORTED",
          4: "QAP_E_OVERFLOW", 5: "QAP_E_SCHEDULE", 6: "QAP_E_STATE", 7: "QAP_E_CUDA",
          9: "QAP_E_NOMEM"}
QAP_COOL_GEOMETRIC, QAP_COOL_LUNDY_MEES = 0, 1
QAP_OPT_WINDOW_MAX, QAP_OPT_THREADS, QAP_OPT_FORCE_GLOBAL_DELTA, QAP_OPT_ENSEMBLE_GROUP = 1, 2, 3, 4
QAP_OPT_TENSOR_CORE = 5
QAP_OPT_SCRATCH_PHASE = 6
QAP_OPT_RELABEL = 7
QAP_OPT_RELABEL_CLUSTER = 8
QAP_OPT_CLUSTER_ENGINE = 10
QAP_OPT_ENSEMBLE_SCRATCH4 = 11
QAP_OPT_SWITCH_GAP = 12
QAP_OPT_PROPOSAL = 9
QAP_ENGINE_SHARED_MEMORY, QAP_ENGINE_TENSOR_MEMORY, QAP_ENGINE_RELABEL, QAP_ENGINE_CLUSTER = 0, 1, 2, 3
QAP_NEAR_LOG_CAP = 1024
QAP_ENS_NEAR_LOG_CAP = 65536

# Every symbol include/qapsa.h declares (checked by tests/test_abi.py).
EXPORTS = ("qap_create", "qap_destroy", "qap_trim_memory", "qap_reset", "qap_delta_init", "qap_sa_run", "qap_cost",
           "qap_get_state", "qap_get_near_ties", "qap_schedule_bounds", "qap_ensemble_run",
           "qap_ensemble_near_ties", "qap_start_perms",
           "qap_set_option", "qap_uses_tensor_core", "qap_engine", "qap_last_kernel_time", "qap_last_scratch_time",
           "qap_status_str",
           "qap_last_error", "qap_version")


class QapError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class qap_schedule(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("t0", C.c_double),
                ("tf", C.c_double), ("total_iters", C.c_uint64)]


class qap_stats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("accepted", C.c_uint64), ("near_ties", C.c_uint64),
                ("cost", C.c_int64), ("best_cost", C.c_int64), ("digest", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class qap_chain_result(C.Structure):
    _fields_ = [("cost", C.c_int64), ("best_cost", C.c_int64), ("accepted", C.c_uint64),
                ("near_ties", C.c_uint64), ("digest", C.c_uint64), ("iterations", C.c_uint64)]


_lib = None


def lib(build_if_missing: bool = True):
    """Load libqapsa.so (building it with nvcc if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and "QAPSA_LIB" not in os.environ:
        from . import _build
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise QapError(7, f"{LIB_PATH} missing (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32p = C.c_void_p, C.POINTER(C.c_int32)
    L.qap_create.argtypes = [C.c_int32, i32p, i32p, i32p, C.c_int32, vp, C.POINTER(vp)]
    L.qap_destroy.argtypes = [vp]
    L.qap_destroy.restype = None
    L.qap_trim_memory.argtypes = [C.c_int32]
    L.qap_reset.argtypes = [vp, i32p]
    L.qap_delta_init.argtypes = [vp]
    L.qap_sa_run.argtypes = [vp, C.c_uint64, C.c_uint64, C.POINTER(qap_schedule), C.c_uint64,
                             C.POINTER(qap_stats)]
    L.qap_cost.argtypes = [vp, i32p, C.POINTER(C.c_int64)]
    L.qap_get_state.argtypes = [vp, i32p, i32p, i32p]
    L.qap_get_near_ties.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint8), C.c_int32,
                                    i32p]
    L.qap_schedule_bounds.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.qap_ensemble_run.argtypes = [vp, C.c_uint32, C.c_uint32, i32p, C.c_uint64,
                                   C.POINTER(qap_schedule), C.c_uint64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_uint32), i32p, C.POINTER(qap_stats),
                                   C.POINTER(qap_chain_result)]
    L.qap_ensemble_near_ties.argtypes = [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint8), C.c_int32, i32p]
    L.qap_start_perms.argtypes = [vp, C.c_uint64, C.c_uint32, C.c_uint32, i32p]
    L.qap_set_option.argtypes = [vp, C.c_int32, C.c_int64]
    L.qap_last_kernel_time.argtypes = [vp, C.POINTER(C.c_float), i32p]
    L.qap_last_scratch_time.argtypes = [vp, C.POINTER(C.c_float), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.qap_status_str.argtypes = [C.c_int]
    L.qap_status_str.restype = C.c_char_p
    L.qap_last_error.argtypes = [vp]
    L.qap_last_error.restype = C.c_char_p
    L.qap_version.restype = C.c_int32
    L.qap_uses_tensor_core.argtypes = [vp]
    L.qap_uses_tensor_core.restype = C.c_int32
    L.qap_engine.argtypes = [vp]
    L.qap_engine.restype = C.c_int32
    for name in EXPORTS:
        if name not in ("qap_destroy", "qap_status_str", "qap_last_error", "qap_version",
                        "qap_uses_tensor_core", "qap_engine"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def _check(st, ctx=None):
    if st != QAP_OK:
        msg = lib().qap_last_error(ctx).decode(errors="replace")
        raise QapError(st, msg)


def make_schedule(kind, t0, tf, total_iters) -> qap_schedule:
    return qap_schedule(int(kind), 0, float(t0), float(tf), int(total_iters))


def _stream_ptr(stream):
    if stream is not None:
        return C.c_void_p(int(stream))
    try:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:
        pass
    return C.c_void_p(0)


# ---- same names as the C ABI ------------------------------------------------

def qap_create(A, B, p0, device: int = 0, stream=None):
    """Returns an opaque ctx handle (c_void_p).  A, B: (n,n) ints; p0: (n,) ints."""
    A, pA = _i32(A)
    B, pB = _i32(B)
    p0, pp = _i32(p0)
    n = A.shape[0]
    out = C.c_void_p()
    _check(lib().qap_create(n, pA, pB, pp, device, _stream_ptr(stream), C.byref(out)))
    return out


def qap_destroy(ctx):
    lib().qap_destroy(ctx)


def qap_trim_memory(device=0):
    """Return the unused part of the library's device pool on `device` to the driver."""
    _check(lib().qap_trim_memory(device))


def qap_reset(ctx, perm=None):
    if perm is None:
        _check(lib().qap_reset(ctx, None), ctx)
    else:
        perm, pp = _i32(perm)
        _check(lib().qap_reset(ctx, pp), ctx)


def qap_delta_init(ctx):
    _check(lib().qap_delta_init(ctx), ctx)


def qap_sa_run(ctx, k0, iters, schedule: qap_schedule, seed) -> dict:
    st = qap_stats()
    _check(lib().qap_sa_run(ctx, k0, iters, C.byref(schedule), seed, C.byref(st)), ctx)
    return st.as_dict()


def qap_cost(ctx, perm=None) -> int:
    out = C.c_int64()
    if perm is None:
        _check(lib().qap_cost(ctx, None, C.byref(out)), ctx)
    else:
        perm, pp = _i32(perm)
        _check(lib().qap_cost(ctx, pp, C.byref(out)), ctx)
    return out.value


def qap_get_state(ctx, n, want_delta=True):
    p = np.zeros(n, np.int32)
    bp = np.zeros(n, np.int32)
    D = np.zeros(max(1, n * (n - 1) // 2), np.int32) if want_delta else None
    _check(lib().qap_get_state(ctx, _i32(p)[1], _i32(bp)[1],
                               D.ctypes.data_as(C.POINTER(C.c_int32)) if want_delta else None), ctx)
    return p, bp, D


def qap_get_near_ties(ctx, cap=QAP_NEAR_LOG_CAP):
    ks = np.zeros(max(cap, 1), np.uint64)
    ds = np.zeros(max(cap, 1), np.uint8)
    cnt = C.c_int32()
    _check(lib().qap_get_near_ties(ctx, ks.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   ds.ctypes.data_as(C.POINTER(C.c_uint8)), cap, C.byref(cnt)), ctx)
    m = min(cnt.value, cap)
    return cnt.value, sorted((int(ks[i]), int(ds[i])) for i in range(m))


def qap_schedule_bounds(ctx):
    t0, tf = C.c_double(), C.c_double()
    _check(lib().qap_schedule_bounds(ctx, C.byref(t0), C.byref(tf)), ctx)
    return t0.value, tf.value


def qap_ensemble_run(ctx, chain_begin, p0s, iters, schedule: qap_schedule, seed,
                     per_chain: bool = False, count=None, n=None):
    """p0s: (count, n) start permutations, or None for the device's chain-keyed ones (then
    count and n are required)."""
    if p0s is None:
        pp = None
    else:
        p0s, pp = _i32(p0s)
        count, n = p0s.shape
    best_cost, best_chain = C.c_int64(), C.c_uint32()
    best_perm = np.zeros(n, np.int32)
    st = qap_stats()
    res = (qap_chain_result * count)() if per_chain else None
    _check(lib().qap_ensemble_run(ctx, chain_begin, count, pp, iters, C.byref(schedule), seed,
                                  C.byref(best_cost), C.byref(best_chain), _i32(best_perm)[1],
                                  C.byref(st), res), ctx)
    out = dict(best_cost=best_cost.value, best_chain=best_chain.value, best_perm=best_perm,
               stats=st.as_dict())
    if per_chain:
        out["per_chain"] = [{f: getattr(r, f) for f, _ in r._fields_} for r in res]
    return out


def qap_ensemble_near_ties(ctx, cap=QAP_ENS_NEAR_LOG_CAP):
    """(total flagged, sorted [(chain, k, decision), ...]) of the last qap_ensemble_run."""
    ch = np.zeros(max(cap, 1), np.uint32)
    ks = np.zeros(max(cap, 1), np.uint64)
    ds = np.zeros(max(cap, 1), np.uint8)
    cnt = C.c_int32()
    _check(lib().qap_ensemble_near_ties(ctx, ch.ctypes.data_as(C.POINTER(C.c_uint32)),
                                        ks.ctypes.data_as(C.POINTER(C.c_uint64)),
                                        ds.ctypes.data_as(C.POINTER(C.c_uint8)), cap, C.byref(cnt)), ctx)
    m = min(cnt.value, cap)
    return cnt.value, sorted((int(ch[i]), int(ks[i]), int(ds[i])) for i in range(m))


def qap_start_perms(ctx, seed, chain_begin, count, n):
    """(count, n) chain-keyed start permutations, generated on the device."""
    out = np.zeros((count, n), np.int32)
    _check(lib().qap_start_perms(ctx, seed, chain_begin, count, _i32(out)[1]), ctx)
    return out


def qap_set_option(ctx, key, value):
    _check(lib().qap_set_option(ctx, key, value), ctx)


def qap_uses_tensor_core(ctx) -> bool:
    return bool(lib().qap_uses_tensor_core(ctx))


def qap_engine(ctx) -> int:
    """QAP_ENGINE_* of the next qap_sa_run."""
    return int(lib().qap_engine(ctx))


def qap_last_scratch_time(ctx):
    """(ms, iteration reached, swaps accepted) of the last run's scratch phase."""
    ms, kr, acc = C.c_float(), C.c_uint64(), C.c_uint64()
    _check(lib().qap_last_scratch_time(ctx, C.byref(ms), C.byref(kr), C.byref(acc)), ctx)
    return ms.value, kr.value, acc.value


def qap_last_kernel_time(ctx):
    ms, nl = C.c_float(), C.c_int32()
    _check(lib().qap_last_kernel_time(ctx, C.byref(ms), C.byref(nl)), ctx)
    return ms.value, nl.value


def qap_status_str(st) -> str:
    return lib().qap_status_str(st).decode()


def qap_version() -> int:
    return lib().qap_version()


# ---- convenience object -------------------------------------------------------

@dataclass
class Solver:
    """RAII wrapper: one single-chain context on one device."""
    A: np.ndarray
    B: np.ndarray
    p0: np.ndarray
    device: int = 0
    stream: object = None

    def __post_init__(self):
        self.n = int(np.asarray(self.A).shape[0])
        self.ctx = qap_create(self.A, self.B, self.p0, self.device, self.stream)

    def close(self):
        if getattr(self, "ctx", None):
            qap_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def reset(self, perm=None):
        qap_reset(self.ctx, perm)

    def delta_init(self):
        qap_delta_init(self.ctx)

    def run(self, k0, iters, schedule, seed):
        return qap_sa_run(self.ctx, k0, iters, schedule, seed)

    def cost(self, perm=None):
        return qap_cost(self.ctx, perm)

    def state(self, want_delta=True):
        return qap_get_state(self.ctx, self.n, want_delta)

    def near_ties(self):
        return qap_get_near_ties(self.ctx)

    def schedule_bounds(self):
        return qap_schedule_bounds(self.ctx)

    def set_option(self, key, value):
        qap_set_option(self.ctx, key, value)

    def uses_tensor_core(self) -> bool:
        return qap_uses_tensor_core(self.ctx)

    def engine(self) -> int:
        return qap_engine(self.ctx)

    def ensemble(self, chain_begin, p0s, iters, schedule, seed, per_chain=False, count=None):
        return qap_ensemble_run(self.ctx, chain_begin, p0s, iters, schedule, seed, per_chain,
                                count=count, n=self.n)

    def ensemble_near_ties(self):
        return qap_ensemble_near_ties(self.ctx)

    def start_perms(self, seed, chain_begin, count):
        return qap_start_perms(self.ctx, seed, chain_begin, count, self.n)

    def last_kernel_time(self):
        return qap_last_kernel_time(self.ctx)

    def last_scratch_time(self):
        return qap_last_scratch_time(self.ctx)
