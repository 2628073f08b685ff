"""Dev probe driver: checks one int8 tcgen05 MMA against numpy (not part of the product)."""
import ctypes, os, sys
import numpy as np

M, N, K = 128, 16, 128
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcprobe.so"))
rng = np.random.default_rng(1)
A = rng.integers(-128, 128, size=(M, K), dtype=np.int8)
B = rng.integers(-128, 128, size=(N, K), dtype=np.int8)
D = np.zeros((M, N), dtype=np.int32)
cyc = np.zeros(1, dtype=np.int64)
p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
rc = lib.probe_run(p(A), p(B), p(D), p(cyc))
ref = A.astype(np.int64) @ B.astype(np.int64).T
print("rc", rc, "cycles", cyc[0], "match", bool((D == ref).all()))
if not (D == ref).all():
    bad = np.argwhere(D != ref)
    print("mismatches", len(bad), bad[:8].tolist())
    print("D[0,:8]", D[0, :8].tolist(), "ref", ref[0, :8].tolist())
    sys.exit(1)
