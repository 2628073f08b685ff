"""Dev probe driver: TS-mode (A in TMEM) int8 MMA check and timings (not part of the product)."""
import ctypes, os
import numpy as np
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcprobe3.so"))
rng = np.random.default_rng(3)
A = rng.integers(0, 256, size=(128, 128), dtype=np.uint8)
B = rng.integers(0, 256, size=(16, 128), dtype=np.uint8)
D = np.zeros((128, 16), dtype=np.int32)
out = np.zeros(8, dtype=np.int64)
p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
rc = lib.probe3_run(p(A), p(B), p(D), p(out))
ref = A.astype(np.int64) @ B.astype(np.int64).T
print("rc", rc, "TS match", bool((D == ref).all()))
if not (D == ref).all():
    print("D[0,:4]", D[0, :4].tolist(), "ref", ref[0, :4].tolist(), "mismatch", int((D != ref).sum()))
for n, v in zip(["4x TS 128x16x32", "8x TS (2 chains)", "rank TS 128x128x32", "rank TS + 8 TS", "8 indep TS N=16", "8 indep TS N=8", "1 TS N=16", "rank + 8 indep"], out):
    print(f"{n:24s} {v:6d} cycles")
