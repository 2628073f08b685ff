"""Dev probe driver: parallel vs single-thread MMA issue (not part of the product)."""
import ctypes, os
import numpy as np
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcprobe5.so"))
out = np.zeros(8, dtype=np.int64)
print("rc", lib.probe5_run(out.ctypes.data_as(ctypes.c_void_p)))
for nm, v in zip(["1 thread: rank + 8 touch, wait", "4 warps x (2 touch) + rank, wait", "1 thread: issue only (9)",
                  "1 thread: issue + wait (9)", "rank only SS"], out):
    print(f"{nm:36s} {v:6d} cycles")
