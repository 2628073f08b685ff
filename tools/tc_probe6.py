"""Dev probe driver: TMEM block read throughput (not part of the product)."""
import ctypes, os
import numpy as np
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcprobe6.so"))
out = np.zeros(8, dtype=np.int64)
print("rc", lib.probe6_run(out.ctypes.data_as(ctypes.c_void_p)))
for nm, v in zip(["1 warp: 4 x ld32 (16 KB)", "4 warps: 4 x ld32 each (64 KB)", "8 warps: 4 x ld32 each (128 KB)",
                  "1 warp: 4-chunk RMW", "1 warp: 1 ld32 + wait"], out):
    print(f"{nm:36s} {v:6d} cycles")
