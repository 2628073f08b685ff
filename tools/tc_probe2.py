"""Dev probe driver: warm tcgen05/TMEM latencies (not part of the product)."""
import ctypes, os
import numpy as np
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcprobe2.so"))
out = np.zeros(12, dtype=np.int64)
rc = lib.probe2_run(out.ctypes.data_as(ctypes.c_void_p))
names = ["mma128x128x32+commit+wait", "8x mma128x16x32+commit+wait", "ld.x1+wait",
         "RMW 32x32 (1 warp)", "RMW 32x128 (1 warp)", "RMW 32x128 x4 warps +sync", "st.x1+wait", "bar.sync 128", "8 indep small", "2 chains of 4", "rank + 8 indep", "8 indep + rank"]
print("rc", rc)
for n, v in zip(names, out):
    print(f"{n:32s} {v:6d} cycles")
