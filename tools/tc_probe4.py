"""Dev probe driver: costs of fences / barriers / TMEM stores (not part of the product)."""
import ctypes, os
import numpy as np
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcprobe4.so"))
out = np.zeros(8, dtype=np.int64)
rc = lib.probe4_run(out.ctypes.data_as(ctypes.c_void_p))
names = ["STS + fence.proxy.async", "STTM.x4 + wait::st", "tc fence + bar + tc fence", "bar.sync",
         "int div 127", "commit(empty) + mbar wait", "stage tail (STS,STTM,fences,bar)", "3x LDS.U8"]
print("rc", rc)
for nm, v in zip(names, out):
    print(f"{nm:36s} {v:6d} cycles")
