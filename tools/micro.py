import ctypes as C, os
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmicro.so"))
out = (C.c_longlong * 8)()
print("rc", L.micro_run(100, out))
print("prepare_addr", out[0], "prepare_theta", out[1], "philox", out[2], "temp32", out[3], "tri_pair", out[4])
