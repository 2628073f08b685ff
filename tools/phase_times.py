"""Per-phase cycle breakdown of the single-chain kernel (debug build libqapsa_timers.so)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["QAPSA_LIB"] = os.path.join(ROOT, "paper_1208_2675_b200", "libqapsa_timers.so")
from paper_1208_2675_b200 import qapsa as Q  # noqa: E402
from qap_inputs import SA_SEED, config  # noqa: E402

iters = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**6
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A, B, p0, cfg = config(3)
s = Q.Solver(A, B, p0)
if threads:
    s.set_option(Q.QAP_OPT_THREADS, threads)
s.delta_init()
t0, tf = s.schedule_bounds()
sch = Q.make_schedule(0, t0, tf, cfg["iters"])
L = Q.lib()
buf = (C.c_ulonglong * 128)()
L.qapsa_debug_phase_cycles(buf)
g = s.run(0, iters, sch, SA_SEED)
ms, _ = s.last_kernel_time()
L.qapsa_debug_phase_cycles(buf)
w_acc, w_no, S, U, nacc, nno = buf[0], buf[1], buf[2], buf[3], buf[4], buf[5]
tdone, qdone = buf[6], buf[7]
print(f"iters {iters:.0e} threads {threads or 'auto'}: {ms:.1f} ms, accepts {g['accepted']}, "
      f"{ms*1e6/max(1,g['accepted']):.0f} ns/accept")
print(f"  per accept: W {w_acc/max(1,nacc):.0f} clk, SU {S/max(1,nacc):.0f} clk (stage released {U/max(1,nacc):.0f}, "
      f"W: offset-0 candidate done {tdone/max(1,nacc):.0f}, exchange done {qdone/max(1,nacc):.0f});"
      f"  non-accepting windows: {nno} x {w_no/max(1,nno):.0f} clk")
print(f"  W-phase prepare_addr {buf[8]}, prepare_theta {buf[9]}, exact double path {buf[10]} (of {iters} iterations)")
print(f"  W: thread 0 reaches its candidate at {buf[11]/max(1,nacc):.0f} clk after the loop top")
print(f"  SU: t0 dots done {buf[12]/max(1,nacc):.0f}, t0 incl. prep {buf[13]/max(1,nacc):.0f}, quads done: first thread {buf[14]/max(1,nacc):.0f}, last thread {buf[15]/max(1,nacc):.0f}")
