"""Summarise an ncu source-page CSV (SASS) of a kernel: stall reasons and per-region samples /
instruction counts between landmark instructions (dev helper)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0   # divide instruction counts (e.g. accepts)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = lambda d: float(d[idx["Warp Stall Sampling (All Samples)"]] or 0)
E = lambda d: float(d[idx["Instructions Executed"]] or 0)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(S(d) for d in data)
totr = {r: sum(float(d[idx[r]] or 0) for d in data) for r in reasons}
T = sum(totr.values())
print("stall reasons:", ", ".join(f"{r[6:]} {v/T*100:.1f}%" for r, v in sorted(totr.items(), key=lambda x: -x[1])[:8]))
print(f"warp instructions / norm: {sum(E(d) for d in data)/norm:.1f}")
keys = ["LDTM", "BAR.SYNC", "UTCIMMA", "TRYWAIT", "STTM", "UTCBAR", "BAR.ARV"]
marks = [i for i, d in enumerate(data) if any(k in d[1] for k in keys)]
prev = 0
for i in marks + [len(data)]:
    seg = data[prev:i]
    s, e = sum(S(d) for d in seg), sum(E(d) for d in seg)
    if s / max(tot, 1) > 0.005 or e / norm > 5:
        top = sorted(((r, sum(float(d[idx[r]] or 0) for d in seg)) for r in reasons), key=lambda x: -x[1])[:2]
        print(f"[{data[prev][0][-5:]}..{data[i][0][-5:] if i < len(data) else 'end'}) {data[prev][1].strip()[:38]:38s}"
              f" samples {s/tot*100:5.1f}%  instrs {e/norm:7.1f}  {top[0][0][6:]} {top[1][0][6:]}")
    prev = i
