"""Per CUDA source line stall samples of an ncu report (cuda,sass source view): the top lines
by samples with their dominant stall reasons (dev helper).
  python tools/ncu_lines.py report.ncu-rep [top] [norm]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = defaultdict(lambda: defaultdict(float))
src = {}
fname, line, hdr = "?", None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        line = (fname, int(r[0]))
        src[line] = r[1].strip()
        continue
    if line is None:
        continue
    a = agg[line]
    for h, i in hdr.items():
        if i < 4 or i >= len(r):
            continue
        if h.startswith("stall_") and "Not Issued" not in h or h in ("Warp Stall Sampling (All Samples)",
                                                                      "Instructions Executed"):
            try:
                a[h] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(a["Warp Stall Sampling (All Samples)"] for a in agg.values())
items = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])
for (f, ln), a in items[:top]:
    s = a["Warp Stall Sampling (All Samples)"]
    st = sorted(((k[6:], v) for k, v in a.items() if k.startswith("stall_")), key=lambda x: -x[1])[:3]
    print(f"{s/tot*100:5.1f}% {f}:{ln:<4d} inst/n {a['Instructions Executed']/norm:7.1f} "
          f"{' '.join(f'{k}:{v/max(s,1)*100:.0f}' for k, v in st):40s} {src.get((f, ln), '')[:90]}")
