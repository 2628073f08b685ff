"""Per-kernel totals and shares of an ncu launch list (gpu__time_duration.sum CSV):
python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] in ("ID", '"ID"'))
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.OrderedDict()
cnt = collections.Counter()
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot[name] = tot.get(name, 0.0) + ms
    cnt[name] += 1
allms = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms':>12s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v:12.3f} {100 * v / allms:6.2f}%")
print(f"{'total':60s} {sum(cnt.values()):8d} {allms:12.3f}")
