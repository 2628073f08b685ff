"""Per-kernel histogram of the SASS mnemonics that show which hardware paths the library uses
(tcgen05 MMA / TMEM / TMA bulk copies / mbarriers / dp4a / FP64 ...):
  python tools/sass_histogram.py [libqapsa.so] > profiles/r02_sass_histogram.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1208_2675_b200/libqapsa.so"
KEYS = ["UTCIMMA", "UTCQMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "STTM", "UBLKCP", "SYNCS.ARRIVE", "SYNCS.PHASECHK",
        "IDP.4A", "DFMA", "DMUL", "DADD", "MUFU", "BAR.SYNC", "BAR.RED", "UCGABAR", "ATOMS", "REDUX", "CREDUX",
        "LDS", "STS", "LDG", "STG", "VOTE", "SHFL"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern, counts = None, collections.OrderedDict()
for ln in out.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
    if kern and m:
        op = m.group(1)
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                counts[kern][k] += 1
dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"SASS mnemonic counts per kernel of {lib} (static instruction counts, cuobjdump -sass)")
print("kernel | " + " | ".join(KEYS))
tot = collections.Counter()
for (k, c), name in zip(counts.items(), dem):
    if not sum(c.values()):
        continue
    tot.update(c)
    print(name[:70] + " | " + " | ".join(str(c[x]) for x in KEYS))
print("TOTAL | " + " | ".join(str(tot[x]) for x in KEYS))
