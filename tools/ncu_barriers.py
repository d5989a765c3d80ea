"""Attribute ncu warp-stall samples of mbarrier waits to the barrier being waited on.
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
       python tools/ncu_barriers.py src.csv BASE_HEX name=off,...  (offsets relative to BASE)"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
base = int(sys.argv[2], 16)
names = {}
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    names[int(v, 16)] = k
h = rows[1]
data = rows[2:]
isrc, iss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iss] or 0) for r in data)
agg = collections.Counter()
last, last_i = None, -99
for i, r in enumerate(data):
    m = re.search(r"TRYWAIT P\d, \[([^\]]*)\]", r[isrc])
    if m:
        off = re.search(r"0x([0-9a-f]+)$", m.group(1))
        last = int(off.group(1), 16) - base if off else None
        last_i = i
    if i - last_i <= 3 and last is not None:
        agg[names.get(last, hex(last))] += float(r[iss] or 0)
    elif "TRYWAIT" in r[isrc] or "YIELD" in r[isrc]:
        agg["?"] += float(r[iss] or 0)
print(f"total samples {tot:.0f}")
for k, v in agg.most_common():
    print(f"{k:12s} {v / tot * 100:5.1f}%")
