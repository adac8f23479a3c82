"""Stall-reason breakdown per SASS line range (ncu --page source --csv --print-source sass).

usage: python tools/stall_regions.py f.csv lo-hi [lo-hi ...]   (line ranges as printed by sass_hot.py)
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) == len(hdr)]
tot = Counter()
for r in data:
    for c in cols:
        tot[c] += int(r[hdr.index(c)] or 0)
print("whole kernel:", ", ".join(f"{k[6:]} {v}" for k, v in tot.most_common(8)))
for rng in sys.argv[2:]:
    lo, hi = map(int, rng.split("-"))
    c = Counter()
    for r in data[lo:hi + 1]:
        for k in cols:
            c[k] += int(r[hdr.index(k)] or 0)
    print(rng, ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(8)))
