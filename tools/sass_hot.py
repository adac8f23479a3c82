"""Rank SASS regions of a kernel by executed warp instructions (ncu source page CSV).

usage: ncu -i rep --page source --csv --kernel-name regex:K --launch-count 1 --print-source sass > f.csv
       python tools/sass_hot.py f.csv [window]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:4194]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((r[0], r[1].strip(), int(r[ie] or 0), int(r[st] or 0)))
    except ValueError:
        pass
tot = sum(d[2] for d in data)
tots = sum(d[3] for d in data)
print(f"total warp inst {tot}, stall samples {tots}, sass lines {len(data)}")
w = int(sys.argv[2]) if len(sys.argv) > 2 else 64
# region = contiguous lines sharing the same execution count
regions = []
cur = None
for i, d in enumerate(data):
    if cur and d[2] == cur[2]:
        cur[1] = i
    else:
        cur = [i, i, d[2]]
        regions.append(cur)
regions.sort(key=lambda r: -(r[1] - r[0] + 1) * r[2])
for a, b, c in regions[:25]:
    n = b - a + 1
    ops = Counter(data[k][1].split()[0] if not data[k][1].startswith("@") else data[k][1].split()[1]
                  for k in range(a, b + 1))
    stalls = sum(data[k][3] for k in range(a, b + 1))
    print(f"lines {a}-{b} n={n} exec={c} share={n*c/tot:.3f} stalls={stalls/tots:.3f} "
          + " ".join(f"{k}:{v}" for k, v in ops.most_common(8)))
