"""Summarise an ncu source-page SASS csv: opcode mix and stall reasons."""
import csv, re, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Instructions Executed' in r)
h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(h)]
ie = h.index('Instructions Executed'); src = h.index('Source')
stall_cols = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
op = Counter(); st = Counter(); tot = 0
def f(x):
    try: return float(x.replace(',', ''))
    except Exception: return 0.0
for r in data:
    n = f(r[ie]); tot += n
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[src])
    if m: op[m.group(2)] += n
    for c in stall_cols: st[h[c]] += f(r[c])
print('total warp instrs', tot)
for k, v in op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25): print(f"{k:10s} {v/tot*100:5.1f}%")
s = sum(st.values()) or 1
print('stalls:')
for k, v in st.most_common(10): print(f"  {k:25s} {v/s*100:5.1f}%")
