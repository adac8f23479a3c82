"""Average per-kernel duration / DRAM bytes from an ncu --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i]
d = defaultdict(list)
for r in rows[i + 1:]:
    x = dict(zip(hdr, r))
    d[(x["Kernel Name"].split("(")[0][:48], x["Metric Name"])].append(float(x["Metric Value"].replace(",", "")))
names = sorted({k[0] for k in d})
print(f"{'kernel':50s} {'n':>3s} {'us':>9s} {'rd MB':>9s} {'wr MB':>9s}")
for n in names:
    t = d.get((n, "gpu__time_duration.sum"), [0])
    rd = d.get((n, "dram__bytes_read.sum"), [0])
    wr = d.get((n, "dram__bytes_write.sum"), [0])
    print(f"{n:50s} {len(t):3d} {sum(t)/len(t)/1e3:9.2f} {sum(rd)/len(rd)/1e6:9.2f} {sum(wr)/len(wr)/1e6:9.2f}")
