"""Summarise an ncu report (raw metrics + SASS stall mix) into markdown.

    python tools/summarize_ncu.py gpurun_out/prof.ncu-rep > profiles/rN_ncu_summary.md
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    h, units, data = rows[0], rows[1], rows[2:]
    name_i = h.index("Kernel Name")
    print(f"# ncu summary: `{rep}`\n")
    print("| metric | " + " | ".join(d[name_i].split("(")[0].replace("void ", "") for d in data) + " |")
    print("|---|" + "---|" * len(data))
    for m, label in METRICS:
        if m not in h:
            continue
        i = h.index(m)
        print(f"| {label} ({units[i]}) | " + " | ".join(d[i] for d in data) + " |")
    for d in data:
        kname = d[name_i].split("(")[0].replace("void ", "")
        base = re.sub(r"<.*", "", kname)
        src = ncu(["-i", rep, "--page", "source", "--csv", "-k", f"regex:{base}", "--print-source", "sass"])
        r = list(csv.reader(io.StringIO(src)))
        try:
            hi = next(k for k, x in enumerate(r) if "Instructions Executed" in x)
        except StopIteration:
            continue
        hh = r[hi]
        body = [x for x in r[hi + 1:] if len(x) == len(hh)]
        ie, sc = hh.index("Instructions Executed"), hh.index("Source")
        stall = [k for k, c in enumerate(hh) if c.startswith("stall_") and "Not Issued" not in c]
        op, st, tot = Counter(), Counter(), 0.0
        seen = set()
        for x in body:
            key = (x[hh.index("Address")], x[sc])
            if key in seen:
                continue
            seen.add(key)
            try:
                n = float(x[ie].replace(",", ""))
            except ValueError:
                n = 0.0
            tot += n
            mm = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", x[sc])
            if mm:
                op[mm.group(2)] += n
            for k in stall:
                try:
                    st[hh[k]] += float(x[k].replace(",", ""))
                except ValueError:
                    pass
        print(f"\n## {kname}\n")
        print("opcode mix: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in op.most_common(10)))
        s = sum(st.values()) or 1.0
        print("\nstall reasons: " + ", ".join(f"{k[6:]} {v / s * 100:.1f}%" for k, v in st.most_common(6)))
        tc = [k for k in op if k.startswith(("UTC", "UTMA", "UBLK")) or k in ("LDTM", "STTM")]
        if tc:
            print("\nBlackwell-native instructions executed: " + ", ".join(f"{k} x{int(op[k])}" for k in sorted(tc)))


if __name__ == "__main__":
    main(sys.argv[1])
