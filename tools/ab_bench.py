"""A/B timing of library variants (experiments only): builds variants of the
library with extra -D flags into tools/_trace/, then runs bench.py against each
in turn, alternating, so run-to-run drift hits both arms alike.

    python tools/ab_bench.py --build NAME=-DFLAG[,-DFLAG2] ...     # here
    python tools/ab_bench.py --run NAME[,NAME...] --rounds 3 -- [bench args]   # on the GPU box
"""
from __future__ import annotations

import argparse
import json
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
OUT = ROOT / "tools" / "_trace"


def lib_path(name: str) -> pathlib.Path:
    return ROOT / "paper_2604_23397_b200" / "lib" / "libarches.so" if name == "base" else OUT / f"lib_{name}.so"


def build(spec: str):
    from paper_2604_23397_b200 import build as B
    name, flags = spec.split("=", 1)
    OUT.mkdir(parents=True, exist_ok=True)
    cmd = [B.nvcc(), *B.ARCH, *B.FLAGS, *[f for f in flags.split(",") if f], "-I", str(ROOT / "include"),
           str(B.CSRC / "arches.cu"), "-o", str(lib_path(name))]
    subprocess.run(cmd, check=True)


def run_one(name: str, bench_args: list[str]) -> dict:
    code = ("import sys; sys.argv=['bench.py']+%r; sys.path.insert(0, %r); "
            "from paper_2604_23397_b200 import _lib; import pathlib; _lib.LIB_PATH=pathlib.Path(%r); "
            "import runpy; runpy.run_path(%r, run_name='__main__')"
            % (bench_args, str(ROOT), str(lib_path(name)), str(ROOT / "bench.py")))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if not line:
        raise RuntimeError(r.stderr[-2000:])
    return json.loads(line[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", nargs="*")
    ap.add_argument("--run")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("rest", nargs=argparse.REMAINDER)
    a = ap.parse_args()
    if a.build:
        for spec in a.build:
            build(spec)
        return
    names = a.run.split(",")
    bench_args = [x for x in a.rest if x != "--"]
    res = {n: [] for n in names}
    for _ in range(a.rounds):
        for n in names:
            d = run_one(n, bench_args)
            res[n].append((d["value"], d["roofline"]["kernel_ms"]))
            print(n, round(d["value"]), {k: round(v * 1e3, 1) for k, v in d["roofline"]["kernel_ms"].items()},
                  flush=True)
    for n in names:
        v = sorted(x[0] for x in res[n])
        print(f"{n}: median {v[len(v) // 2]:.0f}  all {[round(x) for x in v]}")


if __name__ == "__main__":
    main()
