"""Per-role K1 timeline (timing analysis only): builds the library with
-DK1T_TRACE into tools/_trace/ (never shipped), runs config-B batches eagerly and
prints, for the first CTAs, each item's globaltimer stamps relative to the
CTA's first copy issue:  P copy issued | C full | C operand buffer free |
C converted | M MMA issued | D0 / D1 accumulator ready (column halves) | D0 done.

    python tools/k1_trace.py --build        # here (nvcc cross-compiles)
    python tools/k1_trace.py                # on the GPU box
"""
from __future__ import annotations

import argparse
import ctypes
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
OUT = ROOT / "tools" / "_trace" / "libarches_trace.so"


def build():
    from paper_2604_23397_b200 import build as B
    OUT.parent.mkdir(parents=True, exist_ok=True)
    cmd = [B.nvcc(), *B.ARCH, *B.FLAGS, "-DK1T_TRACE", "-I", str(ROOT / "include"),
           str(B.CSRC / "arches.cu"), "-o", str(OUT)]
    subprocess.run(cmd, check=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--slots", type=int, default=256)
    ap.add_argument("--ctas", type=int, default=3)
    a = ap.parse_args()
    if a.build:
        build()
        return
    from paper_2604_23397_b200 import _lib
    _lib.LIB_PATH = OUT
    import numpy as np
    import torch
    from bench import make_stream_inputs
    from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    seeds = [1000]
    geo, scens, pil, y, tx, nv, reg = make_stream_inputs(273, 4, a.slots, seeds)
    plan = ArchesPlan(geo, 1.25, PipelineConfig(), ExecutionMode.CONCURRENT, "oracle")
    eng = SlotEngine(plan, 1, a.slots)
    eng.set_streams(pil, seeds)
    eng.load(y=y, tx=tx, noise_var=nv, regime=reg)
    for _ in range(4):
        eng.run()
    torch.cuda.synchronize()
    lib = ctypes.CDLL(str(OUT))
    buf = np.zeros((8, 64, 8), dtype=np.uint64)
    assert lib.arches_k1t_trace(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    span = np.zeros((256, 5), dtype=np.uint64)
    assert lib.arches_k1t_span(span.ctypes.data_as(ctypes.c_void_p)) == 0
    n = int((span[:, 0] > 0).sum())
    sp = span[:n].astype(np.int64)
    t00 = sp[:, 0].min()
    rel = (sp - t00) / 1e3
    print(f"{n} CTAs: entry spread {rel[:, 0].min():.2f}..{rel[:, 0].max():.2f} us, first copy "
          f"{rel[:, 1].min():.2f}..{rel[:, 1].max():.2f}, drain done {rel[:, 2].min():.2f}.."
          f"{rel[:, 2].max():.2f} (median {np.median(rel[:, 2]):.2f})")
    print(f"  zeroed {np.median(rel[:, 3]):.2f}, synced {np.median(rel[:, 4]):.2f} (medians)")
    print("slowest CTAs:", np.argsort(-rel[:, 2])[:8].tolist(), np.sort(rel[:, 2])[-8:].round(2).tolist())
    names = ["P", "Cfull", "Cfree", "Cdone", "M", "D0", "D1", "D0done"]
    t0all = min(int(buf[b, 0, 0]) for b in range(8) if buf[b, 0, 0])
    for b in range(a.ctas):
        t0 = int(buf[b, 0, 0])
        print(f"CTA {b}: first copy at +{(t0 - t0all) / 1e3:.2f} us (relative to the earliest CTA)")
        print("  j  " + " ".join(f"{n:>7}" for n in names))
        for j in range(64):
            if not buf[b, j, 0]:
                break
            print(f" {j:2d}  " + " ".join(f"{(int(v) - t0) / 1e3:7.2f}" if v else "      -" for v in buf[b, j]))


if __name__ == "__main__":
    main()
