"""Run the same slot batch several times and report any bitwise difference
(K1 taps / sigma2 in the workspace, expert outputs, telemetry, KPM records).

    python tools/determinism.py [--n-prb 52] [--slots 300] [--reps 5]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-prb", type=int, default=52)
    ap.add_argument("--slots", type=int, default=300)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch
    from bench import make_inputs
    from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo, scens, pil, y, tx, nv, reg = make_inputs(a.n_prb, 4, a.slots, 7)
    plan = ArchesPlan(geo, 1.25, PipelineConfig(), ExecutionMode.CONCURRENT, "oracle")
    eng = SlotEngine(plan, 1, a.slots)
    eng.set_streams(pil[None], [7])
    eng.load(y=y, tx=tx, noise_var=nv, regime=reg)
    ref = None
    for r in range(a.reps):
        eng.reset()
        eng.run()
        torch.cuda.synchronize()
        cur = {"ws": eng.ws.clone(), "h_mmse": eng.h_mmse.clone(), "h_ai": eng.h_ai.clone(),
               "tel": eng.tel.clone(), "kpm": eng.kpm.clone()}
        if ref is None:
            ref = cur
            continue
        for k in ref:
            d = (ref[k].view(torch.uint8).reshape(-1) != cur[k].view(torch.uint8).reshape(-1)).nonzero().reshape(-1)
            if d.numel():
                print(f"rep {r}: {k} differs in {d.numel()} bytes, first at {d[0].item()}, last at {d[-1].item()}")
    from paper_2604_23397_b200 import _lib
    print("ws bytes", eng.ws.numel(), "coef bytes/unit", 8 * ((4 * 3 * 28 + 1) // 2 * 2))
    print("done")


if __name__ == "__main__":
    main()
