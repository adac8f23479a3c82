"""Run a few eager hot-path steps (no CUDA graph) for ncu captures.

    ncu --set full -k regex:k2_synth -c 1 python tools/profile_step.py --slots 256
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slots", type=int, default=256)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--n-prb", type=int, default=273)
    ap.add_argument("--n-ant", type=int, default=4)
    ap.add_argument("--streams", type=int, default=1)
    ap.add_argument("--tx", default="complex", choices=["packed", "complex"])
    a = ap.parse_args()
    import torch
    from bench import make_stream_inputs
    from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    seeds = [1000 + k for k in range(a.streams)]
    geo, scens, pil, y, tx, nv, reg = make_stream_inputs(a.n_prb, a.n_ant, a.slots, seeds)
    flags = _lib.FLAG_TX_PACKED if a.tx == "packed" and a.n_ant in (1, 2, 4) else 0
    plan = ArchesPlan(geo, 1.25, PipelineConfig(), ExecutionMode.CONCURRENT, "oracle", flags=flags)
    eng = SlotEngine(plan, a.streams, a.slots)
    eng.set_streams(pil, seeds)
    eng.load(y=y, tx=tx, noise_var=nv, regime=reg)
    for _ in range(a.steps):
        eng.run()
    torch.cuda.synchronize()
    print("done", eng.kpm_records()[0]["slot_index"][-1])


if __name__ == "__main__":
    main()
