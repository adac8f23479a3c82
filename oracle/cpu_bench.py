"""Timed CPU baseline: the oracle restatement of the reference hot path.

TEST/BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).  Run as a subprocess
by bench.py so BLAS thread counts can be fixed before numpy loads:

    OPENBLAS_NUM_THREADS=1 python -m oracle.cpu_bench --n-prb 273 --slots 2 --seed 5

Times exactly the hot path of SURVEY.md s8(a) per slot (a1-a12: LS, noise
variance, MMSE incl. the per-slot Wiener rebuild, denoiser, switch, |H|
telemetry, equaliser, link adaptation, TB, CRC, windows, window features and
predict), slot synthesis excluded, concurrent mode, good/poor alternating
every slot with the oracle policy (BASELINE config B).  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-prb", type=int, default=273)
    ap.add_argument("--n-ant", type=int, default=4)
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--window", type=int, default=100)
    a = ap.parse_args(argv)

    from oracle.ref_path import CellLoop
    from paper_2604_23397_b200.config import PipelineConfig
    from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
    from paper_2604_23397_b200.scene import CellScene

    geo = SlotGeometry(n_ant=a.n_ant, n_prb=a.n_prb)
    scens = default_scenarios(a.seed, geo)
    regimes = ["good" if i % 2 == 0 else "poor" for i in range(a.slots)]
    cs = CellScene(geo, scens, regimes[0])
    inputs = [cs.next_slot(r) for r in regimes]          # synthesis: untimed
    loop = CellLoop(geo, scens, policy="oracle", pcfg=PipelineConfig(window_length=a.window))
    per_slot = []
    t_all = time.perf_counter()
    for s, r in zip(inputs, regimes):
        t0 = time.perf_counter()
        loop.run_slot(s.y, s.tx, cs.pilots, r)
        per_slot.append(time.perf_counter() - t0)
    total = time.perf_counter() - t_all
    print(json.dumps({"slots": a.slots, "seconds": total, "per_slot_s": per_slot,
                      "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
                      "n_prb": a.n_prb, "n_ant": a.n_ant}))


if __name__ == "__main__":
    main()
