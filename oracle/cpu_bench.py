"""Timed CPU baseline: the oracle restatement of the reference hot path.

TEST/BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).  Run as a subprocess
by bench.py so BLAS thread counts can be fixed before numpy loads:

    OPENBLAS_NUM_THREADS=1 python -m oracle.cpu_bench --n-prb 273 --slots 2 --seed 5

Default mode times exactly the hot path of SURVEY.md s8(a) per slot (a1-a12:
LS, noise variance, MMSE incl. the per-slot Wiener rebuild, denoiser, switch,
|H| telemetry, equaliser, link adaptation, TB, CRC, windows, window features
and predict), slot synthesis excluded, concurrent mode, good/poor alternating
every slot (BASELINE config B with the oracle policy; config A with
--policy tree --tree FILE).

--policy-stress: BASELINE config D -- per slot boundary, for each of --cells
cells, `Dapp.on_indication` (dapp_control.py:107-120: append the record,
window_features over the last 100 records, predict, message).  Times
`--slots` boundaries over a sample of cells.  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def policy_stress(a):
    from collections import deque

    import numpy as np

    from oracle.ref_path import KpmRecord, predict, tree_from_text, window_features
    root, _ = tree_from_text(open(a.tree).read())
    rng = np.random.default_rng(a.seed)

    def record(n):
        kw = dict(slot_index=n, phy_throughput=float(rng.random() * 40), mcs_index=int(rng.integers(0, 28)),
                  pdu_length=int(rng.integers(0, 3000)), ndi=int(rng.integers(0, 2)),
                  rsrp=float(rng.random()), code_rate=0.5, qam_order=4, num_cb=1,
                  tb_size=int(rng.integers(0, 3000)), snr_db=float(rng.normal(10, 8)),
                  mac_throughput=float(rng.random() * 40), lcid4_throughput=float(rng.random() * 30),
                  mac_rx_bytes=int(rng.integers(0, 3000)), lcid4_rx_bytes=int(rng.integers(0, 2500)))
        return KpmRecord(**kw)

    windows = [deque((record(i) for i in range(a.window)), maxlen=a.window) for _ in range(a.cells)]
    fresh = [[record(a.window + s) for s in range(a.slots)] for _ in range(a.cells)]
    per_boundary = []
    for s in range(a.slots):
        t0 = time.perf_counter()
        for c in range(a.cells):
            w = windows[c]
            w.append(fresh[c][s])
            predict(root, window_features(list(w)))
        per_boundary.append(time.perf_counter() - t0)
    print(json.dumps({"mode": "policy-stress", "cells": a.cells, "boundaries": a.slots,
                      "per_boundary_s": per_boundary}))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-prb", type=int, default=273)
    ap.add_argument("--n-ant", type=int, default=4)
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--window", type=int, default=100)
    ap.add_argument("--policy", default="oracle", choices=["oracle", "tree"])
    ap.add_argument("--tree", default=None, help="tree v1 text (switch_policy.to_text)")
    ap.add_argument("--policy-stress", action="store_true")
    ap.add_argument("--cells", type=int, default=32)
    a = ap.parse_args(argv)
    if a.policy_stress:
        return policy_stress(a)

    from oracle.ref_path import CellLoop
    from paper_2604_23397_b200.config import PipelineConfig
    from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
    from paper_2604_23397_b200.scene import CellScene

    geo = SlotGeometry(n_ant=a.n_ant, n_prb=a.n_prb)
    scens = default_scenarios(a.seed, geo)
    regimes = ["good" if i % 2 == 0 else "poor" for i in range(a.slots)]
    cs = CellScene(geo, scens, regimes[0])
    inputs = [cs.next_slot(r) for r in regimes]          # synthesis: untimed
    loop = CellLoop(geo, scens, policy=a.policy, pcfg=PipelineConfig(window_length=a.window),
                    tree_text=open(a.tree).read() if a.policy == "tree" else None)
    per_slot = []
    t_all = time.perf_counter()
    for s, r in zip(inputs, regimes):
        t0 = time.perf_counter()
        loop.run_slot(s.y, s.tx, cs.pilots, r)
        per_slot.append(time.perf_counter() - t0)
    total = time.perf_counter() - t_all
    print(json.dumps({"slots": a.slots, "seconds": total, "per_slot_s": per_slot,
                      "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
                      "n_prb": a.n_prb, "n_ant": a.n_ant, "policy": a.policy}))


if __name__ == "__main__":
    main()
