"""K1 work-split edge cases vs the oracle, and run-to-run determinism.

K1 cuts its (16-row tile, DMRS symbol, 256-subcarrier chunk) items into one
contiguous range per CTA; a row's bins are the sum of its segments (the tile's
first chunk and every CTA range start inside it), its last chunk's copy runs on
into the next OFDM symbol (or is clamped at the end of the grid), tiles never
straddle streams.  These cases put every one of those boundaries under the
oracle (expert_bank.py:96-214 restated in oracle/ref_path.py), and check that
repeated runs are bit-identical (no order- or race-dependent sums).
"""
import numpy as np
import pytest

from parity import assert_estimate_close, assert_sigma2_close, to_ref_layout
from oracle import ref_path as R
from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
from paper_2604_23397_b200.scene import CellScene, to_device_layout

pytestmark = pytest.mark.gpu


def _run(geo, n_streams, n_slots, seed0=3):
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    scenes, slots = [], []
    for k in range(n_streams):
        cs = CellScene(geo, default_scenarios(seed0 + k, geo), "good")
        scenes.append(cs)
        slots.append([cs.next_slot("good" if i % 2 == 0 else "poor") for i in range(n_slots)])
    plan = ArchesPlan(geo, 1.25, PipelineConfig(), ExecutionMode.CONCURRENT, "oracle")
    eng = SlotEngine(plan, n_streams, n_slots)
    eng.set_streams(np.stack([cs.pilots for cs in scenes]), [seed0 + k for k in range(n_streams)])
    flat = [s for ss in slots for s in ss]
    eng.load(y=np.stack([to_device_layout(s.y) for s in flat]),
             tx=np.stack([s.tx.T for s in flat]).astype(np.complex64),
             noise_var=[s.noise_var for s in flat], regime=[1] * len(flat))
    eng.run()
    return eng, scenes, slots


CASES = [
    # (n_prb, n_ant, dmrs_symbols, streams, slots, checked units)
    (12, 4, (0, 5, 10), 3, 6, None),            # partial tiles (24 rows per stream), N < one chunk
    (273, 4, (0, 5, 10), 1, 37, [0, 1, 17, 35, 36]),  # 390 items on 148 CTAs: several segments per row
    (52, 4, (2, 7, 13), 2, 5, None),            # DMRS symbol last in the slot: the grid-end clamp
    (24, 16, (0, 5, 10), 2, 3, None),           # one unit per tile
    (24, 64, (0, 5, 10), 1, 2, None),           # a unit spans four tiles
]


@pytest.mark.parametrize("n_prb,n_ant,dmrs,n_streams,n_slots,check", CASES,
                         ids=[f"{c[0]}prb-{c[1]}ant-d{c[2][-1]}-{c[3]}x{c[4]}" for c in CASES])
def test_k1_split_edges_match_oracle(n_prb, n_ant, dmrs, n_streams, n_slots, check):
    geo = SlotGeometry(n_ant=n_ant, n_prb=n_prb, dmrs_symbols=dmrs)
    eng, scenes, slots = _run(geo, n_streams, n_slots)
    tel = eng.telemetry()
    for k in range(n_streams):
        for i in (check if check is not None else range(n_slots)):
            s, u = slots[k][i], k * n_slots + i
            ls = R.ls_estimate(s.y, scenes[k].pilots, geo)
            nv = R.estimate_noise_var(ls, 16)
            tag = f"stream {k} slot {i}"
            assert_sigma2_close(tel[k, i]["sigma2_hat"], nv, float(np.mean(np.abs(ls) ** 2)), tag)
            assert_estimate_close(to_ref_layout(eng.h_mmse[u].cpu().numpy()), R.mmse_estimate(ls, nv, 1.25),
                                  tag + " mmse")
            assert_estimate_close(to_ref_layout(eng.h_ai[u].cpu().numpy()), R.denoiser_estimate(ls, 20),
                                  tag + " ai")


@pytest.mark.parametrize("n_prb,n_ant,n_streams,n_slots", [(273, 4, 1, 96), (24, 64, 2, 4)])
def test_k1_repeat_runs_bit_identical(n_prb, n_ant, n_streams, n_slots):
    import torch
    geo = SlotGeometry(n_ant=n_ant, n_prb=n_prb)
    eng, _, _ = _run(geo, n_streams, n_slots)
    first = None
    for _ in range(4):
        eng.reset()
        eng.run()
        torch.cuda.synchronize()
        cur = [t.cpu().numpy().copy() for t in (eng.h_mmse, eng.h_ai, eng.tel, eng.kpm)]
        if first is None:
            first = cur
            continue
        for a, b in zip(first, cur):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
