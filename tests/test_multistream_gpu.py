"""Several independent streams in one batch (BASELINE config C: cells x layers,
each layer an independent single-layer DMRS port, SURVEY.md s7 hard part 6).

Each stream's closed loop must equal the oracle's `CellLoop` (harness.execute_run
restated, pinned to the reference by test_oracle_golden) run on that stream
alone: per-stream pilots, seeds (CRC draw), control state and KPM windows must
not leak across streams -- in particular where a tensor-core K1 row tile or a
K2 work range spans two streams."""
import numpy as np
import pytest

from parity import assert_estimate_close, compare_kpms, to_ref_layout
from oracle import ref_path as R
from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
from paper_2604_23397_b200.scene import CellScene, to_device_layout

pytestmark = pytest.mark.gpu


def _streams(geo, seeds, n_slots):
    out = []
    for k, seed in enumerate(seeds):
        scens = default_scenarios(seed, geo)
        # a different good/poor phase per stream so the modes differ across streams
        regimes = ["good" if ((i + k) // (k + 1)) % 2 == 0 else "poor" for i in range(n_slots)]
        cs = CellScene(geo, scens, regimes[0])
        slots = [cs.next_slot(r) for r in regimes]
        out.append((seed, scens, regimes, cs, slots))
    return out


@pytest.mark.parametrize("n_prb,n_streams,n_slots,exec_mode", [
    (12, 4, 30, ExecutionMode.CONCURRENT),     # 2 cells x 2 layers
    (52, 3, 40, ExecutionMode.CONCURRENT),     # 128-row K1 tiles span two streams
    (52, 2, 24, ExecutionMode.SELECTED_ONLY),
])
def test_streams_match_independent_oracle_loops(n_prb, n_streams, n_slots, exec_mode):
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo = SlotGeometry(n_ant=4, n_prb=n_prb)
    seeds = [101 + 7 * k for k in range(n_streams)]
    streams = _streams(geo, seeds, n_slots)
    pcfg = PipelineConfig()
    plan = ArchesPlan(geo, 1.25, pcfg, exec_mode, "oracle")
    eng = SlotEngine(plan, n_streams, n_slots)
    eng.set_streams(np.stack([s[3].pilots for s in streams]), seeds)
    eng.load(y=np.stack([to_device_layout(sl.y) for s in streams for sl in s[4]]),
             tx=np.stack([sl.tx.T for s in streams for sl in s[4]]).astype(np.complex64),
             noise_var=[sl.noise_var for s in streams for sl in s[4]],
             regime=[1 if r == "good" else 0 for s in streams for r in s[2]])
    eng.run()
    got = eng.kpm_records()
    for k, (seed, scens, regimes, cs, slots) in enumerate(streams):
        loop = R.CellLoop(geo, scens, "oracle", exec_mode=exec_mode, pcfg=pcfg, keep_arrays=True)
        for sl, r in zip(slots, regimes):
            loop.run_slot(sl.y, sl.tx, cs.pilots, r)
        res = loop.finish()
        assert got[k]["mode"].tolist() == res.modes, f"stream {k} modes"
        rows = np.array([rec.row() for rec in res.records], dtype=np.float64)
        compare_kpms(got[k], rows)
        # expert outputs of the first and last slot of the stream
        for i in (0, n_slots - 1):
            u = k * n_slots + i
            if res.slots[i].mmse is not None:
                assert_estimate_close(to_ref_layout(eng.h_mmse[u].cpu().numpy()), res.slots[i].mmse,
                                      f"stream {k} slot {i} mmse")
            if res.slots[i].ai is not None:
                assert_estimate_close(to_ref_layout(eng.h_ai[u].cpu().numpy()), res.slots[i].ai,
                                      f"stream {k} slot {i} ai")
