"""BASELINE config E (massive MIMO: 273 PRB, 64 RX, 4 layers, each layer an
independent single-layer DMRS port): the tensor-core K1 over 128-row tiles of
(unit, antenna) rows and the antenna-group K2 (MRC sums across groups of four
antennas) against the oracle's closed loop run per layer.  The reference path
itself supports any n_ant (radio_scene.py:110-115); layers > 1 are the declared
per-port extension (SURVEY.md s7 hard part 6)."""
import numpy as np
import pytest

from parity import assert_estimate_close, assert_sigma2_close, compare_kpms, to_ref_layout
from oracle import ref_path as R
from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
from paper_2604_23397_b200.scene import CellScene, to_device_layout

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_prb,n_ant,n_layers,n_slots", [
    (12, 16, 3, 10),
    (273, 64, 4, 2),
])
def test_massive_mimo_layers_match_oracle(n_prb, n_ant, n_layers, n_slots):
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo = SlotGeometry(n_ant=n_ant, n_prb=n_prb)
    seeds = [500 + k for k in range(n_layers)]
    layers = []
    for k, seed in enumerate(seeds):
        scens = default_scenarios(seed, geo)
        regimes = ["good" if (i + k) % 2 == 0 else "poor" for i in range(n_slots)]
        cs = CellScene(geo, scens, regimes[0])
        layers.append((scens, regimes, cs, [cs.next_slot(r) for r in regimes]))
    pcfg = PipelineConfig()
    plan = ArchesPlan(geo, 1.25, pcfg, ExecutionMode.CONCURRENT, "oracle")
    eng = SlotEngine(plan, n_layers, n_slots)
    eng.set_streams(np.stack([l[2].pilots for l in layers]), seeds)
    eng.load(y=np.stack([to_device_layout(sl.y) for l in layers for sl in l[3]]),
             tx=np.stack([sl.tx.T for l in layers for sl in l[3]]).astype(np.complex64),
             noise_var=[sl.noise_var for l in layers for sl in l[3]],
             regime=[1 if r == "good" else 0 for l in layers for r in l[1]])
    eng.run()
    got = eng.kpm_records()
    tel = eng.telemetry()
    for k, (scens, regimes, cs, slots) in enumerate(layers):
        loop = R.CellLoop(geo, scens, "oracle", pcfg=pcfg, keep_arrays=True)
        for sl, r in zip(slots, regimes):
            loop.run_slot(sl.y, sl.tx, cs.pilots, r)
        res = loop.finish()
        assert got[k]["mode"].tolist() == res.modes, f"layer {k} modes"
        compare_kpms(got[k], np.array([rec.row() for rec in res.records], dtype=np.float64))
        for i, sr in enumerate(res.slots):
            u = k * n_slots + i
            ls = R.ls_estimate(slots[i].y, cs.pilots, geo)
            assert_sigma2_close(tel[k, i]["sigma2_hat"], sr.nv_est, float(np.mean(np.abs(ls) ** 2)),
                                f"layer {k} slot {i}")
            assert_estimate_close(to_ref_layout(eng.h_mmse[u].cpu().numpy()), sr.mmse,
                                  f"layer {k} slot {i} mmse")
            assert_estimate_close(to_ref_layout(eng.h_ai[u].cpu().numpy()), sr.ai,
                                  f"layer {k} slot {i} ai")


def test_batch_kernel_counts():
    """arches_batch_kernels (the count bench.py reports): RNG + K1 + finalize
    grid(s) + K2 + K3 + K4; many-antenna plans finalise in two grids (rows, taps);
    the CUDA-core forms finalise in line."""
    from paper_2604_23397_b200.engine import ArchesPlan
    pcfg = PipelineConfig()
    geo_b, geo_e = SlotGeometry(n_ant=4, n_prb=273), SlotGeometry(n_ant=64, n_prb=273)
    assert ArchesPlan(geo_b, 1.25, pcfg, ExecutionMode.CONCURRENT, "oracle").batch_kernels() == 6
    assert ArchesPlan(geo_e, 1.25, pcfg, ExecutionMode.CONCURRENT, "oracle").batch_kernels() == 7
    assert ArchesPlan(geo_b, 1.25, pcfg, ExecutionMode.CONCURRENT, "oracle",
                      flags=0x3).batch_kernels() == 4
