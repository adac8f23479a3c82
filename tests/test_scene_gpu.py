"""Device-side slot synthesis (arches_synthesize, scene_gpu.DeviceScene) against
the host scene (scene.CellScene, pinned bit-exact to the reference by
tests/test_oracle_golden.py) and, end to end, against the reference's golden
closed loops (the benched 273-PRB window-100 loop and the config-A tree loop).

Contract: every random BIT is the reference's -- QPSK data / pilots / interferer
symbols exact, so tx and the pilots are bit-identical; y (complex64) agrees to
the fp64 libm / DFT rounding of the fading and AWGN draws:
max |dy| <= Y_TOL * max |y| per slot (measured ~1e-7: one complex64 ulp)."""
import numpy as np
import pytest

from golden_io import loop_setup, loops_long
from parity import compare_kpms
from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
from paper_2604_23397_b200.scene import CellScene, to_device_layout

pytestmark = pytest.mark.gpu
Y_TOL = 1e-6


def _engine(geo, scens, C, S, policy="oracle", pcfg=None, em=None, dcfg=None, tree=None):
    from paper_2604_23397_b200.config import ExecutionMode
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    plan = ArchesPlan(geo, scens["good"].assumed_delay_spread, pcfg,
                      em or ExecutionMode.CONCURRENT, policy, dcfg)
    return SlotEngine(plan, C, S, tree=tree)


@pytest.mark.parametrize("n_prb,n_ant,S,batches", [(273, 4, 6, 2), (52, 4, 8, 3), (12, 8, 5, 2),
                                                   (24, 16, 3, 2)])
def test_device_synthesis_matches_host_scene(n_prb, n_ant, S, batches):
    import torch
    from paper_2604_23397_b200.scene_gpu import DeviceScene
    geo = SlotGeometry(n_ant=n_ant, n_prb=n_prb)
    seeds = [5, 1234]
    scens = default_scenarios(seeds[0], geo)
    eng = _engine(geo, scens, len(seeds), S)
    ds = DeviceScene(eng, {"good": scens["good"], "poor": scens["poor"]}, seeds)
    hosts = [CellScene(geo, default_scenarios(sd, geo), "good") for sd in seeds]
    for c, h in enumerate(hosts):
        assert np.array_equal(ds.pilots[c].cpu().numpy(), h.pilots.astype(np.complex64))
    for b in range(batches):
        reg = [["good" if (i + b + c) % 3 else "poor" for i in range(S)] for c in range(len(seeds))]
        ds.next_batch(reg)
        torch.cuda.synchronize()
        y = eng.y.cpu().numpy().reshape(len(seeds), S, *eng.y.shape[1:])
        tx = eng.tx.cpu().numpy().reshape(len(seeds), S, *eng.tx.shape[1:])
        nv = eng.noise_var.cpu().numpy().reshape(len(seeds), S)
        for c, h in enumerate(hosts):
            for i in range(S):
                sl = h.next_slot(reg[c][i])
                assert np.array_equal(tx[c, i], sl.tx.T.astype(np.complex64)), (b, c, i)
                want = to_device_layout(sl.y)
                err = np.abs(y[c, i] - want).max() / np.abs(want).max()
                assert err <= Y_TOL, (b, c, i, err)
                assert nv[c, i] == sl.noise_var


@pytest.mark.parametrize("lid", ["p273_alt_w100_conc", "p52_tree_default"])
def test_closed_loop_on_device_synthesised_slots(lid):
    """The golden reference loops reproduced with the inputs synthesised on the
    device: integer KPMs, CRC, modes and messages exact; rsrp / SINR within
    tests/parity.py (the synthesis ulps sit far below those tolerances)."""
    import torch
    from paper_2604_23397_b200.policy import from_text
    from golden_io import tree_text
    from paper_2604_23397_b200.scene_gpu import DeviceScene
    m, recs, extra = {m["id"]: (m, r, e) for m, r, e in loops_long()}[lid]
    geo, scen, regimes, em, pcfg, dcfg = loop_setup(m)
    n = len(regimes)
    S = n // 5 if n % 5 == 0 else n // 4
    tree = from_text(tree_text(m["tree"])) if m["tree"] else None
    eng = _engine(geo, scen, 1, S, "tree" if m["policy"] == "tree" else m["policy"], pcfg, em,
                  dcfg, tree)
    ds = DeviceScene(eng, scen, [m["seed"]], first_regime=regimes[0])
    got = []
    for b in range(n // S):
        ds.next_batch([regimes[b * S:(b + 1) * S]])
        eng.run()
        got.append(eng.kpm_records()[0].copy())
    got = np.concatenate(got)
    k = len(got)
    compare_kpms(got, recs[:k], extra[:k])
    assert got["mode"].tolist() == m["modes"][:k]
