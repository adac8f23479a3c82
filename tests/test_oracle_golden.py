"""Pin the CPU oracle (and the input synthesiser) to the reference's own outputs.

Every expectation here was produced by the unmodified reference
(tools/make_golden.py); the oracle must reproduce it bit-for-bit, otherwise it
cannot serve as the checker for the device path.
"""
import hashlib

import numpy as np
import pytest

from golden_io import (case_scenario, experts_large, experts_small, loop_inputs, loop_setup,
                       loops, tree_text)
from oracle import ref_path as R
from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
from paper_2604_23397_b200.scene import CellScene

SMALL = [c["id"] for c, _ in experts_small()]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("cid", SMALL)
def test_oracle_experts_small_bit_exact(cid):
    case, d = dict((c["id"], (c, d)) for c, d in experts_small())[cid]
    geo = SlotGeometry(n_ant=case["n_ant"], n_prb=case["n_prb"])
    scen = case_scenario(case)
    ls = R.ls_estimate(d["y"], d["pilots"], geo)
    assert np.array_equal(ls, d["ls"])
    nv = R.estimate_noise_var(ls, case["guard"])
    assert nv == float(d["nv_est"])
    if "mmse" in d:
        mmse = R.mmse_estimate(ls, nv, scen.assumed_delay_spread)
        assert np.array_equal(mmse, d["mmse"])
    ai = R.denoiser_estimate(ls, case["truncation"])
    assert np.array_equal(ai, d["ai"])
    for name in ("mmse", "ai"):
        if f"sinr_{name}" not in d:
            continue
        _, sinr = R.equalize(d["y"], d[name], case["noise_var"], d["tx"], geo)
        assert sinr == float(d[f"sinr_{name}"])
        assert float(np.mean(np.abs(d[name]) ** 2)) == float(d[f"rsrp_{name}"])


@pytest.mark.parametrize("case", experts_large(), ids=lambda c: c["id"])
def test_oracle_and_scene_large_hash_exact(case):
    geo = SlotGeometry(n_ant=case["n_ant"], n_prb=case["n_prb"])
    scens = default_scenarios(case["seed"], geo)
    cs = CellScene(geo, scens, "good")
    for rec in case["slots"]:
        s = cs.next_slot(rec["regime"])
        assert sha(s.y) == rec["sha_y"]           # scene.py reproduces the reference grid
        ls = R.ls_estimate(s.y, cs.pilots, geo)
        assert sha(ls) == rec["sha_ls"]
        nv = R.estimate_noise_var(ls, 16)
        assert nv == rec["nv_est"]
        mmse = R.mmse_estimate(ls, nv, scens["good"].assumed_delay_spread)
        ai = R.denoiser_estimate(ls, 20)
        assert sha(mmse) == rec["sha_mmse"]
        assert sha(ai) == rec["sha_ai"]
        nv_true = scens[rec["regime"]].noise_var(geo.n_ant)
        for name, est in (("mmse", mmse), ("ai", ai)):
            _, sinr = R.equalize(s.y, est, nv_true, s.tx, geo)
            assert sinr == rec[f"sinr_{name}"]


def run_oracle_loop(m):
    geo, scen, regimes, em, pcfg, dcfg = loop_setup(m)
    policy = m["policy"]
    cs, inputs = loop_inputs(geo, scen, regimes)
    loop = R.CellLoop(geo, scen, policy=policy, exec_mode=em, pcfg=pcfg, dcfg=dcfg,
                      tree_text=tree_text(m["tree"]) if m["tree"] else None)
    for s, reg in zip(inputs, regimes):
        loop.run_slot(s.y, s.tx, cs.pilots, reg)
    return loop.finish()


@pytest.mark.parametrize("lid", [m["id"] for m, _, _ in loops()])
def test_oracle_closed_loop_bit_exact(lid):
    m, recs, extra = dict((m["id"], (m, r, e)) for m, r, e in loops())[lid]
    res = run_oracle_loop(m)
    got = np.array([[float(v) for v in k.row()] for k in res.records])
    assert np.array_equal(got, recs)
    assert res.modes == m["modes"]
    assert [[x.mode, x.decided_at_ns, x.deliverable_at_ns, x.trigger] for x in res.messages] \
        == m["messages"]
    assert res.failsafe_events == m["failsafe_events"]
    assert np.array_equal(np.array([s.sinr_db for s in res.slots]), extra[:, 0])
    assert np.array_equal(np.array([s.est_abs_mean for s in res.slots]), extra[:, 1])


def test_reference_kats_in_oracle():
    # known answers pinned by the reference's own tests
    from paper_2604_23397_b200.config import DEFAULT_MCS_TABLE as T
    a = R.time_interp_weights((0, 5, 10), 14)
    assert np.allclose(a[2], (0.6, 0.4, 0.0)) and np.array_equal(a[13], (0.0, 0.0, 1.0))
    assert R.transport_block(0, 12, T)[0] == 47            # test_phy_pipeline.py:58-67
    assert R.link_adapt(-100.0, T) == 0 and R.link_adapt(1e6, T) == T.n_mcs - 1
    for i in (0, 5, 11, 20):
        assert R.link_adapt(T.thresholds_db[i], T) == i
    w = R.ThroughputWindow(4, 0.0005)
    assert w.push(1000) == pytest.approx(1000 * 8 / 1e6 / 0.0005)
