"""Drop-in functions (reference signatures) on the device vs the reference's
golden outputs, plus the reference's own contract tests restated against them
(test_expert_bank.py, test_phy_pipeline.py:145-168, test_dapp_control.py:60-65,
test_switch_policy.py:151-163)."""
import math

import numpy as np
import pytest

from golden_io import case_scenario, experts_small
from parity import SINR_ABS_TOL_DB, assert_estimate_close, assert_sigma2_close
from paper_2604_23397_b200 import compat as X
from paper_2604_23397_b200.config import PipelineConfig
from paper_2604_23397_b200.errors import (ConfigurationError, ContractViolation,
                                          PipelineStateError)
from paper_2604_23397_b200.geometry import (DmrsEstimate, ExpertId, ResourceGrid, Stage,
                                            SlotGeometry)
from paper_2604_23397_b200.policy import Node, TreeModel

pytestmark = pytest.mark.gpu


def _rx(case, d):
    geo = SlotGeometry(n_ant=case["n_ant"], n_prb=case["n_prb"])
    return geo, ResourceGrid(values=d["y"], known_dmrs=d["pilots"], geometry=geo)


@pytest.mark.parametrize("cid", [c["id"] for c, _ in experts_small()])
def test_compat_experts_match_reference(cid):
    case, d = dict((c["id"], (c, d)) for c, d in experts_small())[cid]
    geo, rx = _rx(case, d)
    scen = case_scenario(case)
    ls = X.ls_estimate(rx, geo)
    assert ls.stage.value == "RawLS" and ls.values.dtype == np.complex128
    assert np.max(np.abs(ls.values - d["ls"])) <= 1e-6 * np.max(np.abs(d["ls"]))
    assert np.array_equal(ls.values[:, :, 1::2, :], ls.values[:, :, 0::2, :])
    nv = X.estimate_noise_var(ls, geo, guard=case["guard"])
    assert_sigma2_close(nv, float(d["nv_est"]), float(np.mean(np.abs(d["ls"]) ** 2)), cid)
    # expert outputs from the reference's own LS input
    ref_ls = DmrsEstimate(d["ls"], Stage.RAW_LS, ls.comb_mask, geo)
    ai = X.denoiser_estimate(ref_ls, geo, truncation=case["truncation"])
    assert ai.stage.value == "Interpolated" and ai.comb_mask.all()
    assert_estimate_close(ai.values, d["ai"], cid + " ai")
    if float(d["nv_est"]) > 1e-10 * float(np.mean(np.abs(d["ls"]) ** 2)):
        mm = X.mmse_estimate(ref_ls, float(d["nv_est"]), scen)
        assert_estimate_close(mm.values, d["mmse"], cid + " mmse")
        est = DmrsEstimate(d["mmse"], Stage.INTERPOLATED, np.ones(geo.n_sc, bool), geo)
        x_hat, sinr = X.equalize(rx, est, case["noise_var"], d["tx"])
        assert x_hat.shape == (geo.n_sc, geo.n_sym)
        assert abs(sinr - float(d["sinr_mmse"])) <= SINR_ABS_TOL_DB


def test_compat_contracts():
    case, d = dict((c["id"], (c, d)) for c, d in experts_small())["good_12prb"]
    geo, rx = _rx(case, d)
    ls = X.ls_estimate(rx, geo)
    bad = ResourceGrid(values=d["y"], known_dmrs=d["pilots"].copy(), geometry=geo)
    bad.known_dmrs[0, 0] = 0.0
    with pytest.raises(ContractViolation):
        X.ls_estimate(bad, geo)
    with pytest.raises(ConfigurationError):
        X.ls_estimate(rx, SlotGeometry(n_ant=4, n_prb=12, n_layers=2))
    est = X.mmse_estimate(ls, 0.01, case_scenario(case))
    with pytest.raises(ContractViolation):
        X.mmse_estimate(est, 0.01, case_scenario(case))       # already interpolated
    with pytest.raises(ConfigurationError):
        X.mmse_estimate(ls, -1.0, case_scenario(case))
    with pytest.raises(ConfigurationError):
        X.denoiser_estimate(ls, geo, truncation=0)
    with pytest.raises(ContractViolation):
        X.denoiser_estimate(est, geo)
    with pytest.raises(ConfigurationError):
        X.estimate_noise_var(ls, geo, guard=0)
    with pytest.raises(ConfigurationError):
        X.estimate_noise_var(ls, geo, guard=geo.n_comb)
    with pytest.raises(ContractViolation):
        X.equalize(rx, ls, 0.0, d["tx"])


def test_compat_denoiser_truncates_the_delay_tail():
    # test_expert_bank.py:103-114 with the fp32 tolerance stated in tests/parity.py
    case, d = dict((c["id"], (c, d)) for c, d in experts_small())["snr5_4prb_1ant"]
    geo, rx = _rx(case, d)
    out = X.denoiser_estimate(X.ls_estimate(rx, geo), geo, truncation=20)
    taps = np.fft.ifft(out.values, axis=2)
    assert np.max(np.abs(taps[:, :, 20:, :])) <= 1e-6 * np.max(np.abs(taps))


class _Costs:
    switch_mmse_us, switch_ai_us = 4.89, 3.36

    def switch_cost_us(self, mode):
        return self.switch_mmse_us if mode == 1 else self.switch_ai_us


class _Mode:
    def __init__(self, m=1):
        self.mode = m


def test_compat_buffers_and_switch_select():
    buf = X.ExpertBuffers((2, 3))
    costs = _Costs()
    mmse_out = np.full((2, 3), 1 + 1j)
    ai_out = np.full((2, 3), 2 - 2j)
    buf.write(ExpertId.MMSE, mmse_out)
    buf.write(ExpertId.AI, ai_out)
    assert X.switch_select(buf, _Mode(1), costs) == costs.switch_mmse_us
    assert np.array_equal(buf.downstream, mmse_out)
    buf.new_slot()
    buf.write(ExpertId.AI, ai_out)
    assert X.switch_select(buf, _Mode(0), costs) == costs.switch_ai_us
    assert np.array_equal(buf.downstream, ai_out)
    assert buf.downstream is buf.buffer_ai
    buf.new_slot()
    with pytest.raises(PipelineStateError):
        X.switch_select(buf, _Mode(1), costs)
    with pytest.raises(PipelineStateError):
        X.switch_select(buf, _Mode(0), costs)


def test_compat_window_features_and_predict():
    class R:
        def __init__(self, mac):
            self.phy_throughput, self.mcs_index, self.pdu_length, self.ndi = 5.0, 12, 500, 0
            self.rsrp, self.snr_db, self.mac_throughput = 1.0, 10.0, mac
            self.lcid4_throughput, self.mac_rx_bytes, self.lcid4_rx_bytes = 0.85 * mac, 500, 425
    vec = X.window_features([R(4.0), R(8.0)])
    assert vec[6] == 6.0 and vec[1] == 12.0
    rng = np.random.default_rng(0)
    rows = rng.normal(size=(100, 10)) * 1e3
    recs = []
    for r in rows:
        o = R(0.0)
        for name, v in zip(("phy_throughput", "mcs_index", "pdu_length", "ndi", "rsrp", "snr_db",
                            "mac_throughput", "lcid4_throughput", "mac_rx_bytes",
                            "lcid4_rx_bytes"), r):
            setattr(o, name, v)
        recs.append(o)
    assert np.array_equal(X.window_features(recs), rows.mean(axis=0))   # bit-exact
    with pytest.raises(ContractViolation):
        X.window_features([])
    # boundary goes left, count tie predicts MMSE (test_switch_policy.py:151-163)
    tree = TreeModel(Node(counts=(3, 3), feature=0, threshold=1.5,
                          left=Node(counts=(2, 0)), right=Node(counts=(1, 1))),
                     feature_names=tuple(f"f{i}" for i in range(10)))
    x = np.zeros(10)
    x[0] = 1.5
    assert X.predict(tree, x) == 0
    x[0] = 1.6
    assert X.predict(tree, x) == 1
    assert list(X.predict(tree, np.array([[1.0] + [0] * 9, [9.0] + [0] * 9]))) == [0, 1]
