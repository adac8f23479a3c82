"""Host-side logic that runs without a GPU: configuration records, the tree
text format, plan-level validation mirrors, the compat install() rebinding
mechanics, and the scene generator's pinned properties."""
import types

import numpy as np
import pytest

from golden_io import GOLDEN, tree_text
from paper_2604_23397_b200 import compat
from paper_2604_23397_b200.config import (DEFAULT_MCS_TABLE, DappConfig, LatencyModel, McsTable,
                                          PipelineConfig)
from paper_2604_23397_b200.errors import ConfigurationError
from paper_2604_23397_b200.geometry import (ScenarioConfig, SlotGeometry, default_scenarios,
                                            pdp_powers)
from paper_2604_23397_b200.policy import from_text, to_device_struct, to_text
from paper_2604_23397_b200.scene import lcid4_jitter, purpose_key


def test_latency_and_dapp_config_kats():
    # test_dapp_control.py:33-48
    assert LatencyModel().total_us() == pytest.approx(139.91, abs=1e-9)
    assert LatencyModel().decision_delay_ns() == 135_410
    assert DappConfig().timeout_ns(500_000) == 10 * 100 * 500_000
    assert DappConfig(failsafe_timeout_us=2.5).timeout_ns(500_000) == 2500
    with pytest.raises(ConfigurationError):
        DappConfig(decision_period_slots=0)
    with pytest.raises(ConfigurationError):
        LatencyModel(framework_overhead_us=-1.0)


def test_mcs_table_validation():
    with pytest.raises(ConfigurationError):
        McsTable(thresholds_db=(0.0, 1.0), qam_order=(2,), code_rate=(0.5, 0.6))
    with pytest.raises(ConfigurationError):
        McsTable(thresholds_db=(1.0, 1.0), qam_order=(2, 2), code_rate=(0.5, 0.6))
    with pytest.raises(ConfigurationError):
        McsTable(thresholds_db=(0.0, 1.0), qam_order=(2, 2), code_rate=(0.6, 0.5))
    assert DEFAULT_MCS_TABLE.n_mcs == 29


def test_geometry_and_scenario():
    g = SlotGeometry()
    assert (g.n_sc, g.n_dmrs, g.n_comb, g.slot_duration_ns) == (144, 3, 72, 500_000)
    with pytest.raises(ConfigurationError):
        SlotGeometry(dmrs_symbols=(0, 14))
    with pytest.raises(ConfigurationError):
        ScenarioConfig(regime="good", interference_prb_mask=(True,))
    s = default_scenarios(5)
    assert s["poor"].interference_prb_mask == (True,) * 12
    assert s["good"].assumed_delay_spread == 1.25
    assert s["good"].noise_var(4) == pytest.approx(0.04)
    p = pdp_powers(3.0)
    assert p.sum() == pytest.approx(1.0) and np.all(np.diff(p) < 0)


def test_tree_text_round_trip():
    for name in ("tree12", "tree52"):
        text = tree_text(name)
        tree = from_text(text)
        assert to_text(tree) == text
        s = to_device_struct(tree)
        assert s.n_nodes == len(tree.nodes())
    with pytest.raises(ConfigurationError):
        from_text("tree v2\nfeatures: a\n0 leaf label=1 counts=0,1\n")


def test_purpose_keys_and_jitter_match_golden():
    import json
    g = json.loads((GOLDEN / "rng.json").read_text())
    for p, k in g["purpose_keys"].items():
        assert purpose_key(p) == k
    for slot, j in g["lcid4_jitter"][:50]:
        assert lcid4_jitter(slot) == j


def test_install_rebinds_by_name_and_restores():
    """install() swaps the names phy_pipeline/dapp_control/expert_bank bound at
    import time and switches to the package's exception classes."""
    class CE(ValueError):
        pass

    class CV(ValueError):
        pass

    def orig(*a, **k):
        return "reference"

    pkg = types.SimpleNamespace(
        phy_pipeline=types.SimpleNamespace(**{n: orig for n in compat.NAMES_PHY}),
        expert_bank=types.SimpleNamespace(**{n: orig for n in compat.NAMES_EXPERT_BANK},
                                          DmrsEstimate=object, Stage=object, ExpertId=object),
        dapp_control=types.SimpleNamespace(**{n: orig for n in compat.NAMES_DAPP}),
        validation=types.SimpleNamespace(ConfigurationError=CE, ContractViolation=CV,
                                         EstimatorError=RuntimeError,
                                         PipelineStateError=RuntimeError))
    saved = compat.install(pkg)
    try:
        assert pkg.phy_pipeline.mmse_estimate is compat.mmse_estimate
        assert pkg.phy_pipeline.ExpertBuffers is compat.ExpertBuffers
        assert pkg.dapp_control.predict is compat.predict
        assert pkg.expert_bank.ls_estimate is compat.ls_estimate
        # contract errors are raised as the reference's classes (no device needed)
        est = types.SimpleNamespace(stage=types.SimpleNamespace(value="Interpolated"))
        with pytest.raises(CV):
            compat.mmse_estimate(est, 0.1, None)
        with pytest.raises(CV):
            compat.window_features([])
    finally:
        compat.uninstall(pkg, saved)
    assert pkg.phy_pipeline.mmse_estimate is orig
