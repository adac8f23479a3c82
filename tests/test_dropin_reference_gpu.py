"""The drop-in claim on the REAL reference.

The unmodified reference package staged under baseline/_ref (tools/fetch_ref.py)
is imported, `compat.install(ranswitch)` rebinds its hot path
(phy_pipeline.{ls_estimate, estimate_noise_var, mmse_estimate, denoiser_estimate,
switch_select, equalize, ExpertBuffers}, dapp_control.{window_features, predict})
onto the B200, and then
  1. the reference's own `harness.execute_run` (harness.py:174-231) reproduces the
     golden closed loops recorded from the pure reference: modes, control
     messages and integer KPMs bit-exact, rsrp / SINR within tests/parity.py;
  2. the reference's own hot-path test modules (test_expert_bank.py,
     test_phy_pipeline.py, test_dapp_control.py, test_switch_policy.py,
     test_harness.py) run with the device rebound.  Every test must pass except
     the ones listed in KNOWN_PRECISION with their reason (bit-exact float64
     asserts that a complex64 device path cannot meet).
  3. compat.equalize's x_hat is value-checked against the reference's.
The staged reference is required: a missing stage is a failure, not a skip.
"""
import os
import pathlib
import subprocess
import sys
import xml.etree.ElementTree as ET

import numpy as np
import pytest

from golden_io import loops
from parity import compare_kpms
from ref_dropin_plugin import REF_TESTS, ROOT, load_staged_reference, staged_reference_missing

pytestmark = pytest.mark.gpu

# reference tests whose assertion is an exact float64 identity (complex128 in,
# complex128 out) that a complex64 device path does not meet bit-for-bit; each
# is covered by a tolerance test in this repo (named in the reason)
KNOWN_PRECISION = {
}

LOOP_IDS = ["tiny_oracle_conc", "tiny_oracle_sel", "tiny_fixed0", "tiny_alt_oracle",
            "p12_oracle_conc", "p12_alt_sel", "p12_tree_failsafe", "p52_alt_oracle"]


def test_reference_is_staged():
    assert staged_reference_missing() is None, staged_reference_missing()


@pytest.fixture(scope="module")
def installed():
    pkg = load_staged_reference()
    from paper_2604_23397_b200 import compat
    saved = compat.install(pkg)
    pkg._arches_originals = saved
    yield pkg
    compat.uninstall(pkg, saved)


@pytest.mark.parametrize("lid", LOOP_IDS)
def test_execute_run_with_device_rebound(installed, lid):
    from paper_2604_23397_b200 import compat
    H, RS, PP, DC, SP = (installed.harness, installed.radio_scene, installed.phy_pipeline,
                         installed.dapp_control, installed.switch_policy)
    assert PP.mmse_estimate is compat.mmse_estimate and DC.predict is compat.predict
    m, recs, extra = {m["id"]: (m, r, e) for m, r, e in loops()}[lid]
    g = m["geometry"]
    geo = RS.SlotGeometry(n_ant=g["n_ant"], n_prb=g["n_prb"])
    scen = {}
    for k, v in m["scenarios"].items():
        kw = dict(v)
        kw["interference_prb_mask"] = tuple(kw.get("interference_prb_mask", ()))
        scen[k] = RS.ScenarioConfig(**kw)
    p = m["pipeline"]
    pcfg = PP.PipelineConfig(window_length=p["window_length"], noise_guard=p["noise_guard"],
                             truncation=p["truncation"], mmse_block_prbs=p["mmse_block_prbs"])
    d = m["dapp"]
    dcfg = DC.DappConfig(decision_period_slots=d["decision_period_slots"],
                         window_length_slots=d["window_length_slots"],
                         failsafe_timeout_us=d["failsafe_timeout_us"])
    tree = None
    if m["tree"]:
        from golden_io import tree_text
        tree = SP.from_text(tree_text(m["tree"]))
    policy = "tree:golden" if m["policy"] == "tree" else m["policy"]
    spec = H.ExperimentSpec(timeline=tuple(tuple(t) for t in m["timeline"]),
                            exec_mode=PP.ExecutionMode(m["exec_mode"]), policy=policy,
                            seed=m["seed"], geometry=geo, scenarios=scen, pipeline_config=pcfg,
                            dapp_config=dcfg)
    run = H.execute_run(spec, tree=tree)
    assert run.modes() == m["modes"]
    assert [[x.mode, x.decided_at_ns, x.deliverable_at_ns, x.trigger] for x in run.messages] \
        == m["messages"]
    assert list(run.failsafe_events) == m["failsafe_events"]
    from paper_2604_23397_b200._lib import KPM_DTYPE
    rows = np.array([[float(v) for v in r.row()] for r in run.records])
    got = np.zeros(len(rows), KPM_DTYPE)
    from parity import REF_COLUMNS
    for i, c in enumerate(REF_COLUMNS):
        got[c] = rows[:, i]
    got["est_abs_mean"] = [o.est_abs_mean for o in run.outcomes]
    got["crc_pass"] = [int(o.crc_pass) for o in run.outcomes]
    compare_kpms(got, recs, extra)


def test_equalize_x_hat_matches_reference(installed):
    """compat.equalize returns the reference's x_hat (phy_pipeline.py:262-266, returned
    at :279) within the fp32 tolerance, and the same SINR."""
    from golden_io import small_case
    from paper_2604_23397_b200 import compat
    RS, EB = installed.radio_scene, installed.expert_bank
    ref_equalize = installed._arches_originals[("phy_pipeline", "equalize")]
    assert ref_equalize is not compat.equalize
    for cid in ("good_12prb", "poor_12prb", "snr5_4prb_1ant", "blocked_64prb"):
        c, dat = small_case(cid)
        geo = RS.SlotGeometry(n_ant=c["n_ant"], n_prb=c["n_prb"])
        rx = RS.ResourceGrid(values=dat["y"], known_dmrs=dat["pilots"], geometry=geo)
        est = EB.DmrsEstimate(dat["mmse"], EB.Stage.INTERPOLATED, np.ones(geo.n_sc, bool), geo)
        xh_dev, s_dev = installed.phy_pipeline.equalize(rx, est, c["noise_var"], dat["tx"])
        xh_ref, s_ref = ref_equalize(rx, est, c["noise_var"], dat["tx"])
        assert xh_dev.shape == xh_ref.shape and xh_dev.dtype == xh_ref.dtype
        d = np.abs(xh_dev - xh_ref)
        assert d.max() <= 1e-4 * np.abs(xh_ref).max(), (cid, d.max())
        nmse = np.sum(d ** 2) / np.sum(np.abs(xh_ref) ** 2)
        assert nmse <= 1e-9, (cid, nmse)
        assert abs(s_dev - s_ref) <= 1e-3


def test_reference_test_suite_with_device_rebound(tmp_path):
    """Run the reference's own hot-path tests with the device rebound."""
    mods = ["test_expert_bank.py", "test_phy_pipeline.py", "test_dapp_control.py",
            "test_switch_policy.py", "test_harness.py"]
    xml = tmp_path / "ref.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(ROOT / "tests"),
                                         env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_dropin_plugin", "-p", "no:cacheprovider",
           "-q", f"--junitxml={xml}", "--rootdir", str(REF_TESTS.parent),
           *[str(REF_TESTS / m) for m in mods]]
    res = subprocess.run(cmd, cwd=REF_TESTS.parent, env=env, capture_output=True, text=True,
                         timeout=1500)
    assert xml.exists(), res.stdout[-3000:] + res.stderr[-3000:]
    results = {}
    for tc in ET.parse(xml).getroot().iter("testcase"):
        name = f"{tc.get('classname').split('.')[-1]}.py::{tc.get('name')}"
        status = "passed"
        for child in tc:
            if child.tag in ("failure", "error"):
                status = "failed"
            elif child.tag == "skipped":
                status = "skipped"
        results[name] = (status, "".join(child.get("message", "") for child in tc)[:300])
    print("\n".join(f"{k}: {v[0]} {v[1]}" for k, v in sorted(results.items())))
    assert len(results) >= 60, res.stdout[-3000:]
    failed = {k: v for k, v in results.items() if v[0] == "failed"}
    unexpected = {k: v for k, v in failed.items() if k not in KNOWN_PRECISION}
    assert not unexpected, unexpected
