"""Switch-semantics property suite (SPEC.md:295-301 invariants, acceptance
criterion 5 at SPEC.md:717) on the device path.

10^4 random mode schedules x 100 slots, run as ONE batch of 10^4 streams x 100
slots through the production executor (arches_run_batch: K1 -> K2 -> K3 -> K4)
and K5 (arches_switch_copy, the reference's aliasing semantics of
switch_select, phy_pipeline.py:81-91).  Each stream replays the same 100-slot
input window (tiny geometry, the reference tests' 2 RX x 4 PRB) under its own
random regime timeline, so the oracle policy (harness.py:205-212) turns each
timeline into a random mode schedule.  Checked per stream and slot:
  * aliasing soundness: the downstream buffer (h_ai after K5) equals the
    selected expert's output element-exact (the MMSE buffer bit-for-bit on
    mode-1 slots, the untouched AI output on mode-0 slots), finite everywhere;
  * slot-boundary semantics: a decision emitted at the end of slot n is
    observable first at n+1 (concurrent); for random mid-slot decision times
    (tree policy, random E3 latency, random period) the mode changes first at
    the slot after the one containing the message time;
  * selected-only lags concurrent by exactly one slot at every switch and
    matches elsewhere -- same-mode slots carry identical per-slot KPMs;
  * control channel off (no decisions in the run) -> every slot MMSE;
  * throughput accounting: sum of tb_size over CRC-pass slots equals the
    cumulative byte count behind phy_throughput.
Budget < 1 min on a B200.
"""
import numpy as np
import pytest

from paper_2604_23397_b200.config import DappConfig, ExecutionMode, LatencyModel, PipelineConfig
from paper_2604_23397_b200.geometry import ScenarioConfig, SlotGeometry
from paper_2604_23397_b200.policy import Node, TreeModel
from paper_2604_23397_b200.scene import CellScene, to_device_layout

pytestmark = pytest.mark.gpu

N_SCHED, N_SLOTS = 10_000, 100
GEO = SlotGeometry(n_ant=2, n_prb=4)
PCFG = PipelineConfig(window_length=5, noise_guard=8)


def _scenarios(seed):
    good = ScenarioConfig(regime="good", seed=seed, interference_excess_delay=8)
    poor = ScenarioConfig(regime="poor", seed=seed, interference_excess_delay=8,
                          interference_prb_mask=(True,) * 4, interference_power_db=0.0)
    return {"good": good, "poor": poor}


_WINDOW = {}


def _window():
    """100 slots of one tiny cell (alternating regimes), device layout."""
    if not _WINDOW:
        scen = _scenarios(3)
        cs = CellScene(GEO, scen, "good")
        sl = [cs.next_slot("good" if (i // 7) % 2 == 0 else "poor") for i in range(N_SLOTS)]
        _WINDOW.update(pilots=cs.pilots, y=np.stack([to_device_layout(s.y) for s in sl]),
                       tx=np.stack([s.tx.T for s in sl]).astype(np.complex64),
                       nv=np.array([s.noise_var for s in sl]))
    return _WINDOW


def _engine(exec_mode, policy, regimes, n_streams, dcfg=None, latency=None, tree=None):
    import torch
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    w = _window()
    plan = ArchesPlan(GEO, 1.25, PCFG, exec_mode, policy, dcfg, latency)
    eng = SlotEngine(plan, n_streams, N_SLOTS, tree=tree, msg_cap=N_SLOTS + 4)
    eng.set_streams(np.broadcast_to(w["pilots"], (n_streams,) + w["pilots"].shape),
                    [7 + 13 * k for k in range(n_streams)])
    dev = eng.y.device
    eng.y.view(n_streams, N_SLOTS, *eng.y.shape[1:]).copy_(
        torch.from_numpy(w["y"]).to(dev)[None].expand(n_streams, *w["y"].shape))
    eng.tx.view(n_streams, N_SLOTS, *eng.tx.shape[1:]).copy_(
        torch.from_numpy(w["tx"]).to(dev)[None].expand(n_streams, *w["tx"].shape))
    eng.noise_var.view(n_streams, N_SLOTS).copy_(
        torch.from_numpy(w["nv"]).to(dev)[None].expand(n_streams, N_SLOTS))
    eng.regime.copy_(torch.from_numpy(regimes.reshape(-1).astype(np.int8)).to(dev))
    return eng


def _random_regimes(rng, n):
    """Per stream a random switching probability, then a random 0/1 timeline."""
    p = rng.uniform(0.0, 0.6, size=(n, 1))
    flips = rng.random((n, N_SLOTS)) < p
    start = rng.integers(0, 2, size=(n, 1))
    return (start ^ (np.cumsum(flips, axis=1) & 1)).astype(np.int8)


@pytest.fixture(scope="module")
def oracle_runs():
    import torch
    rng = np.random.default_rng(2026)
    reg = _random_regimes(rng, N_SCHED)
    out = {}
    for em in (ExecutionMode.CONCURRENT, ExecutionMode.SELECTED_ONLY):
        eng = _engine(em, "oracle", reg, N_SCHED)
        eng.run()
        ai_before = eng.h_ai.clone()
        eng.switch_copy()                      # K5: downstream = buffer_ai (aliasing semantics)
        torch.cuda.synchronize()
        out[em] = dict(kpm=eng.kpm_records(), h_mmse=eng.h_mmse, h_ai_expert=ai_before,
                       downstream=eng.h_ai, eng=eng)
    return reg, out


def test_decisions_apply_at_the_next_boundary(oracle_runs):
    reg, out = oracle_runs
    conc = out[ExecutionMode.CONCURRENT]["kpm"]["mode"]
    sel = out[ExecutionMode.SELECTED_ONLY]["kpm"]["mode"]
    # oracle message at the end of slot n carries regime(n): concurrent applies it at n+1
    want = np.ones_like(conc)
    want[:, 1:] = reg[:, :-1]
    assert np.array_equal(conc, want)
    # ... and selected-only one boundary later
    want_sel = np.ones_like(sel)
    want_sel[:, 2:] = reg[:, :-2]
    assert np.array_equal(sel, want_sel)
    assert (np.diff(conc, axis=1) != 0).sum() > 100_000   # the schedules really switch


def test_selected_only_lags_concurrent_by_exactly_one_slot(oracle_runs):
    _, out = oracle_runs
    kc, ks = out[ExecutionMode.CONCURRENT]["kpm"], out[ExecutionMode.SELECTED_ONLY]["kpm"]
    assert np.array_equal(ks["mode"][:, 1:], kc["mode"][:, :-1])
    # same mode -> same per-slot expert-derived KPMs (the window totals carry history)
    same = ks["mode"] == kc["mode"]
    for f in ("mcs_index", "tb_size", "crc_pass", "snr_db", "rsrp", "est_abs_mean", "num_cb"):
        assert np.array_equal(ks[f][same], kc[f][same]), f


def test_downstream_equals_selected_expert_element_exact(oracle_runs):
    import torch
    _, out = oracle_runs
    for em, r in out.items():
        mode = torch.from_numpy(r["kpm"]["mode"].reshape(-1).copy()).to(r["downstream"].device)
        sel = mode.view(-1, 1, 1, 1) == 1
        want = torch.where(sel, r["h_mmse"], r["h_ai_expert"])
        assert torch.equal(r["downstream"].view(torch.int64), want.view(torch.int64)), em
        assert bool(torch.isfinite(torch.view_as_real(r["downstream"])).all())


def test_throughput_accounting(oracle_runs):
    """sum(tb_size over CRC-pass slots) == cumulative PHY bytes behind phy_throughput
    (phy_pipeline.py:471-480: phy_t = cum * 8 / 1e6 / ((n + 1) * slot_s))."""
    _, out = oracle_runs
    k = out[ExecutionMode.CONCURRENT]["kpm"]
    cum = np.cumsum(np.where(k["crc_pass"] == 1, k["tb_size"], 0), axis=1)
    slot_s = GEO.slot_duration_us * 1e-6
    elapsed = (k["slot_index"] + 1) * GEO.slot_duration_us * 1e-6
    assert np.allclose(k["phy_throughput"] * elapsed * 1e6 / 8.0, cum, rtol=1e-12, atol=1e-6)
    assert slot_s > 0 and (k["crc_pass"] == 1).mean() > 0.2


def test_control_channel_off_runs_all_mmse():
    """No decision inside the run (decision period beyond it): every slot MMSE,
    in both execution modes; the fail-safe never has to act."""
    tree = TreeModel(Node(counts=(5, 1)))   # would say AI -- but is never consulted
    rng = np.random.default_rng(5)
    reg = _random_regimes(rng, 512)
    for em in (ExecutionMode.CONCURRENT, ExecutionMode.SELECTED_ONLY):
        eng = _engine(em, "tree", reg, 512, DappConfig(decision_period_slots=1000,
                                                       window_length_slots=10), tree=tree)
        eng.run()
        k = eng.kpm_records()
        assert (k["mode"] == 1).all()
        assert int(eng.msg_count.sum().item()) == 0


def test_mid_slot_decisions_apply_at_the_next_slot():
    """Tree policy with a random E3 latency and period per configuration: every
    decision lands mid-slot (or on a boundary); the mode it carries is observable
    first at slot ceil(t / slot) (concurrent) and one slot later (selected-only),
    reconstructed from the device's own message log."""
    rng = np.random.default_rng(11)
    slot_ns = GEO.slot_duration_ns
    checked = 0
    for trial in range(6):
        period = int(rng.integers(1, 7))
        lat = LatencyModel(framework_overhead_us=float(rng.uniform(0.0, 900.0)))
        if np.ceil(lat.decision_delay_ns() / (period * slot_ns)) + 2 > 8:
            continue
        feat = 6   # mac_throughput: flips with the channel, so decisions vary
        tree = TreeModel(Node(counts=(4, 4), feature=feat, threshold=float(rng.uniform(0.05, 0.4)),
                              left=Node(counts=(3, 1)), right=Node(counts=(1, 3))))
        reg = _random_regimes(rng, 256)
        for em, extra in ((ExecutionMode.CONCURRENT, 0), (ExecutionMode.SELECTED_ONLY, 1)):
            eng = _engine(em, "tree", reg, 256, DappConfig(decision_period_slots=period,
                                                           window_length_slots=3), lat, tree)
            eng.run()
            k = eng.kpm_records()
            for s in range(256):
                msgs = eng.messages(s)
                mode = np.ones(N_SLOTS, np.int32)
                # SwitchController.begin_slot (phy_pipeline.py:123-139): messages in
                # deliverable order (stable), applied at the first slot n with
                # t <= n * slot (concurrent) or t <= (n - 1) * slot (selected-only)
                # (pending messages first, then forced fail-safe ones, each by time)
                ev = []
                for i, m in enumerate(msgs):
                    t = int(m["deliverable_at_ns"])
                    forced = int(m["trigger"]) == 1       # fail-safe: forced at t, no lag
                    ev.append((-(-t // slot_ns) + (0 if forced else extra), int(forced), t, i))
                for first, _, _, i in sorted(ev):
                    if first < N_SLOTS:
                        mode[first:] = int(msgs[i]["mode"])
                assert np.array_equal(k["mode"][s], mode), (trial, em, s)
                checked += len(msgs)
    assert checked > 1000
