"""The equalised-symbol data path after the switch (K6, arches_downstream):
x_hat of the selected expert as equalize() forms it (phy_pipeline.py:258-266,
returned at :279) and the max-log demapper (oracle.ref_path.demap_llr).

CPU: the oracle's x_hat is the reference's (the oracle equalize is pinned by
tests/test_oracle_golden.py) and its demapper decides exactly the transmitted
QPSK bits on a clean channel.  GPU: the device x_hat / LLRs against the oracle
over a switching closed loop (modes from K4), on 16QAM / 64QAM schedules too."""
import numpy as np
import pytest

from oracle import ref_path as R
from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
from paper_2604_23397_b200.scene import CellScene, to_device_layout

XHAT_ELEM_TOL = 1e-4   # max |d| <= tol * max |x_hat| (fp32 equaliser, tests/parity.py style)
LLR_TOL = 2e-3         # |d LLR| <= tol * max |LLR| per unit


def test_oracle_demapper_recovers_clean_qpsk_bits():
    geo = SlotGeometry(n_ant=4, n_prb=12)
    scens = {k: v.__class__(**{**v.__dict__, "base_snr_db": 40.0})
             for k, v in default_scenarios(3, geo).items()}
    cs = CellScene(geo, scens, "good")
    s = cs.next_slot("good")
    est = s.h_true[:, None, :, None].repeat(len(geo.dmrs_symbols), axis=3)
    xh, _ = R.equalize(s.y, est, s.noise_var, s.tx, geo)
    llr = R.demap_llr(xh, R.equalizer_gain(est, geo), s.noise_var, 2, geo)
    data = R.data_re_mask(geo)
    b0 = (s.tx.real < 0)[data]
    b1 = (s.tx.imag < 0)[data]
    assert np.array_equal(llr[..., 0][data] < 0, b0)
    assert np.array_equal(llr[..., 1][data] < 0, b1)
    assert (llr[~data] == 0).all() and (llr[..., 2:] == 0).all()
    # 16QAM / 64QAM labels: LLR signs follow the nearest level's Gray label
    for qm in (4, 6):
        l2 = R.demap_llr(xh, R.equalizer_gain(est, geo), s.noise_var, qm, geo)
        assert np.isfinite(l2).all() and (l2[..., qm:] == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("n_prb,n_ant,exec_mode", [(12, 4, ExecutionMode.CONCURRENT),
                                                   (52, 4, ExecutionMode.SELECTED_ONLY),
                                                   (12, 8, ExecutionMode.CONCURRENT)])
def test_device_xhat_and_llrs_match_oracle(n_prb, n_ant, exec_mode):
    import torch
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo = SlotGeometry(n_ant=n_ant, n_prb=n_prb)
    scens = default_scenarios(7, geo)
    regimes = ["good" if (i // 3) % 2 == 0 else "poor" for i in range(12)]
    cs = CellScene(geo, scens, "good")
    slots = [cs.next_slot(r) for r in regimes]
    pcfg = PipelineConfig(window_length=4)
    plan = ArchesPlan(geo, 1.25, pcfg, exec_mode, "oracle")
    eng = SlotEngine(plan, 1, len(slots))
    eng.set_streams(cs.pilots[None], [7])
    eng.load(y=np.stack([to_device_layout(s.y) for s in slots]),
             tx=np.stack([s.tx.T for s in slots]).astype(np.complex64),
             noise_var=[s.noise_var for s in slots], regime=[1 if r == "good" else 0 for r in regimes])
    eng.run()
    xh, llr = eng.downstream_symbols()
    torch.cuda.synchronize()
    recs = eng.kpm_records()[0]
    loop = R.CellLoop(geo, scens, "oracle", exec_mode, pcfg=pcfg, keep_arrays=True)
    for s, r in zip(slots, regimes):
        loop.run_slot(s.y, s.tx, cs.pilots, r)
    res = loop.finish()
    assert recs["mode"].tolist() == res.modes and len(set(res.modes)) == 2
    xh, llr = xh.cpu().numpy(), llr.cpu().numpy()
    for i, (sl, sr) in enumerate(zip(res.slots, slots)):
        ref = sl.x_hat.T                                  # (T, N)
        d = np.abs(xh[i] - ref)
        assert d.max() <= XHAT_ELEM_TOL * np.abs(ref).max(), (i, d.max())
        for qm in (int(recs["qam_order"][i]), 4, 6)[:1]:
            want = R.demap_llr(sl.x_hat, R.equalizer_gain(sl.downstream, geo), sr.noise_var,
                               qm, geo).transpose(1, 0, 2)   # (T, N, 6)
            scale = np.abs(want).max()
            assert np.abs(llr[i] - want).max() <= LLR_TOL * scale, (i, qm)
            sig = np.abs(want) > 1e-3 * scale
            assert np.array_equal(np.sign(llr[i][sig]), np.sign(want[sig]))


@pytest.mark.gpu
@pytest.mark.parametrize("qm", [4, 6])
def test_device_higher_order_demapper(qm):
    """16QAM / 64QAM max-log LLRs (force the scheduled order through the KPM record)."""
    import torch
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo = SlotGeometry(n_ant=4, n_prb=12)
    scens = default_scenarios(9, geo)
    cs = CellScene(geo, scens, "good")
    slots = [cs.next_slot("good") for _ in range(3)]
    plan = ArchesPlan(geo, 1.25, PipelineConfig(window_length=4), policy="fixed:1")
    eng = SlotEngine(plan, 1, 3)
    eng.set_streams(cs.pilots[None], [9])
    eng.load(y=np.stack([to_device_layout(s.y) for s in slots]),
             tx=np.stack([s.tx.T for s in slots]).astype(np.complex64),
             noise_var=[s.noise_var for s in slots], regime=[1, 1, 1])
    eng.run()
    k = eng.kpm.view(3, -1).clone()
    rec = k.cpu().numpy().view(_lib.KPM_DTYPE).reshape(3)
    rec["qam_order"] = qm
    eng.kpm.copy_(torch.from_numpy(rec.view(np.uint8).reshape(-1)))
    _, llr = eng.downstream_symbols(x_hat=False)
    llr = llr.cpu().numpy()
    h = eng.h_mmse.cpu().numpy()
    for i, s in enumerate(slots):
        est = np.transpose(h[i], (0, 2, 1))[:, None].astype(np.complex128)
        xh, _ = R.equalize(s.y, est, s.noise_var, s.tx, geo)
        want = R.demap_llr(xh, R.equalizer_gain(est, geo), s.noise_var, qm, geo).transpose(1, 0, 2)
        scale = np.abs(want).max()
        assert np.abs(llr[i] - want).max() <= LLR_TOL * scale
