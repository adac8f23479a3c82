"""Eq. 3 perturbation of the MMSE expert (perturbation_lab.py:92-144; the
Pipeline.perturb hook, phy_pipeline.py:401,444-445).

CPU: the oracle's perturbed loop reproduces the reference's per-slot traces
(tools/make_golden_perturb.py) bit-for-bit, and the reference's own
perturbation_lab.sweep table from those traces.  GPU (K7, arches_perturb_mmse):
one stream per rho, the device traces against the reference (integer KPMs and
CRC exact, rsrp / SINR within tests/parity.py), the perturbed MMSE buffer
within the expert tolerance, rho = 0 bit-identical to an unperturbed run, and
the SPEC acceptance statistics of the injection (E|dH|^2 within 2% of
(rho E|H|)^2 over 1e6 elements)."""
import json
import pathlib

import numpy as np
import pytest

from oracle import ref_path as R
from parity import REF_COLUMNS, assert_estimate_close, compare_kpms
from paper_2604_23397_b200.config import ExecutionMode
from paper_2604_23397_b200.geometry import ScenarioConfig, SlotGeometry
from paper_2604_23397_b200.scene import CellScene, to_device_layout

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def _gold():
    meta = json.loads((GOLD / "perturb.json").read_text())
    arr = np.load(GOLD / "perturb.npz")
    return meta, arr


def _setup():
    meta, arr = _gold()
    kw = dict(meta["scenario"])
    kw["interference_prb_mask"] = tuple(kw.get("interference_prb_mask", ()))
    scen = ScenarioConfig(**kw)
    geo = SlotGeometry(n_prb=meta["n_prb"])
    cs = CellScene(geo, {"good": scen}, "good")
    slots = [cs.next_slot("good") for _ in range(meta["slots"])]
    return meta, arr, geo, scen, cs, slots


def test_oracle_perturbed_loop_matches_reference():
    meta, arr, geo, scen, cs, slots = _setup()
    for i, rho in enumerate(meta["rhos"]):
        loop = R.CellLoop(geo, {"good": scen}, "oracle", ExecutionMode.SELECTED_ONLY,
                          perturb_rho=rho, keep_arrays=True)
        for s in slots:
            loop.run_slot(s.y, s.tx, cs.pilots, "good")
        res = loop.finish()
        rows = np.array([[float(v) for v in k.row()] for k in res.records])
        assert np.array_equal(rows, arr[f"rho{i}__records"]), rho
        ext = np.array([[sl.sinr_db, sl.est_abs_mean, float(sl.crc)] for sl in res.slots])
        assert np.array_equal(ext, arr[f"rho{i}__extra"]), rho
        for s in range(2):
            assert np.array_equal(res.slots[s].mmse, arr[f"rho{i}__mmse_slot{s}"])


def test_reference_sweep_table_from_the_traces():
    """perturbation_lab.sweep's means are per-rho slot means of the same traces."""
    meta, arr, geo, scen, cs, slots = _setup()
    sw = meta["sweep"]
    names = sw["kpm_names"]
    for j, rho in enumerate(sw["rho_values"]):
        loop = R.CellLoop(geo, {"good": scen}, "oracle", ExecutionMode.SELECTED_ONLY,
                          perturb_rho=rho)
        for s in slots[:sw["slots_per_point"]]:
            loop.run_slot(s.y, s.tx, cs.pilots, "good")
        res = loop.finish()
        for i, name in enumerate(names):
            if name == "est_abs_mean":
                col = [sl.est_abs_mean for sl in res.slots]
            elif name == "est_abs_sq":
                col = [sl.est_abs_mean ** 2 for sl in res.slots]
            else:
                col = [getattr(k, name) for k in res.records]
            assert np.mean(col) == pytest.approx(arr["sweep__mean"][i, j], rel=1e-12, abs=1e-12), \
                (name, rho)


@pytest.mark.gpu
def test_device_perturbation_matches_reference():
    import torch
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    meta, arr, geo, scen, cs, slots = _setup()
    rhos = meta["rhos"]
    C, S = len(rhos), meta["slots"]
    plan = ArchesPlan(geo, scen.assumed_delay_spread, exec_mode=ExecutionMode.SELECTED_ONLY,
                      policy="oracle")
    eng = SlotEngine(plan, C, S)
    eng.set_streams(np.stack([cs.pilots] * C), [scen.seed] * C)
    one = [to_device_layout(s.y) for s in slots]
    eng.load(y=np.stack(one * C), tx=np.stack([s.tx.T for s in slots] * C).astype(np.complex64),
             noise_var=[s.noise_var for s in slots] * C, regime=[1] * (C * S))
    eng.run_perturbed(rhos)
    torch.cuda.synchronize()
    recs = eng.kpm_records()
    mm = eng.h_mmse.cpu().numpy().reshape(C, S, *eng.h_mmse.shape[1:])
    for i, rho in enumerate(rhos):
        assert (recs[i]["mode"] == 1).all()
        compare_kpms(recs[i], arr[f"rho{i}__records"], arr[f"rho{i}__extra"])
        for s in range(2):
            dev = np.transpose(mm[i, s], (0, 2, 1))[:, None]
            assert_estimate_close(dev, arr[f"rho{i}__mmse_slot{s}"], f"rho {rho} slot {s}")


@pytest.mark.gpu
def test_rho_zero_is_the_unperturbed_path():
    import torch
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    meta, arr, geo, scen, cs, slots = _setup()
    out = []
    for perturbed in (False, True):
        plan = ArchesPlan(geo, scen.assumed_delay_spread, exec_mode=ExecutionMode.SELECTED_ONLY)
        eng = SlotEngine(plan, 1, 12)
        eng.set_streams(cs.pilots[None], [scen.seed])
        eng.load(y=np.stack([to_device_layout(s.y) for s in slots[:12]]),
                 tx=np.stack([s.tx.T for s in slots[:12]]).astype(np.complex64),
                 noise_var=[s.noise_var for s in slots[:12]], regime=[1] * 12)
        if perturbed:
            eng.run_perturbed([0.0])
        else:
            eng.run()
        torch.cuda.synchronize()
        out.append((eng.kpm.cpu().numpy(), eng.h_mmse.cpu().numpy(), eng.tel.cpu().numpy()))
    for a, b in zip(*out):
        assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("rho", [0.5, 1.0, 2.0])
def test_injection_statistics(rho):
    """SPEC acceptance 1: E|H_noisy - H|^2 within 2% of (rho E|H|)^2 over ~1e6 elements."""
    import torch
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    meta, arr, geo, scen, cs, slots = _setup()
    S = 40   # 40 slots x 4 ant x 144 sc x 3 dmrs x 16 streams = 1.1e6 elements
    C = 16
    plan = ArchesPlan(geo, scen.assumed_delay_spread, exec_mode=ExecutionMode.SELECTED_ONLY)
    eng = SlotEngine(plan, C, S)
    eng.set_streams(np.stack([cs.pilots] * C), [scen.seed + c for c in range(C)])
    eng.load(y=np.stack([to_device_layout(s.y) for s in slots[:S]] * C),
             tx=np.stack([s.tx.T for s in slots[:S]] * C).astype(np.complex64),
             noise_var=[s.noise_var for s in slots[:S]] * C, regime=[1] * (C * S))
    eng.run()
    clean = eng.h_mmse.clone()
    m = torch.from_numpy(eng.telemetry()["abs_mean"][..., 1].reshape(-1).copy()).cuda()
    eng.reset()
    eng.run_perturbed([rho] * C)
    d = (eng.h_mmse - clean).abs() ** 2
    per_unit = d.reshape(C * S, -1).mean(dim=1) / (rho * m) ** 2
    got = float(per_unit.mean())
    assert d.numel() > 1_000_000
    assert abs(got - 1.0) < 0.02, got
