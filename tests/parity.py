"""Shared parity helpers: tolerances (stated once) and engine builders."""
from __future__ import annotations

import numpy as np

# fp32 device path vs the fp64 reference (north star: "within a stated fp32
# tolerance on NMSE and per-element relative error")
NMSE_TOL = 1e-9            # ||d||^2 / ||ref||^2 per expert output
ELEM_TOL = 1e-4            # max |d| <= ELEM_TOL * max |ref|
SIGMA2_REL_TOL = 1e-4      # estimate_noise_var
SIGMA2_ABS_FLOOR = 1e-6    # noiseless slots: absolute floor relative to mean |h|^2
SINR_ABS_TOL_DB = 1e-3     # equalize SINR
RSRP_REL_TOL = 1e-5        # mean |H|^2 telemetry
KPM_INT_FIELDS = ("mcs_index", "pdu_length", "ndi", "qam_order", "num_cb", "tb_size",
                  "mac_rx_bytes", "lcid4_rx_bytes")
# throughput fields are integer-derived and rounded like CPython -> bit-exact
KPM_EXACT_FLOAT_FIELDS = ("phy_throughput", "mac_throughput", "lcid4_throughput", "code_rate")
REF_COLUMNS = ("slot_index", "phy_throughput", "mcs_index", "pdu_length", "ndi", "rsrp",
               "code_rate", "qam_order", "num_cb", "tb_size", "snr_db",
               "mac_throughput", "lcid4_throughput", "mac_rx_bytes", "lcid4_rx_bytes")


def to_ref_layout(dev: np.ndarray) -> np.ndarray:
    """device (A, D, N) -> reference (A, 1, N, D)."""
    return np.transpose(dev, (0, 2, 1))[:, None, :, :]


def assert_estimate_close(got: np.ndarray, ref: np.ndarray, what: str = ""):
    d = got.astype(np.complex128) - ref
    nmse = float(np.sum(np.abs(d) ** 2) / max(np.sum(np.abs(ref) ** 2), 1e-300))
    elem = float(np.max(np.abs(d)) / max(np.max(np.abs(ref)), 1e-300))
    assert nmse <= NMSE_TOL, f"{what}: NMSE {nmse:.3e} > {NMSE_TOL}"
    assert elem <= ELEM_TOL, f"{what}: max|d|/max|ref| {elem:.3e} > {ELEM_TOL}"
    return nmse, elem


def assert_sigma2_close(got: float, ref: float, mean_pow: float, what: str = ""):
    tol = max(SIGMA2_REL_TOL * abs(ref), SIGMA2_ABS_FLOOR * mean_pow)
    assert abs(got - ref) <= tol, f"{what}: sigma2 {got!r} vs {ref!r} (tol {tol:.3e})"


def compare_kpms(got, ref_rows: np.ndarray, ref_extra: np.ndarray | None = None):
    """got: structured KPM_DTYPE records (n,); ref_rows: (n, 15) golden rows."""
    ref = {c: ref_rows[:, i] for i, c in enumerate(REF_COLUMNS)}
    assert np.array_equal(got["slot_index"], ref["slot_index"].astype(np.int64))
    for f in KPM_INT_FIELDS:
        bad = np.nonzero(got[f] != ref[f].astype(np.int64))[0]
        assert bad.size == 0, f"{f} differs at slots {bad[:10]}"
    for f in KPM_EXACT_FLOAT_FIELDS:
        bad = np.nonzero(got[f] != ref[f])[0]
        assert bad.size == 0, f"{f} differs at slots {bad[:10]}: {got[f][bad[:3]]} vs {ref[f][bad[:3]]}"
    rs = np.abs(got["rsrp"] - ref["rsrp"]) / np.abs(ref["rsrp"])
    assert rs.max() <= RSRP_REL_TOL, f"rsrp rel err {rs.max():.3e}"
    sn = np.abs(got["snr_db"] - ref["snr_db"])
    assert sn.max() <= SINR_ABS_TOL_DB, f"snr err {sn.max():.3e} dB"
    if ref_extra is not None:
        am = np.abs(got["est_abs_mean"] - ref_extra[:, 1]) / np.abs(ref_extra[:, 1])
        assert am.max() <= RSRP_REL_TOL
        assert np.array_equal(got["crc_pass"], ref_extra[:, 2].astype(np.int32))
    return {"rsrp_rel": float(rs.max()), "snr_abs_db": float(sn.max())}


def build_engine(geo, scen, regimes, exec_mode, pcfg, dcfg, policy, tree, n_slots_per_batch=None):
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    plan = ArchesPlan(geo, scen["good"].assumed_delay_spread, pcfg, exec_mode, policy, dcfg)
    S = n_slots_per_batch or len(regimes)
    return plan, SlotEngine(plan, 1, S, tree=tree)
