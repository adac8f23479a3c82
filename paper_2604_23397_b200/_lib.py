"""ctypes binding of the native C ABI (`include/arches.h`, `lib/libarches.so`).

The library is the product: there is no Python or CPU fallback.  If the shared
object is missing the import fails loudly (`DeviceError`).
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

from .errors import DeviceError, raise_for_status

LIB_PATH = pathlib.Path(__file__).resolve().parent / "lib" / "libarches.so"

MAX_ANT, MAX_DMRS, MAX_SYM, MAX_BINS, MAX_MCS, MAX_TREE_NODES = 64, 4, 14, 64, 32, 64
EXEC_CONCURRENT, EXEC_SELECTED_ONLY = 0, 1
POLICY_ORACLE, POLICY_FIXED, POLICY_TREE = 0, 1, 2
FLAG_NO_TC_K1, FLAG_NO_TC_K2 = 0x1, 0x2
FLAG_TX_PACKED = 0x4   # tx arguments are the packed QPSK wire format (include/arches.h)
EXPERT_OUT_C128 = 0x100
LLR_STRIDE = 6
TRIGGERS = {0: "policy", 1: "failsafe", 2: "oracle", 3: "fixed"}


class Geom(C.Structure):
    _fields_ = [("n_ant", C.c_int32), ("n_prb", C.c_int32), ("n_sym", C.c_int32),
                ("n_dmrs", C.c_int32), ("dmrs_symbols", C.c_int32 * MAX_DMRS),
                ("slot_duration_us", C.c_double)]


class Params(C.Structure):
    _fields_ = [("noise_guard", C.c_int32), ("truncation", C.c_int32),
                ("mmse_block_prbs", C.c_int32), ("window_length", C.c_int32),
                ("assumed_delay_spread", C.c_double), ("ridge", C.c_double),
                ("sinr_cap_db", C.c_double), ("lcid4_fraction", C.c_double),
                ("lcid4_jitter", C.c_double), ("crc_margin_db", C.c_double),
                ("crc_scale_db", C.c_double), ("mac_header_bytes", C.c_int32),
                ("n_mcs", C.c_int32), ("mcs_threshold_db", C.c_double * MAX_MCS),
                ("mcs_qam", C.c_int32 * MAX_MCS), ("mcs_rate", C.c_double * MAX_MCS),
                ("exec_mode", C.c_int32), ("policy", C.c_int32), ("fixed_mode", C.c_int32),
                ("decision_period_slots", C.c_int32), ("dapp_window_slots", C.c_int32),
                ("flags", C.c_int32), ("decision_delay_ns", C.c_int64),
                ("failsafe_timeout_ns", C.c_int64), ("crc_purpose_key", C.c_uint64)]


class SceneRegime(C.Structure):
    _fields_ = [("noise_var", C.c_double), ("interference_var", C.c_double),
                ("temporal_correlation", C.c_double), ("shadow_sigma_db", C.c_double),
                ("shadow_correlation", C.c_double)]


class TreeNode(C.Structure):
    _fields_ = [("feature", C.c_int32), ("left", C.c_int32), ("right", C.c_int32),
                ("label", C.c_int32), ("threshold", C.c_double)]


class Tree(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("reserved", C.c_int32),
                ("nodes", TreeNode * MAX_TREE_NODES)]


TELEMETRY_DTYPE = np.dtype([
    ("sigma2_hat", "<f8"), ("abs_mean", "<f8", 2), ("rsrp", "<f8", 2), ("sinr_db", "<f8", 2),
    ("mcs", "<i4", 2), ("tb_bytes", "<i4", 2), ("num_cb", "<i4", 2), ("crc", "<i4", 2),
    ("mac_rx", "<i4", 2), ("lcid4_rx", "<i4", 2)])
KPM_DTYPE = np.dtype([
    ("slot_index", "<i8"), ("phy_throughput", "<f8"), ("rsrp", "<f8"), ("code_rate", "<f8"),
    ("snr_db", "<f8"), ("mac_throughput", "<f8"), ("lcid4_throughput", "<f8"),
    ("est_abs_mean", "<f8"), ("mcs_index", "<i4"), ("pdu_length", "<i4"), ("ndi", "<i4"),
    ("qam_order", "<i4"), ("num_cb", "<i4"), ("tb_size", "<i4"), ("mac_rx_bytes", "<i4"),
    ("lcid4_rx_bytes", "<i4"), ("mode", "<i4"), ("crc_pass", "<i4")])
SPLIT_EVAL_DTYPE = np.dtype([("total", "<f8"), ("left_total", "<f8"), ("right_total", "<f8"),
                             ("left_threshold", "<f8"), ("right_threshold", "<f8"),
                             ("left_feature", "<i4"), ("right_feature", "<i4")])
MESSAGE_DTYPE = np.dtype([("decided_at_ns", "<i8"), ("deliverable_at_ns", "<i8"),
                          ("mode", "<i4"), ("trigger", "<i4")])
assert TELEMETRY_DTYPE.itemsize == 104 and KPM_DTYPE.itemsize == 104
assert MESSAGE_DTYPE.itemsize == 24

P = C.c_void_p
_SIGS = {
    "arches_plan_create": (C.c_int, [C.POINTER(Geom), C.POINTER(Params), C.POINTER(P)]),
    "arches_plan_destroy": (C.c_int, [P]),
    "arches_state_bytes": (C.c_size_t, [P, C.c_int32]),
    "arches_workspace_bytes": (C.c_size_t, [P, C.c_int32]),
    "arches_batch_kernels": (C.c_int32, [P]),
    "arches_state_init": (C.c_int, [P, P, C.c_int32, P]),
    "arches_ls_analyze": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P, C.c_int64, P, P, P, P]),
    "arches_experts_equalize": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P, P, C.c_int64, P, P,
                                          P, P, P, P]),
    "arches_kpm_scan": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P, P, P, P, P, C.c_int32, P]),
    "arches_kpm_scan_sequential": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P, P, P, P, P,
                                             C.c_int32, P]),
    "arches_run_batch": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int64, P, P, P, P, P, P, P, P,
                                   P, P, P, P, P, P, C.c_int32, P, P]),
    "arches_run_batch_async": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int64, P, P, P, P, P, P, P,
                                         P, P, P, P, P, P, P, C.c_int32, P, P]),
    "arches_join": (C.c_int, [P, P]),
    "arches_switch_copy": (C.c_int, [P, C.c_int32, P, P, P, P]),
    "arches_switch_copy_one": (C.c_int, [P, P, P, C.c_size_t, P]),
    "arches_ls_materialize": (C.c_int, [P, C.c_int32, P, P, P, P]),
    "arches_expert_from_ls": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P, P, P, P]),
    "arches_equalize": (C.c_int, [P, C.c_int32, P, P, P, P, P, P, P, P, P, P]),
    "arches_downstream": (C.c_int, [P, C.c_int32, P, P, P, P, P, P, P, P]),
    "arches_perturb_mmse": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int64, P, P, P, P, P, P, P,
                                      P, P, P]),
    "arches_tree_eval_splits": (C.c_int, [P, P, P, C.c_int32, C.c_int32, P, P, C.c_int32, P, P]),
    "arches_scene_state_bytes": (C.c_size_t, [P, C.c_int32]),
    "arches_scene_workspace_bytes": (C.c_size_t, [P, C.c_int32]),
    "arches_scene_pilots": (C.c_int, [P, C.c_int32, P, P, P]),
    "arches_synthesize": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P, P, C.c_int32, P, P, P, P,
                                    P, P, P, P, P]),
    "arches_pack_qpsk": (C.c_int, [P, C.c_int32, P, P, P, P]),
    "arches_tx_bits_bytes": (C.c_size_t, [P, C.c_int32]),
    "arches_unpack_qpsk": (C.c_int, [P, C.c_int32, P, P, P]),
    "arches_window_features": (C.c_int, [P, C.c_int32, P, P]),
    "arches_tree_predict": (C.c_int, [P, P, C.c_int32, C.c_int32, P, P]),
    "arches_last_error": (C.c_char_p, []),
    "arches_version": (C.c_char_p, []),
    "arches_host_crc_uniform": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "arches_host_lcid4_jitter": (C.c_double, [C.c_uint64]),
    "arches_host_blake2b64": (C.c_uint64, [C.c_char_p, C.c_size_t]),
    "arches_plan_bins": (C.c_int32, [P]),
    "arches_device_available": (C.c_int32, []),
}
EXPORTED = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """Load libarches.so (build it with `python -m paper_2604_23397_b200.build`)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(f"native library missing: {LIB_PATH} (run the build)")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc:
        raise_for_status(rc, lib().arches_last_error().decode(errors="replace"))


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
