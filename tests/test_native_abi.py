"""The C ABI library loads without a GPU, exports every symbol include/arches.h
declares, and its host-side generators match the reference bit-for-bit."""
import pathlib
import re

import numpy as np

from golden_io import rng_vectors
from paper_2604_23397_b200 import _lib

HEADER = pathlib.Path(__file__).resolve().parents[1] / "include" / "arches.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(arches_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)   # the binding covers the whole header
    assert b"sm_100a" in lib.arches_version()


def test_host_philox_crc_uniform_matches_numpy_stream():
    g = rng_vectors()
    key = g["purpose_keys"]["crc"]
    for seed, slot, u in g["crc_uniform"]:
        assert _lib.lib().arches_host_crc_uniform(seed, key, slot) == u


def test_host_blake2b_and_lcid4_jitter():
    g = rng_vectors()
    L = _lib.lib()
    for purpose, key in g["purpose_keys"].items():
        assert L.arches_host_blake2b64(purpose.encode(), len(purpose)) == key
    for slot, jit in g["lcid4_jitter"]:
        assert L.arches_host_lcid4_jitter(slot) == jit


def test_struct_layouts_match_header():
    import ctypes as C
    assert C.sizeof(_lib.Geom) == 40
    assert C.sizeof(_lib.TreeNode) == 24
    assert _lib.KPM_DTYPE.itemsize == 104 and _lib.TELEMETRY_DTYPE.itemsize == 104


def test_error_codes_map_onto_reference_classes():
    from paper_2604_23397_b200 import errors as E
    for code, cls in ((1, E.ConfigurationError), (2, E.ContractViolation),
                      (3, E.EstimatorError), (4, E.PipelineStateError)):
        try:
            E.raise_for_status(code, "x")
        except cls:
            pass
        else:  # pragma: no cover
            raise AssertionError(cls)
    assert issubclass(E.ConfigurationError, ValueError)
    assert issubclass(E.ContractViolation, ValueError)
    assert issubclass(E.EstimatorError, RuntimeError)


def test_plan_rejects_control_queues_the_device_cannot_hold():
    """A decision delay spanning more decision periods than the device's
    in-flight message queue (ARCHES_MAX_PENDING) is a configuration error at
    plan creation (the check runs before any device call), never a silently
    dropped message (the reference list is unbounded, phy_pipeline.py:114-117)."""
    import pytest
    from paper_2604_23397_b200 import errors as E
    from paper_2604_23397_b200.config import DappConfig, LatencyModel
    from paper_2604_23397_b200.engine import ArchesPlan
    from paper_2604_23397_b200.geometry import SlotGeometry
    geo = SlotGeometry(n_ant=2, n_prb=4)
    # 10 ms of framework latency at a 1-slot decision period: ~20 messages in flight
    lat = LatencyModel(framework_overhead_us=10_000.0)
    with pytest.raises(E.ConfigurationError, match="in flight"):
        ArchesPlan(geo, 1.25, policy="tree", dapp=DappConfig(decision_period_slots=1,
                                                              window_length_slots=1),
                   latency=lat)
