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
