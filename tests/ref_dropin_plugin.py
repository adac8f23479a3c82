"""Test infrastructure: import the STAGED, unmodified reference (`baseline/_ref`,
staged by tools/fetch_ref.py -- /root/reference itself is not on the GPU box)
and, as a pytest plugin (`-p ref_dropin_plugin`), rebind its hot path onto the
device with `compat.install` before the reference's own tests are collected.

The only accommodation is the Python >= 3.11 import fix (harness.py:83 uses a
non-frozen PipelineConfig instance as a dataclass default):
`PipelineConfig` gets an identity hash before the package __init__ imports
harness.  No reference source is modified.
"""
from __future__ import annotations

import importlib
import importlib.util
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
STAGED = ROOT / "baseline" / "_ref"
REF_SRC = STAGED / "ranswitch"
REF_TESTS = STAGED / "refpkg" / "tests"


def staged_reference_missing() -> str | None:
    if not (REF_SRC / "__init__.py").exists() or not REF_TESTS.exists():
        return (f"{STAGED} is not staged: run `python tools/fetch_ref.py` (or "
                "__graft_entry__.build()) in the build container")
    return None


def load_staged_reference():
    if "ranswitch" in sys.modules:
        return sys.modules["ranswitch"]
    why = staged_reference_missing()
    if why:
        raise RuntimeError(why)
    sys.dont_write_bytecode = True
    spec = importlib.util.spec_from_file_location(
        "ranswitch", REF_SRC / "__init__.py", submodule_search_locations=[str(REF_SRC)])
    pkg = importlib.util.module_from_spec(spec)
    sys.modules["ranswitch"] = pkg
    importlib.import_module("ranswitch.phy_pipeline").PipelineConfig.__hash__ = object.__hash__
    spec.loader.exec_module(pkg)
    return pkg


def pytest_configure(config):
    sys.path.insert(0, str(ROOT))
    pkg = load_staged_reference()
    from paper_2604_23397_b200 import compat
    config._arches_saved = compat.install(pkg)
