"""Error taxonomy of the drop-in boundary.

Mirrors the four exception classes of the reference
(`pkg/src/ranswitch/validation.py:9-26`) with the same base classes, so code
written against the reference (`except ConfigurationError`, `except ValueError`)
behaves identically.  The C-ABI reports failures as integer status codes
(`include/arches.h`, `ARCHES_E_*`); `raise_for_status` maps them 1:1 onto these
classes.
"""
from __future__ import annotations


class ConfigurationError(ValueError):
    """Invalid configuration (ranges, guard/truncation, n_layers != 1)."""


class ContractViolation(ValueError):
    """Input violates a call contract (shape, NaN, zero pilot, wrong stage)."""


class EstimatorError(RuntimeError):
    """Numerical failure inside an estimator; carries a diagnostic."""

    def __init__(self, msg, condition_number=None):
        super().__init__(msg)
        self.condition_number = condition_number


class PipelineStateError(RuntimeError):
    """A buffer was consumed before the owning expert populated it."""


class DeviceError(RuntimeError):
    """CUDA runtime failure or missing native library (never silently ignored)."""


# status codes shared with include/arches.h
ARCHES_OK = 0
ARCHES_E_CONFIG = 1
ARCHES_E_CONTRACT = 2
ARCHES_E_ESTIMATOR = 3
ARCHES_E_STATE = 4
ARCHES_E_CUDA = 5

_BY_CODE = {
    ARCHES_E_CONFIG: ConfigurationError,
    ARCHES_E_CONTRACT: ContractViolation,
    ARCHES_E_ESTIMATOR: EstimatorError,
    ARCHES_E_STATE: PipelineStateError,
    ARCHES_E_CUDA: DeviceError,
}


def raise_for_status(code: int, message: str) -> None:
    if code == ARCHES_OK:
        return
    raise _BY_CODE.get(code, DeviceError)(message or f"arches status {code}")
