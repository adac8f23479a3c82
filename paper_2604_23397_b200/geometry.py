"""Slot geometry, scenario parameters and estimate containers.

Host-side value types with the reference's attribute names so the drop-in
functions accept either these or the reference objects (duck-typed):
`SlotGeometry` (`radio_scene.py:30-63`), `ScenarioConfig` (`radio_scene.py:66-120`),
`ResourceGrid` (`radio_scene.py:123-127`), `pdp_powers`/`N_TAPS`
(`radio_scene.py:25,130-137`), `Stage`/`ExpertId`/`DmrsEstimate`
(`expert_bank.py:22-37`).
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field, replace
from typing import Any, Optional

import numpy as np

from .errors import ConfigurationError

N_TAPS = 8          # TDL length of the channel model and of the MMSE prior
GOOD, POOR = "good", "poor"


@dataclass(frozen=True)
class SlotGeometry:
    n_ant: int = 4
    n_layers: int = 1
    n_prb: int = 12
    n_sym: int = 14
    dmrs_symbols: tuple = (0, 5, 10)
    slot_duration_us: float = 500.0

    def __post_init__(self):
        if min(self.n_ant, self.n_layers, self.n_prb, self.n_sym) < 1:
            raise ConfigurationError("geometry dimensions must be positive")
        if self.slot_duration_us <= 0:
            raise ConfigurationError("slot_duration_us must be > 0")
        syms = tuple(self.dmrs_symbols)
        if list(syms) != sorted(set(syms)) or any(s >= self.n_sym or s < 0 for s in syms):
            raise ConfigurationError("dmrs_symbols must be strictly increasing and < n_sym")

    @property
    def n_sc(self) -> int:
        return 12 * self.n_prb

    @property
    def n_comb(self) -> int:
        return 6 * self.n_prb

    @property
    def n_dmrs(self) -> int:
        return len(self.dmrs_symbols)

    @property
    def comb(self) -> np.ndarray:
        return np.arange(0, self.n_sc, 2)

    @property
    def slot_duration_ns(self) -> int:
        return int(round(self.slot_duration_us * 1000))


@dataclass(frozen=True)
class ScenarioConfig:
    regime: str = GOOD
    base_snr_db: float = 20.0
    interference_prb_mask: tuple = ()
    interference_power_db: float = 3.0
    delay_spread: float = 3.0
    temporal_correlation: float = 0.9
    shadow_sigma_db: float = 4.0
    shadow_correlation: float = 0.9355
    seed: int = 0
    interference_excess_delay: int = 32
    mmse_assumed_delay_spread: Optional[float] = None

    def __post_init__(self):
        if self.regime not in (GOOD, POOR):
            raise ConfigurationError(f"unknown regime {self.regime!r}")
        for name in ("temporal_correlation", "shadow_correlation"):
            v = getattr(self, name)
            if not (0.0 <= v <= 1.0 - 1e-12):
                raise ConfigurationError(f"{name}={v} outside [0, 1)")
        if self.delay_spread < 0 or self.shadow_sigma_db < 0 or self.interference_excess_delay < 0:
            raise ConfigurationError("delay_spread, shadow_sigma_db, excess delay must be >= 0")
        if self.regime == GOOD and any(self.interference_prb_mask):
            raise ConfigurationError("good regime implies an all-clear interference mask")

    @property
    def assumed_delay_spread(self) -> float:
        return self.delay_spread if self.mmse_assumed_delay_spread is None \
            else self.mmse_assumed_delay_spread

    def noise_var(self, n_ant: int = 4) -> float:
        if math.isinf(self.base_snr_db):
            return 0.0
        return n_ant / 10.0 ** (self.base_snr_db / 10.0)

    def interference_var(self) -> float:
        if self.regime == GOOD or not any(self.interference_prb_mask):
            return 0.0
        return 10.0 ** (self.interference_power_db / 10.0)


def default_scenarios(seed: int, geometry: SlotGeometry | None = None) -> dict:
    """The two-regime setup of `harness.py:39-59`: SNR 20 dB, delay spread 3,
    MMSE prior 1.25; poor adds a full-band 0 dB co-channel interferer."""
    geometry = geometry or SlotGeometry()
    good = ScenarioConfig(regime=GOOD, base_snr_db=20.0, delay_spread=3.0,
                          temporal_correlation=0.9, seed=seed,
                          mmse_assumed_delay_spread=1.25)
    poor = replace(good, regime=POOR, interference_prb_mask=(True,) * geometry.n_prb,
                   interference_power_db=0.0)
    return {GOOD: good, POOR: poor}


def pdp_powers(delay_spread: float, n_taps: int = N_TAPS) -> np.ndarray:
    """Exponential power-delay profile, normalised to unit sum."""
    if delay_spread <= 0:
        out = np.zeros(n_taps)
        out[0] = 1.0
        return out
    e = np.exp(-np.arange(n_taps) / delay_spread)
    return e / e.sum()


@dataclass
class ResourceGrid:
    values: Any            # (n_ant, n_sc, n_sym) received samples
    known_dmrs: Any        # (n_comb, n_dmrs) unit-magnitude pilots
    geometry: SlotGeometry


class Stage(enum.Enum):
    RAW_LS = "RawLS"
    INTERPOLATED = "Interpolated"


class ExpertId(enum.Enum):
    MMSE = 1
    AI = 0


@dataclass
class DmrsEstimate:
    values: Any            # (n_ant, n_layers, n_sc, n_dmrs)
    stage: Stage
    comb_mask: np.ndarray
    geometry: SlotGeometry
    device: Any = field(default=None, repr=False, compare=False)  # device-resident copy
