"""Configuration records of the hot path (host side, plain values).

Same field names and defaults as the reference so configs and call sites carry
over unchanged: `McsTable`/`DEFAULT_MCS_TABLE` (`phy_pipeline.py:149-186`),
`PipelineConfig` (`phy_pipeline.py:353-374`), `ExecutionMode`
(`phy_pipeline.py:28-30`), `LatencyModel` (`dapp_control.py:26-46`),
`DappConfig` (`dapp_control.py:53-68`).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Optional

from .errors import ConfigurationError

CB_SEGMENT_BITS = 8448
N_DATA_SYM = 11


class ExecutionMode(enum.Enum):
    CONCURRENT = "concurrent"
    SELECTED_ONLY = "selected"


@dataclass(frozen=True)
class McsTable:
    thresholds_db: tuple
    qam_order: tuple
    code_rate: tuple

    def __post_init__(self):
        t, q, r = self.thresholds_db, self.qam_order, self.code_rate
        if not (len(t) == len(q) == len(r)):
            raise ConfigurationError("MCS table columns must align")
        if any(b <= a for a, b in zip(t, t[1:])):
            raise ConfigurationError("MCS thresholds must be strictly increasing")
        se = [a * b for a, b in zip(q, r)]
        if any(b < a for a, b in zip(se, se[1:])):
            raise ConfigurationError("spectral efficiency must be non-decreasing")

    @property
    def n_mcs(self) -> int:
        return len(self.thresholds_db)


DEFAULT_MCS_TABLE = McsTable(
    thresholds_db=(-9.0, -7.95, -6.9, -5.85, -4.8, -3.75, -2.7, -1.65, -0.6, 0.45,
                   1.9, 3.6, 5.8, 6.6, 8.5, 10.5, 12.4,
                   14.4, 16.4, 18.3, 19.5, 20.3, 21.1, 21.9, 22.7, 23.5, 24.3, 25.1, 25.9),
    qam_order=(2,) * 10 + (4,) * 7 + (6,) * 12,
    code_rate=(0.12, 0.15, 0.19, 0.24, 0.30, 0.37, 0.44, 0.51, 0.59, 0.66,
               0.34, 0.38, 0.43, 0.48, 0.54, 0.60, 0.64,
               0.43, 0.46, 0.50, 0.54, 0.58, 0.63, 0.67, 0.72, 0.77, 0.82, 0.86, 0.93),
)


@dataclass(eq=False)
class PipelineConfig:
    window_length: int = 100
    lcid4_fraction: float = 0.85
    lcid4_jitter: float = 0.03
    crc_margin_db: float = 6.0
    crc_scale_db: float = 2.0
    truncation: int = 20
    mac_header_bytes: int = 3
    sinr_cap_db: float = 60.0
    mmse_block_prbs: int = 32
    noise_guard: int = 16
    mcs_table: McsTable = field(default_factory=lambda: DEFAULT_MCS_TABLE)

    @classmethod
    def from_dict(cls, cfg: dict) -> "PipelineConfig":
        p = cfg.get("pipeline", {})
        keys = ("window_length", "lcid4_fraction", "lcid4_jitter", "crc_margin_db",
                "crc_scale_db", "truncation", "mac_header_bytes", "sinr_cap_db",
                "mmse_block_prbs", "noise_guard")
        return cls(**{k: p[k] for k in keys if k in p})


@dataclass(frozen=True)
class LatencyModel:
    framework_overhead_us: float = 135.0
    policy_inference_us: float = 0.41
    switch_exec_us: float = 4.5

    def __post_init__(self):
        if min(self.framework_overhead_us, self.policy_inference_us, self.switch_exec_us) < 0:
            raise ConfigurationError("latency components must be >= 0")

    def total_us(self) -> float:
        return self.framework_overhead_us + self.policy_inference_us + self.switch_exec_us

    def decision_delay_ns(self) -> int:
        return int(round((self.framework_overhead_us + self.policy_inference_us) * 1000.0))


@dataclass(frozen=True)
class DappConfig:
    decision_period_slots: int = 100
    window_length_slots: int = 100
    failsafe_timeout_us: Optional[float] = None

    def __post_init__(self):
        if self.decision_period_slots < 1 or self.window_length_slots < 1:
            raise ConfigurationError("periods must be positive")
        if self.failsafe_timeout_us is not None and self.failsafe_timeout_us <= 0:
            raise ConfigurationError("failsafe timeout must be positive")

    def timeout_ns(self, slot_duration_ns: int) -> int:
        if self.failsafe_timeout_us is not None:
            return int(round(self.failsafe_timeout_us * 1000.0))
        return 10 * self.decision_period_slots * slot_duration_ns
