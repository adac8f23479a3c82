"""Host-side synthetic uplink slots (input generation, NOT the hot path).

Produces the reference's received grids bit-for-bit so the device path and the
CPU reference process identical inputs.  Restates `rng.py:17-55` (counter
Philox streams, Box-Muller CN(0,1), QPSK) and `radio_scene.py:140-306` (TDL
AR(1) fading with log-normal shadow, delayed co-channel interferer, pilots,
`Y = H*X + Hi*Xi + W`).  Every floating-point expression keeps the reference's
operation order because bit-exact reproduction depends on it.

Layouts:
  * reference layout  y[a, k, t]  complex128  (`ResourceGrid.values`)
  * device layout     y[a, t, k]  complex64   (frequency-contiguous rows)
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, ContractViolation
from .geometry import GOOD, N_TAPS, ScenarioConfig, SlotGeometry, pdp_powers

_U64 = (1 << 64) - 1


def purpose_key(purpose: str) -> int:
    """blake2b-64 little-endian digest of the purpose string (`rng.py:17-21`)."""
    d = hashlib.blake2b(purpose.encode("utf-8"), digest_size=8).digest()
    return int.from_bytes(d, "little")


def stream(seed: int, purpose: str, slot_index: int = 0) -> np.random.Generator:
    """numpy Philox4x64-10, key=(seed, purpose_key), counter=(0, slot, 0, 0)
    (`rng.py:24-34`)."""
    if slot_index < 0:
        raise ValueError("slot_index must be >= 0")
    bitgen = np.random.Philox(counter=np.array([0, slot_index, 0, 0], dtype=np.uint64),
                              key=np.array([seed & _U64, purpose_key(purpose)], dtype=np.uint64))
    return np.random.Generator(bitgen)


def complex_normal(gen: np.random.Generator, shape) -> np.ndarray:
    """Box-Muller CN(0,1) from two uniform blocks (`rng.py:37-47`)."""
    u1 = gen.random(shape)
    u2 = gen.random(shape)
    return np.sqrt(-np.log1p(-u1)) * np.exp(2j * np.pi * u2)


def qpsk(gen: np.random.Generator, shape) -> np.ndarray:
    """(+-1 +-1j)/sqrt(2) from bounded integer draws (`rng.py:50-55`)."""
    b = gen.integers(0, 2, size=(2,) + tuple(shape))
    return ((2 * b[0] - 1) + 1j * (2 * b[1] - 1)) / np.sqrt(2.0)


def pilots(geo: SlotGeometry, seed: int) -> np.ndarray:
    """(n_comb, n_dmrs) fixed pilots (`radio_scene.py:233-237`)."""
    return qpsk(stream(seed, "pilot"), (geo.n_comb, geo.n_dmrs))


def _grid_with_pilots(geo: SlotGeometry, seed: int, purpose: str, slot: int,
                      pil: np.ndarray) -> np.ndarray:
    x = qpsk(stream(seed, purpose, slot), (geo.n_sc, geo.n_sym))
    for j, sym in enumerate(geo.dmrs_symbols):
        x[0::2, sym] = pil[:, j]
    return x


def transmit_grid(geo: SlotGeometry, seed: int, slot: int, pil=None) -> np.ndarray:
    """(n_sc, n_sym) QPSK data with pilots on the comb of DMRS symbols
    (`radio_scene.py:240-249`)."""
    return _grid_with_pilots(geo, seed, "data", slot,
                             pilots(geo, seed) if pil is None else pil)


class _Fading:
    """Sequential AR(1) TDL tap process (`radio_scene.py:156-192`)."""

    def __init__(self, geo: SlotGeometry, scen: ScenarioConfig, purpose: str,
                 excess_delay: int, shadowed: bool):
        self.geo, self.scen, self.purpose = geo, scen, purpose
        self.excess, self.shadowed = excess_delay, shadowed
        self.sqrt_p = np.sqrt(pdp_powers(scen.delay_spread))
        self.taps = None
        self.shadow_db = 0.0
        self.next = 0

    def step(self) -> np.ndarray:
        n, s = self.next, self.scen
        z = complex_normal(stream(s.seed, self.purpose, n),
                           (self.geo.n_ant, self.geo.n_layers, len(self.sqrt_p)))
        innov = z * self.sqrt_p
        phi = s.temporal_correlation
        self.taps = innov if self.taps is None else \
            phi * self.taps + math.sqrt(1.0 - phi * phi) * innov
        self.next += 1
        if not self.shadowed or s.shadow_sigma_db == 0:
            return self.taps
        g = s.shadow_sigma_db * float(stream(s.seed, "shadow", n).standard_normal())
        phi_s = s.shadow_correlation
        self.shadow_db = g if n == 0 else \
            phi_s * self.shadow_db + math.sqrt(1.0 - phi_s * phi_s) * g
        return self.taps * 10.0 ** (self.shadow_db / 20.0)

    def freq(self) -> np.ndarray:
        """(n_ant, n_layers, n_sc) frequency response of the next slot."""
        h = np.fft.fft(self.step(), n=self.geo.n_sc, axis=-1)
        if self.excess:
            k = np.arange(self.geo.n_sc)
            h = h * np.exp(-2j * np.pi * self.excess * k / self.geo.n_sc)
        return h


@dataclass
class SlotInput:
    """One synthesised slot of one single-layer stream."""
    y: np.ndarray            # (A, N, T) complex128, reference layout
    tx: np.ndarray           # (N, T) complex128
    h_true: np.ndarray       # (A, N) complex128 true channel (constant over the slot)
    noise_var: float         # true per-antenna thermal variance (equaliser input)
    regime: str


class CellScene:
    """Sequential slot source for one cell (= one single-layer DMRS port).

    Mirrors `Pipeline.run_slot` input generation (`phy_pipeline.py:430-433,459`)
    including mid-run regime changes (`Pipeline.set_scenario`, `:406-420`): the
    fading and interferer processes advance every slot regardless of regime.
    """

    def __init__(self, geo: SlotGeometry, scenarios: dict, first_regime: str = GOOD):
        if geo.n_layers != 1:
            raise ConfigurationError("a CellScene is one single-layer stream")
        self.geo = geo
        self.scenarios = scenarios
        s0 = scenarios[first_regime]
        if s0.interference_excess_delay + N_TAPS > geo.n_comb:
            raise ConfigurationError("interference_excess_delay does not fit the comb span")
        self.seed = s0.seed
        self.channel = _Fading(geo, s0, "channel", 0, True)
        self.interferer = _Fading(geo, s0, "interferer", s0.interference_excess_delay, False)
        self.pilots = pilots(geo, self.seed)
        self.slot = 0

    def next_slot(self, regime: str) -> SlotInput:
        geo, n = self.geo, self.slot
        scen = self.scenarios[regime]
        self.channel.scen = scen
        self.interferer.scen = scen
        h = self.channel.freq()[:, 0, :]            # (A, N)
        h_i = self.interferer.freq()[:, 0, :]
        x = _grid_with_pilots(geo, self.seed, "data", n, self.pilots)
        y = h[:, :, None] * x[None, :, :]
        nv = scen.noise_var(geo.n_ant)
        if nv > 0:
            w = complex_normal(stream(self.seed, "awgn", n), y.shape)
            y = y + math.sqrt(nv) * w
        iv = scen.interference_var()
        if iv > 0:
            mask = np.repeat(np.asarray(scen.interference_prb_mask, dtype=bool), 12)
            if mask.size != geo.n_sc:
                raise ConfigurationError("interference mask does not cover the PRBs")
            x_i = _grid_with_pilots(geo, self.seed, "interferer-data", n, self.pilots)
            y[:, mask, :] += math.sqrt(iv) * h_i[:, mask, None] * x_i[None, mask, :]
        self.slot += 1
        return SlotInput(y=y, tx=x, h_true=h, noise_var=nv, regime=regime)


def to_device_layout(y_ref: np.ndarray) -> np.ndarray:
    """(A, N, T) complex -> (A, T, N) complex64 (frequency-contiguous rows)."""
    return np.ascontiguousarray(np.transpose(y_ref, (0, 2, 1))).astype(np.complex64)


def lcid4_jitter(slot: int) -> float:
    """Seed-independent traffic wobble in [-1, 1) (`phy_pipeline.py:347-350`)."""
    d = hashlib.blake2b(f"lcid4:{slot}".encode(), digest_size=8).digest()
    return int.from_bytes(d, "little") / float(1 << 64) * 2.0 - 1.0


QPSK_AMP = np.float32(1.0 / np.sqrt(2.0))   # the complex64 of qpsk() (rng.py:50-55)
TX_TILE, TX_ROW_BYTES = 128, 32


def pack_qpsk(tx: np.ndarray) -> np.ndarray:
    """Transmit grids (U, T, N) complex -> packed QPSK codes (U, n_tiles, T, 32) uint8,
    the packed wire format of include/arches.h (arches_unpack_qpsk): RE (t, 128 * tile + j) is
    byte j // 4 of row t, bits 2 (j % 4): bit 0 = Re > 0, bit 1 = Im > 0.  Every RE
    must be exactly a qpsk() symbol in complex64 (the whole grid is QPSK, pilots
    included: radio_scene.py:240-249)."""
    x = np.asarray(tx)
    if x.ndim != 3:
        raise ContractViolation(f"tx shape {x.shape}, expected (units, n_sym, n_sc)")
    x = x.astype(np.complex64, copy=False)
    re, im = x.real, x.imag
    if not (np.all(np.abs(re) == QPSK_AMP) and np.all(np.abs(im) == QPSK_AMP)):
        raise ContractViolation("tx grid is not QPSK (+-1 +-1j)/sqrt(2) in complex64: "
                                "load it as a complex grid")
    U, T, N = x.shape
    n_tiles = -(-N // TX_TILE)
    code = np.zeros((U, T, n_tiles * TX_TILE), np.uint8)
    code[:, :, :N] = (re > 0).astype(np.uint8) | ((im > 0).astype(np.uint8) << 1)
    q = code.reshape(U, T, n_tiles, TX_ROW_BYTES, 4)
    packed = q[..., 0] | (q[..., 1] << 2) | (q[..., 2] << 4) | (q[..., 3] << 6)
    return np.ascontiguousarray(packed.transpose(0, 2, 1, 3))   # (U, n_tiles, T, 32)
