"""Device-side slot synthesis (csrc/k_scene.cuh, `arches_synthesize`): the
reference scene for many cells at once, written straight into a SlotEngine's
input buffers -- no host synthesis, no H2D of the grids.

Same streams and operation order as the host `scene.CellScene` (itself pinned
to the reference): AR(1) TDL channel + log-normal shadow and the delayed
interferer (`ChannelProcess`, radio_scene.py:156-196), pilots
(`pilot_sequence`, :233-237), QPSK data (`transmit_grid`, :240-249) and
Y = H X + sqrt(nv) W + sqrt(iv) H_i X_i (`synthesize_uplink_slot`, :277-306).
The one host draw per cell-slot is the shadow's standard normal (numpy's
ziggurat, `stream(seed, "shadow", slot).standard_normal()`).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import ConfigurationError
from .geometry import GOOD, N_TAPS, POOR, pdp_powers
from .scene import stream


class DeviceScene:
    """Sequential slot source for the engine's streams (cells), on the device."""

    def __init__(self, engine, scenarios: dict, seeds, first_regime: str = GOOD):
        import torch
        self.eng = engine
        geo = engine.plan.geometry
        if engine.C != len(seeds):
            raise ConfigurationError("one seed per engine stream")
        s0 = scenarios[first_regime]
        if s0.interference_excess_delay + N_TAPS > geo.n_comb:
            raise ConfigurationError("interference_excess_delay does not fit the comb span")
        self.geo, self.scenarios = geo, scenarios
        self.seeds = [int(s) for s in seeds]
        dev = engine.device
        plan = engine.plan.handle
        L = _lib.lib()
        regs = (_lib.SceneRegime * 2)()
        masks = np.zeros((2, geo.n_prb), np.uint8)
        for code, name in ((0, POOR), (1, GOOD)):
            sc = scenarios[name]
            regs[code].noise_var = sc.noise_var(geo.n_ant)
            regs[code].interference_var = sc.interference_var()
            regs[code].temporal_correlation = sc.temporal_correlation
            regs[code].shadow_sigma_db = sc.shadow_sigma_db
            regs[code].shadow_correlation = sc.shadow_correlation
            m = np.asarray(sc.interference_prb_mask, dtype=bool)
            if m.size not in (0, geo.n_prb):
                raise ConfigurationError("interference mask does not cover the PRBs")
            if m.size:
                masks[code] = m
        self._regs = regs
        self._sqrt_p = (C.c_double * N_TAPS)(*np.sqrt(pdp_powers(s0.delay_spread)))
        self._excess = int(s0.interference_excess_delay)
        self._mask = torch.from_numpy(masks).to(dev)
        self.state = torch.zeros(L.arches_scene_state_bytes(plan, engine.C), dtype=torch.uint8,
                                 device=dev)
        self.ws = torch.empty(L.arches_scene_workspace_bytes(plan, engine.U), dtype=torch.uint8,
                              device=dev)
        self._seeds = torch.from_numpy(np.array(self.seeds, dtype=np.uint64).view(np.int64)).to(dev)
        self.pilots = torch.empty((engine.C, engine.M, engine.D), dtype=torch.complex64, device=dev)
        _lib.check(L.arches_scene_pilots(plan, engine.C, _lib.ptr(self._seeds),
                                         _lib.ptr(self.pilots), torch.cuda.current_stream().cuda_stream))
        engine.pilots.copy_(self.pilots)
        engine.seeds.copy_(self._seeds)
        self.slot = 0

    def next_batch(self, regimes):
        """Synthesise the next n_slots slots of every stream into the engine;
        regimes: (n_streams, n_slots) of "good"/"poor" (or 1/0)."""
        import torch
        eng = self.eng
        r = np.asarray(regimes)
        if r.dtype.kind in "US":
            r = (r == GOOD).astype(np.int8)
        r = np.ascontiguousarray(r.astype(np.int8).reshape(eng.C, eng.S))
        slots = range(self.slot, self.slot + eng.S)
        z = np.array([[float(stream(sd, "shadow", n).standard_normal()) for n in slots]
                      for sd in self.seeds])
        eng._settle()
        eng.regime.copy_(torch.from_numpy(r.reshape(-1)))
        zd = torch.from_numpy(z.reshape(-1)).to(eng.device)
        tx = (torch.empty((eng.U, eng.T, eng.N), dtype=torch.complex64, device=eng.device)
              if eng.tx_packed else eng.tx)
        _lib.check(_lib.lib().arches_synthesize(
            eng.plan.handle, eng.C, eng.S, _lib.ptr(self._seeds), self._regs, _lib.ptr(self._mask),
            self._sqrt_p, self._excess, _lib.ptr(eng.regime), _lib.ptr(zd), _lib.ptr(self.pilots),
            _lib.ptr(self.state), _lib.ptr(self.ws), _lib.ptr(eng.y), _lib.ptr(tx),
            _lib.ptr(eng.noise_var), torch.cuda.current_stream().cuda_stream))
        if eng.tx_packed:   # synthesis writes the complex grid; the engine keeps its codes
            eng._pack_into(tx, eng.tx)
        self.slot += eng.S
