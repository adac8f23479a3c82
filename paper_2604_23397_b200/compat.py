"""Drop-in replacements for the reference's hot-path call surface.

Same names, signatures, argument meaning and error behaviour as the reference
(`/root/reference/pkg/src/ranswitch`); every numeric step runs on the device
through the C ABI (no CPU fallback):

  ls_estimate          expert_bank.py:96-116
  estimate_noise_var   expert_bank.py:199-214
  mmse_estimate        expert_bank.py:153-177
  denoiser_estimate    expert_bank.py:182-196
  equalize             phy_pipeline.py:253-279
  ExpertBuffers        phy_pipeline.py:55-78   (device-resident buffers)
  switch_select        phy_pipeline.py:81-91   (K5 mode-predicated copy)
  window_features      dapp_control.py:85-90
  predict              switch_policy.py:237-248

`install()` rebinds these names inside an imported `ranswitch` (the rebinding
rule of SURVEY.md s8b: phy_pipeline and dapp_control import them by name) and
switches this module to raise the reference's own exception classes.

Numerics: the device path computes in complex64 with fp64 scalars; returned
arrays are upcast to complex128 so callers see the reference dtypes.  The
stated tolerances are in tests/parity.py.
"""
from __future__ import annotations

import sys
import types

import numpy as np

from . import _lib
from . import errors as _own_errors
from .config import PipelineConfig
from .geometry import DmrsEstimate as _OwnDmrsEstimate
from .geometry import ExpertId as _OwnExpertId
from .geometry import Stage as _OwnStage
from .policy import FEATURE_ORDER, tree_tensor

_E = _own_errors                       # exception namespace (switched by install())
_CLASSES = {"DmrsEstimate": _OwnDmrsEstimate, "Stage": _OwnStage, "ExpertId": _OwnExpertId}
_PLANS: dict = {}


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise _own_errors.DeviceError("the ARCHES device path needs a CUDA device")
    return torch


def _stage_value(stage) -> str:
    return getattr(stage, "value", stage)


def _stage(value: str, like=None):
    cls = type(like) if like is not None and hasattr(like, "value") else _CLASSES["Stage"]
    return cls(value)


def _estimate(values, stage_value, comb_mask, geometry, like=None):
    cls = type(like) if like is not None else _CLASSES["DmrsEstimate"]
    st = _stage(stage_value, getattr(like, "stage", None))
    return cls(values=values, stage=st, comb_mask=comb_mask, geometry=geometry)


class _PlanEntry:
    def __init__(self, plan, ws_units: int):
        torch = _torch()
        self.plan = plan
        self.ws = torch.empty(plan.workspace_bytes(ws_units), dtype=torch.uint8, device="cuda")


def _plan(geometry, guard=None, truncation=20, block_prbs=32, ds=1.25, sinr_cap_db=60.0):
    from .engine import ArchesPlan
    if guard is None:  # unused by the caller: any valid value
        guard = max(1, min(16, 6 * geometry.n_prb - 1))
    key = (geometry.n_ant, geometry.n_prb, geometry.n_sym, tuple(geometry.dmrs_symbols),
           float(geometry.slot_duration_us), int(guard), int(truncation), int(block_prbs), float(ds),
           float(sinr_cap_db))
    ent = _PLANS.get(key)
    if ent is None:
        pc = PipelineConfig(noise_guard=guard, truncation=truncation, mmse_block_prbs=block_prbs,
                            sinr_cap_db=float(sinr_cap_db))
        try:
            plan = ArchesPlan(geometry, ds, pc, policy="fixed:1")
        except _own_errors.ConfigurationError as e:
            raise _E.ConfigurationError(str(e)) from None
        ent = _PLANS[key] = _PlanEntry(plan, 1)
    return ent


def _dev_ls(values: np.ndarray):
    """(A, 1, N, D) complex -> device (1, A, D, N) complex64."""
    torch = _torch()
    v = np.asarray(values)
    host = np.ascontiguousarray(np.transpose(v[:, 0, :, :], (0, 2, 1))).astype(np.complex64)
    return torch.from_numpy(host[None]).to("cuda")


def _host_est(dev) -> np.ndarray:
    """device (1, A, D, N) complex -> (A, 1, N, D) complex128."""
    arr = dev[0].cpu().numpy()
    return np.ascontiguousarray(np.transpose(arr, (0, 2, 1))[:, None, :, :]).astype(np.complex128)


def _stream():
    return _torch().cuda.current_stream().cuda_stream


def _check(rc):
    if rc:
        msg = _lib.lib().arches_last_error().decode(errors="replace")
        cls = {1: _E.ConfigurationError, 2: _E.ContractViolation, 3: _E.EstimatorError,
               4: _E.PipelineStateError}.get(rc, _own_errors.DeviceError)
        raise cls(msg)


# ------------------------------------------------------------------ experts

def ls_estimate(rx, geometry):
    """Per-pilot Y/X at comb REs, gaps filled by the lower even neighbour."""
    if geometry.n_layers != 1:
        raise _E.ConfigurationError("estimators support a single layer")
    pil = np.asarray(rx.known_dmrs)
    if np.any(np.abs(pil) == 0):
        raise _E.ContractViolation("pilot magnitude 0")
    torch = _torch()
    ent = _plan(geometry)
    y = np.asarray(rx.values)
    y_dev = torch.from_numpy(np.ascontiguousarray(np.transpose(y, (0, 2, 1)))
                             .astype(np.complex64)[None]).to("cuda")
    p_dev = torch.from_numpy(pil.astype(np.complex64)[None]).to("cuda")
    out = torch.empty((1, geometry.n_ant, len(geometry.dmrs_symbols), geometry.n_sc),
                      dtype=torch.complex64, device="cuda")
    _check(_lib.lib().arches_ls_materialize(ent.plan.handle, 1, _lib.ptr(y_dev), _lib.ptr(p_dev),
                                            _lib.ptr(out), _stream()))
    mask = np.zeros(geometry.n_sc, dtype=bool)
    mask[0::2] = True
    return _estimate(_host_est(out), "RawLS", mask, geometry)


def _require_raw(ls, who):
    if _stage_value(ls.stage) != "RawLS":
        raise _E.ContractViolation(f"{who} expects a RawLS input")


def estimate_noise_var(ls, geometry, guard: int = 16) -> float:
    _require_raw(ls, "estimate_noise_var")
    n_comb = len(np.arange(0, geometry.n_sc, 2))
    if not 1 <= guard < n_comb:
        raise _E.ConfigurationError(f"guard {guard} outside 1..{n_comb - 1}")
    torch = _torch()
    ent = _plan(geometry, guard=guard)
    sig = torch.empty(1, dtype=torch.float64, device="cuda")
    _check(_lib.lib().arches_expert_from_ls(ent.plan.handle, 1, 0, _lib.ptr(_dev_ls(ls.values)),
                                            None, _lib.ptr(sig), None, _lib.ptr(ent.ws),
                                            _stream()))
    return float(sig.item())


def mmse_estimate(ls, noise_var: float, scenario, block_prbs: int = 32):
    _require_raw(ls, "mmse_estimate")
    if noise_var < 0:
        raise _E.ConfigurationError("noise_var must be >= 0")
    torch = _torch()
    geo = ls.geometry
    ent = _plan(geo, block_prbs=block_prbs, ds=float(scenario.assumed_delay_spread))
    nv = torch.tensor([float(noise_var)], dtype=torch.float64, device="cuda")
    out = torch.empty((1, geo.n_ant, len(geo.dmrs_symbols), geo.n_sc), dtype=torch.complex128,
                      device="cuda")   # fp64 synthesis: the reference's output dtype
    _check(_lib.lib().arches_expert_from_ls(ent.plan.handle, 1, 1 | _lib.EXPERT_OUT_C128,
                                            _lib.ptr(_dev_ls(ls.values)),
                                            _lib.ptr(nv), None, _lib.ptr(out), _lib.ptr(ent.ws),
                                            _stream()))
    return _estimate(_host_est(out), "Interpolated", np.ones(geo.n_sc, dtype=bool), geo, like=ls)


def denoiser_estimate(ls, geometry, truncation: int = 20):
    _require_raw(ls, "denoiser_estimate")
    if not 1 <= truncation <= geometry.n_sc:
        raise _E.ConfigurationError(f"truncation {truncation} outside 1..{geometry.n_sc}")
    torch = _torch()
    ent = _plan(geometry, truncation=truncation)
    out = torch.empty((1, geometry.n_ant, len(geometry.dmrs_symbols), geometry.n_sc),
                      dtype=torch.complex128, device="cuda")   # fp64 synthesis
    _check(_lib.lib().arches_expert_from_ls(ent.plan.handle, 1, 2 | _lib.EXPERT_OUT_C128,
                                            _lib.ptr(_dev_ls(ls.values)),
                                            None, None, _lib.ptr(out), _lib.ptr(ent.ws),
                                            _stream()))
    return _estimate(_host_est(out), "Interpolated", np.ones(geometry.n_sc, dtype=bool),
                     geometry, like=ls)


def equalize(rx, estimate, noise_var: float, tx_grid, sinr_cap_db: float = 60.0):
    """Returns (equalised grid (n_sc, n_sym), post-equalisation SINR in dB)."""
    if _stage_value(estimate.stage) != "Interpolated":
        raise _E.ContractViolation("equalize expects an Interpolated estimate")
    torch = _torch()
    geo = estimate.geometry
    ent = _plan(geo, sinr_cap_db=sinr_cap_db)   # cached per cap like every compat plan
    y = np.asarray(rx.values)
    y_dev = torch.from_numpy(np.ascontiguousarray(np.transpose(y, (0, 2, 1)))
                             .astype(np.complex64)[None]).to("cuda")
    tx = torch.from_numpy(np.ascontiguousarray(np.asarray(tx_grid).T).astype(np.complex64)[None]).to("cuda")
    nv = torch.tensor([float(noise_var)], dtype=torch.float64, device="cuda")
    sinr = torch.empty(1, dtype=torch.float64, device="cuda")
    xh = torch.empty((1, geo.n_sym, geo.n_sc), dtype=torch.complex64, device="cuda")
    _check(_lib.lib().arches_equalize(ent.plan.handle, 1, _lib.ptr(y_dev),
                                      _lib.ptr(_dev_ls(estimate.values)), _lib.ptr(tx),
                                      _lib.ptr(nv), _lib.ptr(sinr), None, None, _lib.ptr(xh),
                                      _lib.ptr(ent.ws), _stream()))
    x_hat = xh[0].cpu().numpy().T.astype(np.complex128)
    return x_hat, float(sinr.item())


# ---------------------------------------------------------- switch plumbing

class DeviceArray:
    """A device-resident complex128 buffer (the reference buffers' dtype, so a
    written expert output reads back element-exact) that numpy can read
    (`__array__` copies device -> host)."""

    def __init__(self, shape):
        torch = _torch()
        self.shape = tuple(shape)
        self.tensor = torch.zeros(self.shape, dtype=torch.complex128, device="cuda")

    dtype = np.dtype(np.complex128)

    def __array__(self, dtype=None, copy=None):
        a = self.tensor.cpu().numpy()
        return a if dtype is None else a.astype(dtype)

    def __len__(self):
        return self.shape[0]

    def __getitem__(self, idx):
        return np.asarray(self)[idx]

    def __setitem__(self, idx, values):
        torch = _torch()
        if isinstance(values, DeviceArray):
            src = values.tensor
        else:
            src = torch.from_numpy(np.asarray(values, dtype=np.complex128)).to("cuda")
        self.tensor[idx] = src


class ExpertBuffers:
    """Per-expert device buffers; `downstream` aliases the AI buffer and
    selecting MMSE copies its output into it (phy_pipeline.py:55-78)."""

    def __init__(self, shape, dtype=complex):
        self.buffer_mmse = DeviceArray(shape)
        self.buffer_ai = DeviceArray(shape)
        self._populated = {1: False, 0: False}

    @staticmethod
    def _key(expert) -> int:
        return int(getattr(expert, "value", expert))

    def write(self, expert, values):
        buf = self.buffer_mmse if self._key(expert) == 1 else self.buffer_ai
        buf[...] = values
        self._populated[self._key(expert)] = True

    def populated(self, expert) -> bool:
        return self._populated[self._key(expert)]

    def new_slot(self):
        self._populated = {1: False, 0: False}

    @property
    def downstream(self):
        return self.buffer_ai


def switch_select(buffers, mode, costs) -> float:
    """mode 1: device copy MMSE -> AI buffer (K5); mode 0: no-op."""
    m = int(mode.mode)
    if m == 1:
        if not buffers.populated(1):
            raise _E.PipelineStateError("MMSE buffer unpopulated at switch_select")
        torch = _torch()
        flag = torch.tensor([1], dtype=torch.int32, device="cuda")
        src, dst = buffers.buffer_mmse.tensor, buffers.buffer_ai.tensor
        # complex128 buffers: 2 interleaved float2 per element
        _check(_lib.lib().arches_switch_copy_one(_lib.ptr(flag), _lib.ptr(src), _lib.ptr(dst),
                                                 2 * src.numel(), _stream()))
    elif not buffers.populated(0):
        raise _E.PipelineStateError("AI buffer unpopulated at switch_select")
    return costs.switch_cost_us(m)


# ------------------------------------------------------------- dApp policy

def window_features(records, names=FEATURE_ORDER) -> np.ndarray:
    """Per-KPM window mean (sequential fp64 sum / n, on the device)."""
    if not records:
        raise _E.ContractViolation("empty KPM window")
    names = tuple(names)
    rows = np.array([[float(getattr(r, n)) for n in names] for r in records], dtype=np.float64)
    return _device_means(rows)


def _device_means(rows: np.ndarray) -> np.ndarray:
    torch = _torch()
    ncol = rows.shape[1]
    out = np.empty(ncol)
    for c0 in range(0, ncol, 10):
        block = np.zeros((rows.shape[0], 10))
        w = min(10, ncol - c0)
        block[:, :w] = rows[:, c0:c0 + w]
        d = torch.from_numpy(np.ascontiguousarray(block)).to("cuda")
        o = torch.empty(10, dtype=torch.float64, device="cuda")
        _check(_lib.lib().arches_window_features(_lib.ptr(d), rows.shape[0], _lib.ptr(o), _stream()))
        out[c0:c0 + w] = o.cpu().numpy()[:w]
    return out


def predict(tree, x):
    """Root-to-leaf descent (device); values equal to a threshold go left."""
    from .policy import predict as _predict
    try:
        return _predict(tree, x)
    except _own_errors.ContractViolation as e:
        raise _E.ContractViolation(str(e)) from None


def train(data, max_depth: int = 2):
    """switch_policy.train (switch_policy.py:173-234) with the exhaustive root
    search on the device (paper_2604_23397_b200.train); same tree, same errors,
    the caller's Node / TreeModel classes."""
    from . import train as _train
    from .policy import Node as _Node
    if len(data) == 0:
        raise _E.ContractViolation("cannot train on an empty dataset")
    try:
        tree = _train.train(data.x, data.y, max_depth=max_depth,
                            feature_names=tuple(data.feature_names))
    except _own_errors.ConfigurationError as e:
        raise _E.ConfigurationError(str(e)) from None
    except _own_errors.ContractViolation as e:
        raise _E.ContractViolation(str(e)) from None
    node_cls, model_cls = _CLASSES.get("Node", _Node), _CLASSES.get("TreeModel", type(tree))

    def conv(n):
        if n is None:
            return None
        return node_cls(counts=tuple(n.counts), feature=n.feature, threshold=n.threshold,
                        left=conv(n.left), right=conv(n.right))
    return model_cls(conv(tree.root), tuple(data.feature_names))


# ---------------------------------------------------------------- install

NAMES_PHY = ("ls_estimate", "estimate_noise_var", "mmse_estimate", "denoiser_estimate",
             "switch_select", "equalize", "ExpertBuffers")
NAMES_EXPERT_BANK = ("ls_estimate", "estimate_noise_var", "mmse_estimate", "denoiser_estimate")
NAMES_DAPP = ("window_features", "predict")
NAMES_POLICY = ("train",)


def install(package=None) -> dict:
    """Rebind the hot-path names inside an imported `ranswitch` package (or a
    namespace with the same submodules).  Returns the replaced originals."""
    global _E
    pkg = package if package is not None else sys.modules.get("ranswitch")
    if pkg is None:
        raise ImportError("import ranswitch before calling install()")
    me = sys.modules[__name__]
    saved = {}
    for modname, names in (("phy_pipeline", NAMES_PHY), ("expert_bank", NAMES_EXPERT_BANK),
                           ("dapp_control", NAMES_DAPP), ("switch_policy", NAMES_POLICY)):
        mod = getattr(pkg, modname, None)
        if mod is None:
            continue
        for n in names:
            if hasattr(mod, n):
                saved[(modname, n)] = getattr(mod, n)
                setattr(mod, n, getattr(me, n))
    val = getattr(pkg, "validation", None)
    if val is not None:
        _E = types.SimpleNamespace(
            ConfigurationError=val.ConfigurationError, ContractViolation=val.ContractViolation,
            EstimatorError=val.EstimatorError, PipelineStateError=val.PipelineStateError)
    eb = getattr(pkg, "expert_bank", None)
    if eb is not None:
        _CLASSES.update(DmrsEstimate=eb.DmrsEstimate, Stage=eb.Stage, ExpertId=eb.ExpertId)
    sp = getattr(pkg, "switch_policy", None)
    if sp is not None:
        _CLASSES.update(Node=sp.Node, TreeModel=sp.TreeModel)
    return saved


def uninstall(package, saved: dict):
    global _E
    for (modname, n), fn in saved.items():
        setattr(getattr(package, modname), n, fn)
    _E = _own_errors
    _CLASSES.update(DmrsEstimate=_OwnDmrsEstimate, Stage=_OwnStage, ExpertId=_OwnExpertId)
    _CLASSES.pop("Node", None)
    _CLASSES.pop("TreeModel", None)
