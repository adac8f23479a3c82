"""numpy/scipy restatement of the reference hot path (TEST INFRASTRUCTURE).

Checker and timed CPU baseline only -- see `oracle/__init__.py`.  Each function
follows the cited reference lines of `/root/reference/pkg/src/ranswitch`
(fp64 / complex128 throughout, same numpy/scipy kernels, same operation order).
Pinned bit-for-bit against the reference by `tests/test_oracle_golden.py`.

Layouts are the reference's: y[a, k, t] (A, N, T); estimates (A, 1, N, D).
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
from scipy.linalg import cho_factor, cho_solve

from paper_2604_23397_b200.config import (CB_SEGMENT_BITS, N_DATA_SYM, DappConfig,
                                          ExecutionMode, LatencyModel, PipelineConfig)
from paper_2604_23397_b200.errors import (ConfigurationError, ContractViolation,
                                          EstimatorError, PipelineStateError)
from paper_2604_23397_b200.geometry import GOOD, N_TAPS, pdp_powers
from paper_2604_23397_b200.scene import complex_normal, lcid4_jitter, stream

RIDGE = 1e-12                          # expert_bank.py:19
FEATURE_ORDER = ("phy_throughput", "mcs_index", "pdu_length", "ndi", "rsrp", "snr_db",
                 "mac_throughput", "lcid4_throughput", "mac_rx_bytes", "lcid4_rx_bytes")
KPM_FIELDS = ("slot_index", "phy_throughput", "mcs_index", "pdu_length", "ndi", "rsrp",
              "code_rate", "qam_order", "num_cb", "tb_size", "snr_db",
              "mac_throughput", "lcid4_throughput", "mac_rx_bytes", "lcid4_rx_bytes")


# ------------------------------------------------------------------ experts

def ls_estimate(y: np.ndarray, pil: np.ndarray, geo) -> np.ndarray:
    """expert_bank.py:96-116 -- comb Y/X, odd subcarriers copy the even one below."""
    if geo.n_layers != 1:
        raise ConfigurationError("estimators support a single layer")
    if np.any(np.abs(pil) == 0):
        raise ContractViolation("pilot magnitude 0")
    rows = y[:, np.arange(0, geo.n_sc, 2), :][:, :, list(geo.dmrs_symbols)]   # (A, M, D)
    ratio = rows / pil[None, :, :]
    out = np.empty((geo.n_ant, 1, geo.n_sc, geo.n_dmrs), dtype=complex)
    out[:, 0, :, :] = ratio[:, np.arange(geo.n_sc) // 2, :]
    return out


def estimate_noise_var(ls: np.ndarray, guard: int = 16) -> float:
    """expert_bank.py:199-214 -- mean tail power of the comb IFFT, times n_comb."""
    comb = ls[:, :, np.arange(0, ls.shape[2], 2), :]   # fancy index: same layout as the reference
    m = comb.shape[2]
    if not 1 <= guard < m:
        raise ConfigurationError(f"guard {guard} outside 1..{m - 1}")
    taps = np.fft.ifft(comb, axis=2)
    return float(np.mean(np.abs(taps[:, :, guard:, :]) ** 2) * m)


def _corr(delay_spread: float, n_sc: int, lags: np.ndarray) -> np.ndarray:
    """expert_bank.py:121-124 -- R(lag) = sum_l p_l exp(-2 pi i l lag / N)."""
    p = pdp_powers(delay_spread)
    l = np.arange(N_TAPS)
    return (p[None, :] * np.exp(-2j * np.pi * l[None, :] * lags[:, None] / n_sc)).sum(axis=1)


@lru_cache(maxsize=16)
def _block_corr(n_sc: int, block: int, ds: float):
    """expert_bank.py:127-136 -- (R_hp, R_pp) of one block, full-band exponent."""
    pos = np.arange(0, block, 2)
    lag_hp = np.arange(block)[:, None] - pos[None, :]
    lag_pp = pos[:, None] - pos[None, :]
    r_hp = _corr(ds, n_sc, lag_hp.ravel()).reshape(lag_hp.shape)
    r_pp = _corr(ds, n_sc, lag_pp.ravel()).reshape(lag_pp.shape)
    return r_hp, r_pp


def wiener_matrix(n_sc: int, block: int, noise_var: float, ds: float) -> np.ndarray:
    """expert_bank.py:139-150 -- W = R_hp (R_pp + (s + ridge) I)^-1 by Cholesky."""
    r_hp, r_pp = _block_corr(n_sc, block, ds)
    a = r_pp + (noise_var + RIDGE) * np.eye(r_pp.shape[0])
    try:
        c = cho_factor(a)
    except np.linalg.LinAlgError as e:
        raise EstimatorError("regularized pilot Gram matrix is not positive definite",
                             condition_number=float(np.linalg.cond(a))) from e
    return r_hp @ cho_solve(c, np.eye(r_pp.shape[0]))


def mmse_block(n_sc: int, block_prbs: int = 32) -> int:
    """expert_bank.py:166-168 -- block width; uneven splits fall back to one block."""
    block = min(n_sc, 12 * block_prbs)
    return n_sc if n_sc % block else block


def mmse_estimate(ls: np.ndarray, noise_var: float, assumed_ds: float,
                  block_prbs: int = 32) -> np.ndarray:
    """expert_bank.py:153-177 -- blocked Wiener interpolation from the comb."""
    if noise_var < 0:
        raise ConfigurationError("noise_var must be >= 0")
    n_sc = ls.shape[2]
    block = mmse_block(n_sc, block_prbs)
    w = wiener_matrix(n_sc, block, float(noise_var), float(assumed_ds))
    mask = np.zeros(n_sc, dtype=bool)
    mask[0::2] = True
    comb = ls[:, :, mask, :]
    out = np.empty_like(ls)
    half = block // 2
    for b in range(n_sc // block):
        seg = comb[:, :, b * half:(b + 1) * half, :]
        out[:, :, b * block:(b + 1) * block, :] = np.einsum("sp,alpd->alsd", w, seg)
    return out


def denoiser_estimate(ls: np.ndarray, truncation: int = 20) -> np.ndarray:
    """expert_bank.py:182-196 -- keep the first `truncation` delay taps."""
    n_sc = ls.shape[2]
    if not 1 <= truncation <= n_sc:
        raise ConfigurationError(f"truncation {truncation} outside 1..{n_sc}")
    taps = np.fft.ifft(ls, axis=2)
    taps[:, :, truncation:, :] = 0.0
    return np.fft.fft(taps, axis=2)


# ---------------------------------------------------------------- equaliser

@lru_cache(maxsize=8)
def time_interp_weights(dmrs_symbols: tuple, n_sym: int) -> np.ndarray:
    """phy_pipeline.py:227-242 -- linear between DMRS symbols, hold outside."""
    xp = np.asarray(dmrs_symbols, dtype=float)
    a = np.zeros((n_sym, len(xp)))
    for s in range(n_sym):
        if s <= xp[0]:
            a[s, 0] = 1.0
        elif s >= xp[-1]:
            a[s, -1] = 1.0
        else:
            k = int(np.searchsorted(xp, s, side="right")) - 1
            f = (s - xp[k]) / (xp[k + 1] - xp[k])
            a[s, k], a[s, k + 1] = 1.0 - f, f
    return a


def data_re_mask(geo) -> np.ndarray:
    """phy_pipeline.py:245-250 -- everything except comb REs of DMRS symbols."""
    m = np.ones((geo.n_sc, geo.n_sym), dtype=bool)
    for sym in geo.dmrs_symbols:
        m[0::2, sym] = False
    return m


def equalize(y: np.ndarray, est: np.ndarray, noise_var: float, tx: np.ndarray, geo,
             sinr_cap_db: float = 60.0):
    """phy_pipeline.py:253-279 -- interpolated MRC, SINR vs the known symbols."""
    a = time_interp_weights(tuple(geo.dmrs_symbols), geo.n_sym)
    h = np.einsum("asd,td->ast", est[:, 0, :, :], a)
    num = np.einsum("ast,ast->st", np.conj(h), y)
    den = np.einsum("ast,ast->st", np.conj(h), h).real + noise_var
    x_hat = num / den
    mask = data_re_mask(geo)
    xd, xh = tx[mask], x_hat[mask]
    ref = np.vdot(xd, xd).real
    alpha = np.vdot(xd, xh) / ref
    err = xh - alpha * xd
    err_p = np.vdot(err, err).real
    sinr = sinr_cap_db if err_p <= 0 else 10.0 * math.log10(abs(alpha) ** 2 * ref / err_p)
    return x_hat, min(sinr, sinr_cap_db)


def equalizer_gain(est: np.ndarray, geo) -> np.ndarray:
    """den - noise_var of equalize() (phy_pipeline.py:262-264): sum_a |h_interp|^2, (N, T)."""
    a = time_interp_weights(tuple(geo.dmrs_symbols), geo.n_sym)
    h = np.einsum("asd,td->ast", est[:, 0, :, :], a)
    return np.einsum("ast,ast->st", np.conj(h), h).real


# Gray PAM levels per dimension of TS 38.211 s5.1.3-5.1.5 (QPSK / 16QAM / 64QAM):
# label bits (b_i, b_{i+2}, b_{i+4}) -> amplitude
def _pam_levels(qm: int):
    nb = qm // 2
    scale = {2: 1 / math.sqrt(2.0), 4: 1 / math.sqrt(10.0), 6: 1 / math.sqrt(42.0)}[qm]
    out = []
    for lab in range(1 << nb):
        c = [1 - 2 * ((lab >> i) & 1) for i in range(3)]
        lev = c[0] if nb == 1 else c[0] * (2 - c[1]) if nb == 2 else c[0] * (4 - c[1] * (2 - c[2]))
        out.append((lab, lev * scale))
    return nb, out


def demap_llr(x_hat: np.ndarray, gain: np.ndarray, noise_var: float, qm: int, geo) -> np.ndarray:
    """Max-log LLRs log P(b=0)/P(b=1) of the data REs (the device K6 contract,
    include/arches.h arches_downstream): z = x_hat / beta, beta = g / (g + nv),
    noise variance nv / g; bit 2i from Re, 2i+1 from Im; (N, T, 6), zero on the
    pilot REs (data_re_mask) and beyond qm."""
    out = np.zeros(x_hat.shape + (6,))
    if qm not in (2, 4, 6):
        return out
    nb, levels = _pam_levels(qm)
    beta = gain / (gain + noise_var)
    s2 = noise_var / gain
    for comp, off in ((x_hat.real, 0), (x_hat.imag, 1)):
        z = comp / beta
        for i in range(nb):
            d0 = np.min([(z - lev) ** 2 for lab, lev in levels if not (lab >> i) & 1], axis=0)
            d1 = np.min([(z - lev) ** 2 for lab, lev in levels if (lab >> i) & 1], axis=0)
            out[..., 2 * i + off] = (d1 - d0) / s2
    out[~data_re_mask(geo)] = 0.0
    return out


def inject_values(values: np.ndarray, rho: float, seed: int, slot: int):
    """perturbation_lab.py:92-98 -- Eq. 3: out = in + rho * mean|in| * CN(0,1)."""
    m = float(np.mean(np.abs(values)))
    if rho == 0.0:
        return values.copy(), m
    z = complex_normal(stream(seed, "inject", slot), values.shape)
    return values + rho * m * z, m


# ---------------------------------------------------------------- KPM layer

def link_adapt(sinr_db: float, table) -> int:
    """phy_pipeline.py:192-195."""
    return max(int(np.searchsorted(table.thresholds_db, sinr_db, side="right")) - 1, 0)


def transport_block(mcs: int, n_prb: int, table):
    """phy_pipeline.py:198-205."""
    if not 0 <= mcs < table.n_mcs:
        raise ConfigurationError(f"mcs {mcs} outside table")
    qam, rate = table.qam_order[mcs], table.code_rate[mcs]
    tb = int(n_prb * 12 * N_DATA_SYM * qam * rate // 8)
    return tb, rate, qam, max(1, math.ceil(tb * 8 / CB_SEGMENT_BITS))


def crc_pass_probability(sinr_db, mcs, table, margin_db=6.0, scale_db=2.0) -> float:
    """phy_pipeline.py:208-214."""
    centre = table.thresholds_db[mcs] - margin_db
    return 1.0 / (1.0 + math.exp(-(sinr_db - centre) / scale_db))


def crc_uniform(seed: int, slot: int) -> float:
    """phy_pipeline.py:221 -- first double of stream(seed, 'crc', slot)."""
    return float(stream(seed, "crc", slot).random())


def crc_outcome(sinr_db, mcs, slot, seed, table, margin_db=6.0, scale_db=2.0) -> bool:
    """phy_pipeline.py:217-222."""
    return crc_uniform(seed, slot) < crc_pass_probability(sinr_db, mcs, table, margin_db,
                                                          scale_db)


class ThroughputWindow:
    """phy_pipeline.py:325-344 -- integer byte total over the last `window` slots."""

    def __init__(self, window: int, slot_s: float):
        self.window, self.slot_s = int(window), slot_s
        self.hist: list = []
        self.total = 0

    def push(self, n: int) -> float:
        self.hist.append(n)
        self.total += n
        if len(self.hist) > self.window:
            self.total -= self.hist[-self.window - 1]
        filled = min(len(self.hist), self.window)
        return self.total * 8.0 / 1e6 / (filled * self.slot_s)


@dataclass(frozen=True)
class KpmRecord:
    slot_index: int
    phy_throughput: float
    mcs_index: int
    pdu_length: int
    ndi: int
    rsrp: float
    code_rate: float
    qam_order: int
    num_cb: int
    tb_size: int
    snr_db: float
    mac_throughput: float
    lcid4_throughput: float
    mac_rx_bytes: int
    lcid4_rx_bytes: int

    def row(self) -> list:
        return [getattr(self, f) for f in KPM_FIELDS]


# ----------------------------------------------------- control + policy

@dataclass
class ControlMessage:
    mode: int
    decided_at_ns: int
    deliverable_at_ns: int
    trigger: str = "policy"


class SwitchController:
    """phy_pipeline.py:94-144 -- slot-boundary application of control traffic."""

    def __init__(self, exec_mode: ExecutionMode, slot_ns: int):
        self.exec_mode, self.slot_ns = exec_mode, int(slot_ns)
        self.mode = 1
        self.pending: list = []
        self.forced: list = []
        self.applied: list = []

    def deliver(self, msg: ControlMessage):
        self.pending.append(msg)
        self.pending.sort(key=lambda m: m.deliverable_at_ns)

    def force_mode(self, mode: int, at_ns: int, trigger: str = "failsafe"):
        self.forced.append((int(at_ns), mode, trigger))
        self.forced.sort(key=lambda f: f[0])

    def begin_slot(self, n: int) -> int:
        t0 = n * self.slot_ns
        cut = t0 - self.slot_ns if self.exec_mode is ExecutionMode.SELECTED_ONLY else t0
        while self.pending and self.pending[0].deliverable_at_ns <= cut:
            m = self.pending.pop(0)
            if m.mode != self.mode:
                self.applied.append((n, m.mode, m.trigger))
            self.mode = m.mode
        while self.forced and self.forced[0][0] <= t0:
            _, mode, trig = self.forced.pop(0)
            if mode != self.mode:
                self.applied.append((n, mode, trig))
            self.mode = mode
        return self.mode


@dataclass
class Node:
    counts: tuple
    feature: int | None = None
    threshold: float | None = None
    left: "Node | None" = None
    right: "Node | None" = None

    @property
    def label(self) -> int:
        """switch_policy.py:76-78 -- a count tie predicts MMSE (1)."""
        return 0 if self.counts[0] > self.counts[1] else 1


def tree_from_text(text: str):
    """switch_policy.py:350-384 -- the 'tree v1' text format; returns (root, names)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0].strip() != "tree v1" or not lines[1].startswith("features:"):
        raise ConfigurationError("unrecognized tree format")
    names = tuple(lines[1].split(":", 1)[1].strip().split(","))
    spec = {}
    for ln in lines[2:]:
        p = ln.split()
        nid = int(p[0])
        if p[1] == "leaf":
            spec[nid] = (tuple(int(v) for v in p[3].split("=")[1].split(",")), None)
        elif p[1] == "split":
            spec[nid] = (tuple(int(v) for v in p[5].split("=")[1].split(",")),
                         (names.index(p[2]), float(p[4]), int(p[6].split("=")[1]),
                          int(p[7].split("=")[1])))
        else:
            raise ConfigurationError(f"bad tree line: {ln}")

    def build(nid):
        counts, split = spec[nid]
        if split is None:
            return Node(counts)
        f, t, l, r = split
        return Node(counts, f, t, build(l), build(r))
    return build(0), names


def predict(root: Node, x) -> int:
    """switch_policy.py:237-248 -- values equal to a threshold go left."""
    node = root
    while node.feature is not None:
        node = node.left if x[node.feature] <= node.threshold else node.right
    return node.label


def window_features(records, names=FEATURE_ORDER) -> np.ndarray:
    """dapp_control.py:85-90 -- per-KPM column mean over the window."""
    if not records:
        raise ContractViolation("empty KPM window")
    return np.array([[float(getattr(r, n)) for n in names] for r in records]).mean(axis=0)


class FailsafeMonitor:
    """dapp_control.py:123-144."""

    def __init__(self, timeout_ns: int):
        self.timeout_ns, self.last, self.tripped, self.events = timeout_ns, 0, False, []

    def note_delivery(self, at_ns: int):
        self.last = max(self.last, int(at_ns))
        self.tripped = False

    def check(self, now_ns: int, mode: int):
        if self.tripped or now_ns - self.last <= self.timeout_ns or mode == 1:
            return None
        self.tripped = True
        self.events.append(int(now_ns))
        return 1


# ----------------------------------------------------------- closed loop

@dataclass
class SlotResult:
    mode: int
    sinr_db: float
    est_abs_mean: float
    rsrp: float
    nv_est: float | None
    crc: bool
    kpm: KpmRecord
    downstream: np.ndarray | None = None
    mmse: np.ndarray | None = None
    ai: np.ndarray | None = None
    x_hat: np.ndarray | None = None


@dataclass
class CellResult:
    slots: list = field(default_factory=list)
    messages: list = field(default_factory=list)
    applied: list = field(default_factory=list)
    failsafe_events: list = field(default_factory=list)

    @property
    def modes(self):
        return [s.mode for s in self.slots]

    @property
    def records(self):
        return [s.kpm for s in self.slots]


class CellLoop:
    """One cell's closed loop: `Pipeline.run_slot` (phy_pipeline.py:422-493) plus the
    policy plumbing of `harness.execute_run` (harness.py:174-231), over
    pre-synthesised inputs (slot synthesis is outside the hot path)."""

    def __init__(self, geo, scenarios, policy="oracle", exec_mode=ExecutionMode.CONCURRENT,
                 pcfg: PipelineConfig | None = None, dcfg: DappConfig | None = None,
                 latency: LatencyModel | None = None, tree_text: str | None = None,
                 keep_arrays: bool = False, perturb_rho: float | None = None):
        self.geo, self.scenarios = geo, scenarios
        self.pcfg = pcfg or PipelineConfig()
        self.dcfg = dcfg or DappConfig()
        self.lat = latency or LatencyModel()
        self.exec_mode = exec_mode
        self.keep = keep_arrays
        # Pipeline.perturb hook (phy_pipeline.py:401,444-445) as perturbation_lab.sweep
        # installs it (perturbation_lab.py:127-133): Eq. 3 on the MMSE output
        self.perturb_rho = perturb_rho
        self.slot_ns = geo.slot_duration_ns
        slot_s = geo.slot_duration_us * 1e-6
        self.ctl = SwitchController(exec_mode, self.slot_ns)
        self.mac_w = ThroughputWindow(self.pcfg.window_length, slot_s)
        self.l4_w = ThroughputWindow(self.pcfg.window_length, slot_s)
        self.cum = 0
        self.ndi = 0
        self.n = 0
        self.buf = {1: None, 0: None}
        self.result = CellResult()
        self.kind, self.arg = policy, None
        if policy.startswith("fixed:"):
            self.kind, self.arg = "fixed", int(policy.split(":")[1])
            self.ctl.force_mode(self.arg, at_ns=0, trigger="fixed")
            self.result.messages.append(ControlMessage(self.arg, 0, 0, "fixed"))
        elif policy == "tree":
            self.root, _ = tree_from_text(tree_text)
            self.window: deque = deque(maxlen=self.dcfg.window_length_slots)
            self.since = 0
            self.monitor = FailsafeMonitor(self.dcfg.timeout_ns(self.slot_ns))
        elif policy != "oracle":
            raise ConfigurationError(f"unknown policy source: {policy!r}")

    def run_slot(self, y, tx, pil, regime: str) -> SlotResult:
        geo, cfg, n = self.geo, self.pcfg, self.n
        scen = self.scenarios[regime]
        mode = self.ctl.begin_slot(n)
        populated = {1: False, 0: False}
        ls = ls_estimate(y, pil, geo)
        nv = scen.noise_var(geo.n_ant)
        if self.exec_mode is ExecutionMode.CONCURRENT:
            to_run = (1, 0)
        else:
            to_run = (mode,)
        nv_est = mmse = ai = None
        est_abs_mean = None
        for e in to_run:
            if e == 1:
                nv_est = estimate_noise_var(ls, cfg.noise_guard)
                mmse = mmse_estimate(ls, nv_est, scen.assumed_delay_spread, cfg.mmse_block_prbs)
                if self.perturb_rho is not None:
                    mmse, est_abs_mean = inject_values(mmse, self.perturb_rho, scen.seed, n)
                self.buf[1] = mmse.copy()
            else:
                ai = denoiser_estimate(ls, min(cfg.truncation, geo.n_sc))
                self.buf[0] = ai.copy()
            populated[e] = True
        # switch_select (phy_pipeline.py:81-91): mode 1 copies MMSE into the AI buffer
        if not populated[mode]:
            raise PipelineStateError("selected expert did not run this slot")
        if mode == 1:
            self.buf[0] = self.buf[1].copy()
        down = self.buf[0]
        if est_abs_mean is None:
            est_abs_mean = float(np.mean(np.abs(down)))
        rsrp = float(np.mean(np.abs(down) ** 2))
        x_hat, sinr = equalize(y, down, nv, tx, geo, cfg.sinr_cap_db)
        tab = cfg.mcs_table
        mcs = link_adapt(sinr, tab)
        tb, rate, qam, ncb = transport_block(mcs, geo.n_prb, tab)
        crc = crc_outcome(sinr, mcs, n, scen.seed, tab, cfg.crc_margin_db, cfg.crc_scale_db)
        pdu = max(tb - cfg.mac_header_bytes, 0)
        mac_rx = pdu if crc else 0
        frac = min(max(cfg.lcid4_fraction + cfg.lcid4_jitter * lcid4_jitter(n), 0.0), 1.0)
        l4_rx = int(mac_rx * frac)
        if crc:
            self.cum += tb
        mac_t = self.mac_w.push(mac_rx)
        l4_t = self.l4_w.push(l4_rx)
        elapsed = (n + 1) * geo.slot_duration_us * 1e-6
        phy_t = self.cum * 8.0 / 1e6 / elapsed
        ndi = self.ndi
        if crc:
            self.ndi = 1 - self.ndi
        kpm = KpmRecord(n, phy_t, mcs, pdu, ndi, rsrp, rate, qam, ncb, tb, sinr,
                        mac_t, l4_t, mac_rx, l4_rx)
        res = SlotResult(mode, sinr, est_abs_mean, rsrp, nv_est, crc, kpm,
                         down.copy() if self.keep else None,
                         mmse if self.keep else None, ai if self.keep else None,
                         x_hat if self.keep else None)
        self.result.slots.append(res)
        self._control(regime, kpm)
        self.n += 1
        return res

    def _control(self, regime: str, kpm: KpmRecord):
        end_ns = (self.n + 1) * self.slot_ns
        msgs = self.result.messages
        if self.kind == "oracle":
            want = 1 if regime == GOOD else 0
            if want != (msgs[-1].mode if msgs else 1):
                m = ControlMessage(want, end_ns, end_ns, "oracle")
                self.ctl.deliver(m)
                msgs.append(m)
        elif self.kind == "tree":
            # Dapp.on_indication (dapp_control.py:107-120), one record per indication
            self.window.append(kpm)
            self.since += 1
            if self.since >= self.dcfg.decision_period_slots:
                self.since = 0
                vec = window_features(list(self.window))
                decided = end_ns + self.lat.decision_delay_ns()
                m = ControlMessage(int(predict(self.root, vec)), decided, decided, "policy")
                self.ctl.deliver(m)
                self.monitor.note_delivery(m.deliverable_at_ns)
                msgs.append(m)
            forced = self.monitor.check(end_ns, self.ctl.mode)
            if forced is not None:
                self.ctl.force_mode(forced, at_ns=end_ns)
                msgs.append(ControlMessage(forced, end_ns, end_ns, "failsafe"))
                self.result.failsafe_events.append(end_ns)

    def finish(self) -> CellResult:
        self.result.applied = list(self.ctl.applied)
        return self.result
