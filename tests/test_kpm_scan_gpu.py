"""The block-parallel K4 scan equals the one-thread-per-stream restatement
(both checked against the reference by test_engine_gpu) on randomised
telemetry, for windows shorter and longer than a warp, every policy and both
execution modes, across several batches, batches longer than one 256-slot
chunk, and BASELINE config D (policy stress: 1024 cells per slot boundary)."""
import numpy as np
import pytest

from paper_2604_23397_b200 import _lib
from paper_2604_23397_b200.config import DappConfig, ExecutionMode, PipelineConfig
from paper_2604_23397_b200.engine import ArchesPlan
from paper_2604_23397_b200.geometry import SlotGeometry
from paper_2604_23397_b200.policy import Node, TreeModel, to_device_struct

pytestmark = pytest.mark.gpu


def random_tel(rng, n_units, table):
    t = np.zeros(n_units, dtype=_lib.TELEMETRY_DTYPE)
    t["sigma2_hat"] = rng.random(n_units)
    for e in (0, 1):
        t["rsrp"][:, e] = rng.random(n_units) + 0.5
        t["abs_mean"][:, e] = rng.random(n_units)
        t["sinr_db"][:, e] = rng.normal(10, 8, n_units)
        t["mcs"][:, e] = rng.integers(0, table.n_mcs, n_units)
        t["tb_bytes"][:, e] = rng.integers(0, 3000, n_units)
        t["num_cb"][:, e] = 1 + t["tb_bytes"][:, e] // 1056
        t["crc"][:, e] = rng.random(n_units) < 0.7
        t["mac_rx"][:, e] = np.where(t["crc"][:, e], np.maximum(t["tb_bytes"][:, e] - 3, 0), 0)
        t["lcid4_rx"][:, e] = (t["mac_rx"][:, e] * 0.85).astype(np.int32)
    return t


def tree_on_mac(cut):
    leaf0, leaf1 = Node(counts=(5, 1)), Node(counts=(1, 5))
    return TreeModel(Node(counts=(6, 6), feature=6, threshold=cut, left=leaf0, right=leaf1))


@pytest.mark.parametrize("policy", ["oracle", "fixed:0", "tree"])
@pytest.mark.parametrize("window,period,dwin,timeout", [(100, 100, 100, None), (5, 3, 7, 2000.0),
                                                       (1, 1, 1, None), (40, 17, 33, 9000.0)])
@pytest.mark.parametrize("em", [ExecutionMode.CONCURRENT, ExecutionMode.SELECTED_ONLY])
@pytest.mark.parametrize("n_streams,n_slots", [(3, 77), (2, 300)])
def test_block_scan_equals_sequential(policy, window, period, dwin, timeout, em, n_streams, n_slots):
    _compare_scans(policy, window, period, dwin, timeout, em, n_streams, n_slots, batches=3)


def test_policy_stress_1024_cells():
    """Config D: 1024 cells, reference dApp defaults (100-slot windows, a
    decision every 100 slots), depth-2 tree, one batch of 250 slots per cell."""
    _compare_scans("tree", 100, 100, 100, None, ExecutionMode.CONCURRENT, 1024, 250, batches=2)


def _compare_scans(policy, window, period, dwin, timeout, em, C_, S, batches):
    import torch
    rng = np.random.default_rng(window * 1000 + period)
    geo = SlotGeometry(n_ant=2, n_prb=4)
    pcfg = PipelineConfig(window_length=window, noise_guard=8)
    dcfg = DappConfig(decision_period_slots=period, window_length_slots=dwin,
                      failsafe_timeout_us=timeout)
    plan = ArchesPlan(geo, 1.25, pcfg, em, policy, dcfg)
    L = _lib.lib()
    dev = torch.device("cuda")
    tree = torch.frombuffer(bytearray(bytes(to_device_struct(tree_on_mac(6.5e6 * 8 / 1e6 * 1e-3)))),
                            dtype=torch.uint8).to(dev)
    states, kpms, logs, counts = [], [], [], []
    for _ in range(2):
        st = torch.zeros(plan.state_bytes(C_), dtype=torch.uint8, device=dev)
        _lib.check(L.arches_state_init(plan.handle, _lib.ptr(st), C_, None))
        states.append(st)
        kpms.append(torch.zeros(C_ * S * 104, dtype=torch.uint8, device=dev))
        logs.append(torch.zeros(C_ * 512 * 24, dtype=torch.uint8, device=dev))
        counts.append(torch.zeros(C_, dtype=torch.int32, device=dev))
    for batch in range(batches):
        tel = random_tel(rng, C_ * S, pcfg.mcs_table)
        # make the MAC rate regime-dependent so the tree flips
        reg = (rng.random(C_ * S) < (0.9 if batch % 2 else 0.1)).astype(np.int8)
        tel_d = torch.from_numpy(tel.view(np.uint8).copy()).to(dev)
        reg_d = torch.from_numpy(reg).to(dev)
        for k, fn in enumerate((L.arches_kpm_scan, L.arches_kpm_scan_sequential)):
            _lib.check(fn(plan.handle, C_, S, _lib.ptr(tel_d), _lib.ptr(reg_d), _lib.ptr(tree),
                          _lib.ptr(states[k]), _lib.ptr(kpms[k]), _lib.ptr(logs[k]),
                          _lib.ptr(counts[k]), 512, None))
        torch.cuda.synchronize()
        a = kpms[0].cpu().numpy().view(_lib.KPM_DTYPE)
        b = kpms[1].cpu().numpy().view(_lib.KPM_DTYPE)
        for f in _lib.KPM_DTYPE.names:
            assert np.array_equal(a[f], b[f]), (batch, f)
        assert torch.equal(counts[0], counts[1])
        assert torch.equal(logs[0], logs[1])
        assert torch.equal(states[0], states[1])
