"""Packed QPSK wire format of the transmit grids (include/arches.h,
arches_pack_qpsk / arches_unpack_qpsk): 2 bits per RE over PCIe.

CPU: the host packer is exact and refuses non-QPSK grids.  GPU: unpacking on
the device restores the complex64 grid bit-for-bit and the device packer
equals the host packer."""
import numpy as np
import pytest

from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
from paper_2604_23397_b200.errors import ContractViolation
from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
from paper_2604_23397_b200.scene import QPSK_AMP, CellScene, pack_qpsk, to_device_layout


def _unpack(bits, N):
    U, nt, T, _ = bits.shape
    codes = np.stack([(bits >> (2 * r)) & 3 for r in range(4)], -1)
    codes = codes.transpose(0, 2, 1, 3, 4).reshape(U, T, nt * 128)[:, :, :N]
    return (np.where(codes & 1, QPSK_AMP, -QPSK_AMP)
            + 1j * np.where(codes & 2, QPSK_AMP, -QPSK_AMP)).astype(np.complex64)


def _slots(geo, n, seed):
    cs = CellScene(geo, default_scenarios(seed, geo), "good")
    return cs, [cs.next_slot("good" if i % 2 == 0 else "poor") for i in range(n)]


@pytest.mark.parametrize("n_prb", [4, 12, 273])
def test_host_pack_round_trip(n_prb):
    geo = SlotGeometry(n_ant=1, n_prb=n_prb)
    _, sl = _slots(geo, 3, 9) if n_prb >= 12 else (None, None)
    if sl is None:
        rng = np.random.default_rng(0)
        b = rng.integers(0, 2, size=(2, 3, 14, 12 * n_prb))
        tx = ((2 * b[0] - 1) + 1j * (2 * b[1] - 1)) / np.sqrt(2.0)
    else:
        tx = np.stack([s.tx.T for s in sl])
    bits = pack_qpsk(tx)
    assert bits.shape == (tx.shape[0], -(-geo.n_sc // 128), 14, 32) and bits.dtype == np.uint8
    assert np.array_equal(_unpack(bits, geo.n_sc), tx.astype(np.complex64))


def test_host_pack_rejects_non_qpsk():
    tx = np.full((1, 14, 48), (1 + 1j) / np.sqrt(2.0))
    tx[0, 3, 7] = 0.5 + 0.5j
    with pytest.raises(ContractViolation):
        pack_qpsk(tx)


@pytest.mark.gpu
@pytest.mark.parametrize("n_prb,n_ant,C,S", [(273, 4, 1, 6), (52, 4, 3, 4), (12, 2, 2, 3)])
def test_wire_format_round_trip_on_device(n_prb, n_ant, C, S):
    """host pack -> H2D -> arches_unpack_qpsk gives the complex64 grid bit-for-bit,
    and the device packer (arches_pack_qpsk) gives the host packer's codes."""
    import torch
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo = SlotGeometry(n_ant=n_ant, n_prb=n_prb)
    plan = ArchesPlan(geo, 1.25, PipelineConfig(window_length=8), ExecutionMode.CONCURRENT, "oracle")
    eng = SlotEngine(plan, C, S)
    tx = np.concatenate([np.stack([s.tx.T for s in _slots(geo, S, 40 + c)[1]]) for c in range(C)])
    tx = tx.astype(np.complex64)
    eng.load(tx=pack_qpsk(tx))
    torch.cuda.synchronize()
    assert np.array_equal(eng.tx.cpu().numpy(), tx)
    eng.load(tx=tx)
    assert np.array_equal(eng.pack_tx(), pack_qpsk(tx))
    # pinned host bits, asynchronous copy (bench.py's e2e form)
    eng.tx.zero_()
    eng.load(tx=torch.from_numpy(pack_qpsk(tx)).pin_memory(), non_blocking=True)
    torch.cuda.synchronize()
    assert np.array_equal(eng.tx.cpu().numpy(), tx)


@pytest.mark.gpu
def test_device_pack_flags_non_qpsk():
    import torch
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo = SlotGeometry(n_ant=2, n_prb=12)
    eng = SlotEngine(ArchesPlan(geo, 1.25), 1, 2)
    eng.tx.copy_(torch.full((2, 14, geo.n_sc), complex(QPSK_AMP, -QPSK_AMP), dtype=torch.complex64))
    assert eng.pack_tx().shape == (2, 2, 14, 32)
    eng.tx[1, 5, 100] = 0.25
    with pytest.raises(ContractViolation):
        eng.pack_tx()
