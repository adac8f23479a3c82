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


def _engine_pair(geo, C, S, policy="oracle", exec_mode=ExecutionMode.CONCURRENT, seed=70):
    """The same batch on a complex-tx plan and on a FLAG_TX_PACKED plan."""
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    pcfg = PipelineConfig(window_length=8)
    slots = [_slots(geo, S, seed + c) for c in range(C)]
    y = np.concatenate([np.stack([to_device_layout(s.y) for s in sl]) for _, sl in slots])
    tx = np.concatenate([np.stack([s.tx.T for s in sl]) for _, sl in slots]).astype(np.complex64)
    nv = np.concatenate([[s.noise_var for s in sl] for _, sl in slots])
    reg = np.tile([1 if i % 2 == 0 else 0 for i in range(S)], C)
    pil = np.stack([cs.pilots for cs, _ in slots])
    out = []
    for flags, txin in ((0, tx), (_lib.FLAG_TX_PACKED, pack_qpsk(tx))):
        plan = ArchesPlan(geo, 1.25, pcfg, exec_mode, policy, flags=flags)
        eng = SlotEngine(plan, C, S)
        eng.set_streams(pil, [seed + c for c in range(C)])
        eng.load(y=y, tx=txin, noise_var=nv, regime=reg)
        out.append(eng)
    return out, tx


def _same_outputs(a, b):
    import torch
    torch.cuda.synchronize()
    for name in ("h_mmse", "h_ai", "tel", "kpm", "msg_count"):
        assert torch.equal(getattr(a, name).view(torch.uint8) if getattr(a, name).is_complex()
                           else getattr(a, name),
                           getattr(b, name).view(torch.uint8) if getattr(b, name).is_complex()
                           else getattr(b, name)), name


@pytest.mark.gpu
@pytest.mark.parametrize("n_prb,n_ant,C,S", [(273, 4, 1, 8), (52, 4, 3, 6), (12, 2, 2, 5), (24, 1, 2, 4)])
def test_packed_plan_matches_complex_plan(n_prb, n_ant, C, S):
    """K2 reading the 2-bit codes (ARCHES_FLAG_TX_PACKED) gives bit-identical expert
    outputs, telemetry, KPMs and messages to the complex64 grid -- sequential and
    pipelined executors, over two consecutive batches."""
    (ref, pk), _ = _engine_pair(SlotGeometry(n_ant=n_ant, n_prb=n_prb), C, S)
    assert pk.tx.dtype.is_floating_point is False and tuple(pk.tx.shape)[-1] == 32
    for pipelined in (False, True):
        for _ in range(2):
            ref.run(pipelined=pipelined)
            pk.run(pipelined=pipelined)
        ref.join()
        pk.join()
        _same_outputs(ref, pk)


@pytest.mark.gpu
def test_packed_plan_perturbation_and_loading_forms():
    """K7 (Eq. 3 perturbation) decodes the codes the same way; loading a complex
    grid into a packed engine packs it on the device; pack_tx returns the codes."""
    import torch
    geo = SlotGeometry(n_ant=4, n_prb=24)
    (ref, pk), tx = _engine_pair(geo, 2, 4)
    for rho in (0.0, 0.3):
        ref.run_perturbed(rho)
        pk.run_perturbed(rho)
        _same_outputs(ref, pk)
    assert np.array_equal(pk.pack_tx(), pack_qpsk(tx))
    pk.tx.zero_()
    pk.load(tx=tx)                       # complex grid -> device packer
    torch.cuda.synchronize()
    assert np.array_equal(pk.tx.cpu().numpy(), pack_qpsk(tx))


@pytest.mark.gpu
def test_packed_flag_rejected_where_k2_cannot_read_codes():
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.engine import ArchesPlan
    from paper_2604_23397_b200.errors import ConfigurationError
    for geo, flags in ((SlotGeometry(n_ant=64, n_prb=12), _lib.FLAG_TX_PACKED),
                       (SlotGeometry(n_ant=4, n_prb=12), _lib.FLAG_TX_PACKED | _lib.FLAG_NO_TC_K2),
                       (SlotGeometry(n_ant=3, n_prb=12), _lib.FLAG_TX_PACKED)):
        with pytest.raises(ConfigurationError):
            ArchesPlan(geo, 1.25, flags=flags)


@pytest.mark.gpu
def test_device_scene_feeds_a_packed_engine():
    """Device synthesis into a FLAG_TX_PACKED engine: the complex grid it writes is
    packed on the device; the codes equal the host packer's of a complex engine's
    grid and the batch runs bit-identically."""
    import torch
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    from paper_2604_23397_b200.scene_gpu import DeviceScene
    geo = SlotGeometry(n_ant=4, n_prb=24)
    seeds = [5, 77]
    scens = default_scenarios(seeds[0], geo)
    engs = []
    for flags in (0, _lib.FLAG_TX_PACKED):
        eng = SlotEngine(ArchesPlan(geo, 1.25, PipelineConfig(window_length=8), flags=flags), 2, 4)
        ds = DeviceScene(eng, {"good": scens["good"], "poor": scens["poor"]}, seeds)  # sets pilots, seeds
        ds.next_batch([["good", "poor", "good", "poor"]] * 2)
        eng.run()
        engs.append(eng)
    torch.cuda.synchronize()
    assert np.array_equal(engs[1].tx.cpu().numpy(), pack_qpsk(engs[0].tx.cpu().numpy()))
    _same_outputs(*engs)
