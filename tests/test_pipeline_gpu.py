"""Cross-batch pipeline (arches_run_batch_async): the control tail of batch n
(RNG, K3, K4) runs on the plan's internal stream next to batch n+1's K1.  The
results must be bit-identical to the sequential arches_run_batch over the same
batch sequence -- KPM records, telemetry, expert outputs, the control state and
the message log (which carries the history of every batch)."""
import numpy as np
import pytest

from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
from paper_2604_23397_b200.scene import CellScene, to_device_layout

pytestmark = pytest.mark.gpu


def _engine(geo, n_streams, n_slots, exec_mode, seeds, flags=0, pcfg=None):
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    streams = []
    for k, seed in enumerate(seeds):
        scens = default_scenarios(seed, geo)
        regimes = ["good" if ((i + k) // 3) % 2 == 0 else "poor" for i in range(n_slots)]
        cs = CellScene(geo, scens, regimes[0])
        streams.append((cs, regimes, [cs.next_slot(r) for r in regimes]))
    plan = ArchesPlan(geo, 1.25, pcfg or PipelineConfig(window_length=8), exec_mode, "oracle",
                      flags=flags)
    eng = SlotEngine(plan, n_streams, n_slots)
    eng.set_streams(np.stack([s[0].pilots for s in streams]), seeds)
    eng.load(y=np.stack([to_device_layout(sl.y) for s in streams for sl in s[2]]),
             tx=np.stack([sl.tx.T for s in streams for sl in s[2]]).astype(np.complex64),
             noise_var=[sl.noise_var for s in streams for sl in s[2]],
             regime=[1 if r == "good" else 0 for s in streams for r in s[1]])
    return eng


def _snapshot(eng):
    return {
        "kpm": eng.kpm.cpu().numpy().copy(),
        "tel": eng.tel.cpu().numpy().copy(),
        "state": eng.state.cpu().numpy().copy(),
        "msg_log": eng.msg_log.cpu().numpy().copy(),
        "msg_count": eng.msg_count.cpu().numpy().copy(),
        "h_mmse": eng.h_mmse.cpu().numpy().copy(),
        "h_ai": eng.h_ai.cpu().numpy().copy(),
    }


FFMA = 0x3   # _lib.FLAG_NO_TC_K1 | FLAG_NO_TC_K2: the CUDA-core K1 and the FFMA K2


@pytest.mark.parametrize("n_prb,n_ant,n_streams,n_slots,n_batches,exec_mode,flags,block", [
    (273, 4, 1, 64, 12, ExecutionMode.CONCURRENT, 0, 32),   # config-B geometry: K3 / K4 overlap a long K1
    (12, 4, 3, 20, 9, ExecutionMode.CONCURRENT, 0, 32),     # several streams, short batches
    (52, 4, 2, 16, 7, ExecutionMode.SELECTED_ONLY, 0, 32),
    (24, 16, 2, 8, 5, ExecutionMode.CONCURRENT, 0, 32),     # antenna-group K2 (massive-MIMO form)
    # FFMA K2 plans (finalise on the caller's stream): routed to the ordered form
    (12, 6, 2, 16, 5, ExecutionMode.CONCURRENT, 0, 32),     # n_ant 6: no tensor-core K2
    (64, 4, 1, 16, 6, ExecutionMode.CONCURRENT, 0, 16),     # tiles straddle 16-PRB MMSE blocks
    (52, 4, 2, 16, 6, ExecutionMode.SELECTED_ONLY, FFMA, 32),
])
def test_pipelined_batches_match_sequential(n_prb, n_ant, n_streams, n_slots, n_batches, exec_mode,
                                            flags, block):
    import torch
    geo = SlotGeometry(n_ant=n_ant, n_prb=n_prb)
    seeds = [31 + 5 * k for k in range(n_streams)]
    pc = PipelineConfig(window_length=8, mmse_block_prbs=block)
    seq = _engine(geo, n_streams, n_slots, exec_mode, seeds, flags, pc)
    pip = _engine(geo, n_streams, n_slots, exec_mode, seeds, flags, pc)
    for _ in range(n_batches):
        seq.run()
    for _ in range(n_batches):
        pip.run(pipelined=True)
    pip.join()
    torch.cuda.synchronize()
    a, b = _snapshot(seq), _snapshot(pip)
    for k in a:
        assert np.array_equal(a[k], b[k]), f"{k} differs between pipelined and sequential runs"
    assert int(a["msg_count"].sum()) > 0


def test_sync_run_after_pipelined_joins_first():
    """A sequential run_batch issued while a pipelined tail is pending must
    order itself after that tail (the library joins it)."""
    import torch
    geo = SlotGeometry(n_ant=4, n_prb=52)
    seeds = [7]
    seq = _engine(geo, 1, 24, ExecutionMode.CONCURRENT, seeds)
    mix = _engine(geo, 1, 24, ExecutionMode.CONCURRENT, seeds)
    for _ in range(6):
        seq.run()
    for i in range(6):
        mix.run(pipelined=(i % 2 == 0))
    mix.join()
    torch.cuda.synchronize()
    a, b = _snapshot(seq), _snapshot(mix)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_graph_captured_pipeline_matches_sequential():
    """The pipelined chain captured as one CUDA graph (bench.py's timed form)."""
    import torch
    geo = SlotGeometry(n_ant=4, n_prb=273)
    seeds = [11]
    seq = _engine(geo, 1, 32, ExecutionMode.CONCURRENT, seeds)
    pip = _engine(geo, 1, 32, ExecutionMode.CONCURRENT, seeds)
    g = pip.capture_pipeline(5)   # the plan's streams exist from creation: nothing runs eagerly
    pip.run_pipeline(g, 5)
    pip.run_pipeline(g, 5)
    for _ in range(10):
        seq.run()
    torch.cuda.synchronize()
    assert pip.next_slot == seq.next_slot == 10 * 32
    a, b = _snapshot(seq), _snapshot(pip)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_streaming_load_between_pipelined_batches():
    """load() of the next batch while the previous batch's tail (K4 reads the
    regime timeline) may still run: the engine joins the tail first, so a
    streaming loop (load, run pipelined, load, ...) equals the sequential one."""
    import torch
    geo = SlotGeometry(n_ant=4, n_prb=52)
    seeds = [19]
    scens = default_scenarios(seeds[0], geo)
    n_slots, n_batches = 16, 6
    regimes = ["good" if (i // 5) % 2 == 0 else "poor" for i in range(n_slots * n_batches)]
    cs = CellScene(geo, scens, regimes[0])
    slots = [cs.next_slot(r) for r in regimes]

    def batch(b):
        sl = slots[b * n_slots:(b + 1) * n_slots]
        rg = regimes[b * n_slots:(b + 1) * n_slots]
        return dict(y=np.stack([to_device_layout(x.y) for x in sl]),
                    tx=np.stack([x.tx.T for x in sl]).astype(np.complex64),
                    noise_var=[x.noise_var for x in sl], regime=[1 if r == "good" else 0 for r in rg])

    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    out = []
    for pipelined in (False, True):
        plan = ArchesPlan(geo, 1.25, PipelineConfig(window_length=8), ExecutionMode.CONCURRENT,
                          "oracle")
        eng = SlotEngine(plan, 1, n_slots)
        eng.set_streams(cs.pilots[None], seeds)
        for b in range(n_batches):   # nothing read back in between: only load() joins
            eng.load(**batch(b))
            eng.run(pipelined=pipelined)
        torch.cuda.synchronize()
        out.append((eng.kpm_records().copy(), eng.messages().copy(), eng.state.cpu().numpy()))
    for x, y in zip(out[0], out[1]):
        assert np.array_equal(x, y)
    assert len(out[0][1]) >= 8   # the regime timeline drove mode changes in every batch


@pytest.mark.parametrize("wire", [False, True])
def test_double_buffered_staging_matches_load_then_run(wire):
    """SlotEngine.stage / run_staged (the bench's e2e loop: batch n+1's inputs cross
    PCIe on a copy stream while batch n runs) give, batch by batch, exactly what
    load + run give -- with a different input batch every step, so a stale or
    swapped input set would show."""
    import torch
    from paper_2604_23397_b200.scene import pack_qpsk
    geo = SlotGeometry(n_ant=4, n_prb=52)
    ref = _engine(geo, 1, 16, ExecutionMode.CONCURRENT, [11])
    dbl = _engine(geo, 1, 16, ExecutionMode.CONCURRENT, [11])
    y0, tx0 = ref.y.cpu(), ref.tx.cpu()
    nv0, reg0 = ref.noise_var.cpu(), ref.regime.cpu()
    batches = []
    for k in range(5):
        tx = torch.from_numpy(pack_qpsk(tx0.numpy())) if wire else tx0.clone()
        batches.append(tuple(t.pin_memory() for t in (
            y0 * (1.0 + 0.15 * k), tx, nv0 * (1.0 + 0.05 * k), torch.roll(reg0, k))))
    want = []
    for b in batches:
        ref.load(y=b[0], tx=b[1], noise_var=b[2], regime=b[3])
        ref.run()
        want.append(_snapshot(ref))
    dbl.stage(*batches[0])
    for k in range(len(batches)):
        dbl.run_staged()
        got = _snapshot(dbl)
        if k + 1 < len(batches):
            dbl.stage(*batches[k + 1])
        for key in want[k]:
            assert np.array_equal(got[key], want[k][key]), (k, key)
