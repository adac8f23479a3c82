"""The benched shapes themselves against the unmodified reference.

Golden loops from tools/make_golden_long.py (harness.execute_run, harness.py:
174-231; Pipeline.run_slot, phy_pipeline.py:422-493):
  * p273_alt_w100_conc / _sel -- config B: 273 PRB, 4 RX, good/poor alternating
    every slot, oracle policy, DEFAULT 100-slot KPM windows, 320 / 300 slots
    (windows wrap; K4's 256-slot chunk and the bench's 256-slot batch crossed);
  * p52_tree_default -- config A: 52 PRB, tree policy, default dApp (100/100).
Each is run the three ways the product runs it: SlotEngine batches of S = 256
(the bench's batch) continued by a second engine, the cross-batch pipeline
captured as one CUDA graph (bench.py's timed form), and several streams of
the same cell in one batch (config C's structure; each stream must reproduce
the reference).  KPM integer fields, throughputs, CRC, modes and control
messages bit-exact; rsrp / SINR / |H| within tests/parity.py tolerances.
"""
import functools

import numpy as np
import pytest

from golden_io import loop_inputs, loop_setup, loops_long, tree_text
from parity import compare_kpms
from paper_2604_23397_b200.policy import from_text
from paper_2604_23397_b200.scene import to_device_layout

pytestmark = pytest.mark.gpu

IDS = [m["id"] for m, _, _ in loops_long()]
TRIG = {0: "policy", 1: "failsafe", 2: "oracle", 3: "fixed"}


@functools.lru_cache(maxsize=None)
def _case(lid):
    m, recs, extra = {m["id"]: (m, r, e) for m, r, e in loops_long()}[lid]
    geo, scen, regimes, em, pcfg, dcfg = loop_setup(m)
    cs, inputs = loop_inputs(geo, scen, regimes)
    arrays = dict(y=np.stack([to_device_layout(s.y) for s in inputs]),
                  tx=np.stack([s.tx.T for s in inputs]).astype(np.complex64),
                  noise_var=np.array([s.noise_var for s in inputs]),
                  regime=np.array([1 if s.regime == "good" else 0 for s in inputs], np.int8))
    return m, recs, extra, geo, scen, em, pcfg, dcfg, cs, arrays


def _engine(lid, n_streams, n_slots):
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    m, _, _, geo, scen, em, pcfg, dcfg, cs, _ = _case(lid)
    tree = from_text(tree_text(m["tree"])) if m["tree"] else None
    policy = "tree" if m["policy"] == "tree" else m["policy"]
    plan = ArchesPlan(geo, scen["good"].assumed_delay_spread, pcfg, em, policy, dcfg)
    eng = SlotEngine(plan, n_streams, n_slots, tree=tree)
    eng.set_streams(np.stack([cs.pilots] * n_streams), [m["seed"]] * n_streams)
    return eng


def _slice(arrays, lo, hi, n_streams=1):
    return {k: np.concatenate([v[lo:hi]] * n_streams) for k, v in arrays.items()}


def _check(lid, got, msgs):
    m, recs, extra = _case(lid)[:3]
    compare_kpms(got, recs, extra)
    assert got["mode"].tolist() == m["modes"]
    assert [[int(x["mode"]), int(x["decided_at_ns"]), int(x["deliverable_at_ns"]),
             TRIG[int(x["trigger"])]] for x in msgs] == m["messages"]


@pytest.mark.parametrize("lid", IDS)
def test_bench_batches_of_256(lid):
    """S = 256 (bench.py's default batch), the rest of the loop in a second
    engine that continues the device-resident control state."""
    arrays = _case(lid)[-1]
    n = len(arrays["regime"])
    first = _engine(lid, 1, 256)
    first.load(**_slice(arrays, 0, 256))
    first.run()
    rest = _engine(lid, 1, n - 256)
    rest.state.copy_(first.state)
    rest.msg_count.copy_(first.msg_count)
    rest.msg_log.copy_(first.msg_log)
    rest.load(**_slice(arrays, 256, n))
    rest.run()
    got = np.concatenate([first.kpm_records()[0], rest.kpm_records()[0]])
    _check(lid, got, rest.messages(0))


@pytest.mark.parametrize("lid", IDS)
def test_graph_captured_pipeline(lid):
    """The cross-batch pipeline captured as a CUDA graph (bench.py's timed form,
    there K batches per replay over a resident input pool): here one batch per
    replay so each of the loop's 5 batches can be loaded before its replay."""
    import torch
    arrays = _case(lid)[-1]
    n = len(arrays["regime"])
    S = n // 5
    eng = _engine(lid, 1, S)
    g = eng.capture_pipeline(1)
    recs = []
    for b in range(5):
        eng.load(**_slice(arrays, b * S, (b + 1) * S))
        eng.run_pipeline(g, 1)
        recs.append(eng.kpm_records()[0].copy())
    torch.cuda.synchronize()
    _check(lid, np.concatenate(recs), eng.messages(0))


@pytest.mark.parametrize("lid", IDS)
def test_async_pipeline_streaming(lid):
    """Eager cross-batch pipeline (arches_run_batch_async): 5 batches, each
    loaded while the previous batch's control tail may still run."""
    import torch
    arrays = _case(lid)[-1]
    n = len(arrays["regime"])
    S = n // 5
    eng = _engine(lid, 1, S)
    kpm_log = []
    for b in range(5):
        eng.load(**_slice(arrays, b * S, (b + 1) * S))   # joins the pending tail first
        eng.run(pipelined=True)
        kpm_log.append(eng.kpm_records()[0].copy())       # joins, then reads
    torch.cuda.synchronize()
    _check(lid, np.concatenate(kpm_log), eng.messages(0))


@pytest.mark.parametrize("lid", IDS)
def test_multistream_same_cell(lid):
    """Three streams of the same cell in one batch: every stream reproduces the
    reference (stream-major unit indexing, per-stream control state)."""
    arrays = _case(lid)[-1]
    n = len(arrays["regime"])
    C = 3 if n <= 320 else 2
    eng = _engine(lid, C, n)
    eng.load(**_slice(arrays, 0, n, C))
    eng.run()
    recs = eng.kpm_records()
    for c in range(C):
        _check(lid, recs[c], eng.messages(c))
