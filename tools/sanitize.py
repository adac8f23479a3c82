"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck) over every kernel of the library: RNG, K1 (tcgen05 and
CUDA-core), K1 finalize, K2 (tcgen05 and FFMA), K3, K4 (block and sequential),
K5, the compat forms, and the cross-batch pipeline (two streams, event hand-offs).

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    from paper_2604_23397_b200.geometry import SlotGeometry, default_scenarios
    from paper_2604_23397_b200.scene import CellScene, to_device_layout

    def engine(geo, C, S, flags=0, em=ExecutionMode.CONCURRENT):
        scens = default_scenarios(5, geo)
        cs = CellScene(geo, scens, "good")
        sl = [cs.next_slot("good" if i % 2 == 0 else "poor") for i in range(S)]
        plan = ArchesPlan(geo, 1.25, PipelineConfig(window_length=4), em, "oracle", flags=flags)
        eng = SlotEngine(plan, C, S)
        eng.set_streams(np.stack([cs.pilots] * C), list(range(C)))
        eng.load(y=np.concatenate([np.stack([to_device_layout(s.y) for s in sl])] * C),
                 tx=np.concatenate([np.stack([s.tx.T for s in sl]).astype(np.complex64)] * C),
                 noise_var=np.tile([s.noise_var for s in sl], C),
                 regime=np.tile([1 if i % 2 == 0 else 0 for i in range(S)], C))
        return eng

    for geo, flags, em in ((SlotGeometry(n_ant=4, n_prb=24), 0, ExecutionMode.CONCURRENT),
                           (SlotGeometry(n_ant=4, n_prb=12), 0x3, ExecutionMode.SELECTED_ONLY),
                           (SlotGeometry(n_ant=16, n_prb=12), 0, ExecutionMode.CONCURRENT),
                           (SlotGeometry(n_ant=64, n_prb=12), 0, ExecutionMode.CONCURRENT)):
        eng = engine(geo, 2, 6, flags, em)
        eng.run()                         # sequential executor (RNG forked on the side stream)
        for _ in range(3):
            eng.run(pipelined=True)       # cross-batch pipeline
        eng.join()
        eng.switch_copy()                 # K5
        torch.cuda.synchronize()
        print("ok", geo.n_ant, geo.n_prb, flags, eng.kpm_records()["mode"].ravel()[:6])
    # compat per-call forms + sequential K4
    from paper_2604_23397_b200 import compat
    geo = SlotGeometry(n_ant=2, n_prb=4)
    scens = default_scenarios(1, geo)
    import dataclasses
    import types
    scens = {k: dataclasses.replace(v, interference_excess_delay=8) for k, v in scens.items()}
    cs = CellScene(geo, scens, "good")
    s = cs.next_slot("good")
    from paper_2604_23397_b200.geometry import ResourceGrid
    rx = ResourceGrid(values=s.y, known_dmrs=cs.pilots, geometry=geo)
    ls = compat.ls_estimate(rx, geo)
    nv = compat.estimate_noise_var(ls, geo, guard=8)
    m = compat.mmse_estimate(ls, nv, scens["good"])
    a = compat.denoiser_estimate(ls, geo)
    xh, sinr = compat.equalize(rx, m, s.noise_var, s.tx)
    rec = types.SimpleNamespace(**{f: 1.0 for f in compat.FEATURE_ORDER})
    print("compat ok", nv, sinr, compat.window_features([rec, rec]))
    L = _lib.lib()
    eng = engine(SlotGeometry(n_ant=4, n_prb=12), 3, 5)
    eng.run()
    _lib.check(L.arches_kpm_scan_sequential(eng.plan.handle, eng.C, eng.S, _lib.ptr(eng.tel),
                                            _lib.ptr(eng.regime), None, _lib.ptr(eng.state),
                                            _lib.ptr(eng.kpm), _lib.ptr(eng.msg_log),
                                            _lib.ptr(eng.msg_count), eng.msg_cap, None))
    torch.cuda.synchronize()
    print("all ok")


if __name__ == "__main__":
    main()
