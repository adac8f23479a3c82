"""Call arches_ls_analyze repeatedly on one batch and diff the workspace."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    n_prb, slots = int(sys.argv[1]), int(sys.argv[2])
    from bench import make_inputs
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo, scens, pil, y, tx, nv, reg = make_inputs(n_prb, 4, slots, 7)
    plan = ArchesPlan(geo, 1.25, PipelineConfig(), ExecutionMode.CONCURRENT, "oracle")
    eng = SlotEngine(plan, 1, slots)
    eng.set_streams(pil[None], [7])
    eng.load(y=y, tx=tx, noise_var=nv, regime=reg)
    L = _lib.lib()
    snaps = []
    for r in range(4):
        if r == 2:
            eng.ws.fill_(0x7F)  # poison the scratch: stale-read detector
        _lib.check(L.arches_ls_analyze(plan.handle, 1, slots, _lib.ptr(eng.y), _lib.ptr(eng.pilots),
                                       None, 0, None, None, _lib.ptr(eng.ws),
                                       torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        snaps.append(eng.ws.cpu().numpy().copy())
    coef_bytes = slots * 2688
    for r in range(1, 4):
        d = np.nonzero(snaps[r][:coef_bytes] != snaps[0][:coef_bytes])[0]
        print(f"run {r}: coef bytes differing {d.size}", (d[:5] // 2688).tolist() if d.size else "")


if __name__ == "__main__":
    main()
