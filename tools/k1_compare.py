"""Compare the tensor-core K1 against the CUDA-core K1 (sigma2, taps) on the GPU.

    python tools/k1_compare.py [--n-prb 273] [--slots 8]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(n_prb, slots, disable_tc):
    import numpy as np
    import torch
    if disable_tc:
        os.environ["ARCHES_DISABLE_K1T"] = "1"
    else:
        os.environ.pop("ARCHES_DISABLE_K1T", None)
    from bench import make_inputs
    from paper_2604_23397_b200 import _lib
    from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    geo, scens, pil, y, tx, nv, reg = make_inputs(n_prb, 4, slots, 1000)
    plan = ArchesPlan(geo, 1.25, PipelineConfig(), ExecutionMode.CONCURRENT, "oracle")
    eng = SlotEngine(plan, 1, slots)
    eng.set_streams(pil[None], [1000])
    eng.load(y=y, tx=tx, noise_var=nv, regime=reg)
    sig = torch.zeros(slots, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    _lib.check(L.arches_ls_analyze(plan.handle, 1, slots, _lib.ptr(eng.y), _lib.ptr(eng.pilots),
                                   None, 0, None, _lib.ptr(sig), _lib.ptr(eng.ws),
                                   torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    A, D, T = 4, 3, 20
    nc = A * D * (8 + T)
    coef = eng.ws[: slots * ((nc + 1) // 2 * 2) * 8].view(torch.complex64).cpu().numpy()
    return sig.cpu().numpy(), coef.reshape(slots, -1)[:, :nc]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-prb", type=int, default=273)
    ap.add_argument("--slots", type=int, default=8)
    a = ap.parse_args()
    import numpy as np
    s_tc, c_tc = run(a.n_prb, a.slots, False)
    import importlib
    s_cc, c_cc = run(a.n_prb, a.slots, True)
    print("sigma2 rel diff", np.max(np.abs(s_tc - s_cc) / np.abs(s_cc)))
    mm = slice(0, 96)
    print("mmse taps max rel", np.max(np.abs(c_tc[:, mm] - c_cc[:, mm])) / np.max(np.abs(c_cc[:, mm])))
    print("ai taps max rel", np.max(np.abs(c_tc[:, 96:] - c_cc[:, 96:])) / np.max(np.abs(c_cc[:, 96:])))
    print("per-tap worst", np.argmax(np.abs(c_tc - c_cc).max(axis=0)))


if __name__ == "__main__":
    main()
