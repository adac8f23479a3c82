"""sigma2 of the golden small expert cases with the tensor-core K1 on and off."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def run(case, d, tc):
    import numpy as np
    if tc:
        os.environ.pop("ARCHES_DISABLE_K1T", None)
    else:
        os.environ["ARCHES_DISABLE_K1T"] = "1"
    from golden_io import case_scenario
    from paper_2604_23397_b200.config import ExecutionMode, PipelineConfig
    from paper_2604_23397_b200.engine import ArchesPlan, SlotEngine
    from paper_2604_23397_b200.geometry import SlotGeometry
    from paper_2604_23397_b200.scene import to_device_layout
    geo = SlotGeometry(n_ant=case["n_ant"], n_prb=case["n_prb"])
    scen = case_scenario(case)
    pcfg = PipelineConfig(noise_guard=case["guard"], truncation=case["truncation"])
    plan = ArchesPlan(geo, scen.assumed_delay_spread, pcfg, ExecutionMode.CONCURRENT, "fixed:1")
    eng = SlotEngine(plan, 1, 1)
    eng.set_streams(d["pilots"][None], [scen.seed])
    eng.load(y=to_device_layout(d["y"])[None], tx=d["tx"].T[None].astype(np.complex64),
             noise_var=[case["noise_var"]], regime=[1])
    eng.run()
    return float(eng.telemetry()[0, 0]["sigma2_hat"])


def main():
    from golden_io import experts_small
    for case, d in experts_small():
        print(case["id"], "tc", run(case, d, True), "cc", run(case, d, False), "ref", float(d["nv_est"]))


if __name__ == "__main__":
    main()
