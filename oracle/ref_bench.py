"""Timed CPU baseline on the UNMODIFIED reference itself (bench.py's reference arm).

TEST/BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).  Imports the staged
reference package (`baseline/_ref/ranswitch`, staged by tools/fetch_ref.py --
/root/reference itself is not on the GPU box; Python >= 3.11 import fix only,
no source change) and runs its own closed loop `harness.execute_run`
(harness.py:174-231) for the bench workload: good / poor alternating every slot,
oracle policy (config B) or a tree policy with the default dApp (config A),
concurrent experts.  Per-slot time = the reference's `Pipeline.run_slot`
(phy_pipeline.py:422-493) plus the control glue of the loop; that includes the
reference's own slot synthesis (~3% of a 273-PRB slot, which spends ~0.5 s in
the per-slot Wiener Cholesky).  Prints one JSON line.

    OPENBLAS_NUM_THREADS=1 python -m oracle.ref_bench --n-prb 273 --slots 3 --seed 5
"""
from __future__ import annotations

import argparse
import importlib
import importlib.util
import json
import os
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF_SRC = ROOT / "baseline" / "_ref" / "ranswitch"


def staged() -> bool:
    return (REF_SRC / "__init__.py").exists()


def load_reference():
    sys.dont_write_bytecode = True
    spec = importlib.util.spec_from_file_location(
        "ranswitch", REF_SRC / "__init__.py", submodule_search_locations=[str(REF_SRC)])
    pkg = importlib.util.module_from_spec(spec)
    sys.modules["ranswitch"] = pkg
    importlib.import_module("ranswitch.phy_pipeline").PipelineConfig.__hash__ = object.__hash__
    spec.loader.exec_module(pkg)
    return pkg


def policy_stress(a, ref):
    """Config D on the reference's own dApp: per slot boundary, for each sampled
    cell, Dapp.on_indication (dapp_control.py:107-120: window append, window_features
    over the last 100 records, predict, ControlMessage), decision every slot."""
    import numpy as np
    PP, SP, DC = ref.phy_pipeline, ref.switch_policy, ref.dapp_control
    tree = SP.from_text(open(a.tree).read())
    rng = np.random.default_rng(a.seed)
    cfg = DC.DappConfig(decision_period_slots=1, window_length_slots=100)

    def record(n):
        return PP.KpmRecord(slot_index=n, phy_throughput=float(rng.random() * 40),
                            mcs_index=int(rng.integers(0, 28)), pdu_length=int(rng.integers(0, 3000)),
                            ndi=int(rng.integers(0, 2)), rsrp=float(rng.random()), code_rate=0.5,
                            qam_order=4, num_cb=1, tb_size=int(rng.integers(0, 3000)),
                            snr_db=float(rng.normal(10, 8)), mac_throughput=float(rng.random() * 40),
                            lcid4_throughput=float(rng.random() * 30),
                            mac_rx_bytes=int(rng.integers(0, 3000)),
                            lcid4_rx_bytes=int(rng.integers(0, 2500)))
    slot_ns = 500_000
    dapps = [DC.Dapp(tree, DC.LatencyModel(), cfg) for _ in range(a.cells)]
    for n in range(100):                      # fill the windows
        for d in dapps:
            d.on_indication(DC.E3Indication((record(n),), (n + 1) * slot_ns))
    fresh = [[record(100 + s) for s in range(a.slots)] for _ in range(a.cells)]
    per_boundary = []
    for s in range(a.slots):
        t0 = time.perf_counter()
        for c, d in enumerate(dapps):
            d.on_indication(DC.E3Indication((fresh[c][s],), (101 + s) * slot_ns))
        per_boundary.append(time.perf_counter() - t0)
    print(json.dumps({"mode": "policy-stress", "cells": a.cells, "boundaries": a.slots,
                      "per_boundary_s": per_boundary,
                      "impl": "reference (staged ranswitch: Dapp.on_indication)"}))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-prb", type=int, default=273)
    ap.add_argument("--n-ant", type=int, default=4)
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--policy", default="oracle", choices=["oracle", "tree"])
    ap.add_argument("--tree", default=None)
    ap.add_argument("--policy-stress", action="store_true")
    ap.add_argument("--cells", type=int, default=16)
    a = ap.parse_args(argv)
    ref = load_reference()
    if a.policy_stress:
        return policy_stress(a, ref)
    H, PP, RS, SP, DC = (ref.harness, ref.phy_pipeline, ref.radio_scene, ref.switch_policy,
                         ref.dapp_control)
    geo = RS.SlotGeometry(n_ant=a.n_ant, n_prb=a.n_prb)
    scens = H.default_scenarios(a.seed, geo)
    regimes = ["good" if i % 2 == 0 else "poor" for i in range(a.slots)]
    # the slot loop of harness.execute_run (harness.py:180-226) around the reference's
    # own Pipeline (an ExperimentSpec would insist on >= 100 slots: the KPM window)
    pipe = PP.Pipeline(geo, scens[regimes[0]], PP.ExecutionMode.CONCURRENT)
    slot_ns = geo.slot_duration_ns
    last = 1
    dapp = monitor = None
    if a.policy == "tree":
        dapp = DC.Dapp(SP.from_text(open(a.tree).read()), DC.LatencyModel(), DC.DappConfig())
        monitor = DC.FailsafeMonitor(timeout_ns=DC.DappConfig().timeout_ns(slot_ns))
    per_slot = []
    current = regimes[0]
    t_all = time.perf_counter()
    for n, regime in enumerate(regimes):
        if regime != current:
            pipe.set_scenario(scens[regime])
            current = regime
        t0 = time.perf_counter()
        out = pipe.run_slot()
        end_ns = (n + 1) * slot_ns
        if dapp is None:   # oracle source (harness.py:205-212)
            mode = 1 if regime == "good" else 0
            if mode != last:
                pipe.deliver(PP.ControlMessage(mode=mode, decided_at_ns=end_ns,
                                               deliverable_at_ns=end_ns, trigger="oracle"))
                last = mode
        else:              # dApp source (harness.py:213-226)
            msg = dapp.on_indication(DC.E3Indication(kpm_window=(out.kpm,), emitted_at_ns=end_ns,
                                                     slot_duration_ns=slot_ns))
            if msg is not None:
                pipe.deliver(msg)
                monitor.note_delivery(msg.deliverable_at_ns)
            forced = H.failsafe_check(monitor, end_ns, pipe.controller.mode_var.mode)
            if forced is not None:
                pipe.controller.force_mode(forced, at_ns=end_ns)
        per_slot.append(time.perf_counter() - t0)
    total = time.perf_counter() - t_all
    print(json.dumps({"slots": a.slots, "seconds": total, "per_slot_s": per_slot,
                      "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
                      "n_prb": a.n_prb, "n_ant": a.n_ant, "policy": a.policy,
                      "impl": "reference (staged ranswitch: Pipeline.run_slot + the execute_run "
                              "control glue)"}))


if __name__ == "__main__":
    main()
