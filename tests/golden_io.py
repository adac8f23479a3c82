"""Loaders for the golden fixtures written by tools/make_golden.py (reference outputs)."""
from __future__ import annotations

import functools
import json
import math
import pathlib

import numpy as np

from paper_2604_23397_b200.config import DappConfig, ExecutionMode, PipelineConfig
from paper_2604_23397_b200.geometry import ScenarioConfig, SlotGeometry
from paper_2604_23397_b200.scene import CellScene

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


@functools.lru_cache(maxsize=None)
def experts_small():
    meta = json.loads((GOLDEN / "experts_small.json").read_text())
    arrs = np.load(GOLDEN / "experts_small.npz")
    cases = []
    for c in meta["cases"]:
        data = {k.split("__", 1)[1]: arrs[k] for k in arrs.files if k.startswith(c["id"] + "__")}
        cases.append((c, data))
    return cases


def small_case(cid):
    for c, d in experts_small():
        if c["id"] == cid:
            return c, d
    raise KeyError(cid)


@functools.lru_cache(maxsize=None)
def experts_large():
    return json.loads((GOLDEN / "experts_large.json").read_text())["cases"]


@functools.lru_cache(maxsize=None)
def loops():
    meta = json.loads((GOLDEN / "loops.json").read_text())["loops"]
    arrs = np.load(GOLDEN / "loops.npz")
    return [(m, arrs[m["id"] + "__records"], arrs[m["id"] + "__extra"]) for m in meta]


@functools.lru_cache(maxsize=None)
def loops_long():
    """Long loops at the benched shapes (tools/make_golden_long.py)."""
    meta = json.loads((GOLDEN / "loops_long.json").read_text())["loops"]
    arrs = np.load(GOLDEN / "loops_long.npz")
    return [(m, arrs[m["id"] + "__records"], arrs[m["id"] + "__extra"]) for m in meta]


def loop_case(lid):
    for m, r, e in loops():
        if m["id"] == lid:
            return m, r, e
    raise KeyError(lid)


@functools.lru_cache(maxsize=None)
def rng_vectors():
    return json.loads((GOLDEN / "rng.json").read_text())


def tree_text(name: str) -> str:
    return (GOLDEN / {"tree12": "tree_12prb.txt", "tree52": "tree_52prb.txt"}[name]).read_text()


def scenario_from_meta(d: dict) -> ScenarioConfig:
    kw = dict(d)
    kw["interference_prb_mask"] = tuple(kw.get("interference_prb_mask", ()))
    return ScenarioConfig(**kw)


def loop_setup(m: dict):
    """(geometry, scenarios, regimes, exec_mode, PipelineConfig, DappConfig) of a golden loop."""
    geo = SlotGeometry(n_ant=m["geometry"]["n_ant"], n_prb=m["geometry"]["n_prb"])
    scen = {k: scenario_from_meta(v) for k, v in m["scenarios"].items()}
    regimes = [r for r, n in m["timeline"] for _ in range(n)]
    p = m["pipeline"]
    pcfg = PipelineConfig(window_length=p["window_length"], noise_guard=p["noise_guard"],
                          truncation=p["truncation"], mmse_block_prbs=p["mmse_block_prbs"])
    d = m["dapp"]
    dcfg = DappConfig(decision_period_slots=d["decision_period_slots"],
                      window_length_slots=d["window_length_slots"],
                      failsafe_timeout_us=d["failsafe_timeout_us"])
    return geo, scen, regimes, ExecutionMode(m["exec_mode"]), pcfg, dcfg


def loop_inputs(geo, scen, regimes):
    """Slot inputs synthesised exactly as the reference Pipeline does."""
    cs = CellScene(geo, scen, regimes[0])
    return cs, [cs.next_slot(r) for r in regimes]


def case_scenario(c: dict) -> ScenarioConfig:
    snr = math.inf if c["snr_db"] == "inf" else c["snr_db"]
    kw = dict(c["scenario"])
    if "interference_prb_mask" in kw:
        kw["interference_prb_mask"] = tuple(kw["interference_prb_mask"])
    return ScenarioConfig(regime=c["regime"], seed=c["seed"], base_snr_db=snr,
                          mmse_assumed_delay_spread=c["assumed_delay_spread"], **kw)
