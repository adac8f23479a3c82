"""Golden vectors for the Eq. 3 perturbation path from the UNMODIFIED reference
(build container only).  Writes tests/golden/perturb.npz / perturb.json.

  * per-slot traces: a Pipeline in SELECTED_ONLY mode (MMSE only, as
    perturbation_lab.sweep runs it, perturbation_lab.py:114-144) with the
    Pipeline.perturb hook (phy_pipeline.py:401,444-445) set to
    perturbation_lab._inject_values (:92-98) at rho in RHOS, 40 slots each:
    KPM rows, post-eq SINR, est_abs_mean, CRC, and the perturbed MMSE buffer of
    the first two slots;
  * perturbation_lab.sweep's DegradationTable (means, ci95) on the same
    geometry and scenario for a 5-point rho grid x 30 slots.
"""
from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import make_golden as MG  # noqa: E402  (loads the reference through ref_shim)
from ranswitch import perturbation_lab as PL  # noqa: E402

PP, RS = MG.PP, MG.RS
RHOS = (0.0, 0.7, 1.6)
N_SLOTS = 40
SEED = 41


def scenario():
    return RS.ScenarioConfig(regime="good", seed=SEED, mmse_assumed_delay_spread=1.25)


def main():
    geo = RS.SlotGeometry(n_prb=12)
    scen = scenario()
    arr, meta = {}, {"versions": MG.versions(), "n_prb": 12, "n_ant": geo.n_ant, "seed": SEED,
                     "rhos": list(RHOS), "slots": N_SLOTS,
                     "scenario": {k: (list(v) if isinstance(v, tuple) else v)
                                  for k, v in vars(scen).items()}}
    for i, rho in enumerate(RHOS):
        pipe = PP.Pipeline(geo, scen, exec_mode=PP.ExecutionMode.SELECTED_ONLY)
        pipe.perturb = lambda slot, values, _r=rho: PL._inject_values(values, _r, scen.seed, slot)
        rows, extra = [], []
        for s in range(N_SLOTS):
            out = pipe.run_slot()
            rows.append([float(v) for v in out.kpm.row()])
            extra.append([out.post_eq_sinr_db, out.est_abs_mean, float(out.crc_pass)])
            if s < 2:
                arr[f"rho{i}__mmse_slot{s}"] = np.array(pipe.buffers.buffer_mmse)
        arr[f"rho{i}__records"] = np.array(rows)
        arr[f"rho{i}__extra"] = np.array(extra)
        print("rho", rho, "mean snr", np.mean([e[0] for e in extra]), flush=True)
    grid = (0.0, 0.5, 1.0, 1.5, 2.0)
    table = PL.sweep(scen, PL.PerturbationConfig(rho_values=grid, slots_per_point=30, seed=SEED),
                     geometry=geo)
    arr["sweep__mean"] = table.mean
    arr["sweep__ci95"] = table.ci95
    meta["sweep"] = {"rho_values": list(grid), "slots_per_point": 30,
                     "kpm_names": list(table.kpm_names)}
    out = MG.OUT
    np.savez_compressed(out / "perturb.npz", **arr)
    (out / "perturb.json").write_text(json.dumps(meta, indent=1))
    print("done")


if __name__ == "__main__":
    main()
