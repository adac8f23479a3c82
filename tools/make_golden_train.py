"""Golden depth-<=2 trees trained by the UNMODIFIED reference (`switch_policy.train`,
switch_policy.py:173-234) for the device trainer (build container only).

Writes tests/golden/train.npz (x, y per case) + train.json (max_depth, feature
names, the reference's `to_text` of the trained tree per case):
  * 40 random datasets: integer grids 0..4 (duplicate values, threshold and
    impurity ties -- the tie rules are part of the contract), continuous
    normals, 20..240 rows, 2..10 features, depths 0 / 1 / 2, pure-label sets;
  * the simulator-labelled dataset the golden tree_12prb was trained on
    (harness.build_labeled_dataset, fixed MMSE, 12 PRB, G/P/G/P x 300 slots).
"""
from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import make_golden as MG  # noqa: E402

SP, H, RS, PP = MG.SP, MG.H, MG.RS, MG.PP


def main():
    rng = np.random.default_rng(2026)
    arr, cases = {}, []
    for i in range(40):
        n = int(rng.integers(20, 241))
        d = int(rng.integers(2, 11))
        kind = ["grid", "normal", "grid", "mixed"][i % 4]
        if kind == "grid":
            x = rng.integers(0, 5, size=(n, d)).astype(float)
        elif kind == "normal":
            x = rng.normal(0, 1, size=(n, d))
        else:
            x = np.concatenate([rng.integers(0, 3, size=(n, d // 2)).astype(float),
                                rng.normal(0, 10, size=(n, d - d // 2))], axis=1)
        y = rng.integers(0, 2, size=n)
        if i % 13 == 12:
            y[:] = i % 2          # pure labels: the root stays a leaf
        depth = [2, 2, 1, 2, 0][i % 5]
        names = tuple(f"f{j}" for j in range(d))
        tree = SP.train(SP.LabeledDataset(x, y, names), max_depth=depth)
        cid = f"r{i:02d}"
        arr[f"{cid}__x"], arr[f"{cid}__y"] = x, y
        cases.append({"id": cid, "max_depth": depth, "features": list(names),
                      "tree": SP.to_text(tree)})
    spec = H.ExperimentSpec(timeline=(("good", 300), ("poor", 300), ("good", 300), ("poor", 300)),
                            exec_mode=PP.ExecutionMode.SELECTED_ONLY, policy="fixed:1", seed=21,
                            geometry=RS.SlotGeometry(n_prb=12),
                            scenarios=H.default_scenarios(21, RS.SlotGeometry(n_prb=12)))
    data = H.build_labeled_dataset(spec)
    tree = SP.train(data, max_depth=2)
    arr["sim12__x"], arr["sim12__y"] = data.x, data.y
    cases.append({"id": "sim12", "max_depth": 2, "features": list(data.feature_names),
                  "tree": SP.to_text(tree)})
    out = MG.OUT
    np.savez_compressed(out / "train.npz", **arr)
    (out / "train.json").write_text(json.dumps({"versions": MG.versions(), "cases": cases},
                                               indent=1))
    print(len(cases), "cases; sim12 rows", len(data), "\n" + SP.to_text(tree))


if __name__ == "__main__":
    main()
