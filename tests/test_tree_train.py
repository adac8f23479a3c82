"""GPU tree training (k_tree_eval_splits, paper_2604_23397_b200.train) against
trees trained by the unmodified reference (switch_policy.train,
switch_policy.py:173-234; tools/make_golden_train.py): the `tree v1` text must
be byte-identical -- split features, thresholds (repr), tie-breaks, counts --
on 40 random datasets (integer grids with ties, continuous, pure, depths
0/1/2) and the simulator-labelled dataset behind the golden tree_12prb."""
import json
import pathlib

import numpy as np
import pytest

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def _cases():
    meta = json.loads((GOLD / "train.json").read_text())["cases"]
    arr = np.load(GOLD / "train.npz")
    return [(c, arr[c["id"] + "__x"], arr[c["id"] + "__y"]) for c in meta]


def test_golden_trees_round_trip_the_text_format():
    from paper_2604_23397_b200.policy import from_text, to_text
    for c, _, _ in _cases():
        assert to_text(from_text(c["tree"])) == c["tree"]


def test_root_candidates_follow_the_reference_scan_order():
    from paper_2604_23397_b200.train import _root_candidates
    x = np.array([[1.0, 5.0], [0.0, 5.0], [1.0, 2.0], [3.0, 7.0]])
    f, t = _root_candidates(x)
    assert f.tolist() == [0, 0, 1, 1] and t.tolist() == [0.5, 2.0, 3.5, 6.0]


@pytest.mark.gpu
def test_device_training_equals_reference():
    from paper_2604_23397_b200.policy import to_text
    from paper_2604_23397_b200.train import train
    for c, x, y in _cases():
        tree = train(x, y, max_depth=c["max_depth"], feature_names=tuple(c["features"]))
        assert to_text(tree) == c["tree"], c["id"]


@pytest.mark.gpu
def test_device_training_scales():
    """5,000-row, 10-feature dataset (the SPEC's >= 5,000-slot labelled set):
    every one of the ~50k root candidates scored on the device."""
    import time
    from paper_2604_23397_b200.train import _root_candidates, eval_splits, train
    rng = np.random.default_rng(1)
    x = rng.normal(size=(5000, 10))
    y = ((x[:, 6] > 0.2) ^ (x[:, 1] < -0.5)).astype(int)
    t0 = time.perf_counter()
    tree = train(x, y)
    dt = time.perf_counter() - t0
    f, _ = _root_candidates(x)
    assert len(f) >= 49_000
    assert tree.depth() == 2 and {tree.root.feature} <= {1, 6}
    assert dt < 30.0
