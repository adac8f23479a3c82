"""Depth-<=2 Gini decision-tree training on the GPU (switch_policy.train,
switch_policy.py:173-234): the exhaustive root search runs as one warp per
root candidate in `k_tree_eval_splits` (csrc/k_tree_train.cuh); the host
enumerates the root candidates and assembles the tree exactly as the
reference does, so the trained model -- thresholds, tie-breaks, counts, and
its `tree v1` text -- is the reference's, byte for byte.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ConfigurationError, ContractViolation
from .policy import FEATURE_ORDER, Node, TreeModel


def _counts(y) -> tuple:
    n0 = int(np.count_nonzero(y == 0))
    return (n0, len(y) - n0)


def _leaf_total(counts) -> float:
    n = counts[0] + counts[1]
    return 0.0 if n == 0 else n - (counts[0] ** 2 + counts[1] ** 2) / n


def _root_candidates(x: np.ndarray):
    """(feature, threshold) of every root split in the reference's scan order:
    features ascending, midpoints of consecutive distinct sorted values ascending
    (`_split_candidates`, switch_policy.py:116-132)."""
    feats, thrs = [], []
    for f in range(x.shape[1]):
        xs = np.sort(x[:, f], kind="stable")
        cut = np.nonzero(xs[:-1] < xs[1:])[0]
        t = 0.5 * (xs[cut] + xs[cut + 1])
        feats.append(np.full(len(t), f, np.int32))
        thrs.append(t)
    return np.concatenate(feats), np.concatenate(thrs)


def eval_splits(x: np.ndarray, y: np.ndarray, feats: np.ndarray, thrs: np.ndarray) -> np.ndarray:
    """Device scores (SPLIT_EVAL_DTYPE per candidate) of the given root splits."""
    import torch
    if not torch.cuda.is_available():
        from .errors import DeviceError
        raise DeviceError("tree training runs on the CUDA device")
    n, F = x.shape
    dev = torch.device("cuda")
    xT = torch.from_numpy(np.ascontiguousarray(x.T, dtype=np.float64)).to(dev)
    order = torch.from_numpy(np.stack([np.argsort(x[:, f], kind="stable") for f in range(F)])
                             .astype(np.int32)).to(dev)
    yd = torch.from_numpy(np.asarray(y, dtype=np.uint8)).to(dev)
    fd = torch.from_numpy(np.ascontiguousarray(feats, dtype=np.int32)).to(dev)
    td = torch.from_numpy(np.ascontiguousarray(thrs, dtype=np.float64)).to(dev)
    out = torch.empty(len(feats) * _lib.SPLIT_EVAL_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().arches_tree_eval_splits(
        _lib.ptr(xT), _lib.ptr(order), _lib.ptr(yd), n, F, _lib.ptr(fd), _lib.ptr(td), len(feats),
        _lib.ptr(out), torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy().view(_lib.SPLIT_EVAL_DTYPE)


def train(x, y, max_depth: int = 2, feature_names=FEATURE_ORDER) -> TreeModel:
    """switch_policy.train on the device; same contract and result."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=int)
    if x.ndim != 2 or x.shape[1] != len(feature_names):
        raise ContractViolation(f"features must be (n, {len(feature_names)})")
    if y.ndim != 1 or len(y) != len(x):
        raise ContractViolation("labels must be 1-D and aligned with rows")
    if not np.all((y == 0) | (y == 1)):
        raise ContractViolation("labels must be 0 or 1")
    if len(y) == 0:
        raise ContractViolation("cannot train on an empty dataset")
    if max_depth not in (0, 1, 2):
        raise ConfigurationError("max_depth must be 0, 1 or 2")
    names = tuple(feature_names)
    root_counts = _counts(y)
    if max_depth == 0 or root_counts[0] == 0 or root_counts[1] == 0:
        return TreeModel(Node(counts=root_counts), names)

    def leaf(mask):
        return Node(counts=_counts(y[mask]))

    if max_depth == 1:
        ev = eval_splits(x, y, np.array([-1], np.int32), np.zeros(1))[0]
        f = int(ev["left_feature"])
        if f < 0:
            return TreeModel(Node(counts=root_counts), names)
        t = float(ev["left_threshold"])
        lm = x[:, f] <= t
        return TreeModel(Node(counts=root_counts, feature=f, threshold=t, left=leaf(lm),
                              right=leaf(~lm)), names)
    feats, thrs = _root_candidates(x)
    if len(feats) == 0:
        return TreeModel(Node(counts=root_counts), names)
    ev = eval_splits(x, y, feats, thrs)
    tot = ev["total"]
    k = int(np.argmin(tot))                   # first minimum in scan order
    if not tot[k] < _leaf_total(root_counts):
        return TreeModel(Node(counts=root_counts), names)
    f, t = int(feats[k]), float(thrs[k])
    lmask = x[:, f] <= t

    def child(mask, cf, ct):
        if cf < 0:
            return leaf(mask)
        sub = mask & (x[:, cf] <= ct)
        return Node(counts=_counts(y[mask]), feature=cf, threshold=ct, left=leaf(sub),
                    right=leaf(mask & ~sub))

    root = Node(counts=root_counts, feature=f, threshold=t,
                left=child(lmask, int(ev["left_feature"][k]), float(ev["left_threshold"][k])),
                right=child(~lmask, int(ev["right_feature"][k]), float(ev["right_threshold"][k])))
    return TreeModel(root, names)
