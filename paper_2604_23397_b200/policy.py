"""Decision-tree policy model: the artefact the hot path loads.

`Node`/`TreeModel` (switch_policy.py:63-98), the `tree v1` text format
(`to_text`/`from_text`, switch_policy.py:324-384) and `predict`
(switch_policy.py:237-248, evaluated on the device).  Training stays offline
in the reference (out of scope).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .errors import ConfigurationError, ContractViolation

FEATURE_ORDER = (
    "phy_throughput", "mcs_index", "pdu_length", "ndi", "rsrp",
    "snr_db", "mac_throughput", "lcid4_throughput", "mac_rx_bytes",
    "lcid4_rx_bytes",
)
LABEL_AI, LABEL_MMSE = 0, 1


@dataclass
class Node:
    counts: tuple
    feature: Optional[int] = None
    threshold: Optional[float] = None
    left: Optional["Node"] = None
    right: Optional["Node"] = None

    @property
    def is_leaf(self) -> bool:
        return self.feature is None

    @property
    def label(self) -> int:
        return LABEL_AI if self.counts[0] > self.counts[1] else LABEL_MMSE


@dataclass
class TreeModel:
    root: Node
    feature_names: tuple = FEATURE_ORDER

    def depth(self) -> int:
        def d(n):
            return 0 if n.is_leaf else 1 + max(d(n.left), d(n.right))
        return d(self.root)

    def nodes(self):
        out, todo = [], [self.root]
        while todo:
            n = todo.pop(0)
            out.append(n)
            if not n.is_leaf:
                todo += [n.left, n.right]
        return out


def to_text(tree) -> str:
    lines = ["tree v1", "features: " + ",".join(tree.feature_names)]
    nid = [0]

    def emit(node):
        me = nid[0]
        nid[0] += 1
        if node.is_leaf:
            lines.append(f"{me} leaf label={node.label} counts={node.counts[0]},{node.counts[1]}")
            return me
        at = len(lines)
        lines.append("")
        lft, rgt = emit(node.left), emit(node.right)
        lines[at] = (f"{me} split {tree.feature_names[node.feature]} <= {node.threshold!r} "
                     f"counts={node.counts[0]},{node.counts[1]} left={lft} right={rgt}")
        return me

    emit(tree.root)
    return "\n".join(lines) + "\n"


def from_text(text: str) -> TreeModel:
    rows = [r for r in text.splitlines() if r.strip()]
    if not rows or rows[0].strip() != "tree v1":
        raise ConfigurationError("unrecognized tree format")
    if len(rows) < 2 or not rows[1].startswith("features:"):
        raise ConfigurationError("missing feature list")
    names = tuple(rows[1].split(":", 1)[1].strip().split(","))
    spec = {}
    for r in rows[2:]:
        f = r.split()
        nid = int(f[0])
        if f[1] == "leaf":
            spec[nid] = {"counts": tuple(int(v) for v in f[3].split("=")[1].split(","))}
        elif f[1] == "split":
            spec[nid] = {"counts": tuple(int(v) for v in f[5].split("=")[1].split(",")),
                         "feature": names.index(f[2]), "threshold": float(f[4]),
                         "left": int(f[6].split("=")[1]), "right": int(f[7].split("=")[1])}
        else:
            raise ConfigurationError(f"bad tree line: {r}")

    def build(i):
        s = spec[i]
        if "feature" not in s:
            return Node(counts=s["counts"])
        return Node(s["counts"], s["feature"], s["threshold"], build(s["left"]),
                    build(s["right"]))

    return TreeModel(build(0), names)


def load_tree(path) -> TreeModel:
    with open(path) as f:
        return from_text(f.read())


def save_tree(tree, path):
    with open(path, "w") as f:
        f.write(to_text(tree))


def to_device_struct(tree) -> _lib.Tree:
    """Flatten a tree (ours or the reference's TreeModel) into `arches_tree`."""
    flat = []

    def visit(node):
        me = len(flat)
        flat.append(None)
        if node.feature is None:
            flat[me] = (-1, -1, -1, int(node.label), 0.0)
        else:
            l = visit(node.left)
            r = visit(node.right)
            flat[me] = (int(node.feature), l, r, int(node.label), float(node.threshold))
        return me

    visit(tree.root)
    if len(flat) > _lib.MAX_TREE_NODES:
        raise ConfigurationError(f"tree has {len(flat)} nodes > {_lib.MAX_TREE_NODES}")
    t = _lib.Tree()
    t.n_nodes = len(flat)
    for i, (f, l, r, lab, thr) in enumerate(flat):
        t.nodes[i] = _lib.TreeNode(f, l, r, lab, thr)
    return t


def tree_tensor(tree, device="cuda"):
    import torch
    raw = bytes(to_device_struct(tree))
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)


def predict(tree, x):
    """Root-to-leaf descent on the device; values equal to a threshold go left."""
    import torch
    arr = np.asarray(x, dtype=float)
    single = arr.ndim == 1
    rows = arr.reshape(1, -1) if single else arr
    if rows.ndim != 2:
        raise ContractViolation(f"expected 2-D feature array, got ndim={rows.ndim}")
    if rows.shape[1] != len(tree.feature_names):
        raise ContractViolation(
            f"expected {len(tree.feature_names)} feature columns, got {rows.shape[1]}")
    if not np.all(np.isfinite(rows)):
        raise ContractViolation("feature array contains NaN or Inf")
    dev = torch.device("cuda")
    xt = torch.from_numpy(np.ascontiguousarray(rows)).to(dev)
    tt = tree_tensor(tree, dev)
    out = torch.empty(len(rows), dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().arches_tree_predict(_lib.ptr(tt), _lib.ptr(xt), len(rows), rows.shape[1],
                                              _lib.ptr(out), s))
    res = out.cpu().numpy().astype(int)
    return int(res[0]) if single else res
