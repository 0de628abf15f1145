"""Spatial-partition config: the reference's tree types, JSON format and host-side
tree building, plus the flattening into the C-ABI ``VrTree``.

Mirrors partitioner.py:51-80 (types), :97-163 (median-split build — one-time host
preprocessing), :166-174 (single-point locate, used for parameter
ownership checks) and :274-324 (JSON).  Batched owner lookup of samples runs in the
K1 kernel; ``locate_many`` here calls the ``vr_locate`` kernel.
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .errors import DegenerateSplitError, InsufficientPointsError, OutOfBoundsError
from .geometry import Aabb, vec3

AXES = "xyz"


@dataclass(frozen=True)
class LeafNode:
    tile_id: int
    box: Aabb


@dataclass(frozen=True)
class SplitNode:
    axis: int
    plane: float
    low: object
    high: object


@dataclass(frozen=True)
class PartitionTree:
    """2^depth disjoint leaves, half-open on split planes, numbered depth-first."""

    root_box: Aabb
    root: object
    depth: int
    leaves: tuple

    def __post_init__(self):
        if len(self.leaves) != 2 ** self.depth:
            raise ValueError("leaf count does not match depth")
        if len(self.leaves) > _lib.VR_MAX_REGIONS:
            raise ValueError(f"at most {_lib.VR_MAX_REGIONS} regions are supported")

    def to_c(self) -> _lib.VrTree:
        """Flatten into the C-ABI descriptor (internal nodes pre-order, root = 0)."""
        t = _lib.VrTree()
        for a in range(3):
            t.root_mn[a] = self.root_box.mn[a]
            t.root_mx[a] = self.root_box.mx[a]
        for leaf in self.leaves:
            for a in range(3):
                t.leaf_mn[leaf.tile_id][a] = leaf.box.mn[a]
                t.leaf_mx[leaf.tile_id][a] = leaf.box.mx[a]
        nodes = []

        def rec(node) -> int:
            if isinstance(node, LeafNode):
                return -node.tile_id - 1
            idx = len(nodes)
            nodes.append(node)
            lo = rec(node.low)
            hi = rec(node.high)
            t.node_axis[idx] = node.axis
            t.node_plane[idx] = node.plane
            t.node_low[idx] = lo
            t.node_high[idx] = hi
            return idx

        rec(self.root)
        t.n_leaves = len(self.leaves)
        t.n_nodes = len(nodes)
        return t


def _aspect_score(size: np.ndarray) -> float:
    g = float(np.cbrt(float(np.prod(size))))
    return float(np.abs(np.log(size / g)).sum())


def _median_plane(coords: np.ndarray) -> float:
    c = np.sort(coords)
    n = c.size
    if n % 2 == 1:
        return float(c[(n - 1) // 2])
    return 0.5 * (float(c[n // 2 - 1]) + float(c[n // 2]))


def choose_split(points: np.ndarray, box: Aabb):
    """Median plane per axis, most-cubic children win, ties x<y<z (partitioner.py:97-128)."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    if pts.shape[0] < 2:
        raise InsufficientPointsError("need at least 2 points to split")
    best = None
    for axis in range(3):
        coords = pts[:, axis]
        plane = _median_plane(coords)
        n_low = int(np.count_nonzero(coords <= plane))
        if n_low == 0 or n_low == pts.shape[0]:
            continue
        if not (box.mn[axis] < plane < box.mx[axis]):
            continue
        lo_size = box.size.copy()
        lo_size[axis] = plane - box.mn[axis]
        hi_size = box.size.copy()
        hi_size[axis] = box.mx[axis] - plane
        score = _aspect_score(lo_size) + _aspect_score(hi_size)
        if best is None or score < best[0]:
            best = (score, axis, plane)
    if best is None:
        raise DegenerateSplitError("no axis separates the points inside the box")
    return best[1], best[2]


def build_tree(points, root_box: Aabb, depth: int) -> PartitionTree:
    """Recursive median splits down to 2^depth leaves (partitioner.py:131-163)."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    if depth < 0:
        raise ValueError("depth must be >= 0")
    if pts.shape[0] < 2 ** depth:
        raise InsufficientPointsError(f"{pts.shape[0]} points cannot fill {2 ** depth} tiles")
    leaves = []

    def rec(p, box, d):
        if d == 0:
            leaf = LeafNode(len(leaves), box)
            leaves.append(leaf)
            return leaf
        if p.shape[0] < 2:
            raise InsufficientPointsError("a subtree ran out of points to split")
        axis, plane = choose_split(p, box)
        low_sel = p[:, axis] <= plane
        lo_mx = box.mx.copy()
        lo_mx[axis] = plane
        hi_mn = box.mn.copy()
        hi_mn[axis] = plane
        low = rec(p[low_sel], Aabb(box.mn, lo_mx), d - 1)
        high = rec(p[~low_sel], Aabb(hi_mn, box.mx), d - 1)
        return SplitNode(axis, plane, low, high)

    root = rec(pts, root_box, depth)
    return PartitionTree(root_box, root, depth, tuple(leaves))


def grid_tree(root_box: Aabb, splits) -> PartitionTree:
    """Tree of midpoint splits along a fixed axis sequence, e.g. "xxx" = 8 x-strips,
    "xyx" = a 4x2 grid.  Used for the synthetic street/city workloads."""
    leaves = []

    def rec(box, level):
        if level == len(splits):
            leaf = LeafNode(len(leaves), box)
            leaves.append(leaf)
            return leaf
        axis = AXES.index(splits[level])
        plane = float(0.5 * (box.mn[axis] + box.mx[axis]))
        lo_mx = box.mx.copy()
        lo_mx[axis] = plane
        hi_mn = box.mn.copy()
        hi_mn[axis] = plane
        low = rec(Aabb(box.mn, lo_mx), level + 1)
        high = rec(Aabb(hi_mn, box.mx), level + 1)
        return SplitNode(axis, plane, low, high)

    root = rec(root_box, 0)
    return PartitionTree(root_box, root, len(splits), tuple(leaves))


def locate(tree: PartitionTree, p) -> int:
    """Owner of a single point; planes belong to the high child (partitioner.py:166-174)."""
    p = vec3(p)
    if not tree.root_box.contains(p):
        raise OutOfBoundsError(f"{p} outside root box")
    node = tree.root
    while isinstance(node, SplitNode):
        node = node.low if p[node.axis] < node.plane else node.high
    return node.tile_id


def locate_many(tree: PartitionTree, pts, device=None) -> np.ndarray:
    """Owner ids of many points via the vr_locate kernel (partitioner.py:177-192)."""
    import torch

    pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
    dev = torch.device(device or "cuda")
    p = torch.from_numpy(pts).to(dev)
    out = torch.empty(pts.shape[0], dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    tc = tree.to_c()
    import ctypes

    _lib.call("vr_locate", _lib.addr(tc), _lib.ptr(p), pts.shape[0], _lib.ptr(out),
              _lib.ptr(err), _lib.stream_ptr())
    _lib.raise_flags(int(err.item()), "in locate_many")
    return out.cpu().numpy().astype(np.int64)


def _node_to_json(node) -> dict:
    if isinstance(node, LeafNode):
        return {"tile_id": node.tile_id, "box": node.box.to_json()}
    return {"axis": AXES[node.axis], "plane": float(node.plane),
            "low": _node_to_json(node.low), "high": _node_to_json(node.high)}


def _node_from_json(d: dict, box: Aabb, leaves: list):
    if "tile_id" in d:
        leaf = LeafNode(int(d["tile_id"]), Aabb.from_json(d["box"]))
        if leaf.tile_id != len(leaves):
            raise ValueError("leaf tile_ids must be depth-first sequential")
        leaves.append(leaf)
        return leaf
    axis = AXES.index(d["axis"])
    plane = float(d["plane"])
    lo_mx = box.mx.copy()
    lo_mx[axis] = plane
    hi_mn = box.mn.copy()
    hi_mn[axis] = plane
    low = _node_from_json(d["low"], Aabb(box.mn, lo_mx), leaves)
    high = _node_from_json(d["high"], Aabb(hi_mn, box.mx), leaves)
    return SplitNode(axis, plane, low, high)


def tree_to_json(tree: PartitionTree) -> dict:
    """Same field order as partitioner.tree_to_json (partitioner.py:305-311)."""
    return {"root_box": tree.root_box.to_json(), "depth": tree.depth,
            "root": _node_to_json(tree.root)}


def tree_from_json(d: dict) -> PartitionTree:
    root_box = Aabb.from_json(d["root_box"])
    leaves = []
    root = _node_from_json(d["root"], root_box, leaves)
    return PartitionTree(root_box, root, int(d["depth"]), tuple(leaves))


def save_tree(tree: PartitionTree, path) -> None:
    Path(path).write_text(json.dumps(tree_to_json(tree), indent=2) + "\n")


def load_tree(path) -> PartitionTree:
    return tree_from_json(json.loads(Path(path).read_text()))
