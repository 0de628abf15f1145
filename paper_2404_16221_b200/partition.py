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
from .errors import DegenerateSplitError, InsufficientPointsError, NoPointsError, OutOfBoundsError
from .geometry import Aabb, rays_to_soa, vec3

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


def _halves(box: Aabb, axis: int, plane: float):
    """The (low, high) children of ``box`` cut at ``plane`` on ``axis``."""
    lo_mx, hi_mn = box.mx.copy(), box.mn.copy()
    lo_mx[axis] = plane
    hi_mn[axis] = plane
    return Aabb(box.mn, lo_mx), Aabb(hi_mn, box.mx)


def _cubeness(sizes: np.ndarray) -> np.ndarray:
    """Sum over a box's three extents of |log(extent / geometric-mean extent)| (0 for a
    cube), for every box of ``sizes[..., 3]`` (partitioner.py:83-86)."""
    with np.errstate(divide="ignore", invalid="ignore"):  # (non-candidate axes: 0 extents)
        gm = np.cbrt(np.prod(sizes, axis=-1))
        return np.abs(np.log(sizes / gm[..., None])).sum(axis=-1)


def choose_split(points: np.ndarray, box: Aabb):
    """Split plane of one node (partitioner.py:97-128): on each axis the median of the
    points' coordinates (mean of the two middle ones for an even count); an axis is a
    candidate when the plane lies strictly inside the box and leaves points on both sides
    (low side: coordinate <= plane); of the candidates, the one whose two children are the
    most cube-like wins, the lower axis on a tie.  All three axes are evaluated at once."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    if n < 2:
        raise InsufficientPointsError("need at least 2 points to split")
    srt = np.sort(pts, axis=0)
    planes = srt[(n - 1) // 2] if n % 2 else 0.5 * (srt[n // 2 - 1] + srt[n // 2])
    n_low = np.count_nonzero(pts <= planes, axis=0)
    ok = (n_low > 0) & (n_low < n) & (box.mn < planes) & (planes < box.mx)
    if not ok.any():
        raise DegenerateSplitError("no axis separates the points inside the box")
    # children extents per candidate axis: [axis][low/high][extent]
    ext = np.broadcast_to(box.size, (3, 2, 3)).copy()
    ax = np.arange(3)
    ext[ax, 0, ax] = planes - box.mn
    ext[ax, 1, ax] = box.mx - planes
    cube = _cubeness(ext)
    score = np.where(ok, cube[:, 0] + cube[:, 1], np.inf)
    axis = int(np.argmin(score))
    return axis, float(planes[axis])


def _grow(root_box: Aabb, depth: int, cut, payload) -> PartitionTree:
    """Complete binary tree built one level at a time.  ``cut(payload, box, level)`` returns
    (axis, plane) of a node; ``payload`` (e.g. the node's points) is handed to the children
    split by the same rule as the points' owner lookup: low child iff coordinate <= plane
    for the build, i.e. the reference's median split (partitioner.py:131-163).  In a
    complete tree the depth-first leaf order is the bottom level's left-to-right order,
    which numbers the tiles.  A node whose cut fails stops its subtree; the error raised is
    the one the reference's depth-first recursion meets first (smallest pre-order key)."""
    level = [(root_box, payload)]
    cuts = []  # per level: (axis, plane) of each node, left to right
    failed = []  # (pre-order key, exception)
    for d in range(depth):
        row, nxt = [], []
        for i, (box, pl) in enumerate(level):
            if box is None:  # below a failed node
                row.append(None)
                nxt += [(None, None), (None, None)]
                continue
            try:
                axis, plane = cut(pl, box, d)
            except (InsufficientPointsError, DegenerateSplitError) as e:
                failed.append(((i << (depth - d), d), e))
                row.append(None)
                nxt += [(None, None), (None, None)]
                continue
            row.append((axis, plane))
            lo_box, hi_box = _halves(box, axis, plane)
            if pl is None:
                nxt += [(lo_box, None), (hi_box, None)]
            else:
                sel = pl[:, axis] <= plane
                nxt += [(lo_box, pl[sel]), (hi_box, pl[~sel])]
        cuts.append(row)
        level = nxt
    if failed:
        raise min(failed, key=lambda f: f[0])[1]
    nodes = [LeafNode(i, box) for i, (box, _) in enumerate(level)]
    leaves = tuple(nodes)
    for row in reversed(cuts):  # assemble bottom-up
        nodes = [SplitNode(a, p, nodes[2 * i], nodes[2 * i + 1]) for i, (a, p) in enumerate(row)]
    return PartitionTree(root_box, nodes[0], depth, leaves)


def build_tree(points, root_box: Aabb, depth: int) -> PartitionTree:
    """Median-split tree with 2^depth leaves over ``points`` (partitioner.py:131-163)."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    if depth < 0:
        raise ValueError("depth must be >= 0")
    if pts.shape[0] < 2 ** depth:
        raise InsufficientPointsError(f"{pts.shape[0]} points cannot fill {2 ** depth} tiles")

    def cut(p, box, d):
        if p.shape[0] < 2:
            raise InsufficientPointsError("a subtree ran out of points to split")
        return choose_split(p, box)

    return _grow(root_box, depth, cut, pts)


def grid_tree(root_box: Aabb, splits) -> PartitionTree:
    """Tree of midpoint splits along a fixed axis sequence, e.g. "xxx" = 8 x-strips,
    "xyx" = a 4x2 grid.  Used for the synthetic street/city workloads."""
    axes = [AXES.index(c) for c in splits]

    def cut(_, box, d):
        a = axes[d]
        return a, float(0.5 * (box.mn[a] + box.mx[a]))

    return _grow(root_box, len(axes), cut, None)


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


# ---- sample-balanced partitioning --------------------------------

@dataclass(frozen=True)
class PointCloud:
    """partitioner.PointCloud: points (n, 3) float64 and their source tag."""

    points: np.ndarray
    source: str


def _k1_all_leaves(tree: PartitionTree, rays, dt: float, device=None):
    """K1 (vr_sample_count / vr_scan_offsets / vr_sample_fill) over every leaf of ``tree``;
    returns (rays_dev, t0, t1, ray_id, per-leaf sample totals) on the device."""
    import torch

    if not dt > 0.0:
        raise ValueError("dt must be > 0")
    if not isinstance(rays, (np.ndarray, torch.Tensor)):
        rays = rays_to_soa(list(rays))
    dev = torch.device(device or "cuda")
    r = torch.as_tensor(np.ascontiguousarray(rays, dtype=np.float64) if isinstance(rays, np.ndarray)
                        else rays, dtype=torch.float64).to(dev).contiguous()
    R, K = r.shape[1], len(tree.leaves)
    s = _lib.stream_ptr()
    tc = tree.to_c()
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    counts = torch.empty(K * R, dtype=torch.int32, device=dev)
    first = torch.empty(K * R, dtype=torch.int32, device=dev)
    te = torch.empty(R, dtype=torch.float64, device=dev)
    _lib.call("vr_sample_count", _lib.addr(tc), _lib.ptr(r), R, R, float(dt), 0, K,
              _lib.ptr(counts), _lib.ptr(first), _lib.ptr(te), None, None, None, _lib.ptr(err), s)
    off = torch.empty(K * R + 1, dtype=torch.int64, device=dev)
    ws = torch.empty(int(_lib.load().vr_scan_workspace_bytes(K * R)), dtype=torch.uint8, device=dev)
    _lib.call("vr_scan_offsets", _lib.ptr(counts), K * R, _lib.ptr(off), _lib.ptr(ws), ws.numel(),
              s)
    bounds = off[torch.arange(K + 1, device=dev) * R].cpu().numpy().astype(np.int64)
    n = int(bounds[-1])
    t0 = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    t1 = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    rid = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    if n:
        _lib.call("vr_sample_fill", _lib.addr(tc), _lib.ptr(r), R, R, float(dt), 0, K,
                  _lib.ptr(off), _lib.ptr(first), _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(rid),
                  n, None, _lib.ptr(err), s)
    # an out-of-root midpoint (rounding at a grazing exit) only matters to owner lookup
    flags = int(err.item()) & ~_lib.VR_FLAG_OOB
    _lib.raise_flags(flags, "in sampling")
    return r, t0[:n], t1[:n], rid[:n], np.diff(bounds)


def rays_to_points(rays, root: Aabb, dt: float, max_points: int, seed: int,
                   device=None) -> PointCloud:
    """Discretize rays on the global dt grid (generate_samples, quadrature.py:66-88, as
    K1 over a one-leaf tree) and subsample the midpoints (partitioner.py:209-229): same
    points, same numpy subsample as the reference.  Raises NoPointsError when no ray
    intersects the root box."""
    if max_points <= 0:
        raise ValueError("max_points must be > 0")
    r, t0, t1, rid, _ = _k1_all_leaves(grid_tree(root, ""), rays, dt, device)
    if t0.numel() == 0:
        raise NoPointsError("no ray intersects the root box")
    t0n, t1n, idx = t0.cpu().numpy(), t1.cpu().numpy(), rid.cpu().numpy().astype(np.int64)
    rn = r.cpu().numpy()
    m = 0.5 * (t0n + t1n)  # SampleInterval.m (quadrature.py:40)
    arr = rn[0:3, idx].T + m[:, None] * rn[3:6, idx].T  # Ray.points_at (geometry.py:96-97)
    if arr.shape[0] > max_points:
        rng = np.random.default_rng(seed)
        keep = np.sort(rng.choice(arr.shape[0], size=max_points, replace=False))
        arr = arr[keep]
    return PointCloud(arr, "ray_discretized")


def default_root_box(points: np.ndarray) -> Aabb:
    """Bounding box of the points grown by 0.5 % of its extent on each side (1e-3 on a flat
    axis), partitioner.py:232-239."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    grow = np.where(hi - lo > 0.0, 0.005 * (hi - lo), 1e-3)
    return Aabb(lo - grow, hi + grow)


def balance_report(tree: PartitionTree, points, rays=None, dt: float = None,
                   device=None) -> dict:
    """Per-leaf point counts and, with rays, per-leaf render-time sample counts
    (partitioner.py:242-271): owner lookup by the vr_locate kernel, sample counts from K1
    over all leaves.  Ratios are max/min, or None when some leaf is empty."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    mn, mx = tree.root_box.mn, tree.root_box.mx
    inside = np.all((pts >= mn) & (pts <= mx), axis=1)
    tids = locate_many(tree, pts[inside], device) if inside.any() else np.zeros(0, np.int64)
    counts = np.bincount(tids, minlength=len(tree.leaves))
    report = {
        "num_tiles": len(tree.leaves),
        "leaf_point_counts": [int(c) for c in counts],
        "points_outside_root": int(np.count_nonzero(~inside)),
        "point_max_min_ratio": float(counts.max() / counts.min()) if counts.min() > 0 else None,
    }
    if rays is not None:
        if dt is None or dt <= 0.0:
            raise ValueError("sample counting needs dt > 0")
        _, _, _, _, per_leaf = _k1_all_leaves(tree, rays, dt, device)
        report["leaf_sample_counts"] = [int(c) for c in per_leaf]
        report["sample_max_min_ratio"] = (
            float(per_leaf.max() / per_leaf.min()) if per_leaf.min() > 0 else None)
    return report


def tree_to_json(tree: PartitionTree) -> dict:
    """The reference's tree JSON (partitioner.py:274-311): {root_box, depth, root}; a split
    node is {axis: "x"|"y"|"z", plane, low, high}, a leaf {tile_id, box}."""

    def enc(node):
        if isinstance(node, SplitNode):
            return {"axis": AXES[node.axis], "plane": float(node.plane),
                    "low": enc(node.low), "high": enc(node.high)}
        return {"tile_id": node.tile_id, "box": node.box.to_json()}

    return {"root_box": tree.root_box.to_json(), "depth": tree.depth, "root": enc(tree.root)}


def tree_from_json(d: dict) -> PartitionTree:
    """Inverse of tree_to_json; leaves must be numbered depth-first (partitioner.py:282-324).
    Split boxes are recomputed from the planes, leaf boxes read as stored."""
    root_box = Aabb.from_json(d["root_box"])
    leaves = []

    def dec(nd, box):
        if "tile_id" not in nd:
            axis = AXES.index(nd["axis"])
            plane = float(nd["plane"])
            lo_box, hi_box = _halves(box, axis, plane)
            low = dec(nd["low"], lo_box)
            return SplitNode(axis, plane, low, dec(nd["high"], hi_box))
        if int(nd["tile_id"]) != len(leaves):
            raise ValueError("leaf tile_ids must be depth-first sequential")
        leaves.append(LeafNode(len(leaves), Aabb.from_json(nd["box"])))
        return leaves[-1]

    root = dec(d["root"], root_box)
    return PartitionTree(root_box, root, int(d["depth"]), tuple(leaves))


def save_tree(tree: PartitionTree, path) -> None:
    Path(path).write_text(json.dumps(tree_to_json(tree), indent=2) + "\n")


def load_tree(path) -> PartitionTree:
    return tree_from_json(json.loads(Path(path).read_text()))
