"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy (float64) restatement of the reference ``volray`` tile-protocol path, used
as the parity checker for the CUDA kernels.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may import this module; the
product package never does.

Pinned: tests/test_oracle_golden.py checks every function here against golden
vectors produced by the unmodified reference (tests/golden/make_golden.py, run in
the build container where /root/reference is importable).

Restated reference functions (file:line under /root/reference/pkg/src/volray):
  slab test ............ geometry.py:109-128      -> box_hit
  bin grid ............. quadrature.py:66-88      -> grid_edges
  cut distances ........ partitioner.py:195-206   -> cut_distances
  split at cuts ........ quadrature.py:91-114     -> split_bins
  owner lookup ......... partitioner.py:166-192   -> Tree.owner
  analytic fields ...... field.py:88-240          -> AnalyticField
  masked ownership ..... field.py:243-273         (implicit: owner-only evaluation)
  segment composite .... quadrature.py:141-188    -> segment_packet
  compose render/dist .. segrender.py:93-142      -> fold_packets
  tile protocol ray .... distsim.py:395-454       -> render_ray_tile
  loss ................. segrender.py:198-207     -> ray_loss

Occupancy grid (SURVEY §8(f) 4 — the paper's empty-space skipping; the
reference has none, so this part is the specification the CUDA path follows,
parity unpinned): occupied / sample_ray(occ=...) drop the sub-bins whose midpoint falls
in an empty cell of its owner's res^3 grid (include/vr_capi.h VrOccupancy);
occupancy_points restates the grid update's jittered cell points.
"""
from __future__ import annotations

import math

import numpy as np

SLIVER = 1e-12
INF = math.inf


class NonFinite(ValueError):
    pass


class NegativeLoss(ValueError):
    pass


class OutOfBounds(ValueError):
    pass


# ---------------------------------------------------------------------------------
# geometry
# ---------------------------------------------------------------------------------

def box_hit(o, d, tn, tf, mn, mx):
    """(t_enter, t_exit) of the ray interval clipped to a closed box, or None."""
    o = np.asarray(o, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    axis_zero = d == 0.0
    outside = (o < mn) | (o > mx)
    if bool(np.any(axis_zero & outside)):
        return None
    with np.errstate(divide="ignore", invalid="ignore"):
        t_a = (mn - o) / d
        t_b = (mx - o) / d
    lo = np.where(axis_zero, -INF, np.minimum(t_a, t_b))
    hi = np.where(axis_zero, INF, np.maximum(t_a, t_b))
    a = float(lo.max())
    b = float(hi.min())
    enter = a if a > tn else tn
    leave = b if b < tf else tf
    return (enter, leave) if enter < leave else None


class Tree:
    """Partition tree parsed from the reference tree JSON (partitioner.py:274-316)."""

    AX = "xyz"

    def __init__(self, doc: dict):
        self.root_mn = np.array(doc["root_box"]["min"], dtype=np.float64)
        self.root_mx = np.array(doc["root_box"]["max"], dtype=np.float64)
        self.leaf_mn, self.leaf_mx = [], []
        self.root = self._parse(doc["root"])
        self.n_leaves = len(self.leaf_mn)

    def _parse(self, node):
        if "tile_id" in node:
            tid = int(node["tile_id"])
            assert tid == len(self.leaf_mn)
            self.leaf_mn.append(np.array(node["box"]["min"], dtype=np.float64))
            self.leaf_mx.append(np.array(node["box"]["max"], dtype=np.float64))
            return ("leaf", tid)
        return ("split", self.AX.index(node["axis"]), float(node["plane"]),
                self._parse(node["low"]), self._parse(node["high"]))

    def owner(self, p) -> int:
        if not (np.all(p >= self.root_mn) and np.all(p <= self.root_mx)):
            raise OutOfBounds(f"{p} outside root box")
        node = self.root
        while node[0] == "split":
            _, axis, plane, low, high = node
            node = low if p[axis] < plane else high
        return node[1]


def grid_edges(te: float, tx: float, dt: float):
    """Bin edges anchored at te with width dt, last edge forced to tx."""
    span = tx - te
    if span <= SLIVER:
        return []
    count = int(math.floor(span / dt))
    edges = [te + k * dt for k in range(count + 1)]
    if tx - edges[-1] > SLIVER:
        edges.append(tx)
    else:
        edges[-1] = tx
    return [(a, b) for a, b in zip(edges[:-1], edges[1:]) if b - a > SLIVER]


def cut_distances(tree: Tree, o, d, tn, tf):
    hit = box_hit(o, d, tn, tf, tree.root_mn, tree.root_mx)
    if hit is None:
        return []
    te, tx = hit
    found = set()
    for k in range(tree.n_leaves):
        h = box_hit(o, d, tn, tf, tree.leaf_mn[k], tree.leaf_mx[k])
        if h is not None:
            found.add(h[0])
            found.add(h[1])
    return sorted(t for t in found if te < t < tx)


def split_bins(bins, cuts):
    if not cuts:
        return list(bins)
    cuts = np.asarray(cuts, dtype=np.float64)
    out = []
    for a, b in bins:
        inner = cuts[(cuts > a) & (cuts < b)]
        if inner.size == 0:
            if b - a > SLIVER:
                out.append((a, b))
            continue
        pts = [a] + inner.tolist() + [b]
        for u, v in zip(pts[:-1], pts[1:]):
            if v - u > SLIVER:
                out.append((u, v))
    return out


def occupancy_cell(tree: Tree, tile: int, p, res: int):
    """Cell (cx, cy, cz) of p in leaf ``tile``'s res^3 grid: floor(((p - mn) / (mx - mn)) *
    res) clamped to [0, res - 1], float64 (the kernel's op order, no FMA)."""
    mn, mx = tree.leaf_mn[tile], tree.leaf_mx[tile]
    u = (np.asarray(p, dtype=np.float64) - mn) / (mx - mn)
    return np.clip(np.floor(u * float(res)), 0.0, float(res - 1)).astype(np.int64)


def occupied(tree: Tree, occ, tile: int, p) -> bool:
    """occ = (bits [n_leaves][words] uint32, res): the bit of p's cell in its owner's grid."""
    bits, res = occ
    c = occupancy_cell(tree, tile, p, res)
    idx = int(c[0] + res * (c[1] + res * c[2]))
    return bool((int(bits[tile][idx >> 5]) >> (idx & 31)) & 1)


def _lowbias32(x):
    x = np.asarray(x, dtype=np.uint64) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & np.uint64(0xFFFFFFFF)
    x ^= x >> np.uint64(16)
    return x


def occupancy_points(mn, mx, res: int, seed: int) -> np.ndarray:
    """(res^3, 3) jittered cell points of the grid update (csrc/occupancy.cu): cell c =
    cx + res (cy + res cz), u_a = (lowbias32(seed * 0x9E3779B9 + 3 c + a) >> 8) * 2^-24,
    point = mn + ((cell + u) / res) * (mx - mn)."""
    n = res ** 3
    c = np.arange(n, dtype=np.uint64)
    cells = np.stack([c % res, (c // res) % res, c // (res * res)], axis=1).astype(np.float64)
    out = np.empty((n, 3))
    base = (np.uint64(seed) * np.uint64(0x9E3779B9)) & np.uint64(0xFFFFFFFF)
    for a in range(3):
        h = _lowbias32((base + c * np.uint64(3) + np.uint64(a)) & np.uint64(0xFFFFFFFF))
        u = (h >> np.uint64(8)).astype(np.float64) * (1.0 / 16777216.0)
        out[:, a] = mn[a] + ((cells[:, a] + u) / float(res)) * (mx[a] - mn[a])
    return out


def sample_ray(tree: Tree, o, d, tn, tf, dt, occ=None):
    """All sub-bins of one ray in t order: arrays t0, t1, tile (distsim.py:369-373, :406-414);
    with ``occ`` (occupancy grid) only the sub-bins whose midpoint cell is occupied."""
    if dt <= 0.0:
        raise ValueError("dt must be > 0")
    o = np.asarray(o, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    hit = box_hit(o, d, tn, tf, tree.root_mn, tree.root_mx)
    if hit is None:
        return np.zeros(0), np.zeros(0), np.zeros(0, dtype=np.int64)
    bins = grid_edges(hit[0], hit[1], dt)
    if bins:
        bins = split_bins(bins, cut_distances(tree, o, d, tn, tf))
    if not bins:
        return np.zeros(0), np.zeros(0), np.zeros(0, dtype=np.int64)
    t0 = np.array([b[0] for b in bins])
    t1 = np.array([b[1] for b in bins])
    mid = 0.5 * (t0 + t1)
    pts = o + mid[:, None] * d
    tile = np.array([tree.owner(p) for p in pts], dtype=np.int64)
    if occ is not None:
        keep = np.array([occupied(tree, occ, k, p) for k, p in zip(tile, pts)], dtype=bool)
        return t0[keep], t1[keep], tile[keep]
    return t0, t1, tile


def participants(tree: Tree, o, d, tn, tf):
    """Leaves whose closed box the ray crosses with positive length (distsim.py:415-419)."""
    return [k for k in range(tree.n_leaves)
            if box_hit(o, d, tn, tf, tree.leaf_mn[k], tree.leaf_mx[k]) is not None]


def root_entry(tree: Tree, o, d, tn, tf) -> float:
    h = box_hit(o, d, tn, tf, tree.root_mn, tree.root_mx)
    return 0.0 if h is None else h[0]


# ---------------------------------------------------------------------------------
# analytic fields (scene JSON schema, field.py:7-23)
# ---------------------------------------------------------------------------------

class AnalyticField:
    def __init__(self, doc: dict):
        self.doc = doc

    def eval(self, pts):
        return _eval_field(self.doc, np.asarray(pts, dtype=np.float64).reshape(-1, 3))


def _inside(pts, box):
    mn = np.array(box["min"], dtype=np.float64)
    mx = np.array(box["max"], dtype=np.float64)
    return np.all(pts >= mn, axis=1) & np.all(pts <= mx, axis=1)


def _eval_field(doc, pts):
    kind = doc["type"]
    n = pts.shape[0]
    if kind == "gaussian_blobs":
        cols = np.array([b["color"] for b in doc["blobs"]], dtype=np.float64)
        sig = np.zeros((len(doc["blobs"]), n))
        for i, b in enumerate(doc["blobs"]):
            c = np.array(b["center"], dtype=np.float64)
            r2 = np.sum((pts - c) ** 2, axis=1)
            sig[i] = b["amplitude"] * np.exp(-0.5 * r2 / (b["scale"] * b["scale"]))
        tot = sig.sum(axis=0)
        mixed = sig.T @ cols
        safe = np.where(tot > 0.0, tot, 1.0)
        rgb = np.where(tot[:, None] > 0.0, mixed / safe[:, None], cols.mean(axis=0))
        return tot, rgb
    if kind == "constant_box":
        ins = _inside(pts, doc["box"])
        sig = np.where(ins, float(doc["density"]), 0.0)
        rgb = np.where(ins[:, None], np.array(doc["color"], dtype=np.float64), 0.0)
        return sig, rgb
    if kind == "voxel_grid":
        return _eval_voxel(doc, pts)
    if kind == "sum":
        parts = [_eval_field(c, pts) for c in doc["children"]]
        sigs = np.array([p[0] for p in parts])
        rgbs = np.array([p[1] for p in parts])
        tot = sigs.sum(axis=0)
        mixed = np.einsum("kn,knc->nc", sigs, rgbs)
        safe = np.where(tot > 0.0, tot, 1.0)
        rgb = np.where(tot[:, None] > 0.0, mixed / safe[:, None], rgbs.mean(axis=0))
        return tot, rgb
    raise ValueError(kind)


def voxel_stencil(doc, pts):
    """Cell-centred clamped trilinear stencil (field.py:176-195): corner ids (n,8,3)
    and weights (n,8), plus the nearest-cell ids (n,3) and the inside mask."""
    mn = np.array(doc["box"]["min"], dtype=np.float64)
    mx = np.array(doc["box"]["max"], dtype=np.float64)
    res = np.array(doc["resolution"], dtype=np.int64)
    cell = (mx - mn) / res.astype(np.float64)
    u = (pts - mn) / cell
    nearest = np.clip(np.floor(u).astype(np.int64), 0, res - 1)
    u = u - 0.5
    i0 = np.clip(np.floor(u).astype(np.int64), 0, np.maximum(res - 2, 0))
    i1 = np.minimum(i0 + 1, res - 1)
    f = np.clip(u - i0, 0.0, 1.0)
    ids, ws = [], []
    for cx in (0, 1):
        for cy in (0, 1):
            for cz in (0, 1):
                sel = np.array([cx, cy, cz])
                idx = np.where(sel == 1, i1, i0)
                w = np.where(sel[0] == 1, f[:, 0], 1.0 - f[:, 0]) * \
                    np.where(sel[1] == 1, f[:, 1], 1.0 - f[:, 1]) * \
                    np.where(sel[2] == 1, f[:, 2], 1.0 - f[:, 2])
                ids.append(idx)
                ws.append(w)
    inside = np.all(pts >= mn, axis=1) & np.all(pts <= mx, axis=1)
    return np.stack(ids, axis=1), np.stack(ws, axis=1), nearest, inside


def _eval_voxel(doc, pts, densities=None):
    res = tuple(doc["resolution"])
    dens = np.asarray(doc["densities"] if densities is None else densities,
                      dtype=np.float64).reshape(res)
    cols = np.asarray(doc["colors"], dtype=np.float64).reshape(res + (3,))
    ids, ws, nearest, inside = voxel_stencil(doc, pts)
    if doc.get("interpolation", "trilinear") == "nearest":
        sig = dens[nearest[:, 0], nearest[:, 1], nearest[:, 2]]
        rgb = cols[nearest[:, 0], nearest[:, 1], nearest[:, 2]]
    else:
        sig = np.zeros(pts.shape[0])
        rgb = np.zeros((pts.shape[0], 3))
        for c in range(8):
            ix = ids[:, c]
            sig = sig + dens[ix[:, 0], ix[:, 1], ix[:, 2]] * ws[:, c]
            rgb = rgb + cols[ix[:, 0], ix[:, 1], ix[:, 2]] * ws[:, c][:, None]
    sig = np.where(inside, sig, 0.0)
    rgb = np.where(inside[:, None], np.clip(rgb, 0.0, 1.0), 0.0)
    return sig, rgb


# ---------------------------------------------------------------------------------
# compositing
# ---------------------------------------------------------------------------------

def segment_packet(t0, t1, sigma, rgb):
    """(T, C[3], A, D, L) of one contiguous run, local T starting at 1."""
    if len(t0) == 0:
        return (1.0, np.zeros(3), 0.0, 0.0, 0.0)
    t0 = np.asarray(t0, dtype=np.float64)
    t1 = np.asarray(t1, dtype=np.float64)
    mids = 0.5 * (t0 + t1)
    alpha = 1.0 - np.exp(-np.asarray(sigma, dtype=np.float64) * (t1 - t0))
    trans = np.cumprod(np.concatenate(([1.0], 1.0 - alpha)))
    w = trans[:-1] * alpha
    color = (w[:, None] * np.asarray(rgb, dtype=np.float64)).sum(axis=0)
    gaps = np.abs(mids[:, None] - mids[None, :])
    dist = float(w @ gaps @ w)
    return (float(trans[-1]), color, float(w.sum()), float((w * mids).sum()), dist)


def fold_packets(packets):
    """Compose ordered packets: colour/opacity/depth/T and distortion with error checks."""
    for p in packets:
        vals = (p[0], p[2], p[3], p[4], *p[1])
        if not all(math.isfinite(v) for v in vals):
            raise NonFinite(str(p))
    T, A, D, L = 1.0, 0.0, 0.0, 0.0
    C = np.zeros(3)
    for (Tk, Ck, Ak, Dk, Lk) in packets:
        L += T * T * Lk + 2.0 * T * (Dk * A - Ak * D)
        C = C + T * Ck
        A += T * Ak
        D += T * Dk
        T *= Tk
    if L < 0.0:
        if L < -1e-12:
            raise NegativeLoss(str(L))
        L = 0.0
    return C, A, D, T, L


def ray_segments(tree: Tree, field_eval, o, d, tn, tf, dt):
    """Per-owner (order_t, tile, packet) list of a ray under the tile protocol.

    ``field_eval(tile, pts, dir) -> (sigma, rgb)`` is the owner's field.
    Segments are split at exact edge breaks (contiguous_runs, quadrature.py:191-206)."""
    t0, t1, tile = sample_ray(tree, o, d, tn, tf, dt)
    segs = []
    for k in sorted(set(tile.tolist())):
        sel = np.nonzero(tile == k)[0]
        a, b = t0[sel], t1[sel]
        mids = 0.5 * (a + b)
        pts = np.asarray(o) + mids[:, None] * np.asarray(d)
        sig, rgb = field_eval(k, pts, d)
        start = 0
        for j in range(1, len(sel) + 1):
            if j == len(sel) or a[j] != b[j - 1]:
                pk = segment_packet(a[start:j], b[start:j], sig[start:j], rgb[start:j])
                segs.append((float(a[start]), k, pk))
                start = j
    segs.sort(key=lambda s: (s[0], s[1]))
    return segs


def render_ray_tile(tree: Tree, field_eval, o, d, tn, tf, dt):
    """(C, A, D, T, L) of one ray under the tile protocol (distsim.py:395-454)."""
    segs = ray_segments(tree, field_eval, o, d, tn, tf, dt)
    return fold_packets([s[2] for s in segs])


def render_ray_samples(tree: Tree, field_eval, o, d, tn, tf, dt):
    """(C, A, D, T, L) under the sample-broadcast / mono protocols: every bin, owner-
    evaluated, in t0 order, one composite_samples over the whole ray (_compose_samples
    distsim.py:385-392, mono distsim.py:398-404)."""
    t0, t1, tile = sample_ray(tree, o, d, tn, tf, dt)
    if len(t0) == 0:
        return np.zeros(3), 0.0, 0.0, 1.0, 0.0
    sig = np.zeros(len(t0))
    rgb = np.zeros((len(t0), 3))
    for k in sorted(set(tile.tolist())):
        sel = np.nonzero(tile == k)[0]
        mids = 0.5 * (t0[sel] + t1[sel])
        sig[sel], rgb[sel] = field_eval(k, np.asarray(o) + mids[:, None] * np.asarray(d), d)
    order = np.argsort(t0, kind="stable")
    T, C, A, D, L = segment_packet(t0[order], t1[order], sig[order], rgb[order])
    return C, A, D, T, L


def ray_loss(C, T, L, bg, target, lambda_dist=1.0):
    pix = np.asarray(C) + T * np.asarray(bg)
    err = pix - np.asarray(target)
    return float(err @ err) + lambda_dist * L


def scene_field_eval(scene_doc):
    """Owner-evaluated field of a reference scene doc: every owner sees the base field
    (MaskedField half-open masking == owner-only evaluation)."""
    f = AnalyticField(scene_doc["field"])

    def ev(tile, pts, d):
        return f.eval(pts)

    return ev


def camera_rays(cam: dict, root_mn, root_mx):
    """Reference camera rays (distsim.py:116-127, :515-526) as an (R, 8) array."""
    pos = np.array(cam["position"], dtype=np.float64)
    look = np.array(cam["look_at"], dtype=np.float64)
    up0 = np.array(cam["up"], dtype=np.float64)
    f = look - pos
    f = f / float(np.linalg.norm(f))
    r = np.cross(f, up0)
    r = r / float(np.linalg.norm(r))
    up = np.cross(r, f)
    hh = math.tan(math.radians(cam["vertical_fov_deg"]) / 2.0)
    hw = hh * cam["width"] / cam["height"]
    i = (np.arange(cam["width"]) + 0.5) / cam["width"] * 2.0 - 1.0
    j = 1.0 - (np.arange(cam["height"]) + 0.5) / cam["height"] * 2.0
    xs, ys = np.meshgrid(i * hw, j * hh)
    dirs = f + xs.reshape(-1, 1) * r + ys.reshape(-1, 1) * up
    dirs = dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    root_mn = np.asarray(root_mn, dtype=np.float64)
    root_mx = np.asarray(root_mx, dtype=np.float64)
    center = 0.5 * (root_mn + root_mx)
    t_far = float(np.linalg.norm(center - pos)) + float(np.linalg.norm(root_mx - root_mn)) + 1.0
    out = np.empty((dirs.shape[0], 8))
    out[:, 0:3] = pos
    out[:, 3:6] = dirs
    out[:, 6] = 0.0
    out[:, 7] = t_far
    return out
