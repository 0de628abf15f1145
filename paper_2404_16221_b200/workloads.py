"""Synthetic workloads of BASELINE.json's configs (random-init fields, seeded rays).

  c1  single region [-1,1]^3, 4096 rays, T=2^14, dt=2^-5 (64 bins on axis rays)
  c2  same scene split into 2 regions (equivalence check; parity-test case)
  c3  8-region x-strip street, root [0,16]x[0,1]x[0,2], 1M rays, T=2^19 per region
  c4  8-region 4x2 city grid, root [0,16]x[0,16]x[0,1], 4M rays, T=2^22 per region
  c4  dt chosen for ~64 samples/ray (measured 64.7); c5 for ~128 (measured 129)
  c5  c4's tree, render-only 1920x1080 frame, ~128 samples/ray
Partitions: the sample-balanced trees in data/ (scripts/make_trees.py: the reference's
rays_to_points + build_tree recipe on a 4096-ray sample) — c3 stays a 1D strip along x,
c4 a 4 x 2 arrangement of median splits; per-region samples max/mean 1.03 / 1.07 (uniform
grids: 1.04 / 1.20), which bounds the parallel efficiency of the 8-GPU run.

Seeds: rays default_rng(0), params seed 1 (+region), targets rng(2).
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .geometry import Aabb
from .partition import grid_tree

DATA = Path(__file__).resolve().parent / "data"


@dataclass
class Workload:
    name: str
    root: Aabb
    splits: str
    n_rays: int
    log2_T: int
    dt: float
    max_res: int = 2048
    train: bool = True
    interlevel: float = 0.0  # > 0: per-region proposal fields + interlevel loss weight
    prop_log2_T: int = 17
    prop_max_res: int = 512

    # "grid": uniform splits; a file name: a committed sample-balanced tree (data/, made
    # by scripts/make_trees.py with the reference's rays_to_points + build_tree recipe)
    partition: str = "grid"

    @property
    def tree(self):
        if self.partition != "grid":
            from .partition import tree_from_json

            return tree_from_json(json.loads((DATA / self.partition).read_text()))
        return grid_tree(self.root, self.splits)


CONFIGS = {
    "c1": Workload("c1-single-region-4096rays-T2^14", Aabb([-1, -1, -1], [1, 1, 1]), "", 4096, 14,
                   2.0 ** -5, 512),
    "c2": Workload("c2-two-region-4096rays-T2^14", Aabb([-1, -1, -1], [1, 1, 1]), "x", 4096, 14,
                   2.0 ** -5, 512),
    "c3": Workload("c3-street-8strip-1Mrays-T2^19", Aabb([0, 0, 0], [16, 1, 2]), "xxx", 1 << 20, 19,
                   0.09, partition="c3_tree.json"),
    "c4": Workload("c4-city-4x2-4Mrays-T2^22", Aabb([0, 0, 0], [16, 16, 1]), "xyx", 1 << 22, 22,
                   0.056, interlevel=1.0, partition="c4_tree.json"),
    # rendering uses the trained model's partition (c4's tree)
    "c5": Workload("c5-render-1080p-8region", Aabb([0, 0, 0], [16, 16, 1]), "xyx", 1920 * 1080, 22,
                   0.028, train=False, partition="c4_tree.json"),
}


def _unit_rows(v):
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def make_rays(w: Workload, seed: int = 0, n: int | None = None) -> np.ndarray:
    """Float64 SoA [8][R] rays for a workload."""
    rng = np.random.default_rng(seed)
    R = w.n_rays if n is None else n
    mn, mx = w.root.mn, w.root.mx
    size = mx - mn
    if w.name.startswith(("c1", "c2")):
        o = rng.uniform(-2.4, 2.4, size=(R, 3))
        tgt = rng.uniform(-0.8, 0.8, size=(R, 3))
        d = _unit_rows(tgt - o)
        tn, tf = 0.0, 20.0
    elif w.name.startswith("c3"):
        # street.py-style rays (scenes.py:97-104) scaled to the strip, plus 1/4 rays
        # travelling along the street (long multi-region traversals)
        n_along = R // 4
        n_side = R - n_along
        o1 = np.stack([rng.uniform(0.5, 15.5, n_side), rng.uniform(0.3, 0.7, n_side),
                       np.full(n_side, -1.2)], axis=1)
        t1 = np.stack([o1[:, 0] + rng.uniform(-1.0, 1.0, n_side), rng.uniform(0.2, 0.8, n_side),
                       rng.uniform(0.4, 1.6, n_side)], axis=1)
        o2 = np.stack([np.full(n_along, -1.0), rng.uniform(0.2, 0.8, n_along),
                       rng.uniform(0.3, 1.7, n_along)], axis=1)
        t2 = np.stack([np.full(n_along, 17.0), rng.uniform(0.2, 0.8, n_along),
                       rng.uniform(0.3, 1.7, n_along)], axis=1)
        o = np.concatenate([o1, o2])
        d = _unit_rows(np.concatenate([t1, t2]) - o)
        tn, tf = 0.0, 30.0
    else:
        # aerial oblique cameras over the city slab (MatrixCity-like, normalised units)
        o = np.stack([rng.uniform(-2.0, 18.0, R), rng.uniform(-2.0, 18.0, R),
                      rng.uniform(2.0, 4.0, R)], axis=1)
        tgt = np.stack([rng.uniform(0.0, 16.0, R), rng.uniform(0.0, 16.0, R),
                        rng.uniform(0.0, 0.3, R)], axis=1)
        d = _unit_rows(tgt - o)
        tn, tf = 0.0, 30.0
    out = np.empty((8, R), dtype=np.float64)
    out[0:3] = o.T
    out[3:6] = d.T
    out[6] = tn
    out[7] = tf
    return out


def make_targets(n: int, seed: int = 2) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 1.0, size=(n, 3)).astype(np.float32)
