"""Sample-balanced partition trees of the benchmark workloads.

The reference's own recipe (partitioner.rays_to_points + build_tree, partitioner.py:131-229):
discretise a sample of the workload's rays on its dt grid, subsample the midpoints, and
split at medians down to 8 leaves (the aspect rule keeps c3 a 1D strip along x and makes
c4 a 4 x 2 arrangement; c5 renders with c4's tree).  Balanced leaves give every GPU of the scaling run the same number of
samples (uniform grids: c4 max/mean 1.20).  Midpoints come from the CPU restatement of the
sampler (bit-identical to K1), so this runs without a GPU; the trees are committed under
paper_2404_16221_b200/data/.

    python scripts/make_trees.py
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2404_16221_b200 as vr  # noqa: E402
from oracle import volray_oracle as vo  # noqa: E402
from paper_2404_16221_b200.workloads import CONFIGS, make_rays  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "paper_2404_16221_b200" / "data"


def main():
    for name in ("c3", "c4"):  # c5 renders with c4's tree
        w = CONFIGS[name]
        root = w.root
        one = vo.Tree(vr.tree_to_json(vr.grid_tree(root, "")))
        rays = make_rays(w, n=4096).T
        pts = []
        for r in rays:
            t0, t1, _ = vo.sample_ray(one, r[0:3], r[3:6], r[6], r[7], w.dt)
            m = 0.5 * (t0 + t1)
            pts.append(r[0:3][None, :] + m[:, None] * r[3:6][None, :])
        pts = np.concatenate(pts)
        if pts.shape[0] > 200000:
            keep = np.sort(np.random.default_rng(3).choice(pts.shape[0], 200000, replace=False))
            pts = pts[keep]
        tree = vr.build_tree(pts, root, 3)
        (OUT / f"{name}_tree.json").write_text(json.dumps(vr.tree_to_json(tree), indent=1))
        print(name, len(tree.leaves), "leaves:",
              [[round(x, 3) for x in (*lf.box.mn, *lf.box.mx)] for lf in tree.leaves])


if __name__ == "__main__":
    main()
