"""Small training steps through every backward variant, for compute-sanitizer or the
checked build (compute-sanitizer is closed on this GPU pool):

    VR_CHECKED=1 python scripts/sanitize.py [variant ...]
    compute-sanitizer --tool memcheck python scripts/sanitize.py [variant ...]

Variants: fused (sample-major tcgen05 MLP backward + fused hash scatter), split (MLP
backward + side-stream scatter), level (level-major hash kernels), density (density-only
proposal fields + the interlevel loss), cuda (CUDA-core reference MLP), render (the render
path), sample (the sample-broadcast protocol).  Each runs two training steps of a 2-region
hash-grid pool on 96 rays and checks the loss is finite.  c4 (not in the default list): two
steps of the c4 bench pool (8 regions at full model size, level-major kernels, proposal
fields, interlevel loss, sparse backward, TMA K4, record-index K5) on 65,536 of its rays.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_16221_b200 as vr  # noqa: E402

VARIANTS = ("fused", "split", "level", "density", "cuda", "render", "sample")


def pool_for(variant):
    root = vr.Aabb([-1, -1, -1], [1, 1, 1])
    tree = vr.grid_tree(root, "x")
    cfg = vr.HashGridConfig(log2_T=14, max_res=256)
    impl = "cuda" if variant == "cuda" else "fused"
    order = "level" if variant == "level" else "sample"
    fields = [vr.HashGridMLP(cfg, tree.leaves[k].box, "cuda", seed=k, table_init=0.3,
                             mlp_impl=impl, hash_order=order) for k in range(2)]
    if variant == "fused":
        for f in fields:
            f.SPLIT_BELOW_BYTES = 0
    props = None
    if variant == "density":
        pcfg = vr.HashGridConfig(log2_T=12, max_res=128)
        props = [vr.HashGridMLP(pcfg, tree.leaves[k].box, "cuda", seed=9 + k, table_init=0.3,
                                density_only=True) for k in range(2)]
    return vr.VolumePool(tree, fields, (0.1, 0.2, 0.3), "cuda", proposals=props)


def rays(n=96, seed=0):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        o = rng.uniform(-2.4, 2.4, size=3)
        d = rng.uniform(-0.8, 0.8, size=3) - o
        out.append([*o, *(d / np.linalg.norm(d)), 0.0, 20.0])
    return np.asarray(out).T.copy()


def main():
    todo = sys.argv[1:] or list(VARIANTS)
    r = rays()
    tg = np.random.default_rng(1).uniform(0, 1, size=(r.shape[1], 3))
    for v in todo:
        if v == "c4":
            import bench
            from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets
            w = CONFIGS["c4"]
            pool = bench.build_pool(w, 0, 1, "cuda:0", None)
            rr = torch.from_numpy(make_rays(w, seed=0, n=65536)).to("cuda:0")
            tt = torch.from_numpy(make_targets(65536, seed=100)).to("cuda:0")
            for step in (1, 2):
                loss = pool.train_step(rr, tt, w.dt, lr=1e-2, step=step,
                                       lambda_interlevel=w.interlevel)
            assert np.isfinite(loss.item())
            print(f"{v}: ok loss {loss.item():.6f}", flush=True)
            del pool
            torch.cuda.empty_cache()
            continue
        pool = pool_for(v)
        if v == "render":
            out, _ = pool.render_rays(r, 0.03)
            torch.cuda.synchronize()
            pool.check()
            assert torch.isfinite(out).all()
            print(f"{v}: ok", flush=True)
            continue
        lam = 0.5 if v == "density" else 0.0
        proto = "sample" if v == "sample" else "tile"
        for step in (1, 2):
            loss = pool.train_step(r, tg, 0.03, lr=1e-2, step=step, lambda_interlevel=lam,
                                   protocol=proto)
        assert np.isfinite(loss.item())
        print(f"{v}: ok loss {loss.item():.6f}", flush=True)
    if os.environ.get("VR_CHECKED") == "1":
        fails = vr._lib.load().vr_check_failures()
        print(f"checked build: {fails} range-check failures", flush=True)
        if fails != 0:
            raise SystemExit(1)


if __name__ == "__main__":
    main()
