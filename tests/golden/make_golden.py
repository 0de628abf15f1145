"""Generate golden vectors by running the UNMODIFIED reference (volray) in this
build container (/root/reference is importable here, it does not exist on the GPU
box).  Output: small .npz / .json fixtures next to this script, committed.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Fixtures
  sampler_*.npz   bin edges (t0, t1), owner tile ids, participants and root entry t
                  of every ray: generate_samples + tile_cut_distances + split_at_planes
                  + locate_many (quadrature.py:66-114, partitioner.py:177-206,
                  distsim.py:369-373, :406-419)
  render_*.npz    per-ray RayAggregate of distsim.render_ray(..., "tile_aggregate")
  image_three_blobs.npz   distsim.render_image of the builtin 64x64 camera, K=4
  image_three_blobs_{sample,mono}.npz   the same image and CommStats under the
                  sample-broadcast and mono protocols (distsim.py:311-316, :385-404);
                  `make_golden.py protocols` regenerates only these two files
  partition_*.npz rays_to_points + build_tree + balance_report (partitioner.py:
                  209-271) on the street and voxel_room scenes (`make_golden.py partition`)
  grad_voxel_room.json    DistributedLossProbe.gradient_pair (local, global) FD
                  gradients of the voxel_room loss (segrender.py:153-251)
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

from volray import distsim, partitioner, quadrature, scenes, segrender, verify  # noqa: E402
from volray.field import scene_to_json  # noqa: E402
from volray.geometry import Aabb, Ray, ray_box_intersect, unit  # noqa: E402

OUT = Path(__file__).resolve().parent


def ray_row(r: Ray):
    return [*r.origin, *r.dir, r.t_near, r.t_far]


def sample_reference(tree, rays, dt):
    counts, t0s, t1s, tiles, parts, tes = [], [], [], [], [], []
    for ray in rays:
        samples = quadrature.generate_samples(ray, tree.root_box, dt)
        if samples:
            samples = quadrature.split_at_planes(samples, partitioner.tile_cut_distances(tree, ray))
        if samples:
            mids = np.array([s.m for s in samples])
            tid = partitioner.locate_many(tree, ray.points_at(mids))
        else:
            tid = np.zeros(0, dtype=np.int64)
        counts.append(len(samples))
        t0s.extend(s.t0 for s in samples)
        t1s.extend(s.t1 for s in samples)
        tiles.extend(int(t) for t in tid)
        mask = 0
        for leaf in tree.leaves:
            if ray_box_intersect(ray, leaf.box) is not None:
                mask |= 1 << leaf.tile_id
        parts.append(mask)
        hit = ray_box_intersect(ray, tree.root_box)
        tes.append(hit[0] if hit else 0.0)
    return dict(counts=np.array(counts, dtype=np.int64), t0=np.array(t0s, dtype=np.float64),
                t1=np.array(t1s, dtype=np.float64), tile=np.array(tiles, dtype=np.int64),
                part=np.array(parts, dtype=np.int64), te=np.array(tes, dtype=np.float64))


def special_rays(root: Aabb, tree, rng):
    """Edge cases: axis-aligned through split planes, grazing faces, truncated
    t ranges, misses, origins inside, exact-division spans."""
    rays = []
    c = root.center
    size = root.size
    planes = []

    def walk(node):
        if isinstance(node, partitioner.SplitNode):
            planes.append((node.axis, node.plane))
            walk(node.low)
            walk(node.high)

    walk(tree.root)
    for axis in range(3):
        for sgn in (1.0, -1.0):
            d = np.zeros(3)
            d[axis] = sgn
            o = c.copy()
            o[axis] = c[axis] - sgn * (size[axis] * 0.5 + 0.75)
            rays.append(Ray(o, d, 0.0, 50.0))
            # along a split plane / on a face
            for (pa, pv) in planes:
                if pa != axis:
                    o2 = o.copy()
                    o2[pa] = pv
                    rays.append(Ray(o2, d, 0.0, 50.0))
            o3 = o.copy()
            o3[(axis + 1) % 3] = root.mn[(axis + 1) % 3]
            rays.append(Ray(o3, d, 0.0, 50.0))  # grazing a face of the root box
            o4 = o.copy()
            o4[(axis + 1) % 3] = root.mx[(axis + 1) % 3] + 0.5
            rays.append(Ray(o4, d, 0.0, 50.0))  # parallel miss
    for _ in range(20):
        r = verify.random_ray(rng, root)
        tn = float(rng.uniform(0.0, 2.0))
        tf = tn + float(rng.uniform(0.1, 4.0))
        rays.append(Ray(r.origin, r.dir, tn, tf))  # truncated ranges
    for _ in range(10):
        o = rng.uniform(root.mn, root.mx)
        d = unit(rng.normal(size=3))
        rays.append(Ray(o, d, 0.0, 30.0))  # origin inside
    # diagonal through a corner (corner graze is a miss for that box)
    rays.append(Ray(root.mn - 1.0, unit(np.ones(3)), 0.0, 50.0))
    return rays


def dump_sampler(name, tree, rays, dt):
    ref = sample_reference(tree, rays, dt)
    np.savez_compressed(OUT / f"sampler_{name}.npz", rays=np.array([ray_row(r) for r in rays]),
                        dt=np.float64(dt), tree=json.dumps(partitioner.tree_to_json(tree)), **ref)
    print(f"sampler_{name}: {len(rays)} rays, {ref['t0'].size} samples")


def dump_render(name, bundle_scene, tree, rays, dt):
    pool = distsim.spawn(tree, bundle_scene)
    rows = []
    for ray in rays:
        agg, _ = distsim.render_ray(pool, ray, "tile_aggregate", dt)
        rows.append([*agg.color, agg.alpha, agg.depth, agg.transmittance, agg.distortion])
    np.savez_compressed(OUT / f"render_{name}.npz", rays=np.array([ray_row(r) for r in rays]),
                        dt=np.float64(dt), tree=json.dumps(partitioner.tree_to_json(tree)),
                        scene=json.dumps(scene_to_json(bundle_scene)), out=np.array(rows))
    print(f"render_{name}: {len(rays)} rays")


def main():
    rng = np.random.default_rng(2024)

    # --- sampler: builtin scenes and their trees ---------------------------------------
    b = scenes.three_blobs()
    tree_tb = partitioner.build_tree(b.points, b.scene.root_box, b.depth)
    cam_rays = [Ray(b.camera.position, d, 0.0, 8.0) for d in distsim.camera_ray_dirs(b.camera)]
    sel = [cam_rays[i] for i in rng.choice(len(cam_rays), 300, replace=False)]
    rays = sel + [verify.random_ray(rng) for _ in range(300)] + special_rays(b.scene.root_box, tree_tb, rng)
    dump_sampler("three_blobs_k4", tree_tb, rays, 0.028)

    tree3 = partitioner.build_tree(b.points, b.scene.root_box, 3)
    rays = [verify.random_ray(rng) for _ in range(400)] + special_rays(b.scene.root_box, tree3, rng)
    dump_sampler("three_blobs_k8", tree3, rays, 0.05)

    s = scenes.street()
    pts = partitioner.rays_to_points(s.rays, s.scene.root_box, s.dt, 4000, seed=3).points
    tree_st = partitioner.build_tree(pts, s.scene.root_box, 3)
    rays = list(s.rays) + special_rays(s.scene.root_box, tree_st, rng)
    dump_sampler("street_k8", tree_st, rays, s.dt)

    v = scenes.voxel_room()
    tree_v = partitioner.build_tree(v.points, v.scene.root_box, v.depth)
    rays = list(v.rays) + special_rays(v.scene.root_box, tree_v, rng)
    dump_sampler("voxel_room_k4", tree_v, rays, v.dt)

    # random trees (uniform points), dyadic dt -> exact-division edge cases
    for depth, dt in ((0, 2.0 ** -5), (1, 0.0625), (2, 0.1), (3, 0.03)):
        pts = rng.uniform(-1.0, 1.0, size=(512, 3))
        tree = partitioner.build_tree(pts, verify.ROOT, depth)
        rays = [verify.random_ray(rng) for _ in range(150)] + special_rays(verify.ROOT, tree, rng)
        dump_sampler(f"random_d{depth}", tree, rays, dt)

    # --- render: tile protocol on analytic scenes ---------------------------------------
    rays = [verify.random_ray(rng) for _ in range(200)]
    dump_render("three_blobs_k4", b.scene, tree_tb, rays, 0.028)
    rays = [verify.random_ray(rng) for _ in range(200)]
    dump_render("three_blobs_k8", b.scene, tree3, rays, 0.05)
    for i in range(3):
        sc = verify.random_scene(np.random.default_rng(100 + i))
        pts = rng.uniform(-1.0, 1.0, size=(256, 3))
        tree = partitioner.build_tree(pts, verify.ROOT, 2)
        rays = [verify.random_ray(rng) for _ in range(120)]
        dump_render(f"random_scene{i}", sc, tree, rays, float(rng.uniform(0.02, 0.08)))
    dump_render("voxel_room_k4", v.scene, tree_v, list(v.rays), v.dt)
    dump_render("street_k8", s.scene, tree_st, list(s.rays), s.dt)

    # --- full image (render_image, 64x64, K=4, white background) ---------------------
    pool = distsim.spawn(tree_tb, b.scene)
    img, st = distsim.render_image(pool, b.camera, "tile", b.dt)
    np.savez_compressed(OUT / "image_three_blobs.npz", image=img,
                        tree=json.dumps(partitioner.tree_to_json(tree_tb)),
                        scene=json.dumps(scene_to_json(b.scene)),
                        camera=json.dumps(b.camera.to_json()), dt=np.float64(b.dt),
                        stats=json.dumps(distsim.stats_json(st, "tile_aggregate", 4)))
    print("image_three_blobs: scalars", st.scalars_sent_total)

    # --- FD gradients on voxel_room (the reference's only gradient oracle) ------------
    probe = segrender.DistributedLossProbe(v.scene, tree_v, v.rays, v.dt)
    grid = v.scene.field
    base_loss = probe._loss(probe._collect())
    entries = []
    grng = np.random.default_rng(3)
    seen = set()
    while len(entries) < 24:
        ray = v.rays[grng.integers(0, len(v.rays))]
        p = ray.point_at(float(grng.uniform(0.4, 2.2)))
        if not grid.box.contains(p):
            continue
        cell = grid.box.size / np.array(grid.resolution)
        idx = tuple(int(q) for q in np.clip(np.floor((p - grid.box.mn) / cell), 0,
                                            np.array(grid.resolution) - 1))
        if idx in seen:
            continue
        seen.add(idx)
        owner = partitioner.locate(tree_v, grid.voxel_center(idx))
        local, glob = probe.gradient_pair(owner, segrender.ParamRef(owner, idx), 1e-4)
        entries.append({"tile": owner, "index": list(idx), "local": local, "global": glob})
    # an untouched voxel (ceiling corner) has zero gradient (test_segrender.py:223-229)
    idx = (0, grid.resolution[1] - 1, grid.resolution[2] - 1)
    owner = partitioner.locate(tree_v, grid.voxel_center(idx))
    local, glob = probe.gradient_pair(owner, segrender.ParamRef(owner, idx), 1e-4)
    entries.append({"tile": owner, "index": list(idx), "local": local, "global": glob})
    doc = {"tree": partitioner.tree_to_json(tree_v), "scene": scene_to_json(v.scene),
           "rays": [ray_row(r) for r in v.rays], "dt": v.dt, "target": 0.5,
           "loss": base_loss, "h": 1e-4, "entries": entries}
    (OUT / "grad_voxel_room.json").write_text(json.dumps(doc))
    print("grad_voxel_room:", len(entries), "entries, loss", base_loss)


def protocols():
    """render_image of the builtin three_blobs camera under the per-sample protocols."""
    b = scenes.three_blobs()
    tree_tb = partitioner.build_tree(b.points, b.scene.root_box, b.depth)
    for proto in ("sample_broadcast", "mono"):
        pool = distsim.spawn(tree_tb, b.scene)
        img, st = distsim.render_image(pool, b.camera, proto, b.dt)
        short = "sample" if proto == "sample_broadcast" else proto
        np.savez_compressed(OUT / f"image_three_blobs_{short}.npz", image=img,
                            tree=json.dumps(partitioner.tree_to_json(tree_tb)),
                            scene=json.dumps(scene_to_json(b.scene)),
                            camera=json.dumps(b.camera.to_json()), dt=np.float64(b.dt),
                            stats=json.dumps(distsim.stats_json(st, proto, 4)))
        print(f"image_three_blobs_{short}: scalars", st.scalars_sent_total)


def partition():
    """Sample-balanced partitioning from ray-discretized points."""
    s = scenes.street()
    v = scenes.voxel_room()
    for name, sc, rays, dt, n_pts, depth in (("street", s.scene, list(s.rays), s.dt, 4000, 3),
                                             ("voxel_room", v.scene, list(v.rays), v.dt, 10 ** 6,
                                              2)):
        pc = partitioner.rays_to_points(rays, sc.root_box, dt, n_pts, seed=3)
        tree = partitioner.build_tree(pc.points, sc.root_box, depth)
        rep = partitioner.balance_report(tree, pc.points, rays, dt)
        np.savez_compressed(OUT / f"partition_{name}.npz", points=pc.points,
                            rays=np.array([ray_row(r) for r in rays]), dt=np.float64(dt),
                            root=json.dumps(sc.root_box.to_json()), max_points=n_pts,
                            tree=json.dumps(partitioner.tree_to_json(tree)),
                            report=json.dumps(rep))
        print(f"partition_{name}: {len(pc.points)} points, report {rep}")


if __name__ == "__main__":
    if sys.argv[1:] == ["protocols"]:
        protocols()
    elif sys.argv[1:] == ["partition"]:
        partition()
    else:
        main()
        protocols()
        partition()
