"""CPU: host-side logic — partition config, C-struct flattening, region ownership,
hash-grid level parameters, workloads, accounting.  No GPU."""
import json

import numpy as np
import pytest

import paper_2404_16221_b200 as vr
from conftest import load_npz, sampler_fixtures
from oracle import hashmlp_oracle as hmo


def _descend_c(tc, p):
    if tc.n_nodes == 0:
        return 0
    node = 0
    while True:
        a = tc.node_axis[node]
        c = tc.node_low[node] if p[a] < tc.node_plane[node] else tc.node_high[node]
        if c < 0:
            return -c - 1
        node = c


@pytest.mark.parametrize("name", sampler_fixtures())
def test_tree_json_roundtrip_and_flattening(name):
    doc = load_npz(name)["tree"]
    tree = vr.tree_from_json(doc)
    assert json.dumps(vr.tree_to_json(tree)) == json.dumps(doc)  # byte-stable
    tc = tree.to_c()
    assert tc.n_leaves == len(tree.leaves) and tc.n_nodes == len(tree.leaves) - 1
    rng = np.random.default_rng(0)
    pts = rng.uniform(tree.root_box.mn, tree.root_box.mx, size=(500, 3))
    for p in pts:
        assert _descend_c(tc, p) == vr.locate(tree, p)
    for leaf in tree.leaves:
        assert list(tc.leaf_mn[leaf.tile_id]) == list(leaf.box.mn)
        assert list(tc.leaf_mx[leaf.tile_id]) == list(leaf.box.mx)


def test_locate_half_open_and_oob():
    tree = vr.grid_tree(vr.Aabb([0, 0, 0], [2, 1, 1]), "x")
    assert vr.locate(tree, [1.0, 0.5, 0.5]) == 1  # plane belongs to the high child
    assert vr.locate(tree, [np.nextafter(1.0, 0), 0.5, 0.5]) == 0
    assert vr.locate(tree, [2.0, 1.0, 1.0]) == 1  # closed root faces
    with pytest.raises(vr.OutOfBoundsError):
        vr.locate(tree, [2.0 + 1e-9, 0.5, 0.5])


def test_grid_tree_shapes():
    t = vr.grid_tree(vr.Aabb([0, 0, 0], [16, 16, 1]), "xyx")
    assert len(t.leaves) == 8 and t.depth == 3
    sizes = {tuple(l.box.size) for l in t.leaves}
    assert sizes == {(4.0, 8.0, 1.0)}
    assert vr.grid_tree(vr.Aabb([0, 0, 0], [1, 1, 1]), "").leaves[0].tile_id == 0


def test_build_tree_balanced_and_errors():
    rng = np.random.default_rng(1)
    pts = rng.uniform(-1, 1, size=(1024, 3))
    tree = vr.build_tree(pts, vr.Aabb([-1, -1, -1], [1, 1, 1]), 3)
    counts = np.bincount([vr.locate(tree, p) for p in pts], minlength=8)
    assert counts.max() - counts.min() <= 8
    with pytest.raises(vr.InsufficientPointsError):
        vr.build_tree(pts[:3], vr.Aabb([-1, -1, -1], [1, 1, 1]), 2)
    with pytest.raises(vr.DegenerateSplitError):
        vr.choose_split(np.zeros((4, 3)), vr.Aabb([-1, -1, -1], [1, 1, 1]))


@pytest.mark.parametrize("k,world", [(8, 1), (8, 2), (8, 4), (8, 8), (4, 2)])
def test_owned_regions_partition_all_regions(k, world):
    seen = []
    for r in range(world):
        lo, cnt = vr.owned_regions(k, r, world)
        seen.extend(range(lo, lo + cnt))
    assert seen == list(range(k))
    with pytest.raises(ValueError):
        vr.owned_regions(6, 0, 4)


@pytest.mark.parametrize("log2_T,max_res", [(12, 128), (14, 512), (19, 2048), (22, 2048)])
def test_hash_levels_agree_with_oracle(log2_T, max_res):
    cfg = vr.HashGridConfig(log2_T=log2_T, max_res=max_res)
    scales, res, dense, offs = cfg.level_params()
    olv, total = hmo.levels(log2_T, max_res=max_res)
    assert offs[-1] == total
    for lv, (s, r, dn, off) in enumerate(olv):
        assert np.float32(scales[lv]) == s and res[lv] == r and dense[lv] == dn
        assert offs[lv] == off
    d = vr.fields.hash_desc(cfg, vr.Aabb([0, 0, 0], [1, 1, 1]))
    assert d.offset[16] == total and np.float32(d.scale[15]) == olv[15][0]


def test_hash_indices_oracle_properties():
    rng = np.random.default_rng(0)
    pts = rng.uniform(0, 1, size=(64, 3))
    idx = hmo.all_indices(pts, [0, 0, 0], [1, 1, 1], 14)
    assert idx.shape == (16, 64, 8)
    assert idx.min() >= 0 and idx.max() < (1 << 14)
    olv, _ = hmo.levels(14)
    for lv, (s, r, dn, off) in enumerate(olv):
        if dn:
            assert idx[lv].max() < r ** 3


@pytest.mark.parametrize("cfg", ["c1", "c3", "c4", "c5"])
def test_workload_rays(cfg):
    from paper_2404_16221_b200.workloads import CONFIGS, make_rays

    w = CONFIGS[cfg]
    rays = make_rays(w, 0, 1000)
    assert rays.shape == (8, 1000) and rays.dtype == np.float64
    assert np.allclose(np.linalg.norm(rays[3:6], axis=0), 1.0, atol=1e-12)
    assert np.all(rays[6] < rays[7])
    assert len(w.tree.leaves) in (1, 2, 8)


def test_comm_stats_shape():
    st = vr.CommStats()
    st.rays = 2
    st.record(0, -1, 9)
    st.record(1, -1, 9)
    doc = vr.stats_json(st, "tile_aggregate", 2)
    assert doc["scalars_sent_total"] == 18 and len(doc["per_worker"]) == 2
    assert st.scalars_sent_total == st.scalars_received_total


def test_geometry_validation():
    with pytest.raises(ValueError):
        vr.Ray([0, 0, 0], [1, 1, 0], 0, 1)
    with pytest.raises(ValueError):
        vr.Aabb([0, 0, 0], [1, 0, 1])
    with pytest.raises(ValueError):
        vr.soa_rays([[0, 0, 0]], [[1, 0, 0]], 1.0, 0.5)
    soa = vr.rays_to_soa([vr.Ray([0, 0, 0], [0, 0, 1], 0.5, 2.0)])
    assert soa.shape == (8, 1) and soa[5, 0] == 1.0 and soa[6, 0] == 0.5


@pytest.mark.parametrize("name", ["partition_street.npz", "partition_voxel_room.npz"])
def test_build_tree_from_ray_points_matches_reference(name):
    """Sample-balanced partitioning: the median-split tree built from
    the reference's ray-discretized points is the reference's tree."""
    g = load_npz(name)
    root = vr.Aabb.from_json(g["root"])
    depth = {"partition_street.npz": 3, "partition_voxel_room.npz": 2}[name]
    tree = vr.build_tree(g["points"], root, depth)
    assert vr.tree_to_json(tree) == g["tree"]
    box = vr.default_root_box(g["points"])
    assert np.all(box.mn <= g["points"].min(axis=0)) and np.all(box.mx >= g["points"].max(axis=0))


def test_reference_value_type_methods():
    """Ray.points_at / to_json / from_json, Aabb.contains_many (geometry.py:59-106) and
    CommStats.merge (distsim.py:250-265): the reference surface on the host value types."""
    import paper_2404_16221_b200 as vr

    r = vr.Ray([0.0, 1.0, 2.0], [0.0, 0.6, 0.8], 0.5, 9.0)
    pts = r.points_at([0.0, 1.0, 2.5])
    np.testing.assert_array_equal(pts[2], [0.0, 1.0 + 2.5 * 0.6, 2.0 + 2.5 * 0.8])
    r2 = vr.Ray.from_json(json.loads(json.dumps(r.to_json())))
    assert np.array_equal(r2.origin, r.origin) and r2.t_far == r.t_far
    box = vr.Aabb([0, 0, 0], [1, 1, 1])
    assert box.contains_many(np.array([[0, 0, 0], [1, 1, 1], [1.0001, 0, 0]])).tolist() == \
        [True, True, False]
    a, b = vr.CommStats(), vr.CommStats()
    a.rays, b.rays = 3, 4
    a.record(0, -1, 9)
    b.record(0, -1, 18, 2)
    b.record(1, -1, 9)
    b.add_time("compose", 0.5)
    a.merge(b)
    assert a.rays == 7 and a.workers[0].scalars_sent == 27 and a.workers[0].messages_sent == 3
    assert a.workers[1].scalars_sent == 9 and a.compositor.scalars_received == 36
    assert a.phase_seconds["compose"] == 0.5
