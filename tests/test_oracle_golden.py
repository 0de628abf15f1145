"""CPU: pin the oracle against the reference's golden vectors and hand cases.

Fixtures come from the unmodified reference (tests/golden/make_golden.py).  These
tests need no GPU; they establish that oracle/ is a faithful restatement before it
is used as the checker for the CUDA kernels."""
import json
import math

import numpy as np
import pytest
import torch

from conftest import GOLDEN, load_npz, render_fixtures, sampler_fixtures
from oracle import grad_oracle, volray_oracle as vo


@pytest.mark.parametrize("name", sampler_fixtures())
def test_sampler_bit_exact_vs_reference(name):
    g = load_npz(name)
    tree = vo.Tree(g["tree"])
    off = 0
    for i, r in enumerate(g["rays"]):
        t0, t1, tile = vo.sample_ray(tree, r[0:3], r[3:6], r[6], r[7], float(g["dt"]))
        n = int(g["counts"][i])
        assert t0.size == n, f"ray {i}: {t0.size} vs {n}"
        assert np.array_equal(t0, g["t0"][off:off + n])
        assert np.array_equal(t1, g["t1"][off:off + n])
        assert np.array_equal(tile, g["tile"][off:off + n])
        part = sum(1 << k for k in vo.participants(tree, r[0:3], r[3:6], r[6], r[7]))
        assert part == int(g["part"][i])
        assert vo.root_entry(tree, r[0:3], r[3:6], r[6], r[7]) == g["te"][i]
        off += n


@pytest.mark.parametrize("name", render_fixtures())
def test_tile_render_matches_reference(name):
    g = load_npz(name)
    tree = vo.Tree(g["tree"])
    ev = vo.scene_field_eval(g["scene"])
    for i, r in enumerate(g["rays"]):
        C, A, D, T, L = vo.render_ray_tile(tree, ev, r[0:3], r[3:6], r[6], r[7], float(g["dt"]))
        got = np.array([*C, A, D, T, L])
        np.testing.assert_allclose(got, g["out"][i], rtol=1e-10, atol=1e-12)


def test_image_matches_reference():
    g = load_npz("image_three_blobs.npz")
    tree = vo.Tree(g["tree"])
    ev = vo.scene_field_eval(g["scene"])
    rays = vo.camera_rays(g["camera"], g["scene"]["root_box"]["min"], g["scene"]["root_box"]["max"])
    bg = np.array(g["scene"]["background"])
    img = np.zeros((rays.shape[0], 3))
    for i in range(0, rays.shape[0], 7):  # every 7th pixel keeps the CPU suite fast
        r = rays[i]
        C, A, D, T, L = vo.render_ray_tile(tree, ev, r[0:3], r[3:6], r[6], r[7], float(g["dt"]))
        img[i] = np.clip(C + T * bg, 0.0, 1.0)
        np.testing.assert_allclose(img[i], g["image"].reshape(-1, 3)[i], atol=1e-12)


@pytest.mark.parametrize("proto", ["sample", "mono"])
def test_sample_protocol_image_matches_reference(proto):
    """The per-sample protocols (one composite over all of a ray's bins) against the
    reference's render_image under that protocol; they agree with the tile image to
    ~1e-10 as the reference promises (distsim.render_ray docstring)."""
    g = load_npz(f"image_three_blobs_{proto}.npz")
    tile = load_npz("image_three_blobs.npz")
    np.testing.assert_allclose(g["image"], tile["image"], rtol=0, atol=1e-9)
    tree = vo.Tree(g["tree"])
    ev = vo.scene_field_eval(g["scene"])
    rays = vo.camera_rays(g["camera"], g["scene"]["root_box"]["min"], g["scene"]["root_box"]["max"])
    bg = np.array(g["scene"]["background"])
    for i in range(0, rays.shape[0], 11):
        r = rays[i]
        C, A, D, T, L = vo.render_ray_samples(tree, ev, r[0:3], r[3:6], r[6], r[7], float(g["dt"]))
        np.testing.assert_allclose(np.clip(C + T * bg, 0.0, 1.0), g["image"].reshape(-1, 3)[i],
                                   atol=1e-12)


def test_voxel_grad_oracle_matches_reference_fd():
    doc = json.loads((GOLDEN / "grad_voxel_room.json").read_text())
    tree = vo.Tree(doc["tree"])
    grid = doc["scene"]["field"]
    res = tuple(grid["resolution"])
    base = np.asarray(grid["densities"], dtype=np.float64).reshape(res)
    dens = [torch.tensor(base.copy(), requires_grad=True) for _ in range(tree.n_leaves)]
    rays = np.asarray(doc["rays"])
    targets = np.full((rays.shape[0], 3), doc["target"])
    loss, _ = grad_oracle.voxel_loss(tree, grid, dens, rays, targets, doc["scene"]["background"],
                                     doc["dt"])
    assert loss.item() == pytest.approx(doc["loss"], rel=1e-12)
    loss.backward()
    for e in doc["entries"]:
        g = dens[e["tile"]].grad[tuple(e["index"])].item()
        fd = e["global"]
        assert abs(e["local"] - fd) <= 1e-6 * (1 + abs(fd))
        assert abs(g - fd) <= 1e-6 * (1.0 + abs(fd)), (e, g)


# ---- reference hand cases (pkg/tests/test_segrender.py, test_quadrature.py) ----------

def test_fold_hand_cases():
    pk = lambda T=1.0, C=(0, 0, 0), A=0.0, D=0.0, L=0.0: (T, np.asarray(C, float), A, D, L)
    C, A, D, T, L = vo.fold_packets([pk(T=0.5, C=(0.3, 0, 0)), pk(T=1.0, C=(0.2, 0, 0))])
    assert C[0] == pytest.approx(0.4, rel=1e-15) and T == pytest.approx(0.5)
    C, A, D, T, L = vo.fold_packets([pk(T=0.0, C=(1, 0, 0), A=1.0), pk(T=0.5, C=(0, 1, 0), A=0.5)])
    assert list(C) == [1, 0, 0] and A == 1.0 and T == 0.0
    # distortion cross term: two point masses w=[.5,.5] at m=[1,3] -> 1.0
    _, _, _, _, L = vo.fold_packets([pk(T=0.5, A=0.5, D=0.5), pk(T=0.0, A=1.0, D=3.0)])
    assert L == pytest.approx(1.0, rel=1e-15)
    with pytest.raises(vo.NonFinite):
        vo.fold_packets([pk(T=math.nan)])
    with pytest.raises(vo.NegativeLoss):
        vo.fold_packets([pk(L=-1.0)])
    assert vo.fold_packets([pk(L=-1e-13)])[4] == 0.0


def test_segment_hand_cases():
    ln2 = math.log(2.0)
    T, C, A, D, L = vo.segment_packet([0.75], [1.25], [ln2 / 0.5], [[1, 0, 0]])
    assert A == pytest.approx(0.5, rel=1e-15) and T == pytest.approx(0.5, rel=1e-15)
    assert D == pytest.approx(0.5, rel=1e-15) and L == 0.0
    T, C, A, D, L = vo.segment_packet([0, 1], [1, 2], [ln2, ln2], [[1, 0, 0], [0, 0, 1]])
    np.testing.assert_allclose(C, [0.5, 0, 0.25], rtol=1e-14)
    assert T == pytest.approx(0.25, rel=1e-14)


def test_grid_edges_hand_cases():
    # test_quadrature.py:54-69
    assert vo.grid_edges(1.0, 2.0, 0.25) == [(1.0, 1.25), (1.25, 1.5), (1.5, 1.75), (1.75, 2.0)]
    assert vo.grid_edges(1.0, 1.9, 0.25) == [(1.0, 1.25), (1.25, 1.5), (1.5, 1.75), (1.75, 1.9)]
    assert vo.split_bins([(1.0, 2.0)], [1.5]) == [(1.0, 1.5), (1.5, 2.0)]
    assert vo.split_bins([(1.0, 2.0)], [1.0 + 1e-14]) == [(1.0 + 1e-14, 2.0)]


# ---- hash encoding: hand-worked vectors from the published algorithm ---------------------

def test_hash_oracle_matches_hand_vectors():
    """oracle/hashmlp_oracle.py against tests/golden/hash_hand.json (Instant-NGP's hash,
    dense/hash switch and trilinear weights restated with Python ints and struct float32
    rounding, tests/golden/make_hash_hand.py): indices bit-exact, weights bit-exact."""
    from oracle import hashmlp_oracle as hmo

    g = json.loads((GOLDEN / "hash_hand.json").read_text())
    u = np.asarray(g["points"], dtype=np.float32)
    for case in g["cases"]:
        lv, _ = hmo.levels(case["log2_T"], max_res=case["max_res"])
        assert len(lv) == len(case["levels"]) == 16
        for (scale, res, dense, _), hand in zip(lv, case["levels"]):
            assert float(scale) == hand["scale"] and res == hand["res"] and dense == hand["dense"]
            idx, w = hmo.corners(u, scale, res, dense, case["log2_T"])
            assert np.array_equal(idx.astype(np.int64), np.asarray(hand["idx"], dtype=np.int64))
            assert np.array_equal(w, np.asarray(hand["w"], dtype=np.float32))


def test_hash_config_levels_match_hand_vectors():
    """The product's level derivation (HashGridConfig.level_params) gives the same scales,
    resolutions and dense/hashed split as the hand vectors."""
    import paper_2404_16221_b200 as vr

    g = json.loads((GOLDEN / "hash_hand.json").read_text())
    for case in g["cases"]:
        scales, res, dense, _ = vr.HashGridConfig(log2_T=case["log2_T"],
                                                  max_res=case["max_res"]).level_params()
        for l, hand in enumerate(case["levels"]):
            assert float(scales[l]) == hand["scale"]
            assert res[l] == hand["res"] and dense[l] == hand["dense"]
