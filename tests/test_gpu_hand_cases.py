"""The reference's hand-worked cases run through the CUDA path (K1 sampling, K4 segment
composite, K5 fold) — the same cases test_oracle_golden.py pins the oracle with:
grid edges / truncation / miss (test_quadrature.py:31-76), split and sliver
(test_quadrature.py:81-115), the ln2 closed forms and the two-bin colour case
(test_quadrature.py:126-141), occlusion (test_segrender.py:62-83)."""
import math

import numpy as np
import pytest
import torch

import paper_2404_16221_b200 as vr
from oracle import volray_oracle as vo

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _leaf(i, mn, mx):
    return {"tile_id": i, "box": {"min": list(mn), "max": list(mx)}}


def _tree(x_lo, x_hi, plane=None):
    """Root [x_lo, x_hi] x [0,1] x [0,1], optionally split once along x."""
    root = {"min": [x_lo, 0.0, 0.0], "max": [x_hi, 1.0, 1.0]}
    if plane is None:
        node, depth = _leaf(0, root["min"], root["max"]), 0
    else:
        node = {"axis": "x", "plane": plane,
                "low": _leaf(0, [x_lo, 0.0, 0.0], [plane, 1.0, 1.0]),
                "high": _leaf(1, [plane, 0.0, 0.0], [x_hi, 1.0, 1.0])}
        depth = 1
    return vr.tree_from_json({"root_box": root, "depth": depth, "root": node})


def _pool(tree, field=None):
    fields = [vr.AnalyticRegion(field if field is not None
                                else vr.ConstantBox(lf.box, 0.0, (0, 0, 0)))
              for lf in tree.leaves]
    return vr.VolumePool(tree, fields, (0.0, 0.0, 0.0), DEV)


def _ray(o, d, tn=0.0, tf=10.0):
    return np.array([[*o, *d, tn, tf]], dtype=np.float64).T.copy()


def _samples(pool, rays, dt):
    b = pool.sample(pool.rays_to_device(rays), dt)
    torch.cuda.synchronize()
    pool.check()
    n = b.n_samples
    off = b.offsets.cpu().numpy()
    owner = np.repeat(np.arange(b.region_cnt * b.n_rays), np.diff(off)) // b.n_rays
    edges = list(zip(b.t0[:n].cpu().tolist(), b.t1[:n].cpu().tolist()))
    return edges, owner.tolist()


@pytest.mark.parametrize("x_hi, tf, dt", [(2.0, 10.0, 0.25), (1.9, 10.0, 0.25),
                                            (2.0, 1.6, 0.25), (2.0, 10.0, 0.3)])
def test_grid_edges_and_truncation(x_hi, tf, dt):
    """Bins te + k dt, the last one cut at tx (box face or t_far), as grid_edges."""
    edges, owner = _samples(_pool(_tree(1.0, x_hi)), _ray((0, 0.5, 0.5), (1, 0, 0), tf=tf), dt)
    assert edges == vo.grid_edges(1.0, min(x_hi, tf), dt)
    assert owner == [0] * len(edges)


def test_split_at_plane_and_owners():
    edges, owner = _samples(_pool(_tree(1.0, 2.0, 1.5)), _ray((0, 0.5, 0.5), (1, 0, 0)), 1.0)
    assert edges == vo.split_bins([(1.0, 2.0)], [1.5]) == [(1.0, 1.5), (1.5, 2.0)]
    assert owner == [0, 1]


def test_sliver_dropped():
    """A cut 1e-14 after the entry leaves a sub-bin <= SLIVER: dropped (quadrature.py:106)."""
    plane = 1.0 + 1e-14
    edges, owner = _samples(_pool(_tree(1.0, 2.0, plane)), _ray((0, 0.5, 0.5), (1, 0, 0)), 1.0)
    assert edges == vo.split_bins([(1.0, 2.0)], [plane]) == [(plane, 2.0)]
    assert owner == [1]


@pytest.mark.parametrize("o, d", [((0, 2.0, 0.5), (1, 0, 0)),      # passes beside the box
                                  ((0, 0.5, 0.5), (-1, 0, 0)),     # points away
                                  ((1.5, 1.5, 0.5), (0, 0, 1))])   # d.y == 0, outside slab
def test_miss_gives_no_samples(o, d):
    edges, _ = _samples(_pool(_tree(1.0, 2.0)), _ray(o, d), 0.25)
    assert edges == []


def _render(pool, rays, dt):
    out, _ = pool.render_rays(rays, dt, clip=False)
    torch.cuda.synchronize()
    pool.check()
    return out[:, 0].cpu().numpy().astype(np.float64)  # r, g, b, alpha, depth, T, L


def test_ln2_closed_form_one_bin():
    """sigma = ln2 / 0.5 over one bin of length 0.5: alpha = T = 1/2, depth = the midpoint
    weight (test_quadrature.py:126-133)."""
    ln2 = math.log(2.0)
    tree = _tree(0.75, 1.25)
    field = vr.ConstantBox(vr.Aabb([0.75, 0, 0], [1.25, 1, 1]), ln2 / 0.5, (1, 0, 0))
    out = _render(_pool(tree, field), _ray((0, 0.5, 0.5), (1, 0, 0)), 0.5)
    T, C, A, D, L = vo.segment_packet([0.75], [1.25], [ln2 / 0.5], [[1, 0, 0]])
    np.testing.assert_allclose(out[[0, 1, 2]], C, atol=1e-6)
    assert out[3] == pytest.approx(A, abs=1e-6) and out[5] == pytest.approx(T, abs=1e-6)
    assert out[4] == pytest.approx(D, abs=1e-6) and out[6] == pytest.approx(0.0, abs=1e-7)


def test_two_bins_colour_and_occlusion():
    """Two bins of sigma = ln2: C = 0.5 red + 0.25 blue, T = 1/4 (test_quadrature.py:134-141);
    the second region is behind the first, so its colour is attenuated by the first's T
    (the fold of test_segrender.py:62-83) — here across two regions and their packets."""
    ln2 = math.log(2.0)
    tree = _tree(0.0, 2.0, 1.0)
    field = vr.SumField((vr.ConstantBox(vr.Aabb([0, 0, 0], [1, 1, 1]), ln2, (1, 0, 0)),
                         vr.ConstantBox(vr.Aabb([1, 0, 0], [2, 1, 1]), ln2, (0, 0, 1))))
    out = _render(_pool(tree, field), _ray((-1, 0.5, 0.5), (1, 0, 0)), 1.0)
    T, C, A, D, L = vo.segment_packet([1, 2], [2, 3], [ln2, ln2], [[1, 0, 0], [0, 0, 1]])
    np.testing.assert_allclose(out[[0, 1, 2]], [0.5, 0.0, 0.25], atol=1e-6)
    np.testing.assert_allclose(out[[0, 1, 2]], C, atol=1e-6)
    assert out[5] == pytest.approx(0.25, abs=1e-6)
    assert out[3] == pytest.approx(A, abs=1e-6) and out[4] == pytest.approx(D, abs=1e-5)
    assert out[6] == pytest.approx(L, abs=1e-5)


def test_opaque_front_region_hides_the_back():
    """An opaque first region (T = 0 to float precision) leaves nothing of the second."""
    tree = _tree(0.0, 2.0, 1.0)
    field = vr.SumField((vr.ConstantBox(vr.Aabb([0, 0, 0], [1, 1, 1]), 1e3, (0, 1, 0)),
                         vr.ConstantBox(vr.Aabb([1, 0, 0], [2, 1, 1]), 5.0, (1, 0, 0))))
    out = _render(_pool(tree, field), _ray((-1, 0.5, 0.5), (1, 0, 0)), 0.25)
    np.testing.assert_allclose(out[[0, 1, 2]], [0.0, 1.0, 0.0], atol=1e-6)
    assert out[3] == pytest.approx(1.0, abs=1e-6) and out[5] == pytest.approx(0.0, abs=1e-6)
