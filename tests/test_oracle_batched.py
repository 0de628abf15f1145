"""CPU: the batched oracle (grad_oracle.field_loss_batched, used by the BASELINE-config
parity tests) against the per-ray oracle and the reference's golden render vectors.

The per-ray oracle is pinned to the reference in test_oracle_golden.py; these tests
carry that pin over to the batched restatement: same outputs to 1e-12, same loss to
1e-12 rel, same gradients to 1e-9 rel (float64 summation order only)."""
import numpy as np
import pytest
import torch

from conftest import load_npz, render_fixtures
from oracle import grad_oracle, hashmlp_oracle as hmo, volray_oracle as vo


@pytest.mark.parametrize("name", render_fixtures())
def test_batched_render_matches_reference(name):
    g = load_npz(name)
    tree = vo.Tree(g["tree"])
    f = vo.AnalyticField(g["scene"]["field"])

    def ev(k, pts, dirs):
        s, c = f.eval(pts)
        return torch.from_numpy(s), torch.from_numpy(c)

    rays = np.asarray(g["rays"])
    _, out, _ = grad_oracle.field_loss_batched(tree, ev, rays, np.zeros((len(rays), 3)),
                                               (0, 0, 0), float(g["dt"]))
    np.testing.assert_allclose(out, g["out"], rtol=1e-10, atol=1e-12)


def _rand_rays(rng, n):
    rays = []
    while len(rays) < n:
        o = rng.uniform(-2.4, 2.4, size=3)
        d = rng.uniform(-0.8, 0.8, size=3) - o
        rays.append([*o, *(d / np.linalg.norm(d)), 0.0, 20.0])
    return np.asarray(rays)


def _models(rng, tree_doc_leaves, log2_T=10, max_res=64):
    ms = []
    _, n_entries = hmo.levels(log2_T, max_res=max_res)
    for mn, mx in tree_doc_leaves:
        table = rng.uniform(-0.5, 0.5, size=(n_entries, 2)).astype(np.float32)
        w = np.zeros(hmo.NPARAMS, dtype=np.float32)
        for off, rows, cols in ((0, 64, 32), (2048, 16, 64), (3072, 64, 32), (5120, 64, 64),
                                (9216, 3, 64)):
            w[off:off + rows * cols] = rng.normal(size=rows * cols) / np.sqrt(cols)
        ms.append(hmo.HashMLPModel(table, w, log2_T, mn, mx, max_res=max_res))
    return ms


def _tree(split: str):
    root = {"min": [-1.0, -1.0, -1.0], "max": [1.0, 1.0, 1.0]}
    if not split:
        return {"root_box": root, "depth": 0, "root": {"tile_id": 0, "box": root}}
    return {"root_box": root, "depth": 1, "root": {
        "axis": "x", "plane": 0.0,
        "low": {"tile_id": 0, "box": {"min": [-1.0, -1.0, -1.0], "max": [0.0, 1.0, 1.0]}},
        "high": {"tile_id": 1, "box": {"min": [0.0, -1.0, -1.0], "max": [1.0, 1.0, 1.0]}}}}


@pytest.mark.parametrize("split", ["", "x"])
@pytest.mark.parametrize("interlevel", [False, True])
def test_batched_equals_per_ray_oracle(split, interlevel):
    rng = np.random.default_rng(3)
    tree = vo.Tree(_tree(split))
    leaves = list(zip(tree.leaf_mn, tree.leaf_mx))
    rays = _rand_rays(rng, 12)
    targets = rng.uniform(0, 1, size=(12, 3))
    bg = (0.2, 0.3, 0.4)
    grads = []
    results = []
    for batched in (False, True):
        ms = _models(np.random.default_rng(5), leaves)
        ps = _models(np.random.default_rng(6), leaves, log2_T=9, max_res=32) if interlevel else None
        if batched:
            loss, out, il = grad_oracle.field_loss_batched(
                tree, lambda k, p, d: ms[k].eval_dirs(p, d), rays, targets, bg, 0.05,
                prop_batch=(lambda k, p, d: ps[k].eval_dirs(p, d)) if interlevel else None,
                lambda_int=0.5)
        elif interlevel:
            loss, out, il = grad_oracle.field_loss_interlevel(
                tree, lambda k, p, d: ms[k].eval_t(p, d), lambda k, p, d: ps[k].eval_t(p, d),
                rays, targets, bg, 0.05, 1.0, 0.5)
        else:
            loss, out = grad_oracle.field_loss(tree, lambda k, p, d: ms[k].eval_t(p, d), rays,
                                               targets, bg, 0.05)
        loss.backward()
        results.append((loss.item(), out))
        grads.append([m.grads() for m in ms + (ps or [])])
    (l0, o0), (l1, o1) = results
    assert l1 == pytest.approx(l0, rel=1e-12)
    np.testing.assert_allclose(o1, o0, rtol=1e-12, atol=1e-12)
    for (ta, wa), (tb, wb) in zip(grads[0], grads[1]):
        np.testing.assert_allclose(tb, ta, rtol=1e-9, atol=1e-12 * np.abs(ta).max())
        np.testing.assert_allclose(wb, wa, rtol=1e-9, atol=1e-12 * np.abs(wa).max())


def test_unquantised_model_is_close_to_quantised():
    """The fp16 quantisation points move the output by ~1e-3, not more: the kernels'
    precision choice (fp16 weights/activations, fp32 accumulation) is a bounded model
    choice, measured here against the ideal float64 model."""
    rng = np.random.default_rng(9)
    tree = vo.Tree(_tree(""))
    leaves = list(zip(tree.leaf_mn, tree.leaf_mx))
    rays = _rand_rays(rng, 16)
    q = _models(np.random.default_rng(5), leaves)[0]
    ideal = hmo.HashMLPModel(q.table.detach().numpy(), q.weights.detach().numpy().astype(np.float32),
                             q.log2_T, q.box_mn, q.box_mx, max_res=64, quantize=False)
    outs = []
    for m in (q, ideal):
        _, out, _ = grad_oracle.field_loss_batched(tree, lambda k, p, d: m.eval_dirs(p, d), rays,
                                                   np.zeros((16, 3)), (0, 0, 0), 0.05)
        outs.append(out)
    diff = np.abs(outs[0][:, 0:4] - outs[1][:, 0:4]).max()
    assert 0.0 < diff < 5e-3, diff
