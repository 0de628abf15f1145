"""Sparse backward (vr_active_rows): the row list is exactly the ordered non-zero rows, and
every backward variant given the list produces the same parameter gradients as the dense
backward (a zero upstream row contributes exactly zero; only the float32 summation order of
the weight-gradient tiles and the table atomics differs)."""
import numpy as np
import pytest
import torch

import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _rows(dsr, n):
    ws = torch.empty(max(int(_lib.load().vr_active_rows_workspace_bytes(n)), 256),
                     dtype=torch.uint8, device=DEV)
    rows = torch.full((max(n, 1),), -7, dtype=torch.int32, device=DEV)
    cnt = torch.full((1,), -1, dtype=torch.int32, device=DEV)
    _lib.call("vr_active_rows", _lib.ptr(dsr), n, _lib.ptr(rows), _lib.ptr(cnt), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    torch.cuda.synchronize()
    return rows, cnt


@pytest.mark.parametrize("n", [0, 1, 31, 4095, 4096, 4097, 1_000_003])
def test_active_rows_are_the_ordered_nonzero_rows(n):
    g = torch.Generator(device="cpu").manual_seed(n)
    dsr = torch.randn((max(n, 1), 4), generator=g)
    # runs of zero rows (the samples behind an opaque surface), single-component rows, NaN
    keep = torch.rand(max(n, 1), generator=g) < 0.3
    dsr[~keep] = 0.0
    if n > 10:
        dsr[3] = torch.tensor([0.0, 0.0, -0.0, 1e-38])
        dsr[5] = torch.tensor([0.0, -0.0, 0.0, 0.0])
        dsr[7] = torch.tensor([float("nan"), 0.0, 0.0, 0.0])
    dsr = dsr.to(DEV)
    rows, cnt = _rows(dsr, n)
    want = torch.nonzero((dsr[:n] != 0).any(1) | dsr[:n].isnan().any(1)).flatten()
    assert cnt.item() == want.numel()
    assert torch.equal(rows[:cnt.item()].long(), want)
    if n > 10:
        assert 3 in want and 7 in want and 5 not in want


def _pool(mlp_impl, hash_order, density_only=False, seed=0):
    rng = np.random.default_rng(seed)
    root = vr.Aabb([-1, -1, -1], [1, 1, 1])
    tree = vr.grid_tree(root, "x")
    cfg = vr.HashGridConfig(log2_T=14, max_res=256)
    fields = [vr.HashGridMLP(cfg, tree.leaves[k].box, DEV, seed=k, mlp_impl=mlp_impl,
                             hash_order=hash_order, table_init=0.5, density_only=density_only)
              for k in range(2)]
    pool = vr.VolumePool(tree, fields, (0.2, 0.3, 0.4), DEV)
    rays = []
    while len(rays) < 400:
        o = rng.uniform(-2.4, 2.4, size=3)
        d = rng.uniform(-0.8, 0.8, size=3) - o
        rays.append([*o, *(d / np.linalg.norm(d)), 0.0, 20.0])
    return pool, pool.rays_to_device(np.asarray(rays).T.copy())


@pytest.mark.parametrize("mlp_impl,hash_order,density_only", [
    ("fused", "sample", False),   # vr_field_bwd_tc (MLP backward + fused scatter)
    ("fused_fwd", "sample", False),  # the same, positions recomputed from the rays
    ("tc", "sample", False),      # vr_mlp_bwd_tc + sample-order vr_hash_scatter
    ("fused", "level", False),    # vr_mlp_bwd_tc + level-major vr_hash_scatter
    ("fused", "auto", True),      # density-only proposal: vr_mlp_bwd_tc_density + scatter
])
@pytest.mark.parametrize("overlap", [False, True])
def test_sparse_backward_matches_dense(mlp_impl, hash_order, density_only, overlap):
    pool, rd = _pool(mlp_impl, hash_order, density_only)
    pool.overlap_backward = overlap
    b = pool.sample(rd, 0.02)
    sig = pool.evaluate(rd, b)
    g = torch.Generator(device="cpu").manual_seed(1)
    dsig = torch.randn((b.n_samples, 4), generator=g) * 0.05
    if density_only:
        dsig[:, 1:] = 0.0
    # 70 % of the rows exactly zero (behind opaque surfaces most samples are)
    t = torch.rand(b.n_samples, generator=g)
    dsig[t < 0.7] = 0.0
    dsig = dsig.to(DEV)
    grads = []
    for active in (False, True):
        pool.ACTIVE_ROWS = active
        pool.zero_grad()
        pool.field_backward(rd, b, dsig, sig_rgb=sig)
        torch.cuda.synchronize()
        pool.check()
        grads.append([(f.grad_table.clone(), f.grad_weights.clone()) for f in pool.fields])
    for (ta, wa), (tb, wb) in zip(*grads):
        assert torch.count_nonzero(ta) > 100
        for a, c in ((ta, tb), (wa, wb)):
            rel = ((a - c).norm() / a.norm()).item()
            assert rel < 1e-5, rel
            # element-wise: float32 reordering only
            assert torch.allclose(a, c, rtol=1e-4, atol=1e-6 * a.abs().max().item())
