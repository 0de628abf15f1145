"""Full-size properties (BASELINE.json's c3: 1,048,576 rays, 8 regions): the one-walk K1
equals count + fill bit for bit, 8 simulated ranks reproduce the single-rank samples and
packets bit for bit (restricted walks, prefilter, sparse exchange), the K4 backward from
the forward's totals matches the recomputing one.  The oracle is too slow at this size;
these are the size-independent checks (sortedness, partition of the sample set,
bitwise agreement between decompositions)."""
import numpy as np
import pytest
import torch

import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def c3():
    w = CONFIGS["c3"]
    tree = w.tree
    rays = torch.from_numpy(make_rays(w)).to(DEV)
    return w, tree, rays


def _fields(tree, lo, cnt):
    # distinct constant densities / colours per region: every packet differs
    return [vr.AnalyticRegion(vr.ConstantBox(tree.leaves[k].box, 0.05 * (k + 1),
                                             (0.1 * k, 0.5, 1.0 - 0.1 * k)))
            for k in range(lo, lo + cnt)]


def _pool(tree, rank=0, world=1):
    lo, cnt = vr.owned_regions(len(tree.leaves), rank, world)
    return vr.VolumePool(tree, _fields(tree, lo, cnt), (0.0, 0.0, 0.0), DEV, rank, world)


def test_one_walk_equals_count_fill_and_sorted(c3):
    w, tree, rays = c3
    pool = _pool(tree)
    pool.stage_k1 = False
    ref = pool.sample(rays, w.dt)
    pool.stage_k1 = True
    b = pool.sample(rays, w.dt)
    b = pool.sample(rays, w.dt)  # the staging is sized by now
    torch.cuda.synchronize()
    pool.check()
    assert pool.last_k1 == "stage"
    n = ref.n_samples
    assert b.n_samples == n and n > 60 * rays.shape[1]
    for a, c in ((b.t0, ref.t0), (b.t1, ref.t1), (b.ray_id, ref.ray_id)):
        assert torch.equal(a[:n], c[:n])
    assert torch.equal(b.offsets, ref.offsets) and torch.equal(b.seg_first, ref.seg_first)
    # inside every segment the bins are ordered and contiguous (t0[i+1] == t1[i])
    off = b.offsets
    same = torch.ones(n, dtype=torch.bool, device=DEV)
    same[off[1:-1][off[1:-1] < n]] = False  # first sample of each segment
    t0, t1 = b.t0[:n], b.t1[:n]
    assert bool((t1 > t0).all())
    assert bool((t0[1:][same[1:]] == t1[:-1][same[1:]]).all())


def test_eight_ranks_reproduce_the_single_rank_samples_and_packets(c3):
    w, tree, rays = c3
    full = _pool(tree)
    b1 = full.sample(rays, w.dt)
    pk1 = full.local_packets(b1, full.evaluate(rays, b1))
    world = 8
    bufs, ns = [], []
    for rank in range(world):
        p = _pool(tree, rank, world)
        b = p.sample(rays, w.dt)
        lo, hi = b1.region_slice(rank)
        n = b.n_samples
        assert n == hi - lo
        assert torch.equal(b.t0[:n], b1.t0[lo:hi]) and torch.equal(b.t1[:n], b1.t1[lo:hi])
        assert torch.equal(b.ray_id[:n], b1.ray_id[lo:hi])
        pk = p.local_packets(b, p.evaluate(rays, b))
        assert torch.equal(pk.view(torch.int32), pk1[rank:rank + 1].view(torch.int32))
        # the sparse exchange's records of this rank
        R = b.n_rays
        cap = R
        send = torch.zeros((cap + 1, 9), dtype=torch.float32, device=DEV)
        n_dev = torch.zeros(1, dtype=torch.int32, device=DEV)
        _lib.call("vr_packets_pack", _lib.ptr(pk), None, _lib.ptr(b.counts), R, b.region_lo,
                  b.region_cnt, _lib.ptr(send), cap, _lib.ptr(n_dev), _lib.ptr(p.err),
                  _lib.stream_ptr())
        bufs.append(send)
        ns.append(int(n_dev.item()))
        p.check()
    slab = torch.empty_like(pk1)
    recv = torch.cat(bufs, 0)
    _lib.call("vr_packets_unpack", _lib.ptr(recv), world, bufs[0].shape[0], 9, rays.shape[1],
              len(tree.leaves), _lib.ptr(slab), None, _lib.ptr(full.err), _lib.stream_ptr())
    torch.cuda.synchronize()
    full.check()
    assert torch.equal(slab.view(torch.int32), pk1.view(torch.int32))
    assert sum(ns) == int((b1.counts > 0).sum())
    # the global composite of the rebuilt slab is the single-rank one
    assert torch.equal(full.compose(slab, b1), full.compose(pk1, b1))


def test_segment_backward_from_totals_full_size(c3):
    w, tree, rays = c3
    p = _pool(tree)
    b = p.sample(rays, w.dt)
    sr = p.evaluate(rays, b)
    R = b.n_rays
    totals = p._segment_totals(b.region_cnt * R)
    p.local_packets(b, sr, totals)
    gen = torch.Generator(device=DEV).manual_seed(7)
    dpk = torch.randn((b.region_cnt, R, 8), device=DEV, generator=gen)
    out = []
    for t in (None, totals):
        dsig = torch.empty((max(b.n_samples, 1), 4), dtype=torch.float32, device=DEV)
        _lib.call("vr_segment_bwd", _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(sr),
                  _lib.ptr(b.offsets), _lib.ptr(b.ray_te), R, b.region_cnt, _lib.ptr(dpk),
                  _lib.ptr(t), _lib.ptr(dsig), _lib.stream_ptr())
        out.append(dsig[:b.n_samples])
    torch.cuda.synchronize()
    assert bool(torch.isfinite(out[0]).all())
    torch.testing.assert_close(out[1], out[0], rtol=1e-5, atol=1e-7)
