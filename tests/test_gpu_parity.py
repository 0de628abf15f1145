"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the oracle.

Tolerances (north_star): sample edges / owner ids / hash indices bit-exact;
colour, opacity, depth <= 1e-4 abs; loss <= 1e-5 rel; gradients <= 1e-3 rel.
"""
import json

import numpy as np
import pytest
import torch

import paper_2404_16221_b200 as vr
from conftest import GOLDEN, load_npz, render_fixtures, sampler_fixtures
from oracle import grad_oracle, hashmlp_oracle as hmo, volray_oracle as vo

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


class _NoField(vr.RegionField):
    def forward(self, *a):
        raise AssertionError("not used")


def _pool(tree, fields=None, rank=0, world=1, bg=(0.0, 0.0, 0.0)):
    lo, cnt = vr.owned_regions(len(tree.leaves), rank, world)
    if fields is None:
        fields = [_NoField() for _ in range(cnt)]
    return vr.VolumePool(tree, fields, bg, DEV, rank, world)


def _soa(rows):
    return np.ascontiguousarray(np.asarray(rows, dtype=np.float64).T)


def _flatten_batch(b):
    """(ray, t0, t1, region) of every owned sample, sorted by (ray, t0)."""
    R = b.n_rays
    off = b.offsets.cpu().numpy()
    n = int(off[-1])
    seg = np.repeat(np.arange(b.region_cnt * R), np.diff(off))
    region = seg // R + b.region_lo
    rid = b.ray_id[:n].cpu().numpy().astype(np.int64)
    assert np.array_equal(rid, seg % R)
    t0 = b.t0[:n].cpu().numpy()
    t1 = b.t1[:n].cpu().numpy()
    order = np.lexsort((t0, rid))
    return rid[order], t0[order], t1[order], region[order]


# stats=False: a rank skips the rays / bins that cannot reach its regions (the training
# path); the samples, owners and order keys must stay bit-identical
@pytest.mark.parametrize("stats", [True, False])
@pytest.mark.parametrize("name", sampler_fixtures())
@pytest.mark.parametrize("world", [1, 2, 4])
def test_sampler_bit_exact(name, world, stats):
    g = load_npz(name)
    tree = vr.tree_from_json(g["tree"])
    K = len(tree.leaves)
    if K % world:
        pytest.skip("regions not divisible")
    rays = _soa(g["rays"])
    ref_ray = np.repeat(np.arange(len(g["counts"])), g["counts"])
    for rank in range(world):
        pool = _pool(tree, rank=rank, world=world)
        b = pool.sample(pool.rays_to_device(rays), float(g["dt"]), stats=stats)
        torch.cuda.synchronize()
        pool.check()
        rid, t0, t1, region = _flatten_batch(b)
        sel = (g["tile"] >= pool.region_lo) & (g["tile"] < pool.region_lo + pool.region_cnt)
        assert np.array_equal(rid, ref_ray[sel])
        assert np.array_equal(t0, g["t0"][sel]), "bin edges t0 differ"
        assert np.array_equal(t1, g["t1"][sel]), "bin edges t1 differ"
        assert np.array_equal(region, g["tile"][sel]), "owner tiles differ"
        assert np.array_equal(b.ray_te.cpu().numpy(), g["te"])
        if stats:
            assert np.array_equal(b.ray_total.cpu().numpy(), g["counts"])
            part = b.ray_part.cpu().numpy().astype(np.int64) & 0xFFFFFFFF
            assert np.array_equal(part, g["part"])
        # segment order key = index of the region's first sample along the ray
        sf = b.seg_first.cpu().numpy().reshape(pool.region_cnt, -1)
        starts = np.concatenate([[0], np.cumsum(g["counts"])])
        for r in range(0, len(g["counts"]), 7):
            tiles = g["tile"][starts[r]:starts[r + 1]]
            for kk in range(pool.region_cnt):
                hit = np.nonzero(tiles == pool.region_lo + kk)[0]
                want = hit[0] if hit.size else np.iinfo(np.int32).max
                assert sf[kk, r] == want


@pytest.mark.parametrize("prefilter", [True, False])
@pytest.mark.parametrize("stats", [True, False])
@pytest.mark.parametrize("name", ["sampler_three_blobs_k8.npz", "sampler_random_d2.npz"])
def test_sampler_one_walk_matches_fill(name, stats, prefilter):
    """One-walk K1 (vr_sample_stage + vr_sample_compact, with or without the multi-rank
    ray prefilter) == count + fill, bit for bit, also through the overflow path (staging
    too small: fill pass, staging grown for next call)."""
    g = load_npz(name)
    tree = vr.tree_from_json(g["tree"])
    rays = _soa(g["rays"])
    for rank, world in ((0, 1), (0, 2), (1, 2), (3, 4)):
        if len(tree.leaves) % world:
            continue
        pool = _pool(tree, rank=rank, world=world)
        pool.k1_prefilter = prefilter
        rd = pool.rays_to_device(rays)
        pool.stage_k1 = False
        ref = pool.sample(rd, float(g["dt"]), stats=stats)
        assert pool.last_k1 == "fill"
        pool.stage_k1 = True
        pool.stage_slots_per_ray = 1
        runs = []
        for _ in range(2):
            runs.append((pool.sample(rd, float(g["dt"]), stats=stats), pool.last_k1))
        assert [k for _, k in runs] == ["fill", "stage"]
        torch.cuda.synchronize()
        pool.check()
        n = ref.n_samples
        for b, _ in runs:
            assert b.region_bounds == ref.region_bounds
            for a, c in ((b.t0, ref.t0), (b.t1, ref.t1), (b.ray_id, ref.ray_id)):
                assert torch.equal(a[:n], c[:n])
            for a, c in ((b.counts, ref.counts), (b.seg_first, ref.seg_first),
                         (b.offsets, ref.offsets), (b.ray_te, ref.ray_te),
                         (b.ray_part, ref.ray_part), (b.ray_total, ref.ray_total)):
                assert (a is None and c is None) or torch.equal(a, c)


@pytest.mark.parametrize("capacity", [1, None])
def test_sample_async_matches_sample(capacity):
    """K1 one step ahead (sample_async / resolve_sample on the sampling stream) gives the
    same batch as sample(); a capacity below the sample count is re-filled."""
    g = load_npz("sampler_three_blobs_k8.npz")
    tree = vr.tree_from_json(g["tree"])
    for rank, world in ((0, 1), (1, 2)):
        pool = _pool(tree, rank=rank, world=world)
        rd = pool.rays_to_device(_soa(g["rays"]))
        ref = pool.sample(rd, float(g["dt"]))
        cap = ref.n_samples if capacity is None else capacity
        b = pool.resolve_sample(pool.sample_async(rd, float(g["dt"]), cap))
        torch.cuda.synchronize()
        assert b.region_bounds == ref.region_bounds
        n = ref.n_samples
        for a, c in ((b.t0, ref.t0), (b.t1, ref.t1), (b.ray_id, ref.ray_id)):
            assert torch.equal(a[:n], c[:n])
        assert torch.equal(b.seg_first, ref.seg_first) and torch.equal(b.offsets, ref.offsets)


def test_sampler_empty_and_bad_args(cuda_device):
    g = load_npz("sampler_random_d2.npz")
    tree = vr.tree_from_json(g["tree"])
    pool = _pool(tree)
    b = pool.sample(pool.rays_to_device(np.zeros((8, 0))), 0.1)
    assert b.n_samples == 0
    with pytest.raises(ValueError):
        pool.sample(pool.rays_to_device(_soa(g["rays"][:4])), 0.0)


def _scene_pool(g, world=1, rank=0):
    tree = vr.tree_from_json(g["tree"])
    scene = vr.scene_from_json(g["scene"])
    return vr.spawn(tree, scene, DEV, rank, world), tree, scene


# the reference's protocols all integrate the same bins and agree within 1e-10
# (distsim.render_ray docstring), so every protocol is checked against the tile golden
@pytest.mark.parametrize("protocol", ["tile", "sample", "mono"])
@pytest.mark.parametrize("name", render_fixtures())
def test_render_matches_reference(name, protocol):
    g = load_npz(name)
    pool, tree, scene = _scene_pool(g)
    out, b = pool.render_rays(_soa(g["rays"]), float(g["dt"]), clip=False, protocol=protocol)
    torch.cuda.synchronize()
    pool.check()
    got = out.cpu().numpy().T.astype(np.float64)  # (R, 7): C, A, depth, T, L
    ref = g["out"]
    np.testing.assert_allclose(got[:, 0:3], ref[:, 0:3], atol=1e-4, rtol=0)
    np.testing.assert_allclose(got[:, 3], ref[:, 3], atol=1e-4, rtol=0)
    np.testing.assert_allclose(got[:, 4], ref[:, 4], atol=1e-4, rtol=0)
    np.testing.assert_allclose(got[:, 5], ref[:, 5], atol=1e-4, rtol=0)
    np.testing.assert_allclose(got[:, 6], ref[:, 6], atol=1e-4, rtol=1e-4)


def test_render_image_matches_reference():
    g = load_npz("image_three_blobs.npz")
    pool, tree, scene = _scene_pool(g)
    cam = vr.Camera.from_json(g["camera"])
    img, st = vr.render_image(pool, cam, "tile", float(g["dt"]))
    np.testing.assert_allclose(img, g["image"], atol=1e-4, rtol=0)
    ref_bytes = np.floor(np.clip(g["image"], 0, 1) * 255 + 0.5).astype(np.uint8)
    got_bytes = np.floor(np.clip(img, 0, 1) * 255 + 0.5).astype(np.uint8)
    assert np.mean(ref_bytes == got_bytes) > 0.999
    assert st.scalars_sent_total == g["stats"]["scalars_sent_total"]
    assert [w["scalars_sent"] for w in vr.stats_json(st, "tile_aggregate", 4)["per_worker"]] == \
        [w["scalars_sent"] for w in g["stats"]["per_worker"]]


@pytest.mark.parametrize("proto", ["sample", "mono"])
def test_render_image_other_protocols_match_reference(proto):
    """render_image under the sample-broadcast / mono protocols: image and the reference's
    CommStats scalar counts (1 + 6 per bin per participation; nothing for mono)."""
    g = load_npz(f"image_three_blobs_{proto}.npz")
    pool, tree, scene = _scene_pool(g)
    cam = vr.Camera.from_json(g["camera"])
    img, st = vr.render_image(pool, cam, proto, float(g["dt"]))
    np.testing.assert_allclose(img, g["image"], atol=1e-4, rtol=0)
    assert st.rays == g["stats"]["rays"]
    assert st.scalars_sent_total == g["stats"]["scalars_sent_total"]
    mine = vr.stats_json(st, g["stats"]["protocol"], 4)["per_worker"]
    ref = g["stats"]["per_worker"]
    assert [(w["scalars_sent"], w["messages_sent"]) for w in mine] == \
        [(w["scalars_sent"], w["messages_sent"]) for w in ref]


def test_sample_protocol_multi_rank_exchange_is_bitwise_identical():
    """Sample-broadcast with 2 simulated ranks: each evaluates only its own regions of the
    all-region batch; the filled-in array (what the all-gather delivers) composes exactly
    the single-rank image."""
    g = load_npz("render_three_blobs_k4.npz")
    rays = _soa(g["rays"])
    dt = float(g["dt"])
    pool1, _, _ = _scene_pool(g)
    out1, _ = pool1.render_rays(rays, dt, protocol="sample")
    full = None
    for rank in range(2):
        p, _, _ = _scene_pool(g, world=2, rank=rank)
        rd = p.rays_to_device(rays)
        b = p.sample(rd, dt, all_regions=True)
        sr = p.evaluate(rd, b)
        full = sr if full is None else full + sr  # disjoint blocks, zeros elsewhere
    ray_off = p._ray_major(b)
    rm = [p._permute(b, ray_off, x, True) for x in (b.t0, b.t1, full)]
    out2 = p.compose(p._whole_ray_packets(b, ray_off, *rm), b)
    assert torch.equal(out1, out2)


def test_multi_rank_composite_is_bitwise_identical():
    """Config 2: packets produced by 2 simulated ranks and gathered give exactly the
    single-rank composite (the training-mode agreement check, distsim.py:457-475)."""
    g = load_npz("render_three_blobs_k4.npz")
    rays = _soa(g["rays"])
    dt = float(g["dt"])
    pool1, tree, scene = _scene_pool(g)
    out1, _ = pool1.render_rays(rays, dt)
    parts = []
    for rank in range(2):
        p, _, _ = _scene_pool(g, world=2, rank=rank)
        rd = p.rays_to_device(rays)
        b = p.sample(rd, dt)
        parts.append(p.local_packets(b, p.evaluate(rd, b)))
        if rank == 0:
            b0 = b
    allp = torch.cat(parts, 0)
    p0, _, _ = _scene_pool(g, world=2, rank=0)
    out2 = p0.compose(allp, b0)
    assert torch.equal(out1, out2)


@pytest.mark.parametrize("name", ["render_three_blobs_k8.npz", "render_street_k8.npz"])
def test_segment_bwd_with_forward_totals(name):
    """vr_segment_bwd from the forward's float64 segment totals (no first sweep) gives the
    per-sample gradients of the recomputing path."""
    from paper_2404_16221_b200 import _lib

    g = load_npz(name)
    rays = _soa(g["rays"])
    dt = float(g["dt"])
    p, _, _ = _scene_pool(g)
    rd = p.rays_to_device(rays)
    b = p.sample(rd, dt)
    sr = p.evaluate(rd, b)
    R = b.n_rays
    totals = p._segment_totals(b.region_cnt * R)
    pk = p.local_packets(b, sr, totals)
    # keeping totals leaves the packets alone (bit compare: order keys of empty ones are NaNs)
    assert torch.equal(pk.view(torch.int32), p.local_packets(b, sr).view(torch.int32))
    gen = torch.Generator(device=DEV).manual_seed(5)
    dpk = torch.randn((b.region_cnt, R, 8), device=DEV, generator=gen)
    out = []
    for t in (None, totals):
        dsig = torch.zeros((max(b.n_samples, 1), 4), dtype=torch.float32, device=DEV)
        _lib.call("vr_segment_bwd", _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(sr),
                  _lib.ptr(b.offsets), _lib.ptr(b.ray_te), R, b.region_cnt, _lib.ptr(dpk),
                  _lib.ptr(t), _lib.ptr(dsig), _lib.stream_ptr())
        out.append(dsig)
    torch.cuda.synchronize()
    torch.testing.assert_close(out[1], out[0], rtol=1e-6, atol=1e-9)
    # the transmittance-only kernel (proposal packets) gives the packets' T bit for bit
    T = torch.empty((b.region_cnt, R), dtype=torch.float32, device=DEV)
    _lib.call("vr_segment_transmittance", _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(sr),
              _lib.ptr(b.offsets), R, b.region_cnt, _lib.ptr(T), _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(T, pk[:, :, 0])
    # the forward with its inputs staged by TMA (n_samples given) == per-lane loads, bit for
    # bit, packets and float64 totals
    assert _lib.load().vr_tma_available() == 1
    n_tma = p._tma_n(b.n_samples, b.t0, b.t1, sr)
    assert n_tma == b.n_samples
    res = []
    for n_arg in (0, n_tma):
        pk2 = torch.empty_like(pk)
        tot2 = torch.empty_like(totals)
        _lib.call("vr_segment_fwd", _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(sr),
                  _lib.ptr(b.offsets), _lib.ptr(b.seg_first), _lib.ptr(b.ray_te), R,
                  b.region_cnt, _lib.ptr(pk2), _lib.ptr(tot2), _lib.ptr(p.err), n_arg,
                  _lib.stream_ptr())
        res.append((pk2, tot2))
    torch.cuda.synchronize()
    p.check()
    assert torch.equal(res[0][0].view(torch.int32), res[1][0].view(torch.int32))
    live = (b.counts.reshape(-1) > 0).repeat_interleave(7)  # totals of non-empty segments
    assert torch.equal(res[0][1][live], res[1][1][live])


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("with_extra", [False, True])
def test_sparse_packet_exchange_kernels(world, with_extra):
    """vr_packets_pack / vr_packets_unpack with simulated ranks: the records are the
    non-empty segments' packets (the numpy restatement, as a set), and the unpacked slab is
    the dense all-gather's slab bit for bit; a too-small capacity raises the overflow."""
    import packets_ref as pr
    from paper_2404_16221_b200 import _lib

    g = load_npz("render_street_k8.npz")
    rays = _soa(g["rays"])
    dt = float(g["dt"])
    bufs, dense, dense_e, ns = [], [], [], []
    for rank in range(world):
        p, _, _ = _scene_pool(g, world=world, rank=rank)
        rd = p.rays_to_device(rays)
        b = p.sample(rd, dt)
        local = p.local_packets(b, p.evaluate(rd, b))
        R = b.n_rays
        extra = None
        if with_extra:
            extra = torch.where(b.counts.reshape(b.region_cnt, R) > 0, local[:, :, 0] * 0.25,
                                torch.ones_like(local[:, :, 0])).contiguous()
        cap = b.region_cnt * R
        width = 10 if with_extra else 9
        send = torch.zeros((cap + 1, width), dtype=torch.float32, device=DEV)
        n_dev = torch.zeros(1, dtype=torch.int32, device=DEV)
        _lib.call("vr_packets_pack", _lib.ptr(local), _lib.ptr(extra), _lib.ptr(b.counts), R,
                  b.region_lo, b.region_cnt, _lib.ptr(send), cap, _lib.ptr(n_dev),
                  _lib.ptr(p.err), _lib.stream_ptr())
        torch.cuda.synchronize()
        p.check()
        n = int(n_dev.item())
        rec, n_ref = pr.pack(local.cpu().numpy(), b.counts.cpu().numpy(), b.region_lo,
                             None if extra is None else extra.cpu().numpy())
        assert n == n_ref and int(send[0, 0].view(torch.int32).item()) == n
        got = send[1:n + 1].cpu().numpy()
        order = np.argsort(got[:, 0].copy().view(np.int32))
        assert np.array_equal(got[order].view(np.uint32), rec.view(np.uint32))
        bufs.append(send)
        dense.append(local)
        dense_e.append(extra)
        ns.append(n)
        # capacity below the record count: flagged
        small = torch.zeros((max(n - 1, 0) + 1, width), dtype=torch.float32, device=DEV)
        if n > 0:
            _lib.call("vr_packets_pack", _lib.ptr(local), _lib.ptr(extra), _lib.ptr(b.counts),
                      R, b.region_lo, b.region_cnt, _lib.ptr(small), n - 1, _lib.ptr(n_dev),
                      _lib.ptr(p.err), _lib.stream_ptr())
            with pytest.raises(vr.CapacityError):
                p.check()
    K = world * dense[0].shape[0]
    R = dense[0].shape[1]
    recv = torch.cat(bufs, 0)
    slab = torch.empty((K, R, 8), dtype=torch.float32, device=DEV)
    slab_e = torch.empty((K, R), dtype=torch.float32, device=DEV) if with_extra else None
    _lib.call("vr_packets_unpack", _lib.ptr(recv), world, bufs[0].shape[0], recv.shape[1], R, K,
              _lib.ptr(slab), _lib.ptr(slab_e), _lib.ptr(p.err), _lib.stream_ptr())
    torch.cuda.synchronize()
    p.check()
    assert torch.equal(slab.view(torch.int32), torch.cat(dense, 0).view(torch.int32))
    if with_extra:
        assert torch.equal(slab_e, torch.cat(dense_e, 0))
    assert sum(ns) < K * R
    # the record index (vr_packets_index): every non-empty segment points at its record,
    # empty ones are -1, and K5 / the interlevel prefix through it equal the dense slab's
    index = torch.empty((K, R), dtype=torch.int32, device=DEV)
    _lib.call("vr_packets_index", _lib.ptr(recv), world, bufs[0].shape[0], recv.shape[1], R, K,
              _lib.ptr(index), _lib.ptr(p.err), _lib.stream_ptr())
    torch.cuda.synchronize()
    p.check()
    live = slab.view(torch.int32)[:, :, 7] != 2 ** 31 - 1
    assert torch.equal(index >= 0, live)
    got = recv[index[live].long()]
    assert torch.equal(got[:, 1:9].view(torch.int32), slab[live].view(torch.int32))
    te = torch.zeros(R, dtype=torch.float64, device=DEV)
    tg = torch.rand((R, 3), device=DEV)
    outs = []
    for records in (False, True):
        out = torch.empty((7, R), device=DEV)
        loss = torch.empty(R, dtype=torch.float64, device=DEV)
        dpk = torch.empty((K, R, 8), device=DEV)
        bgv = p._set_bg((0.1, 0.2, 0.3))
        if records:
            _lib.call("vr_global_train_records", _lib.ptr(recv), recv.shape[1], _lib.ptr(index),
                      K, R, _lib.ptr(te), _lib.addr(bgv), _lib.ptr(tg), 0.5, 0, K, _lib.ptr(out),
                      _lib.ptr(loss), _lib.ptr(dpk), _lib.ptr(p.err), _lib.stream_ptr())
        else:
            _lib.call("vr_global_train", _lib.ptr(slab), K, R, _lib.ptr(te), _lib.addr(bgv),
                      _lib.ptr(tg), 0.5, 0, K, _lib.ptr(out), _lib.ptr(loss), _lib.ptr(dpk),
                      _lib.ptr(p.err), _lib.stream_ptr())
        pre = None
        if with_extra:
            pre = torch.empty((K, R, 2), device=DEV)
            if records:
                _lib.call("vr_prefix_train_records", _lib.ptr(recv), _lib.ptr(index), K, R, 0, K,
                          _lib.ptr(pre), _lib.stream_ptr())
            else:
                _lib.call("vr_prefix_train", _lib.ptr(slab), _lib.ptr(slab_e), K, R, 0, K,
                          _lib.ptr(pre), _lib.stream_ptr())
        torch.cuda.synchronize()
        p.check()
        outs.append((out, loss, dpk, pre))
    (o0, l0, d0, p0), (o1, l1, d1, p1) = outs
    assert torch.equal(o0, o1) and torch.equal(l0, l1) and torch.equal(d0, d1)
    if with_extra:
        assert torch.equal(p0, p1)


@pytest.mark.parametrize("name", ["partition_street.npz", "partition_voxel_room.npz"])
def test_rays_to_points_and_balance_report_match_reference(name):
    """rays_to_points (K1 on a one-leaf tree + the reference's numpy subsample) gives the
    reference's points bit for bit; balance_report's point and sample counts match."""
    g = load_npz(name)
    root = vr.Aabb.from_json(g["root"])
    rays = _soa(g["rays"])
    pc = vr.rays_to_points(rays, root, float(g["dt"]), int(g["max_points"]), seed=3, device=DEV)
    assert pc.source == "ray_discretized"
    assert np.array_equal(pc.points, g["points"])
    tree = vr.tree_from_json(g["tree"])
    rep = vr.balance_report(tree, pc.points, rays, float(g["dt"]), device=DEV)
    assert rep == g["report"]


def _grad_setup():
    doc = json.loads((GOLDEN / "grad_voxel_room.json").read_text())
    tree = vr.tree_from_json(doc["tree"])
    scene = vr.scene_from_json(doc["scene"])
    rays = _soa(doc["rays"])
    targets = np.full((rays.shape[1], 3), doc["target"])
    return doc, tree, scene, rays, targets


@pytest.mark.parametrize("protocol", ["tile", "sample"])
def test_voxel_gradients_match_reference_fd(protocol):
    doc, tree, scene, rays, targets = _grad_setup()
    pool = vr.spawn(tree, scene, DEV)
    pool.zero_grad()
    loss, out, b = pool.loss_and_grad(rays, targets, doc["dt"], protocol=protocol)
    torch.cuda.synchronize()
    pool.check()
    assert loss.item() == pytest.approx(doc["loss"], rel=1e-5)
    for e in doc["entries"]:
        g = pool.fields[e["tile"]].grad[tuple(e["index"])].item()
        fd = e["global"]
        assert abs(g - fd) <= 1e-3 * abs(fd) + 1e-6, (e, g)


@pytest.mark.parametrize("world", [2, 4])
def test_voxel_gradients_locality(world):
    """Each rank's gradient equals the corresponding slice of the single-rank gradient
    (no gradient all-reduce needed: segrender.py:209-221 LOCAL == GLOBAL)."""
    doc, tree, scene, rays, targets = _grad_setup()
    full = vr.spawn(tree, scene, DEV)
    full.zero_grad()
    full.loss_and_grad(rays, targets, doc["dt"])
    rd = full.rays_to_device(rays)
    pools = [vr.spawn(tree, scene, DEV, r, world) for r in range(world)]
    batches, sigs, locs = [], [], []
    for p in pools:
        p.zero_grad()
        b = p.sample(rd, doc["dt"])
        s = p.evaluate(rd, b)
        batches.append(b)
        sigs.append(s)
        locs.append(p.local_packets(b, s))
    allp = torch.cat(locs, 0)
    tg = torch.as_tensor(targets, dtype=torch.float32, device=DEV).contiguous()
    import ctypes
    from paper_2404_16221_b200 import _lib
    losses = []
    for p, b, s in zip(pools, batches, sigs):
        R = b.n_rays
        out = torch.empty((7, R), dtype=torch.float32, device=DEV)
        rl = torch.empty(R, dtype=torch.float64, device=DEV)
        dpk = torch.empty((b.region_cnt, R, 8), dtype=torch.float32, device=DEV)
        _lib.call("vr_global_train", _lib.ptr(allp), allp.shape[0], R, _lib.ptr(b.ray_te),
                  _lib.addr(p._set_bg(None)), _lib.ptr(tg), 1.0, p.region_lo, p.region_cnt,
                  _lib.ptr(out), _lib.ptr(rl), _lib.ptr(dpk), _lib.ptr(p.err), _lib.stream_ptr())
        losses.append(rl.sum().item())
        dsig = torch.zeros((max(b.n_samples, 1), 4), dtype=torch.float32, device=DEV)
        _lib.call("vr_segment_bwd", _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(s), _lib.ptr(b.offsets),
                  _lib.ptr(b.ray_te), R, b.region_cnt, _lib.ptr(dpk), None, _lib.ptr(dsig),
                  _lib.stream_ptr())
        p.field_backward(rd, b, dsig)
    assert len(set(losses)) == 1  # bitwise identical loss on every rank
    for p in pools:
        for kk, f in enumerate(p.fields):
            ref = full.fields[p.region_lo + kk].grad
            assert torch.allclose(f.grad, ref, rtol=1e-6, atol=1e-12)


def test_nonfinite_packet_raises():
    g = load_npz("render_three_blobs_k4.npz")
    pool, _, _ = _scene_pool(g)
    rays = pool.rays_to_device(_soa(g["rays"][:16]))
    b = pool.sample(rays, float(g["dt"]))
    pk = pool.local_packets(b, pool.evaluate(rays, b))
    nonempty = (pk[:, :, 7].view(torch.int32) != np.iinfo(np.int32).max).nonzero()
    k, r = nonempty[0].tolist()
    pk[k, r, 0] = float("nan")
    pool.compose(pk, b)
    with pytest.raises(vr.NonFiniteInputError):
        pool.check()


# ---- hash grid + MLP (parity unpinned: checked against oracle/hashmlp_oracle.py) ------

def _hash_setup(log2_T=14, K=2, n_rays=48, seed=0, restriction=False, mlp_impl="fused",
                hash_order="auto"):
    rng = np.random.default_rng(seed)
    root = vr.Aabb([-1, -1, -1], [1, 1, 1])
    tree = vr.grid_tree(root, "x" * int(np.log2(K))) if K > 1 else vr.grid_tree(root, "")
    cfg = vr.HashGridConfig(log2_T=log2_T, max_res=256)
    fields, models = [], []
    table0 = weights0 = None
    for k in range(K):
        box = root if restriction else tree.leaves[k].box
        _, n_entries = hmo.levels(log2_T, max_res=256)
        if table0 is None or not restriction:
            table0 = rng.uniform(-0.3, 0.3, size=(n_entries, 2)).astype(np.float32)
            w = np.zeros(hmo.NPARAMS, dtype=np.float32)
            for off, rows, cols in ((0, 64, 32), (2048, 16, 64), (3072, 64, 32), (5120, 64, 64),
                                    (9216, 3, 64)):
                w[off:off + rows * cols] = rng.normal(size=rows * cols) / np.sqrt(cols)
            weights0 = w
        f = vr.HashGridMLP(cfg, box, DEV, mlp_impl=mlp_impl, table=torch.from_numpy(table0.copy()),
                           weights=torch.from_numpy(weights0.copy()), hash_order=hash_order)
        fields.append(f)
        models.append(hmo.HashMLPModel(table0, weights0, log2_T, box.mn, box.mx, max_res=256))
    pool = vr.VolumePool(tree, fields, (0.2, 0.3, 0.4), DEV)
    rays = np.stack([vo_ray for vo_ray in (_rand_ray(rng) for _ in range(n_rays))], axis=1)
    targets = rng.uniform(0, 1, size=(n_rays, 3))
    return pool, tree, models, rays, targets


def _rand_ray(rng):
    while True:
        o = rng.uniform(-2.4, 2.4, size=3)
        t = rng.uniform(-0.8, 0.8, size=3)
        d = t - o
        n = np.linalg.norm(d)
        if n > 1e-6:
            d = d / n
            return np.array([*o, *d, 0.0, 20.0])


def test_hash_indices_bit_exact():
    pool, tree, models, rays, _ = _hash_setup(log2_T=12, K=2)
    rd = pool.rays_to_device(rays)
    b = pool.sample(rd, 0.03)
    from paper_2404_16221_b200 import _lib
    for kk, f in enumerate(pool.fields):
        lo, hi = b.region_slice(kk)
        n = hi - lo
        idx = torch.empty((16, n, 8), dtype=torch.int32, device=DEV)
        _lib.call("vr_hash_indices", _lib.addr(f.desc), _lib.ptr(rd), rd.shape[1],
                  _lib.ptr(b.t0[lo:]), _lib.ptr(b.t1[lo:]), _lib.ptr(b.ray_id[lo:]), n,
                  _lib.ptr(idx), _lib.stream_ptr())
        t0 = b.t0[lo:hi].cpu().numpy()
        t1 = b.t1[lo:hi].cpu().numpy()
        r = b.ray_id[lo:hi].cpu().numpy()
        m = 0.5 * (t0 + t1)
        pts = rays[0:3, r].T + m[:, None] * rays[3:6, r].T
        want = hmo.all_indices(pts, f.box.mn, f.box.mx, 12, max_res=256)
        assert np.array_equal(idx.cpu().numpy().astype(np.int64), want)


# overlap: split backward (MLP on the main stream, scatter on the side stream) vs the
# fused tensor-core backward / per-field backward
@pytest.mark.parametrize("mlp_impl,hash_order,overlap", [
    ("fused", "sample", False), ("fused", "sample", True), ("fused_fwd", "sample", False),
    ("tc", "sample", False), ("cuda", "sample", False), ("fused", "level", True),
    ("fused", "level", False), ("cuda", "level", False)])
@pytest.mark.parametrize("restriction", [False, True])
def test_hashmlp_loss_and_grads_match_oracle(restriction, mlp_impl, hash_order, overlap):
    pool, tree, models, rays, targets = _hash_setup(log2_T=14, K=2, restriction=restriction,
                                                    mlp_impl=mlp_impl, hash_order=hash_order)
    pool.overlap_backward = overlap  # the split pipeline applies to level-major fields
    dt = 0.04
    pool.zero_grad()
    loss, out, b = pool.loss_and_grad(rays, targets, dt)
    torch.cuda.synchronize()
    pool.check()
    otree = vo.Tree(vr.tree_to_json(tree))
    oloss, oout = grad_oracle.field_loss(otree, lambda k, pts, d: models[k].eval_t(pts, d),
                                         rays.T, targets, (0.2, 0.3, 0.4), dt)
    oloss.backward()
    got = out.cpu().numpy().T
    oo = oout.detach().cpu().numpy() if hasattr(oout, "detach") else np.asarray(oout)
    # colour, opacity, depth, transmittance, distortion (north_star: 1e-4 abs)
    for col in range(7):
        np.testing.assert_allclose(got[:, col], oo[:, col], atol=1e-4, rtol=0, err_msg=str(col))
    assert loss.item() == pytest.approx(oloss.item(), rel=1e-5)
    for kk, f in enumerate(pool.fields):
        gt, gw = models[kk].grads()
        mine_t = f.grad_table.cpu().numpy().astype(np.float64)
        mine_w = f.grad_weights.cpu().numpy().astype(np.float64)
        rel_t = np.linalg.norm(mine_t - gt) / max(np.linalg.norm(gt), 1e-30)
        rel_w = np.linalg.norm(mine_w - gw) / max(np.linalg.norm(gw), 1e-30)
        print(f"region {kk}: grad rel err table {rel_t:.2e} weights {rel_w:.2e}")
        assert rel_t <= 1e-3, rel_t
        assert rel_w <= 1e-3, rel_w


def test_level_major_hash_kernels_match_sample_major():
    """vr_hash_positions + vr_hash_fwd_lm == vr_hash_fwd bit for bit; vr_hash_bwd_lm sums the
    same contributions as vr_hash_bwd (float atomics: order-dependent rounding only)."""
    from paper_2404_16221_b200 import _lib
    pool, tree, models, rays, _ = _hash_setup(log2_T=16, K=1, n_rays=3000)
    f = pool.fields[0]
    rd = pool.rays_to_device(rays)
    b = pool.sample(rd, 0.01)
    n = b.n_samples
    assert n > 100000
    s = _lib.stream_ptr()
    enc_a = torch.empty((16, n), dtype=torch.float32, device=DEV)
    enc_b = torch.empty((16, n), dtype=torch.float32, device=DEV)
    pos = torch.empty((3, n), dtype=torch.float32, device=DEV)
    args = (_lib.ptr(rd), rd.shape[1], _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(b.ray_id), n)
    pos_a = torch.empty((3, n), dtype=torch.float32, device=DEV)
    _lib.call("vr_hash_fwd", _lib.addr(f.desc), _lib.ptr(f.table), *args, _lib.ptr(enc_a),
              _lib.ptr(pos_a), s)
    _lib.call("vr_hash_positions", _lib.addr(f.desc), *args, _lib.ptr(pos), s)
    _lib.call("vr_hash_fwd_lm", _lib.addr(f.desc), _lib.ptr(f.table), _lib.ptr(pos), n,
              _lib.ptr(enc_b), s)
    assert torch.equal(enc_a.view(torch.int32), enc_b.view(torch.int32))
    assert torch.equal(pos_a.view(torch.int32), pos.view(torch.int32))
    denc = torch.randn((16, n, 2), device=DEV)
    ga = torch.zeros_like(f.table)
    gb = torch.zeros_like(f.table)
    ws = f._workspace(rd.device)
    _lib.call("vr_hash_bwd", _lib.addr(f.desc), *args, _lib.ptr(denc), _lib.ptr(ga), _lib.ptr(ws),
              ws.numel(), s)
    _lib.call("vr_hash_bwd_lm", _lib.addr(f.desc), _lib.ptr(pos), n, _lib.ptr(denc),
              _lib.ptr(gb), _lib.ptr(ws), ws.numel(), s)
    gc = torch.zeros_like(f.table)  # sample order from stored positions, co-resident grid
    _lib.call("vr_hash_scatter", _lib.addr(f.desc), _lib.ptr(pos), n, _lib.ptr(denc),
              _lib.ptr(gc), _lib.ptr(ws), ws.numel(), 0, 148, None, None, s)
    torch.cuda.synchronize()
    assert torch.count_nonzero(ga) > 1000
    for g in (gb, gc):
        rel = ((ga - g).norm() / ga.norm()).item()
        assert rel < 1e-5, rel


def test_hash_order_auto_picks_level_major_for_tables_larger_than_l2():
    cfg_small = vr.HashGridConfig(log2_T=19, max_res=2048)
    cfg_big = vr.HashGridConfig(log2_T=22, max_res=2048)
    box = vr.Aabb([0, 0, 0], [1, 1, 1])
    assert vr.HashGridMLP(cfg_small, box, DEV).hash_order == "sample"
    assert vr.HashGridMLP(cfg_big, box, DEV).hash_order == "level"


def test_train_step_decreases_loss():
    pool, tree, models, rays, targets = _hash_setup(log2_T=14, K=2, n_rays=256)
    losses = [pool.train_step(rays, targets, 0.04, lr=1e-2, step=s).item() for s in range(1, 21)]
    assert losses[-1] < losses[0]


@pytest.mark.parametrize("n", [1, 127, 128, 1000, 40000])
def test_mlp_tensor_core_matches_cuda_core(n):
    """tcgen05 MLP (production) vs the CUDA-core reference kernel: same fp16
    quantisation points, fp32 accumulation -> agreement to accumulation order."""
    from paper_2404_16221_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(n)
    w32 = vr.fields.init_mlp_weights(g).to(DEV)
    w16 = w32.half()
    enc = (torch.randn((16, n, 2), generator=g) * 0.5).half().to(DEV).contiguous()
    R = max(n // 7, 1)
    d = torch.randn((R, 3), generator=g, dtype=torch.float64)
    d = d / d.norm(dim=1, keepdim=True)
    rays = torch.zeros((8, R), dtype=torch.float64)
    rays[3:6] = d.T
    rays = rays.to(DEV)
    rid = torch.randint(0, R, (n,), generator=g, dtype=torch.int32).to(DEV)
    s = _lib.stream_ptr()
    outs = []
    for name in ("vr_mlp_fwd", "vr_mlp_fwd_tc"):
        o = torch.empty((n, 4), dtype=torch.float32, device=DEV)
        _lib.call(name, _lib.ptr(w16), _lib.ptr(enc), _lib.ptr(rays), R, _lib.ptr(rid), n,
                  _lib.ptr(o), s)
        outs.append(o)
    torch.cuda.synchronize()
    a, b = outs
    assert torch.isfinite(b).all()
    rel = ((a - b).abs() / (a.abs() + 1e-3)).max().item()
    assert rel < 2e-3, rel
    assert (a - b).abs()[:, 1:].max().item() < 1e-4
    dsr = (torch.randn((n, 4), generator=g) * 0.1).to(DEV)
    grads = []
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    for name in ("vr_mlp_bwd", "vr_mlp_bwd_tc"):
        gw = torch.zeros(_lib.VR_MLP_NPARAMS, dtype=torch.float32, device=DEV)
        de = torch.empty((16, n, 2), dtype=torch.float32, device=DEV)
        args = [_lib.ptr(w16), _lib.ptr(enc), _lib.ptr(rays), R, _lib.ptr(rid), n, _lib.ptr(dsr)]
        if name.endswith("_tc"):  # with the forward's output: per-CTA gradient scaling
            args += [_lib.ptr(b)]
        args += [_lib.ptr(gw), _lib.ptr(de)]
        if name.endswith("_tc"):
            args += [_lib.ptr(err), 0, None, None]
        _lib.call(name, *args, s)
        grads.append((gw, de))
    torch.cuda.synchronize()
    assert err.item() == 0
    (gw_a, de_a), (gw_b, de_b) = grads
    # random (unstructured) inputs: fp16 activation rounding flips between fp32
    # accumulation orders dominate the difference (scripts/debug_mlp.py measures both
    # kernels against a float64 reference: same order of error)
    assert ((gw_a - gw_b).norm() / gw_a.norm()).item() < 5e-3
    assert ((de_a - de_b).norm() / de_a.norm()).item() < 5e-3
    assert gw_b[_lib.VR_MLP_W3C + 3 * 64:].abs().max().item() == 0.0


@pytest.mark.parametrize("density_only", [False, True])
def test_interlevel_loss_and_proposal_grads_match_oracle(density_only):
    """Interlevel (proposal) loss — parity against oracle/grad_oracle.field_loss_interlevel
    (parity unpinned: no reference code).  NeRF gradients must be unaffected (w is
    stop-gradient in the interlevel term).  density_only: the proposal runs only its
    density branch (its colour head gets zero gradient either way)."""
    rng = np.random.default_rng(7)
    pool, tree, models, rays, targets = _hash_setup(log2_T=14, K=2, seed=3)
    cfg = vr.HashGridConfig(log2_T=12, max_res=128)
    props, pmodels = [], []
    for k in range(len(tree.leaves)):
        _, n_entries = hmo.levels(12, max_res=128)
        table = rng.uniform(-0.3, 0.3, size=(n_entries, 2)).astype(np.float32)
        w = np.zeros(hmo.NPARAMS, dtype=np.float32)
        for off, rows, cols in ((0, 64, 32), (2048, 16, 64), (3072, 64, 32), (5120, 64, 64),
                                (9216, 3, 64)):
            w[off:off + rows * cols] = rng.normal(size=rows * cols) / np.sqrt(cols)
        box = tree.leaves[k].box
        props.append(vr.HashGridMLP(cfg, box, DEV, table=torch.from_numpy(table),
                                    weights=torch.from_numpy(w), density_only=density_only))
        pmodels.append(hmo.HashMLPModel(table, w, 12, box.mn, box.mx, max_res=128))
    pool2 = vr.VolumePool(tree, pool.fields, (0.2, 0.3, 0.4), DEV, proposals=props)
    dt = 0.04
    pool2.zero_grad()
    loss, out, b = pool2.loss_and_grad(rays, targets, dt, lambda_interlevel=0.5)
    torch.cuda.synchronize()
    pool2.check()
    otree = vo.Tree(vr.tree_to_json(tree))
    oloss, oout, oil = grad_oracle.field_loss_interlevel(
        otree, lambda k, p, d: models[k].eval_t(p, d), lambda k, p, d: pmodels[k].eval_t(p, d),
        rays.T, targets, (0.2, 0.3, 0.4), dt, 1.0, 0.5)
    oloss.backward()
    assert oil.item() > 0.0
    assert loss.item() == pytest.approx(oloss.item(), rel=1e-5)
    for kk in range(len(tree.leaves)):
        for f, m in ((pool2.fields[kk], models[kk]), (props[kk], pmodels[kk])):
            gt, gw = m.grads()
            rel_t = np.linalg.norm(f.grad_table.cpu().numpy() - gt) / max(np.linalg.norm(gt), 1e-30)
            rel_w = np.linalg.norm(f.grad_weights.cpu().numpy() - gw) / max(np.linalg.norm(gw), 1e-30)
            assert rel_t <= 1e-3 and rel_w <= 1e-3, (kk, rel_t, rel_w)


# ---- optimiser and error gating ---------------------------------------------------------

@pytest.mark.parametrize("n", [1, 7, 4096, 100003])
def test_adam_matches_torch(n):
    """vr_adam_step == torch.optim.Adam (no weight decay) over several steps of the same
    gradient sequence, betas (0.9, 0.99), eps 1e-15 (the training defaults)."""
    from paper_2404_16221_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(n)
    p0 = torch.randn(n, generator=g)
    grads = [torch.randn(n, generator=g) * 10.0 ** (-k) for k in range(6)]
    mine = p0.clone().to(DEV)
    m = torch.zeros_like(mine)
    v = torch.zeros_like(mine)
    ref = p0.clone().to(DEV).requires_grad_(True)
    opt = torch.optim.Adam([ref], lr=1e-2, betas=(0.9, 0.99), eps=1e-15)
    s = _lib.stream_ptr()
    for step, gr in enumerate(grads, start=1):
        gd = gr.to(DEV)
        _lib.call("vr_adam_step", _lib.ptr(mine), _lib.ptr(gd), _lib.ptr(m), _lib.ptr(v), n, 1e-2,
                  0.9, 0.99, 1e-15, step, None, s)
        ref.grad = gd.clone()
        opt.step()
    torch.cuda.synchronize()
    st = opt.state[ref]
    torch.testing.assert_close(mine, ref.detach(), rtol=1e-5, atol=1e-7)
    # the moments to a few float32 ulps of their scale (m cancels where the gradient
    # sequence changes sign: relative error there is meaningless)
    torch.testing.assert_close(m, st["exp_avg"], rtol=4e-6, atol=4e-7 * m.abs().max().item())
    torch.testing.assert_close(v, st["exp_avg_sq"], rtol=4e-6, atol=0)


def test_adam_is_skipped_when_the_error_word_is_set():
    from paper_2404_16221_b200 import _lib
    p = torch.randn(1000, device=DEV)
    p0 = p.clone()
    gr = torch.randn(1000, device=DEV)
    m = torch.zeros_like(p)
    v = torch.zeros_like(p)
    err = torch.full((1,), _lib.VR_FLAG_NONFINITE, dtype=torch.int32, device=DEV)
    _lib.call("vr_adam_step", _lib.ptr(p), _lib.ptr(gr), _lib.ptr(m), _lib.ptr(v), 1000, 1e-2,
              0.9, 0.99, 1e-15, 1, _lib.ptr(err), _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(p, p0) and not m.any() and not v.any()
    err.zero_()
    _lib.call("vr_adam_step", _lib.ptr(p), _lib.ptr(gr), _lib.ptr(m), _lib.ptr(v), 1000, 1e-2,
              0.9, 0.99, 1e-15, 1, _lib.ptr(err), _lib.stream_ptr())
    torch.cuda.synchronize()
    assert not torch.equal(p, p0)


def _poisoned_pool(field, value):
    """A hash+MLP pool whose exchanged packets get one non-empty packet's field set to
    value (mid train_step: after K4, before K5)."""
    pool, tree, models, rays, targets = _hash_setup(log2_T=12, K=2, n_rays=64)
    orig = pool.exchange_packets

    def poisoned(b, local, extra=None, dst=None):
        allp, all_e = orig(b, local, extra, dst)
        live = (allp[:, :, 7].view(torch.int32) != np.iinfo(np.int32).max).nonzero()
        k, r = live[0].tolist()
        allp[k, r, field] = value
        return allp, all_e

    pool.exchange_packets = poisoned
    return pool, rays, targets


@pytest.mark.parametrize("field,value,exc", [
    (0, float("nan"), vr.NonFiniteInputError),   # T
    (1, float("inf"), vr.NonFiniteInputError),   # C.r
    (6, -1.0, vr.NegativeLossError),             # L: composed distortion below -1e-12
])
def test_train_step_raises_and_leaves_parameters_unchanged(field, value, exc):
    """A non-finite packet / negative distortion in the middle of train_step raises the
    reference exception from THAT step (segrender.py:124-141) and Adam does not run."""
    pool, rays, targets = _poisoned_pool(field, value)
    f = pool.fields[0]
    before = [t.clone() for t in (f.table, f.weights)]
    with pytest.raises(exc):
        pool.train_step(rays, targets, 0.04, lr=1e-2, step=1)
    for fl in pool.fields:
        assert fl.adam is None or not any(t.any() for t in fl.adam)  # moments untouched
    assert torch.equal(f.table, before[0]) and torch.equal(f.weights, before[1])
    assert int(pool.err.item()) == 0  # cleared by the raise
    # the next clean step trains normally
    pool.exchange_packets = type(pool).exchange_packets.__get__(pool)
    loss = pool.train_step(rays, targets, 0.04, lr=1e-2, step=1)
    assert np.isfinite(loss.item()) and not torch.equal(f.table, before[0])




def test_a_trainable_field_instance_serves_one_region_only():
    pool, tree, models, rays, targets = _hash_setup(log2_T=12, K=2, n_rays=8)
    with pytest.raises(ValueError):
        vr.VolumePool(tree, [pool.fields[0], pool.fields[0]], (0, 0, 0), DEV)
    scene = vr.Scene(tree.root_box, pool.fields[0], (0, 0, 0))
    with pytest.raises(ValueError):
        vr.spawn(tree, scene, DEV)


@pytest.mark.parametrize("case_i", [0, 1, 2])
def test_hash_kernels_match_hand_vectors(case_i):
    """vr_hash_indices and vr_hash_fwd on the hand-worked points of tests/golden/hash_hand.json
    (the published Instant-NGP hash, make_hash_hand.py): every corner index bit-exact; each
    level's feature = sum of hand weight x table entry (fp16 output: within one fp16 ulp)."""
    from paper_2404_16221_b200 import _lib
    g = json.loads((GOLDEN / "hash_hand.json").read_text())
    case = g["cases"][case_i]
    pts = np.asarray(g["points"], dtype=np.float64)
    n = len(pts)
    cfg = vr.HashGridConfig(log2_T=case["log2_T"], max_res=case["max_res"])
    rng = np.random.default_rng(case_i)
    f = vr.HashGridMLP(cfg, vr.Aabb([0, 0, 0], [1, 1, 1]), DEV, seed=case_i, table_init=1.0)
    table = f.table.cpu().numpy()
    # rays from the points themselves (t0 = t1 = 0: the sample point is the origin)
    rays = np.zeros((8, n))
    rays[0:3] = pts.T
    rays[3] = 1.0
    rays[7] = 1.0
    rd = torch.from_numpy(rays).to(DEV)
    z = torch.zeros(n, dtype=torch.float64, device=DEV)
    rid = torch.arange(n, dtype=torch.int32, device=DEV)
    idx = torch.empty((16, n, 8), dtype=torch.int32, device=DEV)
    s = _lib.stream_ptr()
    _lib.call("vr_hash_indices", _lib.addr(f.desc), _lib.ptr(rd), n, _lib.ptr(z), _lib.ptr(z),
              _lib.ptr(rid), n, _lib.ptr(idx), s)
    enc = torch.empty((16, n), dtype=torch.float32, device=DEV)  # half2 per (level, sample)
    pos = torch.empty((3, n), dtype=torch.float32, device=DEV)
    _lib.call("vr_hash_fwd", _lib.addr(f.desc), _lib.ptr(f.table), _lib.ptr(rd), n, _lib.ptr(z),
              _lib.ptr(z), _lib.ptr(rid), n, _lib.ptr(enc), _lib.ptr(pos), s)
    torch.cuda.synchronize()
    got = idx.cpu().numpy()
    feats = enc.cpu().numpy().view(np.float16).reshape(16, n, 2).astype(np.float64)
    offs = f.desc.offset
    for l, hand in enumerate(case["levels"]):
        want = np.asarray(hand["idx"], dtype=np.int64)
        assert np.array_equal(got[l].astype(np.int64), want), f"level {l}"
        w = np.asarray(hand["w"], dtype=np.float64)
        ref = (w[:, :, None] * table[offs[l] + want]).sum(1)
        ulp = np.maximum(np.spacing(np.abs(ref).astype(np.float16)).astype(np.float64), 2.0 ** -24)
        assert (np.abs(feats[l] - ref) <= ulp * 1.01).all(), f"level {l}"


@pytest.mark.parametrize("name", ["vr_mlp_bwd_tc", "vr_mlp_bwd_tc_density"])
def test_mlp_backward_flags_a_non_finite_gradient(name):
    """A non-finite value in the MLP backward (an fp16 operand overflow, or a NaN upstream)
    reaches d(enc) / the weight gradients and raises VR_FLAG_GRAD_OVERFLOW."""
    from paper_2404_16221_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(3)
    n = 1000
    w16 = vr.fields.init_mlp_weights(g).to(DEV).half()
    enc = (torch.randn((16, n, 2), generator=g) * 0.5).half().to(DEV).contiguous()
    rays = torch.zeros((8, n), dtype=torch.float64, device=DEV)
    rays[3] = 1.0
    rid = torch.arange(n, dtype=torch.int32, device=DEV)
    sig = torch.ones((n, 4), device=DEV)
    for poison, flagged in ((False, False), (True, True)):
        dsr = (torch.randn((n, 4), generator=g) * 0.1).to(DEV)
        if poison:
            dsr[417, 0] = float("nan")
        gw = torch.zeros(_lib.VR_MLP_NPARAMS, device=DEV)
        de = torch.empty((16, n, 2), device=DEV)
        err = torch.zeros(1, dtype=torch.int32, device=DEV)
        _lib.call(name, _lib.ptr(w16), _lib.ptr(enc), _lib.ptr(rays), n, _lib.ptr(rid), n,
                  _lib.ptr(dsr), _lib.ptr(sig), _lib.ptr(gw), _lib.ptr(de), _lib.ptr(err), 0,
                  None, None, _lib.stream_ptr())
        torch.cuda.synchronize()
        assert bool(err.item() & _lib.VR_FLAG_GRAD_OVERFLOW) == flagged
