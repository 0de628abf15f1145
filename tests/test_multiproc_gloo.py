"""CPU, world_size 2 over gloo: the multi-rank exchange path of the engine.

Each rank builds the packets of its own region block (here with the CPU oracle, in
the engine's packet format), exchanges them through the product's comm functions,
and the global fold of the gathered slab must equal — bitwise — the fold of the slab
a single process builds for all regions (the training-mode agreement check,
distsim.py:457-475)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_npz
from oracle import volray_oracle as vo

INT_MAX = np.iinfo(np.int32).max


def oracle_packets(g, region_lo, cnt):
    """[cnt, R, 8] float32 packets {T, C, A, D - A*te, L, order bits}."""
    tree = vo.Tree(g["tree"])
    ev = vo.scene_field_eval(g["scene"])
    rays = g["rays"]
    R = rays.shape[0]
    out = np.zeros((cnt, R, 8), dtype=np.float32)
    out[:, :, 0] = 1.0
    out[:, :, 7] = np.array([INT_MAX], dtype=np.int32).view(np.float32)[0]
    for r in range(R):
        o, d, tn, tf = rays[r, 0:3], rays[r, 3:6], rays[r, 6], rays[r, 7]
        t0, t1, tile = vo.sample_ray(tree, o, d, tn, tf, float(g["dt"]))
        te = vo.root_entry(tree, o, d, tn, tf)
        for kk in range(cnt):
            sel = np.nonzero(tile == region_lo + kk)[0]
            if sel.size == 0:
                continue
            mids = 0.5 * (t0[sel] + t1[sel])
            sig, rgb = ev(region_lo + kk, o + mids[:, None] * d, d)
            T, C, A, D, L = vo.segment_packet(t0[sel], t1[sel], sig, rgb)
            out[kk, r, :7] = [T, *C, A, D - A * te, L]
            out[kk, r, 7] = np.array([sel[0]], dtype=np.int32).view(np.float32)[0]
    return out


def fold_slab(slab):
    """Global fold of a [K, R, 8] slab (K5 restated, float64)."""
    K, R, _ = slab.shape
    res = np.zeros((R, 5))
    keys = slab[:, :, 7].copy().view(np.int32)
    for r in range(R):
        ks = [k for k in range(K) if keys[k, r] != INT_MAX]
        ks.sort(key=lambda k: keys[k, r])
        pk = [(float(slab[k, r, 0]), slab[k, r, 1:4].astype(np.float64), float(slab[k, r, 4]),
               float(slab[k, r, 5]), float(slab[k, r, 6])) for k in ks]
        C, A, D, T, L = vo.fold_packets(pk)
        res[r] = [C.sum(), A, D, T, L]
    return res


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_16221_b200 import comm

        g = load_npz(name)
        K = len(vo.Tree(g["tree"]).leaf_mn)
        lo, cnt = comm.owned_regions(K, rank, world)
        local = torch.from_numpy(oracle_packets(g, lo, cnt))
        allp = comm.all_gather_packets(local, dist.group.WORLD, world)
        gathered = comm.gather_packets(local, dist.group.WORLD, world, rank)
        loss = torch.tensor([float(fold_slab(allp.numpy())[:, 4].sum())], dtype=torch.float64)
        everyone = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(everyone, loss)
        q.put((rank, allp.numpy(), None if gathered is None else gathered.numpy(),
               [float(e.item()) for e in everyone]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["render_three_blobs_k4.npz", "render_street_k8.npz"])
def test_exchange_world2_matches_single_process(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = load_npz(name)
    K = len(vo.Tree(g["tree"]).leaf_mn)
    single = oracle_packets(g, 0, K)
    ref_fold = fold_slab(single)
    for rank, allp, gathered, losses in sorted(results, key=lambda x: x[0]):
        assert np.array_equal(allp.view(np.uint32), single.view(np.uint32))
        assert np.array_equal(fold_slab(allp), ref_fold)
        assert len(set(losses)) == 1  # identical loss on every rank
        if rank == 0:
            assert np.array_equal(gathered.view(np.uint32), single.view(np.uint32))
        else:
            assert gathered is None
    # the folded result equals the reference tile render of these rays
    np.testing.assert_allclose(ref_fold[:, 1], g["out"][:, 3], atol=1e-6)
    np.testing.assert_allclose(ref_fold[:, 3], g["out"][:, 5], atol=1e-6)


def _sparse_worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import packets_ref as pr
        from paper_2404_16221_b200 import comm

        g = load_npz(name)
        K = len(vo.Tree(g["tree"]).leaf_mn)
        lo, cnt = comm.owned_regions(K, rank, world)
        local = oracle_packets(g, lo, cnt)
        counts = (local[:, :, 7].copy().view(np.int32) != INT_MAX).astype(np.int32)
        # stands in for the proposal transmittance (1 on empty segments, as K4 writes)
        extra = np.where(counts > 0, local[:, :, 0] * 0.5, 1.0).astype(np.float32)
        rec, n = pr.pack(local, counts, lo, extra)
        n_max = comm.all_reduce_max_(torch.tensor([n], dtype=torch.int64), dist.group.WORLD,
                                     world)
        buf = torch.from_numpy(pr.buffer(rec, int(n_max.item())))
        allb = comm.all_gather_packets(buf, dist.group.WORLD, world)
        slab, ex = pr.unpack(allb.numpy(), world, K, local.shape[1])
        got = comm.gather_packets(buf, dist.group.WORLD, world, rank)
        q.put((rank, int(n_max.item()), n, slab, ex, None if got is None else got.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["render_three_blobs_k4.npz", "render_street_k8.npz"])
def test_sparse_exchange_world2_matches_dense(name):
    """Sparse packet exchange (records of non-empty segments; VolumePool.exchange_packets):
    the record-count MAX all-reduce, the padded all-gather and the gather, unpacked with the
    numpy restatement of vr_packets_unpack, rebuild the dense single-process slab bit for
    bit on every rank (and on rank 0 for the gather)."""
    import packets_ref as pr

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sparse_worker, args=(r, world, port, name, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = load_npz(name)
    K = len(vo.Tree(g["tree"]).leaf_mn)
    single = oracle_packets(g, 0, K)
    R = single.shape[1]
    counts = [n for _, _, n, _, _, _ in results]
    for rank, n_max, n, slab, ex, got in sorted(results, key=lambda x: x[0]):
        assert n_max == max(counts)
        assert np.array_equal(slab.view(np.uint32), single.view(np.uint32))
        live = single[:, :, 7].copy().view(np.int32) != INT_MAX
        assert np.array_equal(ex, np.where(live, single[:, :, 0] * 0.5, 1.0).astype(np.float32))
        if rank == 0:
            s0, _ = pr.unpack(got, world, K, R)
            assert np.array_equal(s0.view(np.uint32), single.view(np.uint32))
        else:
            assert got is None
    assert sum(counts) < K * R  # fewer records than dense packets


def _sample_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_16221_b200 import comm

        K = 4
        bounds = [0, 5, 5, 17, 30]  # region-major sample offsets (region 1 empty)
        full = torch.arange(30 * 4, dtype=torch.float32).reshape(30, 4) + 0.5
        lo, cnt = comm.owned_regions(K, rank, world)
        mine = torch.zeros_like(full)
        mine[bounds[lo]:bounds[lo + cnt]] = full[bounds[lo]:bounds[lo + cnt]]
        a = mine.clone()
        got_all = comm.exchange_samples(a, bounds, K, dist.group.WORLD, world, rank, None)
        g = mine.clone()
        got_root = comm.exchange_samples(g, bounds, K, dist.group.WORLD, world, rank, 0)
        q.put((rank, got_all, a.numpy(), got_root, g.numpy(), full.numpy()))
    finally:
        dist.destroy_process_group()


def test_sample_exchange_world2():
    """Sample-broadcast protocol exchange (comm.exchange_samples): every rank's region block
    of the per-sample (sigma, rgb) array reaches every rank (training) or rank 0 (render)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sample_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got_all, a, got_root, g, full in results:
        assert got_all and np.array_equal(a, full)
        if rank == 0:
            assert got_root and np.array_equal(g, full)
        else:
            assert not got_root
