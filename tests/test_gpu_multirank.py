"""Two real processes (world_size 2, gloo) sharing cuda:0: the engine's multi-rank paths end
to end — K1 sizing collective, sparse and dense packet exchange, K5 on every rank, the
per-rank gradients.  gloo stages the CUDA tensors through host memory (comm._host_staged),
so neither rank's kernels wait on the other's; this checks the host-side protocol, not
NVLink speed.  Compared with one process owning every region: losses and images bitwise,
gradients of each rank's regions equal to the single-process slices."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _soa(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    import paper_2404_16221_b200 as vr

    doc = json.loads((GOLDEN / "grad_voxel_room.json").read_text())
    tree = vr.tree_from_json(doc["tree"])
    scene = vr.scene_from_json(doc["scene"])
    rays = _soa(doc["rays"])
    targets = np.full((rays.shape[1], 3), doc["target"])
    return vr, doc, tree, scene, rays, targets


def _run(pool, rays, targets, dt):
    pool.zero_grad()
    loss, out, b = pool.loss_and_grad(rays, targets, dt)
    img, _ = pool.render_rays(rays, dt)
    torch.cuda.synchronize()
    pool.check()
    grads = [f.grad.detach().cpu().numpy().copy() for f in pool.fields]
    return (float(loss.item()), out.cpu().numpy(), None if img is None else img.cpu().numpy(),
            grads, b.seg_max)


def _worker(rank, world, port, sparse, q, backend="gloo"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = f"cuda:{rank}" if backend == "nccl" else "cuda:0"
    if backend == "nccl":
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device(dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vr, doc, tree, scene, rays, targets = _setup()
        pool = vr.spawn(tree, scene, dev, rank, world, dist.group.WORLD)
        pool.sparse_exchange = sparse
        q.put((rank, _run(pool, rays, targets, doc["dt"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
@pytest.mark.parametrize("sparse", [True, False])
def test_two_processes_match_single_process(sparse, backend):
    """gloo: both ranks on cuda:0 (tensors staged through the host).  nccl: one GPU per rank,
    the exchange is NCCL's all_gather_into_tensor / gather over the GPUs' link (skipped on a
    single-GPU box)."""
    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("the NCCL path needs 2 GPUs")
    vr, doc, tree, scene, rays, targets = _setup()
    single = _run(vr.spawn(tree, scene, "cuda:0"), rays, targets, doc["dt"])
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sparse, q, backend))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    K = len(tree.leaves)
    per = K // world
    for rank, (loss, out, img, grads, seg_max) in results.items():
        assert loss == single[0]  # identical loss on every rank
        assert np.array_equal(out, single[1])
        if rank == 0:
            assert np.array_equal(img, single[2])
        else:
            assert img is None
        for kk, g in enumerate(grads):
            np.testing.assert_allclose(g, single[3][rank * per + kk], rtol=1e-10, atol=1e-15)
        assert (seg_max is not None) == sparse


# ---- interlevel loss across ranks (proposal fields, width-10 sparse records) ----------------

def _il_pool(rank, world, group, sparse=True):
    """Two regions of hash-grid NeRF + density-only proposal fields (seeded per region, so
    every process builds the same models); rank r owns its block of regions."""
    import paper_2404_16221_b200 as vr

    root = vr.Aabb([-1, -1, -1], [1, 1, 1])
    tree = vr.grid_tree(root, "x")
    lo, cnt = vr.owned_regions(len(tree.leaves), rank, world)
    cfg = vr.HashGridConfig(log2_T=12, max_res=128)
    pcfg = vr.HashGridConfig(log2_T=10, max_res=64)
    fields = [vr.HashGridMLP(cfg, tree.leaves[k].box, "cuda:0", seed=10 + k, table_init=0.3)
              for k in range(lo, lo + cnt)]
    props = [vr.HashGridMLP(pcfg, tree.leaves[k].box, "cuda:0", seed=50 + k, table_init=0.3,
                            density_only=True) for k in range(lo, lo + cnt)]
    pool = vr.VolumePool(tree, fields, (0.2, 0.3, 0.4), "cuda:0", rank, world, group,
                         proposals=props)
    pool.sparse_exchange = sparse
    rng = np.random.default_rng(5)
    rays = []
    while len(rays) < 200:
        o = rng.uniform(-2.4, 2.4, size=3)
        d = rng.uniform(-0.8, 0.8, size=3) - o
        rays.append([*o, *(d / np.linalg.norm(d)), 0.0, 20.0])
    rays = np.asarray(rays).T.copy()
    targets = rng.uniform(0, 1, size=(200, 3))
    return pool, rays, targets


def _il_run(pool, rays, targets):
    pool.zero_grad()
    loss, out, _ = pool.loss_and_grad(rays, targets, 0.04, lambda_interlevel=0.5)
    torch.cuda.synchronize()
    return (float(loss.item()), out.cpu().numpy(),
            [(f.grad_table.cpu().numpy(), f.grad_weights.cpu().numpy())
             for f in pool.fields + pool.proposals])


def _il_worker(rank, world, port, sparse, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pool, rays, targets = _il_pool(rank, world, dist.group.WORLD, sparse)
        q.put((rank, _il_run(pool, rays, targets)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sparse", [True, False])
def test_two_processes_interlevel_match_single_process(sparse):
    """The interlevel loss across 2 real processes: the proposal transmittance travels in the
    width-10 sparse records (or the dense extra slab), vr_prefix_train runs with own_lo > 0
    on rank 1, and the loss each rank reports is the whole batch's (its interlevel part is
    all-reduced) — equal to one process owning both regions; per-rank NeRF and proposal
    gradients equal that process's slices (float atomics: summation order only)."""
    single = _il_run(*_il_pool(0, 1, None))
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_il_worker, args=(r, world, port, sparse, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, (loss, out, grads) in results.items():
        assert loss == pytest.approx(single[0], rel=1e-12)
        assert np.array_equal(out, single[1])
        # rank r owns region r: its NeRF field is single's field r, its proposal single's 2 + r
        for got, want in zip(grads, [single[2][rank], single[2][2 + rank]]):
            for a, b in zip(got, want):
                assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()
