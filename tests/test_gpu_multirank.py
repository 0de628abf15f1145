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


def _worker(rank, world, port, sparse, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vr, doc, tree, scene, rays, targets = _setup()
        pool = vr.spawn(tree, scene, "cuda:0", rank, world, dist.group.WORLD)
        pool.sparse_exchange = sparse
        q.put((rank, _run(pool, rays, targets, doc["dt"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sparse", [True, False])
def test_two_processes_match_single_process(sparse):
    vr, doc, tree, scene, rays, targets = _setup()
    single = _run(vr.spawn(tree, scene, "cuda:0"), rays, targets, doc["dt"])
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sparse, q)) for r in range(world)]
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
