"""Level-major hash kernels vs table size (log2_T) on real c3 samples of one region."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib as L
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

DEV = "cuda:0"
w = CONFIGS["c3"]
tree = w.tree
s = L.stream_ptr()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / reps


for log2_T in (19, 20, 21, 22):
    cfg = vr.HashGridConfig(log2_T=log2_T, max_res=w.max_res)
    fields = [vr.HashGridMLP(cfg, tree.leaves[k].box, DEV, seed=k, hash_order="level")
              if k == 3 else vr.AnalyticRegion(vr.ConstantBox(tree.leaves[k].box, 0.0, (0, 0, 0)))
              for k in range(len(tree.leaves))]
    pool = vr.VolumePool(tree, fields, (0, 0, 0), DEV)
    rays = pool.rays_to_device(make_rays(w))
    b = pool.sample(rays, w.dt)
    lo, hi = b.region_slice(3)
    n = hi - lo
    f = fields[3]
    pos = torch.empty((3, n), device=DEV)
    enc = torch.empty((16, n), dtype=torch.float32, device=DEV)
    denc = torch.randn((16, n, 2), device=DEV) * 1e-3
    L.call("vr_hash_positions", L.addr(f.desc), L.ptr(rays), rays.shape[1], L.ptr(b.t0[lo:]),
           L.ptr(b.t1[lo:]), L.ptr(b.ray_id[lo:]), n, L.ptr(pos), s)
    ws = f._workspace(rays.device)
    tf = timeit(lambda: L.call("vr_hash_fwd_lm", L.addr(f.desc), L.ptr(f.table), L.ptr(pos), n,
                               L.ptr(enc), s))
    tb = timeit(lambda: L.call("vr_hash_bwd_lm", L.addr(f.desc), L.ptr(pos), n, L.ptr(denc),
                               L.ptr(f.grad_table), L.ptr(ws), ws.numel(), s))
    tbs = timeit(lambda: L.call("vr_hash_bwd", L.addr(f.desc), L.ptr(rays), rays.shape[1],
                                L.ptr(b.t0[lo:]), L.ptr(b.t1[lo:]), L.ptr(b.ray_id[lo:]), n,
                                L.ptr(denc), L.ptr(f.grad_table), L.ptr(ws), ws.numel(), s))
    mb = f.n_entries * 8 / 2**20
    print(f"log2_T {log2_T}: table {mb:.0f} MB, {n} samples: fwd_lm {tf:.3f} ms  bwd_lm {tb:.3f} ms"
          f"  bwd(sample order) {tbs:.3f} ms  -> {tb / n * 1e6:.3f} ns/sample", flush=True)
    del pool, fields, f
    torch.cuda.empty_cache()
