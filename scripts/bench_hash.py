"""Per-level cost of the hash-grid kernels on real c3 samples (one region)."""
import sys
sys.path.insert(0, ".")
import ctypes
import torch
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib as L
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

DEV = "cuda:0"
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
w.n_rays = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
tree = w.tree
cfg = vr.HashGridConfig(log2_T=w.log2_T, max_res=w.max_res)
fields = [vr.HashGridMLP(cfg, tree.leaves[k].box, DEV, seed=k) for k in range(len(tree.leaves))]
pool = vr.VolumePool(tree, fields, (0, 0, 0), DEV)
rays = pool.rays_to_device(make_rays(w))
b = pool.sample(rays, w.dt)
k = 3
lo, hi = b.region_slice(k)
n = hi - lo
f = fields[k]
enc = torch.empty((16, n, 2), dtype=torch.float16, device=DEV)
denc = torch.randn((16, n, 2), device=DEV) * 1e-3
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


print(f"{w.name}: region {k}: {n} samples; levels res={list(f.desc.res)[:16]}")
for nl in (1, 2, 4, 8, 12, 16):
    d = L.VrHashGridDesc.from_buffer_copy(f.desc)
    d.n_levels = nl
    tf = timeit(lambda: L.call("vr_hash_fwd", L.addr(d), L.ptr(f.table), L.ptr(rays), rays.shape[1],
                               L.ptr(b.t0[lo:]), L.ptr(b.t1[lo:]), L.ptr(b.ray_id[lo:]), n, L.ptr(enc), None, s))
    nb = int(L.load().vr_hash_bwd_workspace_bytes(L.addr(d)))
    ws = torch.zeros(max(nb, 16), dtype=torch.uint8, device=DEV)
    tb = timeit(lambda: L.call("vr_hash_bwd", L.addr(d), L.ptr(rays), rays.shape[1], L.ptr(b.t0[lo:]),
                               L.ptr(b.t1[lo:]), L.ptr(b.ray_id[lo:]), n, L.ptr(denc), L.ptr(f.grad_table),
                               L.ptr(ws), ws.numel(), s))
    tb0 = timeit(lambda: L.call("vr_hash_bwd", L.addr(d), L.ptr(rays), rays.shape[1], L.ptr(b.t0[lo:]),
                               L.ptr(b.t1[lo:]), L.ptr(b.ray_id[lo:]), n, L.ptr(denc), L.ptr(f.grad_table),
                               None, 0, s))
    print(f"levels 0..{nl-1}: fwd {tf:.3f} ms  bwd {tb:.3f} ms (replicas {nb/1e6:.1f} MB)  bwd plain {tb0:.3f} ms")
