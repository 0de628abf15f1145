"""Experiment: hash-grid kernels on samples in spatial (Morton) order vs ray order.

Coarse levels: lanes of a warp that hit the same sector merge into one L2 request, so
spatially sorted samples need fewer requests per sample.  c3, one region."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib as L
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

DEV = "cuda:0"
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
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


def spread(x):  # 10-bit -> every third bit
    x = x.to(torch.int64) & 0x3FF
    x = (x | (x << 16)) & 0x030000FF
    x = (x | (x << 8)) & 0x0300F00F
    x = (x | (x << 4)) & 0x030C30C3
    x = (x | (x << 2)) & 0x09249249
    return x


cfg = vr.HashGridConfig(log2_T=w.log2_T, max_res=w.max_res)
K = 3
fields = [vr.HashGridMLP(cfg, tree.leaves[k].box, DEV, seed=k, hash_order="sample")
          if k == K else vr.AnalyticRegion(vr.ConstantBox(tree.leaves[k].box, 0.0, (0, 0, 0)))
          for k in range(len(tree.leaves))]
pool = vr.VolumePool(tree, fields, (0, 0, 0), DEV)
rays = pool.rays_to_device(make_rays(w))
b = pool.sample(rays, w.dt)
lo, hi = b.region_slice(K)
n = hi - lo
f = fields[K]
t0, t1, rid = b.t0[lo:hi].contiguous(), b.t1[lo:hi].contiguous(), b.ray_id[lo:hi].contiguous()
pos = torch.empty((3, n), device=DEV)
L.call("vr_hash_positions", L.addr(f.desc), L.ptr(rays), rays.shape[1], L.ptr(t0), L.ptr(t1),
       L.ptr(rid), n, L.ptr(pos), s)
enc = torch.empty((16, n), dtype=torch.float32, device=DEV)
denc = torch.randn((16, n, 2), device=DEV) * 1e-3
ws = f._workspace(rays.device)
print(f"{w.name}: region {K}, {n} samples, table {f.n_entries * 8 / 2**20:.0f} MB")

for bits in (0, 4, 6, 8, 10):
    if bits == 0:
        perm = torch.arange(n, device=DEV)
        label = "ray order"
    else:
        q = (pos.clamp(0, 1 - 1e-7) * (1 << bits)).to(torch.int64)
        code = spread(q[0]) | (spread(q[1]) << 1) | (spread(q[2]) << 2)
        torch.cuda.synchronize()
        ts = timeit(lambda: torch.sort(code))
        perm = torch.sort(code).indices
        label = f"morton {bits} bits/axis (torch.sort {ts:.2f} ms)"
    t0p, t1p, ridp = t0[perm].contiguous(), t1[perm].contiguous(), rid[perm].contiguous()
    posp = pos[:, perm].contiguous()
    dencp = denc[:, perm].contiguous()
    tf = timeit(lambda: L.call("vr_hash_fwd", L.addr(f.desc), L.ptr(f.table), L.ptr(rays),
                               rays.shape[1], L.ptr(t0p), L.ptr(t1p), L.ptr(ridp), n, L.ptr(enc),
                               None, s))
    tb = timeit(lambda: L.call("vr_hash_scatter", L.addr(f.desc), L.ptr(posp), n, L.ptr(dencp),
                               L.ptr(f.grad_table), L.ptr(ws), ws.numel(), 0, 0, s))
    print(f"{label:45s} hash fwd {tf:.3f} ms   scatter {tb:.3f} ms", flush=True)
