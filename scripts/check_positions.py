"""Normalised hash-grid positions of every c4 / c5 sample: vr_hash_positions (division by
reciprocal + one FMA correction, hashgrid.cuh) against torch float64 division, bit for bit."""
import sys

sys.path.insert(0, ".")
import torch

import bench
from paper_2404_16221_b200 import _lib as L
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

total = mism = 0
for cfg in ("c4", "c5", "c3"):
    w = CONFIGS[cfg]
    pool = bench.build_pool(w, 0, 1, "cuda:0", None)
    for seed in (0, 1):
        rays = pool.rays_to_device(make_rays(w, seed=seed))
        b = pool.sample(rays, w.dt)
        for kk, f in enumerate(pool.fields):
            lo, hi = b.region_slice(kk)
            n = hi - lo
            pos = torch.empty(3 * n, dtype=torch.float32, device="cuda")
            L.call("vr_hash_positions", L.addr(f.desc), L.ptr(rays), rays.shape[1],
                   L.ptr(b.t0[lo:]), L.ptr(b.t1[lo:]), L.ptr(b.ray_id[lo:]), n, L.ptr(pos),
                   L.stream_ptr())
            r = b.ray_id[lo:hi].long()
            m = 0.5 * (b.t0[lo:hi] + b.t1[lo:hi])
            for a in range(3):
                p = rays[a, r] + m * rays[3 + a, r]
                u = ((p - f.box.mn[a]) / (f.box.mx[a] - f.box.mn[a])).float()
                got = pos[a * n:(a + 1) * n]
                bad = int((got.view(torch.int32) != u.view(torch.int32)).sum())
                total += n
                mism += bad
        torch.cuda.synchronize()
    print(f"{cfg}: cumulative {total} coordinates, {mism} differ", flush=True)
    del pool
    torch.cuda.empty_cache()
print("positions bit-identical" if mism == 0 else f"MISMATCH {mism}")
