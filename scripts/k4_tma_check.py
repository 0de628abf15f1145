"""K4 forward with and without TMA staging on the same c4 batch: equal outputs, timing."""
import os
import sys
import time

sys.path.insert(0, ".")
import torch

import bench
from paper_2404_16221_b200 import _lib as L
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

w = CONFIGS["c4"]
lib = L.load()
print("tma available:", lib.vr_tma_available())
pool = bench.build_pool(w, 0, 1, "cuda:0", None)
rays = pool.rays_to_device(make_rays(w))
b = pool.sample(rays, w.dt)
sig = pool.evaluate(rays, b)
outs = {}
for n_arg in (0, pool._tma_n(b.n_samples, b.t0, b.t1, sig)):
    pk = torch.empty((b.region_cnt, b.n_rays, 8), device="cuda")
    tot = torch.empty(b.region_cnt * b.n_rays * 7, dtype=torch.float64, device="cuda")
    f = lambda: L.call("vr_segment_fwd", L.ptr(b.t0), L.ptr(b.t1), L.ptr(sig), L.ptr(b.offsets),
                       L.ptr(b.seg_first), L.ptr(b.ray_te), b.n_rays, b.region_cnt, L.ptr(pk),
                       L.ptr(tot), L.ptr(pool.err), n_arg, L.stream_ptr())
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"n_samples arg {n_arg}: {e0.elapsed_time(e1) / 10:.3f} ms")
    outs[n_arg > 0] = (pk.clone(), tot.clone())
print("packets equal:", torch.equal(outs[False][0].view(torch.int32), outs[True][0].view(torch.int32)),
      "totals equal:", torch.equal(outs[False][1], outs[True][1]))
