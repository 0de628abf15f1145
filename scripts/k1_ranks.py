"""K1 time per rank when the c3/c4 region set is split over N ranks (simulated on one GPU:
each rank's VolumePool samples only its own regions; no collective involved)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

DEV = "cuda:0"
for name in sys.argv[1:] or ["c3"]:
    w = CONFIGS[name]
    tree = w.tree
    rays = torch.from_numpy(make_rays(w)).to(DEV)
    for world in (1, 2, 4, 8):
        times = []
        for rank in range(world):
            lo, cnt = vr.owned_regions(len(tree.leaves), rank, world)
            fields = [vr.AnalyticRegion(vr.ConstantBox(tree.leaves[k].box, 0.0, (0, 0, 0)))
                      for k in range(lo, lo + cnt)]
            pool = vr.VolumePool(tree, fields, (0, 0, 0), DEV, rank, world)
            pool.sample(rays, w.dt)
            torch.cuda.synchronize()
            from paper_2404_16221_b200 import _lib
            import bench
            timer = bench.EventTimer()
            _lib.TIMER = timer
            for _ in range(3):
                bb = pool.sample(rays, w.dt)
            torch.cuda.synchronize()
            _lib.TIMER = None
            tot = timer.totals()
            ms = sum(t for t, _ in tot.values()) / 3
            times.append((ms, bb.n_samples, {k: round(t / 3, 2) for k, (t, _) in tot.items()}))
        print(name, "world", world, "K1 kernel ms per rank:", [round(t[0], 2) for t in times],
              "rank 0:", times[0][2], flush=True)
