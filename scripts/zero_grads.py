"""Fraction of samples whose upstream gradient (dsigma, drgb) is exactly zero, per training
step of a workload (c3 by default) — the samples a backward could skip."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets

DEV = torch.device("cuda:0")
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
pool = bench.build_pool(w, 0, 1, DEV, None)
rays = torch.from_numpy(make_rays(w)).to(DEV)
tg = torch.from_numpy(make_targets(w.n_rays)).to(DEV)
orig = vr.VolumePool.field_backward_jobs
fr = []


def spy(self, rays_, b, jobs):
    d = jobs[0][1][: b.n_samples]
    z = (d == 0).all(dim=1)
    # whole 128-sample tiles of zeros, per region
    tiles = []
    for k in range(b.region_cnt):
        lo, hi = b.region_slice(k)
        zz = z[lo:hi]
        n = (hi - lo) // 128 * 128
        tiles.append(zz[:n].view(-1, 128).all(dim=1).float().mean().item())
    fr.append((z.float().mean().item(), sum(tiles) / len(tiles)))
    return orig(self, rays_, b, jobs)


vr.VolumePool.field_backward_jobs = spy
for s in range(1, 15):
    pool.train_step(rays, tg, w.dt, lr=1e-2, step=s, lambda_interlevel=w.interlevel)
    torch.cuda.synchronize()
    print(f"step {s}: zero-gradient samples {fr[-1][0]:.3f}, all-zero 128-tiles {fr[-1][1]:.3f}",
          flush=True)
