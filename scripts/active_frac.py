"""Why samples have a zero upstream gradient in the bench's steady state (c4 by default):
per field set, the fraction of samples with dsig_rgb == 0 (the active-row list skips them),
and of the remaining ones how many the MLP backward still turns into exact zeros (density
clamp of trunc_exp at |od0| >= 15, saturated sigmoid rgb in {0, 1})."""
import sys

sys.path.insert(0, ".")
import torch

import bench
from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets

DEV = "cuda:0"
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
burn = int(sys.argv[2]) if len(sys.argv) > 2 else 27
pool = bench.build_pool(w, 0, 1, DEV, None)
batches = [(torch.from_numpy(make_rays(w, seed=s)).to(DEV),
            torch.from_numpy(make_targets(w.n_rays, seed=100 + s)).to(DEV)) for s in range(4)]
for k in range(burn):
    r, t = batches[k % 4]
    pool.train_step(r, t, w.dt, lr=1e-2, step=k + 1, lambda_interlevel=w.interlevel)
torch.cuda.synchronize()

stats = []
orig_jobs = pool.field_backward_jobs


def jobs(rays, b, js):
    base = pool.region_lo - b.region_lo
    for fields, dsig, sig in js:
        tot = dict(n=0, zero=0, clamp=0, sat=0)
        for kk in range(len(fields)):
            lo, hi = b.region_slice(base + kk)
            d = dsig[lo:hi]
            sg = sig[lo:hi] if sig is not None else None
            z = (d == 0).all(1)
            tot["n"] += hi - lo
            tot["zero"] += int(z.sum())
            if sg is not None:
                s0 = sg[:, 0]
                clamp = (s0 >= torch.exp(torch.tensor(15.0, device=DEV))) | (
                    s0 <= torch.exp(torch.tensor(-15.0, device=DEV)))
                rgb = sg[:, 1:]
                satc = ((rgb == 0) | (rgb == 1) | (d[:, 1:] == 0)).all(1)
                dead = ~z & (clamp | (d[:, 0] == 0)) & satc
                tot["clamp"] += int((~z & clamp).sum())
                tot["sat"] += int(dead.sum())
        stats.append(tot)
    return orig_jobs(rays, b, js)


pool.field_backward_jobs = jobs
r, t = batches[burn % 4]
pool.train_step(r, t, w.dt, lr=1e-2, step=burn + 1, lambda_interlevel=w.interlevel)
torch.cuda.synchronize()
for name, st in zip(("nerf", "proposal"), stats):
    n = st["n"]
    print(f"{name}: {n} samples, upstream zero {st['zero'] / n:.3f}, "
          f"density clamped (non-zero upstream) {st['clamp'] / n:.3f}, "
          f"zero through the MLP's saturations {st['sat'] / n:.3f}")
