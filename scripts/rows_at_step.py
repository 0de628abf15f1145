"""Active-row counts (vr_active_rows) of every region in the step prof_r2b.sh captures: the
bench's sequence (burn-in + warm-up steps over the rotating batches), then one more step
on batch 0 whose row lists are recorded.  Gives the per-launch sample counts the sparse
kernels' ncu captures are normalised by (scripts/ncu_bounds.py).
    python scripts/rows_at_step.py <config> <burnin+warmup> > rows.json"""
import json
import sys

sys.path.insert(0, ".")
import torch

import bench
from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets

DEV = "cuda:0"
w = CONFIGS[sys.argv[1]]
n_pre = int(sys.argv[2])
pool = bench.build_pool(w, 0, 1, DEV, None)
batches = [(torch.from_numpy(make_rays(w, seed=s)).to(DEV),
            torch.from_numpy(make_targets(w.n_rays, seed=100 + s)).to(DEV)) for s in range(4)]
for k in range(n_pre):
    r, t = batches[k % 4]
    pool.train_step(r, t, w.dt, lr=1e-2, step=k + 1, lambda_interlevel=w.interlevel)
rec = []
orig = pool._active_rows


def spy(dsig, n):
    rows, cnt = orig(dsig, n)
    rec.append((cnt, n))
    return rows, cnt


pool._active_rows = spy
r, t = batches[0]
pool.train_step(r, t, w.dt, lr=1e-2, step=n_pre + 1, lambda_interlevel=w.interlevel)
torch.cuda.synchronize()
vals = [(int(c.item()), n) for c, n in rec]
K = len(pool.fields)
print(json.dumps({"config": w.name, "step": n_pre + 1,
                  "nerf": vals[:K], "proposal": vals[K:2 * K]}))
