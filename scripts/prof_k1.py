"""One K1 (vr_sample_stage + compaction) of a config for rank/world (for ncu captures)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

name, rank, world = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
w = CONFIGS[name]
tree = w.tree
rays = torch.from_numpy(make_rays(w)).to("cuda:0")
lo, cnt = vr.owned_regions(len(tree.leaves), rank, world)
fields = [vr.AnalyticRegion(vr.ConstantBox(tree.leaves[k].box, 0.0, (0, 0, 0)))
          for k in range(lo, lo + cnt)]
pool = vr.VolumePool(tree, fields, (0, 0, 0), "cuda:0", rank, world)
for _ in range(2):
    b = pool.sample(rays, w.dt)
torch.cuda.synchronize()
print(name, rank, world, "samples", b.n_samples, pool.last_k1)
