"""Samples per region of a workload's batch (seed 0): the n of the profiled launches."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_16221_b200.workloads import CONFIGS, make_rays  # noqa: E402

for name in sys.argv[1:]:
    w = CONFIGS[name]
    pool = bench.build_pool(w, 0, 1, torch.device("cuda"), None)
    b = pool.sample(torch.from_numpy(make_rays(w, seed=0)).cuda(), w.dt)
    print(name, [b.region_bounds[k + 1] - b.region_bounds[k] for k in range(b.region_cnt)])
    del pool
    torch.cuda.empty_cache()
