#!/bin/bash
# c4 step time vs the MLP backward's grid cap beside the side-stream scatter
for c in 148 185 222 259 296; do
  VR_MLP_BWD_CTAS=$c python bench.py --config c4 --sub none --no-e2e --no-cpu --burnin 20 --steps 6 --warmup 2 > gpurun_out/sweep_$c.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/sweep_$c.json').read().strip().splitlines()[-1]);print($c, round(d['ms_per_step'],2), round(d['kernels']['vr_mlp_bwd_tc']['ms_per_step'],1), round(d['kernels']['vr_hash_scatter']['ms_per_step'],1))"
done
