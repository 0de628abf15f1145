#!/bin/bash
# step time of a config under environment variants:  bash scripts/sweep_env.sh c3 "" "VR_SPLIT_BELOW_MB=64" ...
cfg=$1; shift
for v in "$@"; do
  env $v python bench.py --config $cfg --sub none --no-e2e --no-cpu --burnin 20 --steps 6 --warmup 2 > gpurun_out/sweep_env.json 2>gpurun_out/sweep_env.err
  python -c "import json;d=json.loads(open('gpurun_out/sweep_env.json').read().strip().splitlines()[-1]);print('$cfg', '[$v]', round(d['ms_per_step'],2))" || tail -3 gpurun_out/sweep_env.err
done
