#!/bin/bash
set -u
for mb in 48 64 80; do
  echo "budget $mb"
  VR_LM_BUDGET_MB=$mb timeout 600 python bench.py --config c5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if v['ms_per_step']>2})"
  VR_LM_BUDGET_MB=$mb timeout 600 python bench.py --config c4 --steps 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if v['ms_per_step']>2})"
done
