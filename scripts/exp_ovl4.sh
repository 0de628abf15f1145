#!/bin/bash
set -u
summ() { python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "ms", round(d["ms_per_step"], 2), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items() if v["ms_per_step"] > 1})
PY
}
VR_SCATTER_BLOCKS=0 timeout 900 python bench.py --config c4 --steps 3 --no-cpu --no-e2e > gpurun_out/ov4_on.log 2>&1; summ gpurun_out/ov4_on.log
VR_OVERLAP_BWD=0 timeout 900 python bench.py --config c4 --steps 3 --no-cpu --no-e2e > gpurun_out/ov4_off.log 2>&1; summ gpurun_out/ov4_off.log
